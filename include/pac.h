/*
 * pac.h -- C-ABI of libpac.so: the B200-native (sm_100a) hot path of
 * "SIMD-PAC-DB: Pretty Performant PAC Privacy" (arXiv 2603.15023).
 *
 * One data-parallel path: per-row privacy-unit (PU) key -> 64-bit world mask with
 * exactly 32 bits set (pac_hash, §2, §4); single-pass
 * accumulation of COUNT/SUM/AVG/MIN/MAX for all m = 64 possible worlds per group
 * (pac_agg, Eq. counter, §4; §5); and the
 * noised release pac_noised with the Bayesian posterior update (§4).
 * Readings of ambiguous passages are DESIGN.md R1..R21; the same readings are
 * implemented, independently, by the CPU oracle under oracle/.
 *
 * Conventions (every entry point):
 *  - d_* pointers are DEVICE pointers owned by the caller (e.g. PyTorch tensors);
 *    h_* pointers are host pointers owned by the caller.  The library owns only
 *    pac_session objects (opaque) and never frees caller memory.
 *  - Calls are asynchronous on `stream` unless documented as synchronizing; the
 *    caller keeps every buffer alive until the stream has passed the call.
 *  - Return value: PAC_OK or a negative-free status code below; no exception or
 *    longjmp crosses the ABI.  Device-side conditions that can only be known after
 *    the kernels ran (group capacity, int64 overflow) are reported in the table's
 *    d_status word (see pac_table) and by pac_table_check().
 *  - Layouts are row-major.  "[G][64]" means 64 consecutive elements per group,
 *    element j = world j (world j <-> bit j of the mask, LSB = world 0, R3).
 */
#ifndef PAC_H_
#define PAC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAC_M 64         /* worlds per PU hash, P:L92 (§2) */
#define PAC_MAX_AGGS 8   /* aggregates per pac_agg_grouped call */
#define PAC_MAX_KEYS 4   /* group-by key columns, total width <= 8 bytes (R20) */

typedef struct CUstream_st* pac_stream_t; /* a cudaStream_t; NULL = legacy default stream */

enum {
  PAC_OK = 0,
  PAC_E_INVAL = 1,      /* bad argument: NULL/size mismatch, both or neither mask source,
                           unsupported aggregate combination, unaligned column */
  PAC_E_CAPACITY = 2,   /* more distinct groups than G_cap (pac_table_check) */
  PAC_E_WORKSPACE = 3,  /* ws_bytes smaller than the *_workspace_size() answer */
  PAC_E_CUDA = 4,       /* a CUDA runtime call or kernel launch failed */
  PAC_E_OVERFLOW = 5,   /* an int64 world sum overflowed (R15 precondition violated) */
  PAC_E_MERGE = 6       /* pac_merge_unpack: the ranks' tables were not laid out on one
                           group dictionary (fingerprints differ) */
};

/* Aggregate kinds (agg in {sum, count, avg, min, max}).  Values: SUM_I64 reads
 * an int64 column, the f64 kinds a double column, COUNT none. */
typedef enum {
  PAC_COUNT = 0,
  PAC_SUM_I64 = 1,
  PAC_SUM_F64 = 2,
  PAC_AVG_F64 = 3,
  PAC_MIN_F64 = 4,
  PAC_MAX_F64 = 5
} pac_agg_kind;

typedef struct {
  int32_t kind;          /* pac_agg_kind */
  const void* d_values;  /* [n_rows] int64 or double; NULL for PAC_COUNT */
} pac_agg_spec;

typedef struct {
  const void* d_col;     /* [n_rows] signed integer key column */
  int32_t elem_bytes;    /* 1, 2, 4 or 8 */
} pac_key_col;

/* ------------------------------------------------------------------ session (§8 a1)
 * P:L886 (§4): "sample a secret world index uniformly at random j* ..., initialize ...
 * P = (1/m, ..., 1/m)"; P:L99 (§2): one j* per query shared by all cells; P:L93 /
 * a fresh per-query hash key.  R13: j* = x0 & 63 of Philox4x32-10(seed;
 * 0,0,0,1), salt = x0 | x1<<32 of Philox(seed; 0,0,0,2).  budget_B is the per-release
 * MI budget B (BASELINE uses 1/128).  The session owns a device copy of P and is
 * single-owner and strictly sequential (noising order matters). */
typedef struct pac_session pac_session;

/* Creates a session on the current CUDA device.  Errors: PAC_E_INVAL (out NULL,
 * budget_B <= 0 or not finite), PAC_E_CUDA. */
int pac_session_create(uint64_t seed, double budget_B, pac_session** out);
/* Session over m = 64 or 128 worlds (§8 f4, R29: j* = x0 & (m-1), P = 1/m; the salt is the
 * same as for m = 64).  pac_session_create(...) == pac_session_create_m(..., 64, ...).
 * An m = 128 session finalizes only m = 128 tables; pac_posterior_update / pac_noised_y
 * are m = 64 only (PAC_E_INVAL otherwise). */
int pac_session_create_m(uint64_t seed, double budget_B, int32_t m, pac_session** out);
/* m of the session (0 for NULL). */
int32_t pac_session_worlds(const pac_session* s);
/* Frees the session (synchronizes the device).  NULL is a no-op. */
int pac_session_destroy(pac_session* s);
/* Synchronizing read of the session state.  Any output pointer may be NULL.
 * h_P64: m doubles (64, or 128 for an m = 128 session).  releases: number of non-NULL, non-zero-variance releases so far. */
int pac_session_query(const pac_session* s, uint64_t* salt, int32_t* jstar, double* h_P64,
                      uint64_t* releases, uint64_t* seed, double* budget_B);
/* Overwrites the posterior with 64 host doubles (resume / tests).  Synchronizing. */
int pac_session_set_posterior(pac_session* s, const double* h_P64);
/* Device pointer of the session's posterior P[64] (owned by the session). */
double* pac_session_posterior_device(pac_session* s);

/* ------------------------------------------------------------------ mask (§8 a2)
 * pac_hash (§2; §4; effective hash pac_hash(h(u) XOR q)):
 *   d_mask[i] = balance(fmix64(uint64(d_pu_key[i]) XOR salt))     (R1, R2)
 * popcount(d_mask[i]) == 32 for every i.  n may be 0.  Errors: PAC_E_INVAL (n < 0,
 * NULL pointer with n > 0), PAC_E_CUDA. */
int pac_mask(const int64_t* d_pu_key, int64_t n, uint64_t salt, uint64_t* d_mask,
             pac_stream_t stream);

/* ------------------------------------------------------------------ aggregation (§8 a3-a5)
 * Output table in canonical order: groups ascending by packed key (R20).  Capacity
 * G_cap groups; all arrays caller-allocated with that capacity.
 *
 *   d_num_groups [1]        int64  number of distinct groups (may exceed G_cap: then
 *                                  the table is invalid and d_status has CAPACITY)
 *   d_status     [1]        int32  0 or PAC_E_CAPACITY / PAC_E_OVERFLOW
 *   d_group_key  [G_cap]    uint64 packed composite key (R20); 0 when ungrouped
 *   d_rows       [G_cap]    int64  rows with a nonzero mask in the group (R21)
 *   d_presence   [G_cap]    uint64 K = OR of the group's masks (R5)
 *   d_count      [G_cap][64] int64 per-world row count.  REQUIRED unless every
 *                                  aggregate is MIN/MAX (then NULL)
 *   d_world[a]   [G_cap][64]       per aggregate a: int64 for SUM_I64; double for
 *                                  SUM_F64 / AVG_F64 (the world's value SUM -- AVG
 *                                  divides by d_count at finalize, R6) and MIN/MAX
 *                                  (+inf / -inf for a world with no row); NULL for COUNT
 * Non-finite values (R30, R31): f64 SUM/AVG are IEEE sums (any NaN -> NaN, +inf with -inf
 * -> NaN, else the infinity; finite sums that overflow are out of contract); MIN/MAX use
 * DuckDB's total order on DOUBLE -- NaN above +inf, all NaNs equal (a NaN is written as the
 * canonical quiet NaN).  A world holding only +inf under MIN reads +inf like an empty
 * world; d_presence tells them apart.
 */
typedef struct {
  int64_t* d_num_groups;
  int32_t* d_status;
  uint64_t* d_group_key;
  int64_t* d_rows;
  uint64_t* d_presence;
  int64_t* d_count;
  void* d_world[PAC_MAX_AGGS];
  int32_t m;  /* worlds per group: 0 or 64, or 128 (§8 f4; then d_presence is [G_cap][2] and
                 d_count / d_world are [G_cap][128]) */
} pac_table;

/* Workspace bytes for pac_agg_grouped with these aggregates and capacity (the minimum: rows
 * of groups without a CTA-local slot are then applied with device atomics). */
int pac_agg_workspace_size(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, size_t* bytes);

/* Workspace bytes for pac_agg_grouped over n_rows rows with the deferred HBM tier: rows of
 * groups that miss a CTA-local slot (high-cardinality tables, e.g. BASELINE C3) are recorded
 * (28 B + 8 B per value column each) and folded per group after the pass instead of taking 64
 * device atomics each.  Equal to pac_agg_workspace_size when no row can miss (G_cap within
 * the local slot capacity, or MIN/MAX-only aggregates).  pac_agg_grouped uses whatever room
 * beyond the minimum ws_bytes offers (capacity ~ (ws_bytes - minimum) / record size rows);
 * rows beyond the capacity fall back to atomics, results identical.  Queries the device.
 * Sort-first path (high cardinality, DESIGN.md §5 "k_srt_*"): for COUNT / SUM / AVG tables with
 * G_cap >= 4096 whose packed key is at most 4 bytes, pac_agg_grouped instead radix-sorts the rows
 * by key when ws_bytes also holds two row buffers, 2 x (4 + 8 + 8 x value columns) bytes per
 * row; this function returns at least that.  With less workspace the tile kernels + deferred
 * tier run (identical integers; f64 sums differ only in summation order, R34). */
int pac_agg_workspace_size_rows(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, int64_t n_rows,
                                size_t* bytes);

/* Single-pass 64-world grouped aggregation (§5; PacCountUpdate P:L2254-2258
 * read with ">> j", R4).  For every row r with mask h_r != 0 in group g, and every
 * world j with bit j of h_r set:
 *   count[g][j] += 1; SUM: world[a][g][j] += v_r; AVG: world[a][g][j] += v_r;
 *   MIN/MAX: world[a][g][j] = min/max(world[a][g][j], v_r); rows[g] += 1; K[g] |= h_r.
 * Masks: exactly one of d_pu_key (hashed in-kernel with `salt`, = pac_mask) and d_mask
 * (explicit masks, e.g. pac_select-ed ones) is non-NULL.
 * keys: n_keys in 0..PAC_MAX_KEYS columns (n_keys = 0: one group, R21).
 * Limits: n_aggs <= PAC_MAX_AGGS; at most 2 distinct int64 SUM columns, 2 distinct f64
 * SUM/AVG columns and 1 f64 MIN/MAX column per call (else PAC_E_INVAL).
 * MIN/MAX-only calls take the pruned path: a row that cannot improve a
 * group's bound min_j MAX_j (resp. max_j MIN_j) is skipped without hashing.
 * Integer results are exact and order-independent; f64 sums are order-dependent in the
 * last bits (<= 1e-9 relative to the exact sum, R16).
 * Errors (synchronous): PAC_E_INVAL, PAC_E_WORKSPACE, PAC_E_CUDA.
 * Errors (asynchronous, in *d_status): PAC_E_CAPACITY, PAC_E_OVERFLOW. */
int pac_agg_grouped(const int64_t* d_pu_key, const uint64_t* d_mask, uint64_t salt,
                    const pac_key_col* keys, int n_keys, const pac_agg_spec* aggs, int n_aggs,
                    int64_t n_rows, const pac_table* out, int64_t G_cap, void* d_ws,
                    size_t ws_bytes, pac_stream_t stream);

/* Synchronizing check of a table: *h_num_groups and the status code (PAC_OK,
 * PAC_E_CAPACITY, PAC_E_OVERFLOW). */
int pac_table_check(const pac_table* t, int64_t* h_num_groups, pac_stream_t stream);

/* Re-derives K after a cross-GPU merge (NCCL has no bitwise-OR reduction, §8e):
 * K[g] bit j = (count[g][j] > 0) when d_count is present (R5, exact).  MIN/MAX-only tables
 * have no counts and a world holding only +inf (MIN) / -inf (MAX) looks empty in the f64
 * table, so there the caller must merge d_presence itself (OR across ranks) and this call
 * only ORs in the worlds whose MIN is not +inf or MAX is not -inf (it never clears a bit).
 * Uses the device-side num_groups. */
int pac_table_rederive_presence(const pac_table* t, const pac_agg_spec* aggs, int n_aggs,
                                int64_t G_cap, pac_stream_t stream);

/* Scatters table `in` (G_in groups, keys a subset of d_union_keys) into table `out`
 * laid out by the ascending union dictionary d_union_keys[G_union]; groups absent from
 * `in` get the empty state (count 0, sums 0, MIN +inf, MAX -inf, rows 0, K 0).  Used so
 * that all ranks share one layout before the allreduce.  `in`'s num_groups is read
 * from the device and clamped to G_cap_in; `out`'s status is `in`'s. */
int pac_table_remap(const pac_table* in, const uint64_t* d_union_keys, int64_t G_union,
                    const pac_agg_spec* aggs, int n_aggs, int64_t G_cap_in,
                    const pac_table* out, pac_stream_t stream);

/* ------------------------------------------------------------------ cross-GPU merge (§8 a5/e)
 * The combine of row-sharded partial tables (P:L1777, P:L1966, P:L2010 thread-local states +
 * combine) as three NCCL all_reduce calls over flat buffers, with no host synchronisation.
 * Every rank's table must be laid out on one group dictionary (pac_table_remap onto the sorted
 * union, or identical dense domains); a fingerprint of the dictionary travels with the data
 * and a mismatch is detected on the device.  Buffers (caller-allocated device memory, element
 * counts from pac_merge_sizes; G = G_cap, fixed, so no num_groups read on the host):
 *   d_i64_sum [n_i64_sum] int64  all_reduce SUM: rows [G], count [G][64] (if the table has
 *                                counts), per SUM_I64 aggregate [G][64]
 *   d_f64_sum [n_f64_sum] double all_reduce SUM: per SUM_F64 / AVG_F64 aggregate [G][64]
 *                                (may be NULL when n_f64_sum == 0)
 *   d_i64_min [n_i64_min] int64  all_reduce MIN: dictionary fingerprint f and ~f, ~status,
 *                                per MIN aggregate [G][64] order-preserving encodings of the
 *                                extremes (R31, NaN largest), per MAX aggregate [G][64] their
 *                                bitwise NOT; a world not in K packs the empty sentinel.
 * pac_merge_unpack writes the merged rows, counts, worlds and K back into the table: K =
 * {count > 0} (R5) or, for MIN/MAX-only tables, the worlds whose merged extreme is not the
 * sentinel (the OR of the ranks' K, exact even for worlds holding only +inf / -inf); d_status
 * = the largest status of any rank, or PAC_E_MERGE when the fingerprints differ.  The int64
 * sums wrap like any int64 addition (R15 precondition: |world sum| < 2^63 globally).
 * Errors: PAC_E_INVAL (bad sizes / pointers, m != 64), PAC_E_CUDA. */
int pac_merge_sizes(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, int64_t* n_i64_sum,
                    int64_t* n_f64_sum, int64_t* n_i64_min);
int pac_merge_pack(const pac_table* t, const pac_agg_spec* aggs, int n_aggs, int64_t G_cap,
                   int64_t* d_i64_sum, double* d_f64_sum, int64_t* d_i64_min, pac_stream_t stream);
int pac_merge_unpack(const pac_table* t, const pac_agg_spec* aggs, int n_aggs, int64_t G_cap,
                     const int64_t* d_i64_sum, const double* d_f64_sum, const int64_t* d_i64_min,
                     pac_stream_t stream);

/* ------------------------------------------------------------------ m = 128 worlds (§8 f4)
 * P:L92 (§2): "Extending to m=128 is possible, and worst-case would double the cost".
 * Readings R28 (hash), R29 (aggregation, finalize).  A 128-world mask is two words
 * [n][2] = {lo: worlds 0..63, hi: worlds 64..127}, exactly 64 bits set when hashed. */
int pac_mask128(const int64_t* d_pu_key, int64_t n, uint64_t salt, uint64_t* d_mask2, pac_stream_t stream);
/* Workspace bytes of pac_agg_grouped128 (hashing != 0: masks computed from pu keys). */
int pac_agg_workspace_size128(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, int64_t n_rows, int hashing,
                              size_t* bytes);
/* Grouped aggregation over 128 worlds into an m = 128 table (out->m == 128: d_presence
 * [G_cap][2], d_count and d_world[a] [G_cap][128]).  Same semantics as pac_agg_grouped with
 * 128 worlds; a row is dropped only when both mask words are 0 (R21).  Implemented as the
 * 64-world kernels over the two mask halves plus a group/row-count pass, merged on device.
 * Errors: as pac_agg_grouped. */
int pac_agg_grouped128(const int64_t* d_pu_key, const uint64_t* d_mask2, uint64_t salt, const pac_key_col* keys,
                       int n_keys, const pac_agg_spec* aggs, int n_aggs, int64_t n_rows, const pac_table* out,
                       int64_t G_cap, void* d_ws, size_t ws_bytes, pac_stream_t stream);

/* ------------------------------------------------------------------ finalize (§8 a6-a7)
 * The fused pac_noised step (§2; §4) over every cell of a table
 * (m = 64, or m = 128 with an m = 128 session: NULL iff (x0 >> 25) >= popcount(K), R29),
 * cells in canonical order g*n_aggs + a (R12); one call = one round `round`.
 * Per cell (Philox4x32-10 key = session seed, counter = (cell_lo, cell_hi, round, 0)):
 *   NULL iff (x0 >> 26) >= popcount(K[g])                              (R10)
 *   y_j = 2*count_j | 2*sum_j | fsum_j/count_j | ext_j for K bit j set, else 0 (R7, R9)
 *   s2 = Var_{j~P}[y]; Delta = s2/(2B)                                  (R8)
 *   s2 == 0 (all y_j with P_j > 0 equal): release y_{j*}, no update     (R11)
 *   else release = y_{j*} + sqrt(Delta)*z, z Box-Muller of (x1,x2,x3)   (R13)
 *        P <- P*W/sum(P*W), W_j = exp(-(d_j - min d)/(2 Delta))         (R14)
 * Outputs (caller-allocated, [G_cap][n_aggs] unless noted):
 *   d_release (NaN for NULL cells), d_is_null (0/1), d_flags [G_cap] bit 0 = diversity
 *   check (rows >= 64 and popcount K <= 34, R18), bit 1 = the table's
 *   d_status was nonzero (CAPACITY / OVERFLOW: then every cell is NULL and P is left
 *   unchanged -- nothing is released from an invalid table), d_delta (optional, may be
 *   NULL; NaN for NULL cells).
 * SURVEY §8(b) lists PAC_E_SUSPICIOUS as a return code for a diversity-flagged group; the
 * call is asynchronous (the flags exist only on the device when it returns), so the
 * diversity check is reported in d_flags bit 0 instead and never aborts (R18).
 * The session posterior is updated in place on the device, in cell order.
 * Errors: PAC_E_INVAL, PAC_E_WORKSPACE, PAC_E_CUDA. */
int pac_finalize_workspace_size(int64_t G_cap, int n_aggs, size_t* bytes);
int pac_finalize(pac_session* s, const pac_table* t, const pac_agg_spec* aggs, int n_aggs,
                 int64_t G_cap, uint32_t round, double* d_release, uint8_t* d_is_null,
                 uint8_t* d_flags, double* d_delta, void* d_ws, size_t ws_bytes,
                 pac_stream_t stream);

/* Standalone Bayesian posterior update: with y = d_y64[64] (device),
 *   P <- P*W/sum(P*W), W_j = exp(-((y_tilde - y_j)^2 - min_i d_i)/(2 delta)) over P_j > 0.
 * delta must be > 0 and finite (else PAC_E_INVAL). */
int pac_posterior_update(pac_session* s, const double* d_y64, double y_tilde, double delta,
                         pac_stream_t stream);

/* ------------------------------------------------------------------ categorical path (§8 f1)
 * After the aggregate (§3, §4; R22-R26).
 * A world vector is y[64] (double, released scale, absent worlds 0) plus a presence mask
 * (uint64, bit j = world j present).  Arrays of n vectors are [n][64] doubles + [n]
 * presences.  A pac_wvec operand with d_y == NULL is the broadcast scalar `scalar`
 * (present in every world). */
typedef enum {
  PAC_OP_ADD = 0, PAC_OP_SUB = 1, PAC_OP_MUL = 2, PAC_OP_DIV = 3, PAC_OP_MIN = 4, PAC_OP_MAX = 5
} pac_lift_op;
typedef enum { PAC_CMP_LT = 0, PAC_CMP_LE = 1, PAC_CMP_GT = 2, PAC_CMP_GE = 3, PAC_CMP_EQ = 4 } pac_cmp_kind;
typedef struct {
  const double* d_y;          /* [n][64], or NULL for a scalar */
  const uint64_t* d_presence; /* [n]; required iff d_y != NULL */
  double scalar;
} pac_wvec;
#define PAC_CMP_INDEX_WORDS 130 /* per group: 64 sorted doubles, 65 suffix masks, count */

/* R22: world vector of aggregate a of every group of table t (the y-vector pac_finalize
 * noises: 2*count | 2*sum | fsum/count | ext, absent worlds 0) into d_y [G_cap][64], and
 * its presence K into d_presence [G_cap].  Rows >= num_groups get zeros / presence 0. */
int pac_world_vector(const pac_table* t, const pac_agg_spec* aggs, int n_aggs, int a, int64_t G_cap,
                     double* d_y, uint64_t* d_presence, pac_stream_t stream);
/* R23 (Eq. vectorexpressionlambda): d_out[i][j] = a_ij OP b_ij where both
 * operands are present, else 0; d_presence_out[i] = presence(a) AND presence(b). */
int pac_lift(int op, const pac_wvec* a, const pac_wvec* b, int64_t n, double* d_out,
             uint64_t* d_presence_out, pac_stream_t stream);
/* Lifted comparison: d_bits[i] bit j = present_j and (a_ij CMP b_ij) (R23, R26). */
int pac_lift_cmp(int cmp, const pac_wvec* a, const pac_wvec* b, int64_t n, uint64_t* d_bits,
                 pac_stream_t stream);
/* R24: pac_noised of n given world vectors, cells in index order i, Philox counter
 * (i_lo, i_hi, round, 3): NULL with probability (64 - popcount(presence))/64, y already in
 * the released scale (no *2), then the pac_finalize steps (variance under P, release,
 * Bayesian update of the session posterior).  d_delta may be NULL. */
int pac_noised_y_workspace_size(int64_t n, size_t* bytes);
int pac_noised_y(pac_session* s, const double* d_y, const uint64_t* d_presence, int64_t n, uint32_t round,
                 double* d_release, uint8_t* d_is_null, double* d_delta, void* d_ws, size_t ws_bytes,
                 pac_stream_t stream);
/* Comparison index of G world vectors (d_c [G][64], d_presence [G]) for the fused
 * row-parallel comparisons below: d_index [G][PAC_CMP_INDEX_WORDS] (caller-allocated). */
int pac_cmp_index(const double* d_c, const uint64_t* d_presence, int64_t G, uint64_t* d_index,
                  pac_stream_t stream);
/* pac_select (Eq. pac-select): d_out[i] = d_h[i] AND d_bits[d_gidx[i]] -- the reduced
 * mask of row i for an upstream PAC aggregate (pass it as pac_agg_grouped's d_mask). */
int pac_select(const uint64_t* d_h, const int32_t* d_gidx, const uint64_t* d_bits, int64_t n,
               uint64_t* d_out, pac_stream_t stream);
/* pac_select_<cmp>: d_out[i] = d_h[i] AND b, b_j = present_j and
 * (d_v[i] CMP c_j), c = the world vector of group d_gidx[i] in the comparison index. */
int pac_select_cmp(int cmp, const uint64_t* d_h, const double* d_v, const int32_t* d_gidx,
                   const uint64_t* d_index, int64_t n, uint64_t* d_out, pac_stream_t stream);
/* pac_filter (Eq. pac-filter; R25): d_out[i] = 1 with probability
 * popcount(d_bits[i])/64: r = x0 >> 26 of Philox(session seed; i_lo, i_hi, round, 4),
 * true iff r < popcount. */
int pac_filter(pac_session* s, const uint64_t* d_bits, int64_t n, uint32_t round, uint8_t* d_out,
               pac_stream_t stream);
/* pac_filter_<cmp>: pac_filter of the pac_select_cmp booleans. */
int pac_filter_cmp(pac_session* s, int cmp, const double* d_v, const int32_t* d_gidx, const uint64_t* d_index,
                   int64_t n, uint32_t round, uint8_t* d_out, pac_stream_t stream);

/* ------------------------------------------------------------------ PU-key join (§8 f2)
 * P:L331-357 §3 (Eq. join-addition, Eq. join-elim), §2; reading R27.  A build
 * table maps a primary key to the tuple's next foreign key along the chain
 * T -fk1-> T1 -> ... -> Tk -fkU-> U (e.g. orders: o_orderkey -> o_custkey).  The table is a
 * caller-allocated device buffer of pac_join_table_bytes(n_build) bytes (16-byte aligned):
 * open addressing, load factor <= 1/2, 16-byte {key, next} slots. */
#define PAC_JOIN_MAX_CHAIN 4
int pac_join_table_bytes(int64_t n_build, size_t* bytes);
/* Builds the table from d_pk[n_build] -> d_next[n_build].  A duplicate primary key is
 * recorded in the table status (PAC_E_INVAL) -- see pac_join_table_status. */
int pac_join_build(const int64_t* d_pk, const int64_t* d_next, int64_t n_build, void* d_table,
                   size_t table_bytes, pac_stream_t stream);
/* Synchronizing: PAC_OK, or PAC_E_INVAL if the build saw a duplicate primary key. */
int pac_join_table_status(const void* d_table, pac_stream_t stream);
/* Per row i: x = d_fk[i]; for t = 0..k-1: x = next of x in table t (k <= PAC_JOIN_MAX_CHAIN;
 * d_tables is a HOST array of k device table pointers).  Join elimination (Eq. join-elim):
 * the final x is the PU key; d_mask[i] = pac_hash(x, salt) (R1, R2), or 0 when some lookup
 * finds no match (R27: no PU -> in no world; pac_agg_grouped drops the row, R21).  Either
 * output may be NULL (d_pu_key[i] = x, or 0 without a match).  0 is also a valid PU key, so
 * d_pu_key cannot mark an unmatched row: aggregate joined rows through d_mask (passed as
 * pac_agg_grouped's d_mask, which drops the unmatched rows), never by feeding d_pu_key back
 * as pac_agg_grouped's d_pu_key when some row may be unmatched. */
int pac_join_mask(const void* const* d_tables, int k, const int64_t* d_fk, int64_t n, uint64_t salt,
                  uint64_t* d_mask, int64_t* d_pu_key, pac_stream_t stream);

/* ------------------------------------------------------------------ approximate SUM (§8 f3)
 * P:L1783-1803 (§5 "Approximation", "Two-sided SUM"); readings R35 (two-sided), R36 (single-
 * sided).  Ungrouped 64-world SUM of an int64 column with the paper's approximate state: per
 * world and side 25 levels of 16-bit counters, level k of weight 2^(4k); a value v != 0 of a row
 * in world j goes to side pos (v > 0) or neg (stored negated), is routed to level
 * l = floor((msb(|v|) - 8) / 4) (0 below 2^8) and adds |v| >> 4l; on overflow the counter's upper
 * 12 bits cascade into the next level (C[k+1] += C[k] >> 4) and its low 4 bits are dropped.
 * two_sided == 0: Table 1's "Single Sum" (R36): one state fed the value's 64-bit two's-complement
 * pattern (routed by its msb), decoded modulo 2^64 as a signed int64.  Order (R35): rows in row order inside blocks of block_rows rows, block states
 * combined in block order -- the result is a deterministic function of (rows, block_rows).
 * Masks: exactly one of d_pu_key (hashed with salt, = pac_mask) and d_mask.
 * Outputs: d_counters [2][64][25] uint16 (side, world, level; single-sided: side 1 zeros);
 * d_y [64] = 2 * (dec(pos) - dec(neg)) (R7; single-sided 2 * (int64)(dec mod 2^64)),
 * dec(C) = sum_k C[k] 2^(4k) in double.  Workspace: pac_approx_sum_workspace_size bytes.
 * Errors: PAC_E_INVAL, PAC_E_WORKSPACE, PAC_E_CUDA. */
int pac_approx_sum_workspace_size(int64_t n_rows, int64_t block_rows, size_t* bytes);
int pac_approx_sum(const int64_t* d_pu_key, const uint64_t* d_mask, uint64_t salt, const int64_t* d_values,
                   int64_t n_rows, int32_t two_sided, int64_t block_rows, uint16_t* d_counters, double* d_y,
                   void* d_ws, size_t ws_bytes, pac_stream_t stream);

/* ------------------------------------------------------------------ runtime / profiling
 * Number of kernels this library has launched since load (all entry points). */
uint64_t pac_launch_count(void);
/* When enabled, pac_agg_grouped brackets its aggregation pass (the main kernel, plus the
 * deferred HBM tier's kernels when they run) with CUDA events on `stream` and accumulates the elapsed time; pac_profile_read synchronizes on the
 * recorded events and returns (total ms, number of timed launches), then resets. */
int pac_profile_enable(int on);
int pac_profile_read(double* h_total_ms, int64_t* h_launches);
/* Name of the kernel(s) of the last timed region (e.g. "k_agg_tiles_tm<1,1,0>"; the deferred
 * HBM tier's kernels are inside the region when they ran).  Owned by the library. */
const char* pac_profile_last_kernel(void);
/* Library version string. */
const char* pac_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PAC_H_ */
