/*
 * oracle/pac_oracle.c -- CPU ORACLE for the PAC stochastic-aggregation hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or execute anything under
 * oracle/.  The product path (paper_2603_15023_b200/, libpac.so) never does, and
 * this file shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C in fp64, written from PAPER.md
 * (arxiv 2603.15023, "SIMD-PAC-DB") and the readings frozen in DESIGN.md
 * ("Readings of the paper", R1..R19).  Every function cites the passage it follows
 * as P:L<line> (<section>).  No blocking, fusion or reordering beyond what the
 * definition states.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"):
 *   philox4x32_10   Random123 known-answer vectors (SC'11 generator)        pinned
 *   fmix64          SplitMix64 reference output for seed 0                   pinned
 *   pac_hash        popcount==32 on every key, fixed point, per-bit / pair
 *                   statistics of a uniform balanced word; the exact flip
 *                   selection (draw stream) has no external pin:
 *                   "parity unpinned" beyond those properties  partial
 *   agg_o1/agg_o2   pandas GROUP BY on each world's filtered rows (Eq. counter
 *                   P:L249-253 / P:L956-970 as a library routine), all-ones masks
 *                   -> plain GROUP BY, sum_j count_j == 32*rows, K == {j:count>0}  pinned
 *   finalize        closed forms (single-PU group, y_j=j, constant y), NULL rate,
 *                   noise std, numpy weighted variance, scipy Gaussian Bayes     pinned
 *   posterior       scipy.stats.norm likelihood Bayes update                    pinned
 *   categorical     (R22-R26) cmp bits == numpy comparisons, select truth table,
 *   path            filter rates popcount/64 (binomial), lift identities,
 *                   noised_y closed forms, noise-once beats noise-twice pinned
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_M 64 /* m = 64 worlds, P:L92 (§2) */

/* ------------------------------------------------------------------ Philox4x32-10
 * DESIGN.md R13 (the paper is silent on the RNG).  Salmon, Moraes, Dror, Shaw,
 * "Parallel random numbers: as easy as 1, 2, 3" (SC'11): round function
 *   (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0)),
 * key bumped by the Weyl constants between rounds, 10 rounds. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; r++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Philox block for (seed, counter words).  seed is the 64-bit session seed (key). */
static void philox_block(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                         uint32_t out[4]) {
  uint32_t ctr[4] = {c0, c1, c2, c3};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  orc_philox4x32_10(ctr, key, out);
}

enum { TAG_CELL = 0, TAG_JSTAR = 1, TAG_SALT = 2, TAG_LIFT = 3, TAG_FILTER = 4 }; /* R13, R24, R25 */

/* ------------------------------------------------------------------ fmix64
 * DESIGN.md R1: the base hash the paper wraps ("We wrap DuckDB's hash function",
 * P:L93 §2) is read as the SplitMix64 finalizer (Stafford Mix13 constants). */
uint64_t orc_fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

static int popcount64(uint64_t x) {
  int c = 0;
  for (int j = 0; j < 64; j++) c += (int)((x >> j) & 1u);
  return c;
}

/* ------------------------------------------------------------------ pac_hash
 * P:L93 (§2): pac_hash re-hashes per query with a salt and "cheaply transform[s]
 * the binomially distributed hash number in a random hash that is guaranteed to
 * have 32 0- and 32 1-bits"; P:L949-952 (§4): keyed hash, per-query key K;
 * `\iffalse` P:L1651: effective hash pac_hash(h(u) XOR q).
 * DESIGN.md R1 (mix) + R2 (balancing, "rejection flips"):
 *   x = fmix64(key XOR salt); c = popcount(x); if c == 32 -> x.
 *   maj = (c > 32); k = |c - 32|.
 *   w_0 = fmix64(x XOR 0xD1B54A32D192ED03); w_{i+1} = fmix64(w_i + 0x9E3779B97F4A7C15).
 *   Each word gives 10 draws p = (w >> 6t) & 63, t = 0..9 (top 4 bits unused).
 *   For each draw: if bit p of the current x equals maj, flip it and k--; stop at k = 0.
 *   Safety net (never reached in practice): after 64 words, flip the remaining k
 *   majority bits from the lowest position upward. */
uint64_t orc_pac_hash(int64_t key, uint64_t salt) {
  uint64_t x = orc_fmix64((uint64_t)key ^ salt);
  int c = popcount64(x);
  if (c == 32) return x;
  uint64_t maj = (c > 32) ? 1u : 0u;
  int k = (c > 32) ? (c - 32) : (32 - c);
  uint64_t w = orc_fmix64(x ^ 0xD1B54A32D192ED03ull);
  for (int word = 0; word < 64; word++) {
    for (int t = 0; t < 10; t++) {
      int p = (int)((w >> (6 * t)) & 63u);
      if (((x >> p) & 1u) == maj) {
        x ^= (1ull << p);
        k--;
        if (k == 0) return x;
      }
    }
    w = orc_fmix64(w + 0x9E3779B97F4A7C15ull);
  }
  for (int p = 0; p < 64 && k > 0; p++) {
    if (((x >> p) & 1u) == maj) {
      x ^= (1ull << p);
      k--;
    }
  }
  return x;
}

void orc_pac_hash_n(const int64_t* keys, int64_t n, uint64_t salt, uint64_t* out) {
  for (int64_t i = 0; i < n; i++) out[i] = orc_pac_hash(keys[i], salt);
}

/* ------------------------------------------------------------------ session
 * P:L886 (§4): "sample a secret world index uniformly at random j* <- {1..m},
 * initialize ... P = (1/m, ..., 1/m)"; P:L99 (§2): one j* per query shared by all
 * cells; P:L93 / P:L950: a fresh per-query hash key (salt).
 * DESIGN.md R13: j* = x0 & 63 of Philox(seed; 0,0,0,TAG_JSTAR);
 *                salt = x0 | x1<<32 of Philox(seed; 0,0,0,TAG_SALT). */
void orc_session_init(uint64_t seed, int* jstar, uint64_t* salt, double* P) {
  uint32_t o[4];
  philox_block(seed, 0, 0, 0, TAG_JSTAR, o);
  *jstar = (int)(o[0] & 63u);
  philox_block(seed, 0, 0, 0, TAG_SALT, o);
  *salt = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
  for (int j = 0; j < ORC_M; j++) P[j] = 1.0 / ORC_M;
}

/* ------------------------------------------------------------------ group keys
 * DESIGN.md R20: composite group key = concatenation (first column most
 * significant) of each column's bits with the sign bit flipped, so unsigned order
 * of the packed key == lexicographic order of the signed column values. */
uint64_t orc_pack_key(const void* const* cols, const int32_t* elem_bytes, int n_keys, int64_t row) {
  uint64_t packed = 0;
  for (int c = 0; c < n_keys; c++) {
    int w = elem_bytes[c];
    uint64_t v;
    if (w == 1) v = (uint64_t)(uint8_t)((const int8_t*)cols[c])[row];
    else if (w == 2) v = (uint64_t)(uint16_t)((const int16_t*)cols[c])[row];
    else if (w == 4) v = (uint64_t)(uint32_t)((const int32_t*)cols[c])[row];
    else v = (uint64_t)((const int64_t*)cols[c])[row];
    v ^= 1ull << (8 * w - 1);
    packed = (w == 8) ? v : ((packed << (8 * w)) | v);
  }
  return packed;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* Distinct packed keys (ascending) of rows with a nonzero mask.  DESIGN.md R21:
 * rows whose world mask is 0 belong to no world ("we filter out rows where
 * this updated pu=0") and create no group.  With n_keys == 0 (ungrouped) there is
 * always exactly one group, key 0 (SQL: an ungrouped aggregate returns one row).
 * Returns G; writes min(G, cap) keys. */
int64_t orc_group_keys(const void* const* cols, const int32_t* elem_bytes, int n_keys,
                       const uint64_t* masks, int64_t n, uint64_t* out, int64_t cap) {
  if (n_keys == 0) {
    if (cap > 0) out[0] = 0;
    return 1;
  }
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < n; i++)
    if (masks[i] != 0) tmp[m++] = orc_pack_key(cols, elem_bytes, n_keys, i);
  qsort(tmp, (size_t)m, sizeof(uint64_t), cmp_u64);
  int64_t g = 0;
  for (int64_t i = 0; i < m; i++) {
    if (i == 0 || tmp[i] != tmp[i - 1]) {
      if (g < cap) out[g] = tmp[i];
      g++;
    }
  }
  free(tmp);
  return g;
}

static int64_t find_group(const uint64_t* gkeys, int64_t G, uint64_t key) {
  int64_t lo = 0, hi = G;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (gkeys[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < G && gkeys[lo] == key) ? lo : -1;
}

/* ------------------------------------------------------------------ aggregation
 * Aggregate kinds (agg in {sum, count, avg, min, max}). */
enum { K_COUNT = 0, K_SUM_I64 = 1, K_SUM_F64 = 2, K_AVG_F64 = 3, K_MIN_F64 = 4, K_MAX_F64 = 5 };

/* Neumaier-compensated running sum (oracle-side accuracy only; the definition is
 * the exact sum).  DESIGN.md R30 (non-finite terms): the IEEE-754 sum -- any NaN
 * term gives NaN, +inf and -inf together give NaN, otherwise an infinite term gives
 * that infinity.  Once a term or the running sum is non-finite the compensation is
 * dropped and the plain IEEE addition continues (the compensation of finite terms
 * would otherwise turn inf into inf - inf = NaN). */
typedef struct { double s, c; } csum;
static void csum_add(csum* a, double v) {
  if (!isfinite(v) || !isfinite(a->s)) { a->s += v; return; }
  double t = a->s + v;
  if (!isfinite(t)) { a->s = t; return; }  /* finite overflow: out of contract (R30) */
  if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v; else a->c += (v - t) + a->s;
  a->s = t;
}
static double csum_value(const csum* a) { return isfinite(a->s) ? a->s + a->c : a->s; }

/* DESIGN.md R31: MIN/MAX order doubles by DuckDB's total order (the paper's host system,
 * P:L1966; r_j = agg({...}) P:L957-970 with agg = the DBMS's min/max): NaN is larger than
 * every other value (+inf included) and all NaNs are equal; otherwise IEEE order.
 * tot_less(a, b) is a < b in that order. */
static int tot_less(double a, double b) {
  if (isnan(a)) return 0;
  if (isnan(b)) return 1;
  return a < b;
}

/* Output table, canonical group order (ascending packed key = gkeys):
 *   rows[G]              rows with nonzero mask in the group (int64)
 *   K[G]                 OR of the row masks ("K <- K | h")
 *   count[G*64]          per-world row count (int64), P:L87 / P:L2255
 *   world[a][G*64]       per aggregate a: int64 (SUM_I64) or double (others);
 *                        SUM_F64/AVG_F64 hold the world's value sum (AVG divides at
 *                        finalize, R6); MIN/MAX hold the extreme, +inf / -inf when
 *                        the world is empty.
 * Returns 0, or 1 if some int64 world sum overflowed (checked with __int128, R15). */
static void init_world(int kind, void* w, int64_t G) {
  for (int64_t i = 0; i < G * ORC_M; i++) {
    if (kind == K_SUM_I64) ((int64_t*)w)[i] = 0;
    else if (kind == K_MIN_F64) ((double*)w)[i] = INFINITY;
    else if (kind == K_MAX_F64) ((double*)w)[i] = -INFINITY;
    else if (kind != K_COUNT) ((double*)w)[i] = 0.0;
  }
}

/* O2: single pass.  For every row, for j = 0..63, update world j iff bit j of the
 * row's mask is set -- PacCountUpdate P:L2254-2258 (read with ">> j", R4)
 * generalised to SUM/AVG/MIN/MAX per §5 P:L1737 ("the value at position j
 * accumulates contributions from those rows whose key_hash has bit j set"). */
int orc_agg_o2(const uint64_t* masks, int64_t n, const void* const* cols, const int32_t* elem_bytes,
               int n_keys, const uint64_t* gkeys, int64_t G, const int32_t* kinds,
               const void* const* values, int n_aggs, int64_t* rows, uint64_t* K, int64_t* count,
               void* const* world) {
  int overflow = 0;
  for (int64_t g = 0; g < G; g++) { rows[g] = 0; K[g] = 0; }
  for (int64_t i = 0; i < G * ORC_M; i++) count[i] = 0;
  for (int a = 0; a < n_aggs; a++) if (world[a]) init_world(kinds[a], world[a], G);
  __int128* isum = (__int128*)calloc((size_t)(G * ORC_M * n_aggs + 1), sizeof(__int128));
  csum* fsum = (csum*)calloc((size_t)(G * ORC_M * n_aggs + 1), sizeof(csum));
  for (int64_t r = 0; r < n; r++) {
    uint64_t h = masks[r];
    if (h == 0) continue;
    uint64_t key = n_keys ? orc_pack_key(cols, elem_bytes, n_keys, r) : 0;
    int64_t g = find_group(gkeys, G, key);
    if (g < 0) continue;
    rows[g] += 1;
    K[g] |= h;
    for (int j = 0; j < ORC_M; j++) {
      if (((h >> j) & 1u) == 0) continue;
      int64_t cell = g * ORC_M + j;
      count[cell] += 1;
      for (int a = 0; a < n_aggs; a++) {
        int64_t idx = ((int64_t)a * G) * ORC_M + cell;
        switch (kinds[a]) {
          case K_SUM_I64: isum[idx] += (__int128)((const int64_t*)values[a])[r]; break;
          case K_SUM_F64:
          case K_AVG_F64: csum_add(&fsum[idx], ((const double*)values[a])[r]); break;
          case K_MIN_F64: {
            double v = ((const double*)values[a])[r];
            double* e = &((double*)world[a])[cell];
            if (count[cell] == 1 || tot_less(v, *e)) *e = v;
            break;
          }
          case K_MAX_F64: {
            double v = ((const double*)values[a])[r];
            double* e = &((double*)world[a])[cell];
            if (count[cell] == 1 || tot_less(*e, v)) *e = v;
            break;
          }
          default: break;
        }
      }
    }
  }
  for (int a = 0; a < n_aggs; a++) {
    for (int64_t cell = 0; cell < G * ORC_M; cell++) {
      int64_t idx = ((int64_t)a * G) * ORC_M + cell;
      if (kinds[a] == K_SUM_I64) {
        __int128 s = isum[idx];
        if (s > (__int128)INT64_MAX || s < (__int128)INT64_MIN) overflow = 1;
        ((int64_t*)world[a])[cell] = (int64_t)s;
      } else if (kinds[a] == K_SUM_F64 || kinds[a] == K_AVG_F64) {
        ((double*)world[a])[cell] = csum_value(&fsum[idx]);
      }
    }
  }
  free(isum);
  free(fsum);
  return overflow;
}

/* combine: state.combine(other) of two partial tables over the same groups ("thread-
 * local" states, P:L2010 combine; O2 "merge per-thread states in thread order"):
 * a <- a (+) b.  rows, counts and int64 sums add (returns 1 when an int64 world sum leaves the
 * int64 range, checked with __int128 -- exact when neither partial overflowed), K ORs, f64 sums
 * add (IEEE, R30), MIN/MAX keep the total-order extreme (R31) of the worlds non-empty in a or b
 * (emptiness from the counts).  Used only to time O2 on several host threads (bench.py's CPU
 * leg); the parity tests use the single-pass O2. */
int orc_combine(int64_t G, const int32_t* kinds, int n_aggs, int64_t* rows_a, uint64_t* K_a,
                int64_t* count_a, void* const* world_a, const int64_t* rows_b, const uint64_t* K_b,
                const int64_t* count_b, void* const* world_b) {
  int overflow = 0;
  for (int64_t g = 0; g < G; g++) { rows_a[g] += rows_b[g]; K_a[g] |= K_b[g]; }
  for (int a = 0; a < n_aggs; a++) {
    if (!world_a[a]) continue;
    for (int64_t cell = 0; cell < G * ORC_M; cell++) {
      switch (kinds[a]) {
        case K_SUM_I64: {
          __int128 s = (__int128)((int64_t*)world_a[a])[cell] + ((const int64_t*)world_b[a])[cell];
          if (s > (__int128)INT64_MAX || s < (__int128)INT64_MIN) overflow = 1;
          ((int64_t*)world_a[a])[cell] = (int64_t)s;
          break;
        }
        case K_SUM_F64:
        case K_AVG_F64: ((double*)world_a[a])[cell] += ((const double*)world_b[a])[cell]; break;
        case K_MIN_F64: {
          double vb = ((const double*)world_b[a])[cell];
          double* e = &((double*)world_a[a])[cell];
          if (count_b[cell] > 0 && (count_a[cell] == 0 || tot_less(vb, *e))) *e = vb;
          break;
        }
        case K_MAX_F64: {
          double vb = ((const double*)world_b[a])[cell];
          double* e = &((double*)world_a[a])[cell];
          if (count_b[cell] > 0 && (count_a[cell] == 0 || tot_less(*e, vb))) *e = vb;
          break;
        }
        default: break;
      }
    }
  }
  for (int64_t cell = 0; cell < G * ORC_M; cell++) count_a[cell] += count_b[cell];
  return overflow;
}

/* O1: the PAC-DB m-fold semantics with hash-coupled worlds (§4, coupled
 * per P:L1028-1030): for each world j, the sampled instance I^(j) is the rows whose
 * mask has bit j set; run the plain GROUP BY on it; then List the 64
 * per-world results per group.  Groups absent from world j keep count 0
 * and the empty-aggregate sentinels (NULL mechanism P:L1654, R9). */
int orc_agg_o1(const uint64_t* masks, int64_t n, const void* const* cols, const int32_t* elem_bytes,
               int n_keys, const uint64_t* gkeys, int64_t G, const int32_t* kinds,
               const void* const* values, int n_aggs, int64_t* rows, uint64_t* K, int64_t* count,
               void* const* world) {
  int overflow = 0;
  int64_t* gid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t r = 0; r < n; r++) {
    uint64_t key = n_keys ? orc_pack_key(cols, elem_bytes, n_keys, r) : 0;
    gid[r] = masks[r] ? find_group(gkeys, G, key) : -1;
  }
  for (int64_t g = 0; g < G; g++) { rows[g] = 0; K[g] = 0; }
  for (int64_t r = 0; r < n; r++)
    if (gid[r] >= 0) { rows[gid[r]] += 1; K[gid[r]] |= masks[r]; }
  for (int a = 0; a < n_aggs; a++) if (world[a]) init_world(kinds[a], world[a], G);
  /* per-world plain GROUP BY state */
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(G + 1));
  __int128* is = (__int128*)malloc(sizeof(__int128) * (size_t)(G + 1));
  csum* fs = (csum*)malloc(sizeof(csum) * (size_t)(G + 1));
  double* ex = (double*)malloc(sizeof(double) * (size_t)(G + 1));
  char* seen = (char*)malloc((size_t)(G + 1));
  for (int j = 0; j < ORC_M; j++) {
    /* COUNT(*) over I^(j) */
    for (int64_t g = 0; g < G; g++) cnt[g] = 0;
    for (int64_t r = 0; r < n; r++)
      if (gid[r] >= 0 && ((masks[r] >> j) & 1u)) cnt[gid[r]] += 1;
    for (int64_t g = 0; g < G; g++) count[g * ORC_M + j] = cnt[g];
    for (int a = 0; a < n_aggs; a++) {
      int kind = kinds[a];
      if (kind == K_COUNT) continue;
      for (int64_t g = 0; g < G; g++) {
        is[g] = 0; fs[g].s = 0; fs[g].c = 0;
        ex[g] = (kind == K_MIN_F64) ? INFINITY : -INFINITY;
        seen[g] = 0;
      }
      for (int64_t r = 0; r < n; r++) {
        if (gid[r] < 0 || !((masks[r] >> j) & 1u)) continue;
        int64_t g = gid[r];
        if (kind == K_SUM_I64) is[g] += (__int128)((const int64_t*)values[a])[r];
        else if (kind == K_SUM_F64 || kind == K_AVG_F64) csum_add(&fs[g], ((const double*)values[a])[r]);
        else if (kind == K_MIN_F64) {  /* R31: the world's first value, then the total-order min */
          double v = ((const double*)values[a])[r];
          if (!seen[g] || tot_less(v, ex[g])) ex[g] = v;
          seen[g] = 1;
        } else if (kind == K_MAX_F64) {
          double v = ((const double*)values[a])[r];
          if (!seen[g] || tot_less(ex[g], v)) ex[g] = v;
          seen[g] = 1;
        }
      }
      for (int64_t g = 0; g < G; g++) {
        int64_t cell = g * ORC_M + j;
        if (kind == K_SUM_I64) {
          if (is[g] > (__int128)INT64_MAX || is[g] < (__int128)INT64_MIN) overflow = 1;
          ((int64_t*)world[a])[cell] = (int64_t)is[g];
        } else if (kind == K_SUM_F64 || kind == K_AVG_F64) {
          ((double*)world[a])[cell] = csum_value(&fs[g]);
        } else {
          ((double*)world[a])[cell] = ex[g];
        }
      }
    }
  }
  free(gid); free(cnt); free(is); free(fs); free(ex); free(seen);
  return overflow;
}

/* ------------------------------------------------------------------ finalize
 * The fused pac_noised step (§2; final mechanism P:L841-850 §4).
 *
 * y-vector (R7, R9): for a world j whose K bit is set, COUNT -> 2*count_j,
 * SUM -> 2*sum_j ("count[j*]*2 + noise", "2*(C_pos - C_neg)"),
 * AVG -> fsum_j / count_j (per-world divisor, R6), MIN/MAX -> ext_j; a world whose
 * K bit is unset reads as 0 ("counters corresponding to unset bits are
 * treated as zeros").
 */
void orc_y_vector(int kind, int64_t g, uint64_t Kg, const int64_t* count, const void* world,
                  double y[64]) {
  for (int j = 0; j < ORC_M; j++) {
    int64_t cell = g * ORC_M + j;
    if (((Kg >> j) & 1u) == 0) { y[j] = 0.0; continue; }
    switch (kind) {
      case K_COUNT: y[j] = 2.0 * (double)count[cell]; break;
      case K_SUM_I64: y[j] = 2.0 * (double)((const int64_t*)world)[cell]; break;
      case K_SUM_F64: y[j] = 2.0 * ((const double*)world)[cell]; break;
      case K_AVG_F64: y[j] = ((const double*)world)[cell] / (double)count[cell]; break;
      default: y[j] = ((const double*)world)[cell]; break;
    }
  }
}

/* Var_{j~P}[y_j] (R8): population variance weighted by P, two-pass,
 * j ascending.  R11: exactly 0 when every y_j with P_j > 0 is equal. */
double orc_weighted_var(const double P[64], const double y[64]) {
  int first = -1, all_equal = 1;
  for (int j = 0; j < ORC_M; j++) {
    if (P[j] > 0.0) {
      if (first < 0) first = j;
      else if (y[j] != y[first]) all_equal = 0;
    }
  }
  if (all_equal) return 0.0;
  double mu = 0.0;
  for (int j = 0; j < ORC_M; j++) mu += P[j] * y[j];
  double s2 = 0.0;
  for (int j = 0; j < ORC_M; j++) s2 += P[j] * (y[j] - mu) * (y[j] - mu);
  return s2;
}

/* Standard normal from one Philox block (R13, Box-Muller):
 *   u1 = (((x1 << 21) ^ (x2 >> 11)) + 0.5) * 2^-53,  u2 = (x3 + 0.5) * 2^-32,
 *   z  = sqrt(-2 ln u1) * cos(2 pi u2). */
double orc_normal(const uint32_t x[4]) {
  uint64_t m53 = ((uint64_t)x[1] << 21) ^ (uint64_t)(x[2] >> 11);
  double u1 = ((double)m53 + 0.5) * 0x1.0p-53;
  double u2 = ((double)x[3] + 0.5) * 0x1.0p-32;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* Bayesian posterior update (§4; §2):
 *   P <- (P .* W) / sum(P .* W),  W_j = exp(-(y~ - y_j)^2 / (2 Delta)).
 * R14: over worlds with P_j > 0, W_j = exp(-(d_j - min_i d_i) / (2 Delta)) with
 * d_j = (y~ - y_j)^2 -- identical after normalisation, and never all zero. */
void orc_posterior_update(double P[64], const double y[64], double ytilde, double delta) {
  double d[64], dmin = INFINITY;
  for (int j = 0; j < ORC_M; j++) {
    d[j] = (ytilde - y[j]) * (ytilde - y[j]);
    if (P[j] > 0.0 && d[j] < dmin) dmin = d[j];
  }
  double tot = 0.0;
  for (int j = 0; j < ORC_M; j++) {
    if (P[j] > 0.0) P[j] = P[j] * exp(-(d[j] - dmin) / (2.0 * delta));
    tot += P[j];
  }
  for (int j = 0; j < ORC_M; j++) P[j] = P[j] / tot;
}

/* pac_noised over every cell of a table, canonical order (R12: groups ascending,
 * aggregates in declared order; one call = one round).  Per cell:
 *   x = Philox(seed; cell_lo, cell_hi, round, TAG_CELL), cell = g*A + a
 *   NULL iff (x0 >> 26) >= popcount(K_g)        (R10)
 *   s2 = Var_P[y]; Delta = s2 / (2B)
 *   s2 == 0 -> release y_{j*}, no update         (R11)
 *   else release y_{j*} + sqrt(Delta) * z, then posterior update
 * flags[g] bit 0: diversity check (R18): rows >= 64 and
 * popcount(K) <= 34. */
void orc_finalize(uint64_t seed, double B, int jstar, double P[64], int64_t G, int n_aggs,
                  const int32_t* kinds, const uint64_t* K, const int64_t* rows, const int64_t* count,
                  const void* const* world, uint32_t round, double* release, uint8_t* is_null,
                  uint8_t* flags, double* delta_out) {
  double y[64];
  for (int64_t g = 0; g < G; g++) {
    int pc = popcount64(K[g]);
    if (flags) flags[g] = (uint8_t)((rows[g] >= 64 && pc <= 34) ? 1 : 0);
    for (int a = 0; a < n_aggs; a++) {
      int64_t cell = g * n_aggs + a;
      uint32_t x[4];
      philox_block(seed, (uint32_t)cell, (uint32_t)((uint64_t)cell >> 32), round, TAG_CELL, x);
      if ((int)(x[0] >> 26) >= pc) {
        is_null[cell] = 1;
        release[cell] = NAN;
        if (delta_out) delta_out[cell] = NAN;
        continue;
      }
      is_null[cell] = 0;
      orc_y_vector(kinds[a], g, K[g], count, world[a], y);
      double s2 = orc_weighted_var(P, y);
      double delta = s2 / (2.0 * B);
      if (delta_out) delta_out[cell] = delta;
      if (s2 == 0.0) {
        release[cell] = y[jstar];
        continue;
      }
      double yt = y[jstar] + sqrt(delta) * orc_normal(x);
      release[cell] = yt;
      orc_posterior_update(P, y, yt, delta);
    }
  }
}

/* ------------------------------------------------------------------ categorical path
 * (§8 f1; §3 "pac_filter" / "pac_select", §4 vector-lifted
 * expressions, §6 the ratio lambda; readings DESIGN.md R22-R26.)
 *
 * A world vector is (y[64], presence): y in the released scale (orc_y_vector, R7/R9:
 * absent worlds read 0), presence = K of the group (R22). */

enum { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_DIV = 3, OP_MIN = 4, OP_MAX = 5 };
enum { CMP_LT = 0, CMP_LE = 1, CMP_GT = 2, CMP_GE = 3, CMP_EQ = 4 };

static double lift_op(int op, double a, double b) {
  switch (op) {
    case OP_ADD: return a + b;
    case OP_SUB: return a - b;
    case OP_MUL: return a * b;
    case OP_DIV: return a / b;
    case OP_MIN: return fmin(a, b);
    default: return fmax(a, b);
  }
}

/* R23 (Eq. vectorexpressionlambda): out_j = e(a_j, b_j), pointwise; a
 * NULL vector operand is the scalar broadcast to every world (presence: all worlds);
 * out presence = AND of the operands' presences; an absent world of the output
 * holds 0 (R9). */
void orc_lift(int op, int64_t n, const double* a, const uint64_t* pa, double sa, const double* b,
              const uint64_t* pb, double sb, double* out, uint64_t* pout) {
  for (int64_t i = 0; i < n; i++) {
    uint64_t pres = (a ? pa[i] : ~0ull) & (b ? pb[i] : ~0ull);
    pout[i] = pres;
    for (int j = 0; j < ORC_M; j++) {
      double x = a ? a[i * ORC_M + j] : sa;
      double y = b ? b[i * ORC_M + j] : sb;
      out[i * ORC_M + j] = ((pres >> j) & 1u) ? lift_op(op, x, y) : 0.0;
    }
  }
}

static int cmp_holds(int cmp, double v, double c) {
  switch (cmp) {
    case CMP_LT: return v < c;
    case CMP_LE: return v <= c;
    case CMP_GT: return v > c;
    case CMP_GE: return v >= c;
    default: return v == c;
  }
}

/* R26: b_j = [present_j and (v cmp c_j)] -- an absent world has no value, and a
 * comparison with it is NULL, i.e. false in a filter. */
uint64_t orc_cmp_bits(int cmp, double v, const double c[64], uint64_t presence) {
  uint64_t b = 0;
  for (int j = 0; j < ORC_M; j++)
    if (((presence >> j) & 1u) && cmp_holds(cmp, v, c[j])) b |= 1ull << j;
  return b;
}

/* Lifted comparison of two world vectors (or a vector and a broadcast scalar):
 * bit j = [present_j and (a_j cmp b_j)], present = AND of the presences (R23, R26). */
void orc_lift_cmp(int cmp, int64_t n, const double* a, const uint64_t* pa, double sa, const double* b,
                  const uint64_t* pb, double sb, uint64_t* bits) {
  for (int64_t i = 0; i < n; i++) {
    uint64_t pres = (a ? pa[i] : ~0ull) & (b ? pb[i] : ~0ull), r = 0;
    for (int j = 0; j < ORC_M; j++) {
      double x = a ? a[i * ORC_M + j] : sa;
      double y = b ? b[i * ORC_M + j] : sb;
      if (((pres >> j) & 1u) && cmp_holds(cmp, x, y)) r |= 1ull << j;
    }
    bits[i] = r;
  }
}

/* pac_select (Eq. pac-select): h' = h AND b, b the world booleans of the
 * row's group (gidx). */
void orc_select(int64_t n, const uint64_t* h, const int32_t* gidx, const uint64_t* bits, uint64_t* out) {
  for (int64_t i = 0; i < n; i++) out[i] = h[i] & bits[gidx[i]];
}

/* pac_select_<cmp>: h' = h AND b with b_j = [v cmp c_j] against the
 * world vector of the row's group. */
void orc_select_cmp(int cmp, int64_t n, const uint64_t* h, const double* v, const int32_t* gidx,
                    const double* c, const uint64_t* pres, uint64_t* out) {
  for (int64_t i = 0; i < n; i++)
    out[i] = h[i] & orc_cmp_bits(cmp, v[i], c + (int64_t)gidx[i] * ORC_M, pres[gidx[i]]);
}

/* pac_filter (Eq. pac-filter): true with probability popcount(b)/m.
 * R25: r = x0 >> 26 in [0,64) of Philox(seed; i_lo, i_hi, round, TAG_FILTER);
 * true iff r < popcount(b) -- exactly popcount(b)/64. */
void orc_filter(uint64_t seed, uint32_t round, int64_t n, const uint64_t* bits, uint8_t* out) {
  for (int64_t i = 0; i < n; i++) {
    uint32_t x[4];
    philox_block(seed, (uint32_t)i, (uint32_t)((uint64_t)i >> 32), round, TAG_FILTER, x);
    out[i] = (uint8_t)((int)(x[0] >> 26) < popcount64(bits[i]) ? 1 : 0);
  }
}

/* pac_filter_<cmp>: pac_filter of b_j = [v cmp c_j]. */
void orc_filter_cmp(uint64_t seed, uint32_t round, int cmp, int64_t n, const double* v, const int32_t* gidx,
                    const double* c, const uint64_t* pres, uint8_t* out) {
  for (int64_t i = 0; i < n; i++) {
    uint64_t b = orc_cmp_bits(cmp, v[i], c + (int64_t)gidx[i] * ORC_M, pres[gidx[i]]);
    uint32_t x[4];
    philox_block(seed, (uint32_t)i, (uint32_t)((uint64_t)i >> 32), round, TAG_FILTER, x);
    out[i] = (uint8_t)((int)(x[0] >> 26) < popcount64(b) ? 1 : 0);
  }
}

/* pac_noised of given world vectors (R24; P:L841-850 applied to a vector-lifted
 * expression, "gets noised once"): cells i = 0..n-1 in order, y already in the
 * released scale (no *2), absent worlds read 0 (R9), Philox(seed; i_lo, i_hi, round,
 * TAG_LIFT), then exactly the per-cell steps of orc_finalize. */
void orc_noised_y(uint64_t seed, double B, int jstar, double P[64], int64_t n, const double* yv,
                  const uint64_t* presence, uint32_t round, double* release, uint8_t* is_null,
                  double* delta_out) {
  double y[64];
  for (int64_t i = 0; i < n; i++) {
    int pc = popcount64(presence[i]);
    uint32_t x[4];
    philox_block(seed, (uint32_t)i, (uint32_t)((uint64_t)i >> 32), round, TAG_LIFT, x);
    if ((int)(x[0] >> 26) >= pc) {
      is_null[i] = 1;
      release[i] = NAN;
      if (delta_out) delta_out[i] = NAN;
      continue;
    }
    is_null[i] = 0;
    for (int j = 0; j < ORC_M; j++) y[j] = ((presence[i] >> j) & 1u) ? yv[i * ORC_M + j] : 0.0;
    double s2 = orc_weighted_var(P, y);
    double delta = s2 / (2.0 * B);
    if (delta_out) delta_out[i] = delta;
    if (s2 == 0.0) {
      release[i] = y[jstar];
      continue;
    }
    double yt = y[jstar] + sqrt(delta) * orc_normal(x);
    release[i] = yt;
    orc_posterior_update(P, y, yt, delta);
  }
}

/* ------------------------------------------------------------------ PU-key join (§8 f2)
 * P:L331-357 §3 (Eq. join-addition, Eq. join-elim), §2; reading R27.
 * The chain T -fk1-> T1 -fk2-> ... -> Tk -fkU-> U with join elimination: starting from the
 * row's fk1, look the key up in T1's primary-key column and continue with that tuple's next
 * FK, k times; the last FK (Tk.fk_U == U.pk by referential integrity) is the PU key, and
 * the row's mask is pac_hash(PU key).  A row whose key finds no match has no PU (it would
 * not survive the inserted inner join): mask 0, found 0.  Lookup = binary search of the
 * table's (pk, next) pairs sorted by pk (libc qsort/bsearch). */
typedef struct { int64_t pk, next; } pk_pair;
static int cmp_pair(const void* a, const void* b) {
  int64_t x = ((const pk_pair*)a)->pk, y = ((const pk_pair*)b)->pk;
  return (x > y) - (x < y);
}

void orc_join_chain_mask(int k, const int64_t* const* pk, const int64_t* const* next, const int64_t* n_build,
                         const int64_t* fk, int64_t n, uint64_t salt, uint64_t* mask, uint8_t* found,
                         int64_t* pu) {
  pk_pair* tab[8];
  for (int t = 0; t < k; t++) {
    tab[t] = (pk_pair*)malloc((size_t)(n_build[t] > 0 ? n_build[t] : 1) * sizeof(pk_pair));
    for (int64_t i = 0; i < n_build[t]; i++) {
      tab[t][i].pk = pk[t][i];
      tab[t][i].next = next[t][i];
    }
    qsort(tab[t], (size_t)n_build[t], sizeof(pk_pair), cmp_pair);
  }
  for (int64_t i = 0; i < n; i++) {
    int64_t x = fk[i];
    int ok = 1;
    for (int t = 0; t < k && ok; t++) {
      pk_pair key = {x, 0};
      const pk_pair* hit = (const pk_pair*)bsearch(&key, tab[t], (size_t)n_build[t], sizeof(pk_pair), cmp_pair);
      if (hit) x = hit->next; else ok = 0;
    }
    found[i] = (uint8_t)ok;
    pu[i] = ok ? x : 0;
    mask[i] = ok ? orc_pac_hash(x, salt) : 0;
  }
  for (int t = 0; t < k; t++) free(tab[t]);
}

/* ------------------------------------------------------------------ m = 128 worlds (§8 f4)
 * P:L92 (§2, footnote): "Extending to m=128 is possible, and worst-case would double the
 * cost of our stochastic-aggregates".  Readings R28 (hash), R29 (session, aggregation,
 * finalize).  A mask is two words: lo = worlds 0..63, hi = worlds 64..127 (R3 extended). */
#define ORC_M2 128

static int bit128(const uint64_t x[2], int j) { return (int)((x[j >> 6] >> (j & 63)) & 1u); }
static int popcount128(const uint64_t x[2]) { return popcount64(x[0]) + popcount64(x[1]); }

/* R28: x_lo = fmix64(key XOR salt), x_hi = fmix64(x_lo XOR 0x6A09E667F3BCC909); balance to
 * exactly 64 ones by the rejection flips of R2 with 7-bit draws: w_0 = fmix64(x_lo XOR x_hi
 * XOR 0xD1B54A32D192ED03), w_{i+1} = fmix64(w_i + 0x9E3779B97F4A7C15); each word gives 9 draws
 * p = (w >> 7t) & 127, t = 0..8; a draw flips bit p if it carries the majority value; stop at
 * k = 0; safety net after 64 words as in R2. */
void orc_pac_hash128(int64_t key, uint64_t salt, uint64_t out[2]) {
  uint64_t x[2];
  x[0] = orc_fmix64((uint64_t)key ^ salt);
  x[1] = orc_fmix64(x[0] ^ 0x6A09E667F3BCC909ull);
  int c = popcount128(x);
  if (c != 64) {
    int maj = c > 64 ? 1 : 0;
    int k = c > 64 ? c - 64 : 64 - c;
    uint64_t w = orc_fmix64(x[0] ^ x[1] ^ 0xD1B54A32D192ED03ull);
    for (int word = 0; word < 64 && k > 0; word++) {
      for (int t = 0; t < 9 && k > 0; t++) {
        int p = (int)((w >> (7 * t)) & 127u);
        if (bit128(x, p) == maj) {
          x[p >> 6] ^= 1ull << (p & 63);
          k--;
        }
      }
      w = orc_fmix64(w + 0x9E3779B97F4A7C15ull);
    }
    for (int p = 0; p < ORC_M2 && k > 0; p++) {
      if (bit128(x, p) == maj) {
        x[p >> 6] ^= 1ull << (p & 63);
        k--;
      }
    }
  }
  out[0] = x[0];
  out[1] = x[1];
}

void orc_pac_hash128_n(const int64_t* keys, int64_t n, uint64_t salt, uint64_t* out) {
  for (int64_t i = 0; i < n; i++) orc_pac_hash128(keys[i], salt, out + 2 * i);
}

/* R29 session: j* = x0 & 127 of Philox(seed; 0,0,0,TAG_JSTAR), salt as R13, P = 1/128. */
void orc_session_init128(uint64_t seed, int* jstar, uint64_t* salt, double* P) {
  uint32_t o[4];
  philox_block(seed, 0, 0, 0, TAG_JSTAR, o);
  *jstar = (int)(o[0] & 127u);
  philox_block(seed, 0, 0, 0, TAG_SALT, o);
  *salt = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
  for (int j = 0; j < ORC_M2; j++) P[j] = 1.0 / ORC_M2;
}

/* R29 aggregation: Eq. counter over 128 worlds; a row is in world j iff bit j of
 * its 128-bit mask is set; rows with a zero mask are dropped (R21); K[g] = OR of the masks
 * (two words).  Same output layout as orc_agg_o2 with 128 worlds per group. */
int orc_agg128(const uint64_t* masks, int64_t n, const void* const* cols, const int32_t* elem_bytes,
               int n_keys, const uint64_t* gkeys, int64_t G, const int32_t* kinds, const void* const* values,
               int n_aggs, int64_t* rows, uint64_t* K, int64_t* count, void* const* world) {
  int overflow = 0;
  const int64_t GM = G * ORC_M2;
  for (int64_t g = 0; g < G; g++) { rows[g] = 0; K[2 * g] = K[2 * g + 1] = 0; }
  for (int64_t i = 0; i < GM; i++) count[i] = 0;
  for (int a = 0; a < n_aggs; a++) {
    if (!world[a]) continue;
    for (int64_t i = 0; i < GM; i++) {
      if (kinds[a] == K_SUM_I64) ((int64_t*)world[a])[i] = 0;
      else if (kinds[a] == K_MIN_F64) ((double*)world[a])[i] = INFINITY;
      else if (kinds[a] == K_MAX_F64) ((double*)world[a])[i] = -INFINITY;
      else if (kinds[a] != K_COUNT) ((double*)world[a])[i] = 0.0;
    }
  }
  __int128* isum = (__int128*)calloc((size_t)(GM * n_aggs + 1), sizeof(__int128));
  csum* fsum = (csum*)calloc((size_t)(GM * n_aggs + 1), sizeof(csum));
  for (int64_t r = 0; r < n; r++) {
    const uint64_t* h = masks + 2 * r;
    if ((h[0] | h[1]) == 0) continue;
    uint64_t key = n_keys ? orc_pack_key(cols, elem_bytes, n_keys, r) : 0;
    int64_t g = find_group(gkeys, G, key);
    if (g < 0) continue;
    rows[g] += 1;
    K[2 * g] |= h[0];
    K[2 * g + 1] |= h[1];
    for (int j = 0; j < ORC_M2; j++) {
      if (!bit128(h, j)) continue;
      int64_t cell = g * ORC_M2 + j;
      count[cell] += 1;
      for (int a = 0; a < n_aggs; a++) {
        int64_t idx = (int64_t)a * GM + cell;
        switch (kinds[a]) {
          case K_SUM_I64: isum[idx] += (__int128)((const int64_t*)values[a])[r]; break;
          case K_SUM_F64:
          case K_AVG_F64: csum_add(&fsum[idx], ((const double*)values[a])[r]); break;
          case K_MIN_F64: {
            double v = ((const double*)values[a])[r];
            double* e = &((double*)world[a])[cell];
            if (count[cell] == 1 || tot_less(v, *e)) *e = v;
            break;
          }
          case K_MAX_F64: {
            double v = ((const double*)values[a])[r];
            double* e = &((double*)world[a])[cell];
            if (count[cell] == 1 || tot_less(*e, v)) *e = v;
            break;
          }
          default: break;
        }
      }
    }
  }
  for (int a = 0; a < n_aggs; a++) {
    for (int64_t cell = 0; cell < GM; cell++) {
      int64_t idx = (int64_t)a * GM + cell;
      if (kinds[a] == K_SUM_I64) {
        __int128 v = isum[idx];
        if (v > (__int128)INT64_MAX || v < (__int128)INT64_MIN) overflow = 1;
        ((int64_t*)world[a])[cell] = (int64_t)v;
      } else if (kinds[a] == K_SUM_F64 || kinds[a] == K_AVG_F64) {
        ((double*)world[a])[cell] = csum_value(&fsum[idx]);
      }
    }
  }
  free(isum);
  free(fsum);
  return overflow;
}

static double weighted_var128(const double* P, const double* y) {
  int first = -1, all_equal = 1;
  for (int j = 0; j < ORC_M2; j++) {
    if (P[j] > 0.0) {
      if (first < 0) first = j;
      else if (y[j] != y[first]) all_equal = 0;
    }
  }
  if (all_equal) return 0.0;
  double mu = 0.0;
  for (int j = 0; j < ORC_M2; j++) mu += P[j] * y[j];
  double s2 = 0.0;
  for (int j = 0; j < ORC_M2; j++) s2 += P[j] * (y[j] - mu) * (y[j] - mu);
  return s2;
}

static void posterior_update128(double* P, const double* y, double ytilde, double delta) {
  double d[ORC_M2], dmin = INFINITY;
  for (int j = 0; j < ORC_M2; j++) {
    d[j] = (ytilde - y[j]) * (ytilde - y[j]);
    if (P[j] > 0.0 && d[j] < dmin) dmin = d[j];
  }
  double tot = 0.0;
  for (int j = 0; j < ORC_M2; j++) {
    if (P[j] > 0.0) P[j] = P[j] * exp(-(d[j] - dmin) / (2.0 * delta));
    tot += P[j];
  }
  for (int j = 0; j < ORC_M2; j++) P[j] = P[j] / tot;
}

/* R29 finalize: the per-cell steps of orc_finalize over 128 worlds: NULL iff
 * (x0 >> 25) >= popcount(K) (probability (128 - popcount)/128); y-vectors of R7/R9;
 * variance and posterior over 128 worlds; diversity flag rows >= 128 and popcount(K) <= 68
 * (R18 scaled to m = 128). */
void orc_finalize128(uint64_t seed, double B, int jstar, double* P, int64_t G, int n_aggs, const int32_t* kinds,
                     const uint64_t* K, const int64_t* rows, const int64_t* count, const void* const* world,
                     uint32_t round, double* release, uint8_t* is_null, uint8_t* flags, double* delta_out) {
  double y[ORC_M2];
  for (int64_t g = 0; g < G; g++) {
    const uint64_t* Kg = K + 2 * g;
    int pc = popcount128(Kg);
    if (flags) flags[g] = (uint8_t)((rows[g] >= 128 && pc <= 68) ? 1 : 0);
    for (int a = 0; a < n_aggs; a++) {
      int64_t cell = g * n_aggs + a;
      uint32_t x[4];
      philox_block(seed, (uint32_t)cell, (uint32_t)((uint64_t)cell >> 32), round, TAG_CELL, x);
      if ((int)(x[0] >> 25) >= pc) {
        is_null[cell] = 1;
        release[cell] = NAN;
        if (delta_out) delta_out[cell] = NAN;
        continue;
      }
      is_null[cell] = 0;
      for (int j = 0; j < ORC_M2; j++) {
        int64_t c = g * ORC_M2 + j;
        if (!bit128(Kg, j)) { y[j] = 0.0; continue; }
        switch (kinds[a]) {
          case K_COUNT: y[j] = 2.0 * (double)count[c]; break;
          case K_SUM_I64: y[j] = 2.0 * (double)((const int64_t*)world[a])[c]; break;
          case K_SUM_F64: y[j] = 2.0 * ((const double*)world[a])[c]; break;
          case K_AVG_F64: y[j] = ((const double*)world[a])[c] / (double)count[c]; break;
          default: y[j] = ((const double*)world[a])[c]; break;
        }
      }
      double s2 = weighted_var128(P, y);
      double delta = s2 / (2.0 * B);
      if (delta_out) delta_out[cell] = delta;
      if (s2 == 0.0) {
        release[cell] = y[jstar];
        continue;
      }
      double yt = y[jstar] + sqrt(delta) * orc_normal(x);
      release[cell] = yt;
      posterior_update128(P, y, yt, delta);
    }
  }
}

/* ------------------------------------------------------------------ approximate SUM (§8 f3)
 * P:L1783-1803 (§5 "Approximation", "Two-sided SUM"); readings DESIGN.md R35-R36.
 * Per world and side, 25 levels of 16-bit counters C[k] of weight 2^(4k).  A value v != 0 of a
 * row in world j goes to side pos (v > 0) or neg (v < 0, stored negated); with
 * a = |v|, msb = index of its highest set bit, it is routed to level
 *   l(v) = floor((msb - 8) / 4)   (0 for msb < 8, capped at 24)
 * and adds c = a >> 4l.  Overflow (C[l] + c > 0xFFFF): "only the upper 12 bits of each counter
 * cascade: C[k+1] += C[k] >> 4" -- the counter's low 4 bits are dropped and it restarts
 * at 0 (R35), recursively upward, then c is added.  Result (R7): 2 * (dec(pos) - dec(neg)),
 * dec(C) = sum_k C[k] 2^(4k).  Single-sided variant (Table 1's "Single Sum", R36): one state fed
 * the value's 64-bit two's-complement pattern u = (uint64)v -- routed by msb(u), adding u >> 4l --
 * and decoded modulo 2^64 as a signed int64 (a negative value has msb 63 and loses its low 52
 * bits: the failure Table 1 shows on negative_mixed, which the second, negated state avoids).
 * Execution order (R35): rows in row order within consecutive blocks of block_rows rows (the
 * thread-local states of P:L1966), block states combined in block order by adding each level of
 * the next block's state into the running state with the same add-with-cascade rule. */
#define ORC_AL 25

static void approx_add_u(uint16_t* C, int k, uint32_t c) {
  if (k >= ORC_AL) return; /* beyond 112 bits: out of contract (R35) */
  if ((uint32_t)C[k] + c > 0xFFFFu) {
    approx_add_u(C, k + 1, (uint32_t)(C[k] >> 4));
    C[k] = 0;
  }
  C[k] = (uint16_t)(C[k] + c);
}

static int approx_level(uint64_t a) {
  int msb = 63;
  while (msb > 0 && ((a >> msb) & 1u) == 0) msb--;
  int l = msb < 8 ? 0 : (msb - 8) / 4;
  return l > ORC_AL - 1 ? ORC_AL - 1 : l;
}

/* counters: [2][64][25] uint16 (side 0 = pos, 1 = neg; single-sided: side 0 only).  y[64] = the
 * released-scale world values 2 * (dec(pos) - dec(neg)), resp. 2 * (int64)(dec mod 2^64). */
void orc_approx_sum(const uint64_t* masks, int64_t n, const int64_t* values, int64_t block_rows, int two_sided,
                    uint16_t* counters, double* y) {
  const size_t nc = (size_t)2 * ORC_M * ORC_AL;
  uint16_t* run = (uint16_t*)calloc(nc, sizeof(uint16_t));
  uint16_t* blk = (uint16_t*)calloc(nc, sizeof(uint16_t));
  for (int64_t b0 = 0; b0 < n; b0 += block_rows) {
    memset(blk, 0, nc * sizeof(uint16_t));
    int64_t b1 = b0 + block_rows < n ? b0 + block_rows : n;
    for (int64_t r = b0; r < b1; r++) {
      int64_t v = values[r];
      if (v == 0 || masks[r] == 0) continue;
      uint64_t a = !two_sided ? (uint64_t)v : (v > 0 ? (uint64_t)v : (uint64_t)0 - (uint64_t)v);
      int l = approx_level(a);
      uint32_t c = (uint32_t)(a >> (4 * l));
      int side = two_sided && v < 0 ? 1 : 0;
      for (int j = 0; j < ORC_M; j++) {
        if (((masks[r] >> j) & 1u) == 0) continue;
        approx_add_u(blk + ((size_t)side * ORC_M + j) * ORC_AL, l, c);
      }
    }
    /* combine the block into the running state, level by level, block order */
    for (int s = 0; s < (two_sided ? 2 : 1); s++)
      for (int j = 0; j < ORC_M; j++)
        for (int k = 0; k < ORC_AL; k++) {
          size_t o = ((size_t)s * ORC_M + j) * ORC_AL;
          approx_add_u(run + o, k, blk[o + k]);
        }
  }
  memcpy(counters, run, nc * sizeof(uint16_t));
  for (int j = 0; j < ORC_M; j++) {
    if (two_sided) {
      double d = 0.0, sc = 1.0;
      for (int k = 0; k < ORC_AL; k++, sc *= 16.0)
        d += ((double)run[(size_t)j * ORC_AL + k] - (double)run[((size_t)ORC_M + j) * ORC_AL + k]) * sc;
      y[j] = 2.0 * d;
    } else {
      uint64_t u = 0; /* decode modulo 2^64 (levels >= 16 vanish) */
      for (int k = 0; k < 16; k++) u += (uint64_t)run[(size_t)j * ORC_AL + k] << (4 * k);
      y[j] = 2.0 * (double)(int64_t)u;
    }
  }
  free(run);
  free(blk);
}
