// libpac: sort-first grouped aggregation for high-cardinality tables (BASELINE C3; DESIGN.md §5
// "k_srt_*: sort first").
//
// The paper's engine keeps one aggregate state per group in thread-local hash tables that are
// combined at the end (§5).  On B200 a group table of ~1e6 groups x 64 worlds does not
// fit on chip, and first-touch CTA dictionaries catch only about half of a Zipf stream (the rest
// took the deferred HBM tier: ~16 ms per 1e8 rows).  Here the rows are instead brought into group
// order first, so that every group's rows are contiguous and the 64-world update becomes a
// streaming fold with one table write per group:
//
//   pass b = 0..3   stable LSD radix pass on byte b of the packed group key (R20, <= 4 bytes):
//                   k_srt_hist (per-CTA digit counts) -> k_srt_scan (digit-major exclusive scan
//                   = every CTA's write cursor per digit) -> k_srt_scatter (tile of 2048 rows:
//                   per-warp match_any ranks, tile-local digit order in shared memory, coalesced
//                   runs written to the cursors).  Pass 0 reads the caller's columns and packs
//                   the key; rows with an explicit zero mask are dropped there (R21).  A byte that
//                   is constant over all keys (OR == AND) is skipped on the device (no data moves).
//   k_srt_hash      pac_hash (R1/R2) of the sorted pu keys in place, stragglers compacted per warp.
//   heads           k_srt_heads / k_srt_hscan: group starts per 2048-row chunk, their exclusive
//                   scan = the canonical slot of every chunk's first group; the group count is
//                   the table's num_groups (slots follow ascending packed key, R12/R20, so the
//                   finishing sort is the identity).  k_srt_bzero zeroes the rows of the groups
//                   that span a chunk boundary (they are added with atomics).
//   k_srt_agg       one warp per chunk, 32 rows per window: segments of equal key inside the
//                   window go through run_body (the transposed Four Russians 64-world update of
//                   the tile kernels, agg_tiles.cuh); a group is written with plain stores when it
//                   lies inside the chunk, with atomics when it spans a boundary.
//
// Within a group the row order after the sort is not the input order: f64 sums differ in the
// last bits (R34); integers are exact.
#include "agg_tiles.cuh"

namespace pac {

void note_launch();
void profile_begin(cudaStream_t st, const char* name);
void profile_end(cudaStream_t st);

#ifndef PAC_SRT_BTAB
#define PAC_SRT_BTAB 0  // 1: pass 0 hash draws through the shared-memory table of common.cuh (measured slower on C3: 7.27 -> 7.40 ms)
#endif
#ifndef PAC_SRT_MINB
#define PAC_SRT_MINB 3  // resident k_srt_scatter CTAs per SM the register allocation targets
#endif
#ifndef PAC_SRT_AGG_MINB
#define PAC_SRT_AGG_MINB 4  // resident k_srt_agg CTAs per SM the register allocation targets
#endif
constexpr int kSrtThreads = 256;  // k_srt_hist / k_srt_scatter
constexpr int kSrtW = kSrtThreads / 32;
// rows per thread and tile of k_srt_scatter: 16 (4096-row tiles, 16 rows per digit on average)
// for rows of at most one value column, 8 otherwise (registers)
__host__ __device__ constexpr int srt_rpt(int) { return 8; }  // (16 measured no faster on C3)
constexpr int kSrtTmax = 4096;    // CTA chunks are multiples of every tile size
constexpr int kSrtCH = 2048;      // rows per k_srt_agg work item (one warp)
constexpr int kSrtMaxV = 4;       // value columns moved with the rows

struct SrtPlan {
  int64_t n;                              // input rows
  const long long* pu;                    // pass 0: pu keys (hashed) or NULL
  const unsigned long long* mask_in;      // pass 0: explicit masks (zero rows dropped) or NULL
  uint64_t salt;
  int n_keys, width;                      // key columns, packed key bytes (1..4)
  const void* key_col[PAC_MAX_KEYS];
  int key_bytes[PAC_MAX_KEYS];
  int nv;                                 // value columns (8 bytes each)
  int hash0;                              // 1: pass 0 hashes the pu keys (else k_srt_hash after the passes)
  const unsigned long long* val_in[kSrtMaxV];
  uint32_t* key[2];                       // ping-pong row buffers
  unsigned long long* msk[2];
  unsigned long long* val[2][kSrtMaxV];
  long long* hist;                        // [256][grid] counts, then offsets (in place)
  unsigned long long* dtot;               // [4][256] digit totals per pass (zeroed up front)
  unsigned long long* ctr;                // [0] rows kept, [1] OR of keys, [2] AND of keys
  int grid;                               // CTAs of k_srt_hist / k_srt_scatter
  int* hcnt;                              // [nch] group starts before the chunk within its block of 8
  int* hblk;                              // [nch / 8] group starts per block, then their exclusive scan
  int nch;                                // agg chunks (upper bound, from n)
};

// The output table, written directly by k_srt_agg (the slots are canonical: no gather pass).
struct SrtOut {
  pac_table t;
  int n_aggs;
  int kind[PAC_MAX_AGGS];  // 0 count (no world array), 1 int64 sum src idx, 2 f64 sum src idx
  int idx[PAC_MAX_AGGS];
};

__device__ __forceinline__ uint32_t srt_pack_key(const SrtPlan& q, int64_t r) {
  uint32_t packed = 0;
#pragma unroll
  for (int c = 0; c < PAC_MAX_KEYS; ++c) {
    if (c < q.n_keys) {
      const int w = q.key_bytes[c];
      uint32_t v;
      if (w == 1) v = (uint32_t)__ldg((const uint8_t*)q.key_col[c] + r);
      else if (w == 2) v = (uint32_t)__ldg((const uint16_t*)q.key_col[c] + r);
      else v = __ldg((const uint32_t*)q.key_col[c] + r);
      v ^= 1u << (8 * w - 1);  // R20: sign bit flipped, first column most significant
      packed = w == 4 ? v : ((packed << (8 * w)) | v);
    }
  }
  return packed;
}

// packed keys of rows r[0..R) (r >= r1: 0), one column at a time so the loads of all rows issue
// back to back
template <int R>
__device__ __forceinline__ void srt_pack_keys(const SrtPlan& q, const int64_t* r, int64_t r1, uint32_t* key) {
#pragma unroll
  for (int j = 0; j < R; ++j) key[j] = 0u;
  for (int c = 0; c < q.n_keys; ++c) {
    const int w = q.key_bytes[c];
    const uint32_t flip = 1u << (8 * w - 1);
    uint32_t v[R];
    if (w == 4) {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = r[j] < r1 ? __ldg((const uint32_t*)q.key_col[c] + r[j]) : 0u;
    } else if (w == 2) {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = r[j] < r1 ? (uint32_t)__ldg((const uint16_t*)q.key_col[c] + r[j]) : 0u;
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = r[j] < r1 ? (uint32_t)__ldg((const uint8_t*)q.key_col[c] + r[j]) : 0u;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) key[j] = w == 4 ? (v[j] ^ flip) : ((key[j] << (8 * w)) | (v[j] ^ flip));
  }
}

// passes in [0, upto) that move data (byte 0 always: it packs, hashes and copies)
__device__ __forceinline__ int srt_nactive(const SrtPlan& q, int upto) {
  const uint32_t var = (uint32_t)(q.ctr[1] ^ q.ctr[2]);
  int a = 0;
  for (int b = 0; b < upto; ++b) a += (b == 0 || ((var >> (8 * b)) & 255u)) ? 1 : 0;
  return a;
}
__device__ __forceinline__ bool srt_active(const SrtPlan& q, int b) {
  return b == 0 || ((((uint32_t)(q.ctr[1] ^ q.ctr[2])) >> (8 * b)) & 255u) != 0;
}
__device__ __forceinline__ int64_t srt_rows(const SrtPlan& q, int b) { return b == 0 ? q.n : (int64_t)q.ctr[0]; }
// rows of one CTA's chunk (multiple of the tile), the same in k_srt_hist and k_srt_scatter
__device__ __forceinline__ int64_t srt_chunk(int64_t n, int grid) {
  const int64_t per = (n + grid - 1) / grid;
  return (per + kSrtTmax - 1) / kSrtTmax * kSrtTmax;
}

// per-CTA digit counts of byte b (pass 0: also the OR / AND of the packed keys).  Per-warp
// sub-histograms (no match_any), 4 consecutive rows per thread and step (one 16-byte load of the
// packed keys after pass 0).
constexpr int kHistThreads = 1024;  // k_srt_hist: 4x the scatter's threads per chunk (occupancy)
template <bool P0>
__global__ void __launch_bounds__(kHistThreads) k_srt_hist(SrtPlan q, int b) {
  if (!P0 && !srt_active(q, b)) return;
  constexpr int HW = kHistThreads / 32;
  __shared__ int h[HW][256];
  __shared__ unsigned long long s_or, s_and;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < HW * 256; i += kHistThreads) (&h[0][0])[i] = 0;
  if (tid == 0) {
    s_or = 0;
    s_and = ~0ull;
  }
  __syncthreads();
  const int64_t n = srt_rows(q, b);
  const int64_t ch = srt_chunk(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * ch, r1 = min(n, r0 + ch);
  const int a = P0 ? 0 : srt_nactive(q, b);
  const uint32_t* kin = P0 ? nullptr : q.key[(a - 1) & 1];
  const int sh = 8 * b;
  int* hw = h[wid];
  uint32_t o = 0, an = ~0u;
#pragma unroll 2
  for (int64_t rb = r0 + 4 * tid; rb < r1; rb += 4 * kHistThreads) {
    uint32_t k4[4];
    bool ok[4];
    if (P0) {
      int64_t rr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) rr[i] = rb + i;
      srt_pack_keys<4>(q, rr, r1, k4);
#pragma unroll
      for (int i = 0; i < 4; ++i) ok[i] = rr[i] < r1 && (!q.mask_in || q.mask_in[rr[i]] != 0ull);
    } else if (rb + 4 <= r1) {
      const uint4 x = *(const uint4*)(kin + rb);  // r0 and the buffers are 16-byte aligned
      k4[0] = x.x; k4[1] = x.y; k4[2] = x.z; k4[3] = x.w;
#pragma unroll
      for (int i = 0; i < 4; ++i) ok[i] = true;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t r = rb + i;
        ok[i] = r < r1;
        k4[i] = 0;
        if (ok[i]) {
          k4[i] = P0 ? srt_pack_key(q, r) : kin[r];
          if (P0 && q.mask_in) ok[i] = q.mask_in[r] != 0ull;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!ok[i]) continue;
      if (P0) {
        o |= k4[i];
        an &= k4[i];
      }
      atomicAdd(&hw[(k4[i] >> sh) & 255u], 1);
    }
  }
  if (P0) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      o |= __shfl_xor_sync(0xffffffffu, o, s);
      an &= __shfl_xor_sync(0xffffffffu, an, s);
    }
    if (lane == 0) {
      atomicOr(&s_or, (unsigned long long)o);
      atomicAnd(&s_and, 0xFFFFFFFF00000000ull | an);
    }
  }
  __syncthreads();
  if (tid < 256) {
    int c = 0;
#pragma unroll 8
    for (int w = 0; w < HW; ++w) c += h[w][tid];
    q.hist[(size_t)tid * gridDim.x + blockIdx.x] = c;
    if (c) atomicAdd(&q.dtot[256 * b + tid], (unsigned long long)c);
  }
  if (P0 && tid == 0) {
    atomicOr(&q.ctr[1], s_or);
    atomicAnd(&q.ctr[2], s_and);
  }
}

// exclusive scan of hist in digit-major order, in place: one warp per digit d -- its base is the
// sum of the digit totals below d (accumulated by k_srt_hist), then the CTA counts of d are scanned
// (all of them in flight at once).  Pass 0 also records the rows kept.
constexpr int kScanMaxGrid = 512;
__global__ void __launch_bounds__(32) k_srt_scan(SrtPlan q, int b) {
  if (!srt_active(q, b)) return;
  const int lane = threadIdx.x, d = blockIdx.x, G = q.grid;
  const unsigned long long* tot = q.dtot + 256 * b;
  long long base = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = 32 * k + lane;
    base += i < d ? (long long)tot[i] : 0;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) base += __shfl_xor_sync(0xffffffffu, base, s);
  if (b == 0 && d == 255 && lane == 0) q.ctr[0] = (unsigned long long)base + tot[255];
  constexpr int KMAX = kScanMaxGrid / 32;
  long long* hd = q.hist + (size_t)d * G;
  long long v[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) v[k] = (32 * k + lane < G) ? hd[32 * k + lane] : 0;
  long long carry = base;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    long long x = v[k];
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, s);
      if (lane >= s) x += y;
    }
    if (32 * k + lane < G) hd[32 * k + lane] = carry + x - v[k];
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

// One stable counting pass on byte b.  Warp w of a tile owns rows [256 w, 256 w + 256) and ranks
// them batch by batch (match_any), so the order inside a digit is: warp, batch, lane -- the input
// order.  The tile is reordered by digit in shared memory and written in runs to the cursors.
template <int NV, bool P0>
__global__ void __launch_bounds__(kSrtThreads, NV <= 1 ? PAC_SRT_MINB : 2) k_srt_scatter(SrtPlan q, int b) {
  if (!P0 && !srt_active(q, b)) return;
  constexpr int RPT = srt_rpt(NV), T = kSrtThreads * RPT;  // longer digit runs per tile when the rows are narrow
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* smsk = (unsigned long long*)smem;                 // [T]
  unsigned long long* sval = smsk + T;                              // [NV][T]
  uint32_t* skey = (uint32_t*)(sval + NV * T);                      // [T]
  int* cnt = (int*)(skey + T);                                      // [256][W]
  int* dstart = cnt + 256 * kSrtW;                                      // [256]
  long long* cur = (long long*)(dstart + 256);                          // [256]
  __shared__ int s_wsum[kSrtW];
  __shared__ int s_tn;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#if PAC_SRT_BTAB
  __shared__ __align__(16) unsigned char s_bt[P0 ? kBtabBytes : 16];  // one-hot table of the hash draws (common.cuh)
  const uint32_t bt = btab_addr(s_bt);
  if (P0) btab_fill(bt, tid);  // the barrier below orders it before the first tile
#endif
  const unsigned lt = (1u << lane) - 1u;
  const int64_t n = srt_rows(q, b);
  const int64_t ch = srt_chunk(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * ch, r1 = min(n, r0 + ch);
  const int a = P0 ? 0 : srt_nactive(q, b);
  const int ib = (a - 1) & 1, ob = a & 1;
  cur[tid] = q.hist[(size_t)tid * gridDim.x + blockIdx.x];
#pragma unroll
  for (int w = 0; w < kSrtW; ++w) cnt[tid * kSrtW + w] = 0;
  __syncthreads();
  for (int64_t t0 = r0; t0 < r1; t0 += T) {
    uint32_t key[RPT], rk[RPT];
    unsigned long long m[RPT], v[RPT][NV > 0 ? NV : 1];
    // load (pass 0: pack, hash; explicit zero masks are dropped).  Every load of the tile is
    // issued before any loaded value is used.
    if (P0) {
      const unsigned long long* msrc = q.mask_in ? q.mask_in : (const unsigned long long*)q.pu;
      const bool k4 = q.n_keys == 1 && q.key_bytes[0] == 4;  // the common layout: one int32 key
      const uint32_t* kc = (const uint32_t*)q.key_col[0];
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int64_t r = t0 + wid * (32 * RPT) + 32 * j + lane;
        const bool in = r < r1;
        m[j] = in ? __ldg(msrc + r) : 0ull;
#pragma unroll
        for (int c = 0; c < NV; ++c) v[j][c] = in ? __ldg(q.val_in[c] + r) : 0ull;
        key[j] = (in && k4) ? __ldg(kc + r) : 0u;  // R20 sign flip applied at first use (ranks)
      }
      if (!k4) {
        int64_t rr[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) rr[j] = t0 + wid * (32 * RPT) + 32 * j + lane;
        srt_pack_keys<RPT>(q, rr, r1, key);
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int64_t r = t0 + wid * (32 * RPT) + 32 * j + lane;
        rk[j] = (r < r1 && (!q.mask_in || m[j] != 0ull)) ? 0u : 0xFFFFFFFFu;  // 0xFFFFFFFF: not kept
      }
    } else {
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int64_t r = t0 + wid * (32 * RPT) + 32 * j + lane;
        const bool in = r < r1;
        key[j] = in ? q.key[ib][r] : 0u;
        m[j] = in ? q.msk[ib][r] : 0ull;
#pragma unroll
        for (int c = 0; c < NV; ++c) v[j][c] = in ? q.val[ib][c][r] : 0ull;
        rk[j] = in ? 0u : 0xFFFFFFFFu;
      }
    }
    if (P0 && q.pu && q.hash0) {
      // pac_hash (R1, R2): mix, popcount and draw word 0 branch-free for every row (two rows
      // interleaved); rows that still need flips are queued per warp and finished with all 32
      // lanes busy.  The staging buffer is free until the reorder below.
      unsigned long long* res = smsk + wid * (32 * RPT);
      unsigned long long* qw = sval + wid * (32 * RPT);  // NV >= 1 here (see srt_pass)
      unsigned short* qr = (unsigned short*)(skey) + wid * (32 * RPT);
      int qn = 0;
#pragma unroll
      for (int j = 0; j < RPT; j += 2) {
        HashState ha, hb;
#if PAC_SRT_BTAB
        pac_hash_begin2_bt(m[j], m[j + 1], q.salt, ha, hb, bt);
#else
        pac_hash_begin2(m[j], m[j + 1], q.salt, ha, hb);
#endif
        m[j] = hash_mask_now(ha);
        m[j + 1] = hash_mask_now(hb);
        const bool sa = rk[j] == 0u && ha.k > 0, sb = rk[j + 1] == 0u && hb.k > 0;
        const unsigned ba = __ballot_sync(0xffffffffu, sa);
        if (sa) {
          const int qi = qn + __popc(ba & lt);
          qw[qi] = ha.w0;
          qr[qi] = (unsigned short)(32 * j + lane);
          res[32 * j + lane] = m[j];
        }
        qn += __popc(ba);
        const unsigned bb = __ballot_sync(0xffffffffu, sb);
        if (sb) {
          const int qi = qn + __popc(bb & lt);
          qw[qi] = hb.w0;
          qr[qi] = (unsigned short)(32 * (j + 1) + lane);
          res[32 * (j + 1) + lane] = m[j + 1];
        }
        qn += __popc(bb);
      }
      __syncwarp();
      for (int qi = lane; qi < qn; qi += 32) {
        const int rr = qr[qi];
#if PAC_SRT_BTAB
        res[rr] = pac_hash_continue_bt(res[rr], qw[qi], bt);
#else
        res[rr] = pac_hash_continue(res[rr], qw[qi]);
#endif
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < RPT; ++j)
        if (rk[j] == 0u && __popcll(m[j]) != 32) m[j] = res[32 * j + lane];
      __syncwarp();
    }
    // ranks within (digit, warp), batch by batch
    if (P0 && q.n_keys == 1 && q.key_bytes[0] == 4) {
#pragma unroll
      for (int j = 0; j < RPT; ++j) key[j] ^= 0x80000000u;
    }
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const bool ok = rk[j] == 0u;
      const uint32_t d = (key[j] >> (8 * b)) & 255u;
      const unsigned peers = __match_any_sync(0xffffffffu, ok ? d : 256u + lane);
      int before = 0;
      if (ok) before = cnt[d * kSrtW + wid];
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) cnt[d * kSrtW + wid] = before + __popc(peers);
      __syncwarp();
      if (ok) rk[j] = (d << 16) | (uint32_t)(before + __popc(peers & lt));
    }
    __syncthreads();
    // per digit: offsets of the warps (in place) and the tile total; the digits' tile starts
    int tot = 0;
    {
      const int d = tid;
#pragma unroll
      for (int w = 0; w < kSrtW; ++w) {
        const int c = cnt[d * kSrtW + w];
        cnt[d * kSrtW + w] = tot;
        tot += c;
      }
      int x = tot;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, s);
        if (lane >= s) x += y;
      }
      if (lane == 31) s_wsum[wid] = x;
      __syncthreads();
      int pre = 0;
#pragma unroll
      for (int w = 0; w < kSrtW; ++w) pre += w < wid ? s_wsum[w] : 0;
      dstart[d] = pre + x - tot;
      if (d == 255) s_tn = pre + x;
    }
    __syncthreads();
    // stage the tile in digit order
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (rk[j] == 0xFFFFFFFFu) continue;
      const int d = (int)(rk[j] >> 16);
      const int pos = dstart[d] + cnt[d * kSrtW + wid] + (int)(rk[j] & 0xFFFFu);
      skey[pos] = key[j];
      smsk[pos] = m[j];
#pragma unroll
      for (int c = 0; c < NV; ++c) sval[c * T + pos] = v[j][c];
    }
    __syncthreads();
    // write out: consecutive staged rows of one digit go to consecutive output rows
    const int tvalid = s_tn;
    for (int i = tid; i < tvalid; i += kSrtThreads) {
      const uint32_t k = skey[i];
      const int d = (int)((k >> (8 * b)) & 255u);
      const int64_t g = cur[d] + (i - dstart[d]);
      q.key[ob][g] = k;
      q.msk[ob][g] = smsk[i];
#pragma unroll
      for (int c = 0; c < NV; ++c) q.val[ob][c][g] = sval[c * T + i];
    }
    __syncthreads();
    cur[tid] += tot;
#pragma unroll
    for (int w = 0; w < kSrtW; ++w) cnt[tid * kSrtW + w] = 0;
    __syncthreads();
  }
}

// pac_hash (R1, R2) of the sorted pu keys, in place (pass 0 moved the raw keys).  8 keys per
// thread: mix, popcount and draw word 0 branch-free for all of them, then the keys that still need
// flips are queued per warp and finished with all 32 lanes busy (no per-lane straggler loops).
constexpr int kHashR = 8;
__global__ void __launch_bounds__(256) k_srt_hash(SrtPlan q) {
  __shared__ unsigned long long qm[8][32 * kHashR], qw[8][32 * kHashR];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long* m = q.msk[(srt_nactive(q, q.width) - 1) & 1];
  const int64_t n = (int64_t)q.ctr[0];
  const int64_t step = (int64_t)gridDim.x * 256 * kHashR;
  for (int64_t b0 = (int64_t)blockIdx.x * 256 * kHashR + wid * 32 * kHashR; b0 < n; b0 += step) {
    unsigned long long x[kHashR];
#pragma unroll
    for (int j = 0; j < kHashR; ++j) {
      const int64_t r = b0 + 32 * j + lane;
      x[j] = r < n ? m[r] : 0ull;
    }
    int qn = 0;
#pragma unroll
    for (int j = 0; j < kHashR; j += 2) {
      HashState ha, hb;
      pac_hash_begin2(x[j], x[j + 1], q.salt, ha, hb);
      x[j] = hash_mask_now(ha);
      x[j + 1] = hash_mask_now(hb);
      const unsigned ba = __ballot_sync(0xffffffffu, ha.k > 0);
      if (ha.k > 0) {
        const int qi = qn + __popc(ba & lt);
        qm[wid][qi] = x[j];
        qw[wid][qi] = ha.w0 | 0ull;
      }
      qn += __popc(ba);
      const unsigned bb = __ballot_sync(0xffffffffu, hb.k > 0);
      if (hb.k > 0) {
        const int qi = qn + __popc(bb & lt);
        qm[wid][qi] = x[j + 1];
        qw[wid][qi] = hb.w0;
      }
      qn += __popc(bb);
    }
    __syncwarp();
    for (int qi = lane; qi < qn; qi += 32) qm[wid][qi] = pac_hash_continue(qm[wid][qi], qw[wid][qi]);
    __syncwarp();
    // queue order = (pair, a before b, lane): walk it again to pick up the finished masks
    int qp = 0;
#pragma unroll
    for (int j = 0; j < kHashR; j += 2) {
      const bool sa = __popcll(x[j]) != 32;
      const unsigned ba = __ballot_sync(0xffffffffu, sa);
      if (sa) x[j] = qm[wid][qp + __popc(ba & lt)];
      qp += __popc(ba);
      const bool sb = __popcll(x[j + 1]) != 32;
      const unsigned bb = __ballot_sync(0xffffffffu, sb);
      if (sb) x[j + 1] = qm[wid][qp + __popc(bb & lt)];
      qp += __popc(bb);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kHashR; ++j) {
      const int64_t r = b0 + 32 * j + lane;
      if (r < n) m[r] = x[j];
    }
  }
}

// group starts (row 0, or key != previous key) per agg chunk of the sorted rows: warp = chunk,
// CTA = block of 8 chunks; hcnt[ch] = starts in the block's chunks before ch, hblk = block totals
__global__ void __launch_bounds__(256) k_srt_heads(SrtPlan q) {
  __shared__ int wc[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ch = blockIdx.x * 8 + wid;
  const int64_t n = (int64_t)q.ctr[0];
  const uint32_t* key = q.key[(srt_nactive(q, q.width) - 1) & 1];
  const int64_t c0 = (int64_t)ch * kSrtCH, c1 = min(n, c0 + kSrtCH);
  int h = 0;
  if (ch < q.nch) {
#pragma unroll 8
    for (int64_t b = c0; b < c1; b += 32) {
      const int64_t r = b + lane;
      bool hd = false;
      if (r < c1) hd = r == 0 || key[r] != key[r - 1];
      h += __popc(__ballot_sync(0xffffffffu, hd));
    }
  }
  if (lane == 0) wc[wid] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int w = 0; w < 8; ++w) {
      if (blockIdx.x * 8 + w < q.nch) q.hcnt[blockIdx.x * 8 + w] = run;
      run += wc[w];
    }
    q.hblk[blockIdx.x] = run;
  }
}

// exclusive scan of the block totals (one CTA); the group count -> the dictionary counter
__global__ void __launch_bounds__(1024) k_srt_hscan(SrtPlan q, int* gcounter) {
  __shared__ int ws[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nb = (q.nch + 7) / 8;
  const int per = (nb + 1023) / 1024;
  const int e0 = min(nb, tid * per), e1 = min(nb, e0 + per);
  int s = 0;
#pragma unroll 8
  for (int i = e0; i < e1; ++i) s += q.hblk[i];
  int x = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int v = ws[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += y;
    }
    ws[lane] = v;
  }
  __syncthreads();
  int run = (wid > 0 ? ws[wid - 1] : 0) + x - s;
#pragma unroll 8
  for (int i = e0; i < e1; ++i) {
    const int c = q.hblk[i];
    q.hblk[i] = run;
    run += c;
  }
  if (tid == 1023) *gcounter = ws[31];
}
// group starts before chunk ch (after k_srt_hscan)
__device__ __forceinline__ int srt_chunk_base(const SrtPlan& q, int ch) { return q.hblk[ch >> 3] + q.hcnt[ch]; }

// rows of the groups that span a chunk boundary start at zero (their chunks add with atomics)
__global__ void __launch_bounds__(256) k_srt_bzero(SrtPlan q, SrtOut o, int64_t G_cap) {
  const int lane = threadIdx.x & 31;
  const int ch = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (ch >= q.nch || ch == 0) return;
  const int64_t n = (int64_t)q.ctr[0];
  const int64_t c0 = (int64_t)ch * kSrtCH;
  if (c0 >= n) return;
  const uint32_t* key = q.key[(srt_nactive(q, q.width) - 1) & 1];
  if (key[c0] != key[c0 - 1]) return;
  const int slot = srt_chunk_base(q, ch) - 1;
  if (slot < 0 || slot >= G_cap) return;
  const size_t bw = (size_t)slot * kM;
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 32 * h;
    o.t.d_count[bw + j] = 0;
    for (int a = 0; a < o.n_aggs; ++a) {
      if (o.kind[a] == 1) ((int64_t*)o.t.d_world[a])[bw + j] = 0;
      else if (o.kind[a] == 2) ((double*)o.t.d_world[a])[bw + j] = 0.0;
    }
  }
  if (lane == 0) o.t.d_rows[slot] = 0;
}

// K of the groups that span a chunk boundary, from their finished counts (R5)
__global__ void __launch_bounds__(256) k_srt_bpresence(SrtPlan q, SrtOut o, int64_t G_cap) {
  const int lane = threadIdx.x & 31;
  const int ch = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (ch >= q.nch || ch == 0) return;
  const int64_t n = (int64_t)q.ctr[0];
  const int64_t c0 = (int64_t)ch * kSrtCH;
  if (c0 >= n) return;
  const uint32_t* key = q.key[(srt_nactive(q, q.width) - 1) & 1];
  if (key[c0] != key[c0 - 1]) return;
  const int slot = srt_chunk_base(q, ch) - 1;
  if (slot < 0 || slot >= G_cap) return;
  const size_t bw = (size_t)slot * kM;
  const uint64_t K = (uint64_t)__ballot_sync(0xffffffffu, o.t.d_count[bw + lane] != 0) |
                     ((uint64_t)__ballot_sync(0xffffffffu, o.t.d_count[bw + lane + 32] != 0) << 32);
  if (lane == 0) o.t.d_presence[slot] = K;
}

// R15 overflow bound over the finished table (after k_finish_count wrote the status)
__global__ void k_srt_overflow(const unsigned long long* gmaxabs, pac_table t, int64_t G_cap) {
  const unsigned long long ma = *gmaxabs;
  if (!ma) return;
  const int64_t G = min((int64_t)*t.d_num_groups, G_cap);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x)
    if ((unsigned long long)t.d_rows[g] > (0x7FFFFFFFFFFFFFFFull / ma)) atomicExch(t.d_status, PAC_E_OVERFLOW);
}

// Streaming 64-world fold over the sorted rows.  Per warp: one chunk of kSrtCH rows, windows of
// 32 rows staged twice in shared memory (row l at A[l] and at B[l + 1], so a segment starting at
// an odd row is 16-byte aligned in B, as run_body's row-pair loads need); rows past the window are
// zero (finite padding, run_body's contract).
constexpr int kSrtS = 48;  // staged rows per copy
template <int NI, int NF>
__global__ void __launch_bounds__(256, NI + NF <= 1 ? PAC_SRT_AGG_MINB : 2) k_srt_agg(SrtPlan q, AggPlan p, SrtOut o) {
  constexpr int NV = NI + NF;
  constexpr int ROWW = 1 + NV;  // 8-byte words per staged row (mask, values)
  __shared__ __align__(16) unsigned long long stage[8][2][ROWW * kSrtS];
  __shared__ uint4 xcs[32];
  __shared__ uint2 xcs2[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < 32) store_xpose(xcs, xcs2, threadIdx.x);
  for (int i = threadIdx.x; i < 8 * 2 * ROWW * kSrtS; i += blockDim.x) (&stage[0][0][0])[i] = 0ull;
  __syncthreads();
  const XposeConst xc = load_xpose(xcs, xcs2, lane);
  unsigned long long* A = stage[wid][0];
  unsigned long long* B = stage[wid][1];
  const int64_t n = (int64_t)q.ctr[0];
  const int fb = (srt_nactive(q, q.width) - 1) & 1;
  const uint32_t* key = q.key[fb];
  const unsigned long long* msk = q.msk[fb];
  const unsigned long long* vals[NV > 0 ? NV : 1];
#pragma unroll
  for (int c = 0; c < NV; ++c) vals[c] = q.val[fb][c];
  const int64_t G_cap = p.G_cap;
  unsigned long long maxabs = 0;
  WarpAcc<NI, NF, 0> acc;
  const int nwarps = gridDim.x * 8;
  for (int ch = blockIdx.x * 8 + wid; ch < q.nch; ch += nwarps) {
    const int64_t c0 = (int64_t)ch * kSrtCH;
    if (c0 >= n) break;
    const int64_t c1 = min(n, c0 + kSrtCH);
    uint32_t prev = c0 > 0 ? key[c0 - 1] : ~key[0];
    const bool end_cont = c1 < n && key[c1] == key[c1 - 1];
    int slot = srt_chunk_base(q, ch) - 1;  // group of the row before the first head of the chunk
    bool cur_ok = c0 > 0 && key[c0] == prev;  // a group continuing from the previous chunk
    bool cur_here = false;                   // the current group's first row is in this chunk
    uint32_t cur_key = key[c0];
    unsigned long long rows = 0;
    acc.reset();
    auto flush = [&](bool atomic) {
      if (slot < 0 || slot >= G_cap) return;
      const size_t bw = (size_t)slot * kM;
      if (!atomic) {
        o.t.d_count[bw + lane] = (int64_t)acc.c0;
        o.t.d_count[bw + lane + 32] = (int64_t)acc.c1;
        for (int a = 0; a < o.n_aggs; ++a) {
          const int kd = o.kind[a], ix = o.idx[a];
          if (kd == 1) {
            int64_t* w = (int64_t*)o.t.d_world[a];
            w[bw + lane] = ix == 0 ? acc.ia0[0] : acc.ia0[NI > 1 ? 1 : 0];
            w[bw + lane + 32] = ix == 0 ? acc.ia1[0] : acc.ia1[NI > 1 ? 1 : 0];
          } else if (kd == 2) {
            double* w = (double*)o.t.d_world[a];
            w[bw + lane] = ix == 0 ? acc.fa0[0] : acc.fa0[NF > 1 ? 1 : 0];
            w[bw + lane + 32] = ix == 0 ? acc.fa1[0] : acc.fa1[NF > 1 ? 1 : 0];
          }
        }
        const uint64_t K = (uint64_t)__ballot_sync(0xffffffffu, acc.c0 != 0) |
                           ((uint64_t)__ballot_sync(0xffffffffu, acc.c1 != 0) << 32);
        if (lane == 0) {
          o.t.d_rows[slot] = (int64_t)rows;
          o.t.d_presence[slot] = K;
        }
      } else {
        if (acc.c0) atomicAdd((unsigned long long*)&o.t.d_count[bw + lane], (unsigned long long)acc.c0);
        if (acc.c1) atomicAdd((unsigned long long*)&o.t.d_count[bw + lane + 32], (unsigned long long)acc.c1);
        for (int a = 0; a < o.n_aggs; ++a) {
          const int kd = o.kind[a], ix = o.idx[a];
          if (kd == 1) {
            unsigned long long* w = (unsigned long long*)o.t.d_world[a];
            const long long x0 = ix == 0 ? acc.ia0[0] : acc.ia0[NI > 1 ? 1 : 0];
            const long long x1 = ix == 0 ? acc.ia1[0] : acc.ia1[NI > 1 ? 1 : 0];
            if (x0) atomicAdd(&w[bw + lane], (unsigned long long)x0);
            if (x1) atomicAdd(&w[bw + lane + 32], (unsigned long long)x1);
          } else if (kd == 2) {
            double* w = (double*)o.t.d_world[a];
            if (acc.c0) atomicAdd(&w[bw + lane], ix == 0 ? acc.fa0[0] : acc.fa0[NF > 1 ? 1 : 0]);
            if (acc.c1) atomicAdd(&w[bw + lane + 32], ix == 0 ? acc.fa1[0] : acc.fa1[NF > 1 ? 1 : 0]);
          }
        }
        if (lane == 0 && rows) atomicAdd((unsigned long long*)&o.t.d_rows[slot], rows);
      }
      if (cur_here && lane == 0) o.t.d_group_key[slot] = (uint64_t)cur_key;
    };
    for (int64_t wb = c0; wb < c1; wb += 32) {
      const int64_t r = wb + lane;
      const bool valid = r < c1;
      const uint32_t k = valid ? key[r] : 0u;
      const unsigned long long mk = valid ? msk[r] : 0ull;
      unsigned long long v[NV > 0 ? NV : 1];
#pragma unroll
      for (int c = 0; c < NV; ++c) v[c] = valid ? vals[c][r] : 0ull;
      const int nv = (int)min((int64_t)32, c1 - wb);
      uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
      if (lane == 0) kp = prev;
      const unsigned H = __ballot_sync(0xffffffffu, valid && k != kp);
      prev = __shfl_sync(0xffffffffu, k, nv - 1);
      // runtime contracts of run_body's fast tables
      bool sm = true, fi = true;
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        const long long x = (long long)v[c];
        const unsigned long long ax = x < 0 ? 0ull - (unsigned long long)x : (unsigned long long)x;
        maxabs = ax > maxabs ? ax : maxabs;
        sm = sm && ax < (1ull << 26);
      }
#pragma unroll
      for (int c = 0; c < NF; ++c) fi = fi && finite_bits(__longlong_as_double((long long)v[c]));
      const bool small = NI == 0 || __all_sync(0xffffffffu, sm);
      const bool fin = NF == 0 || __all_sync(0xffffffffu, fi);
      // stage: A[l] = row l, B[l + 1] = row l (masks, then the value columns, stride kSrtS)
      A[lane] = mk;
#pragma unroll
      for (int c = 0; c < NV; ++c) A[(1 + c) * kSrtS + lane] = v[c];
      if (H & ~1u) {  // a segment may start at an odd row: the shifted copy
        B[lane + 1] = mk;
#pragma unroll
        for (int c = 0; c < NV; ++c) B[(1 + c) * kSrtS + lane + 1] = v[c];
      }
      __syncwarp();
      int s = 0;
      while (s < nv) {
        if ((H >> s) & 1u) {  // a new group starts at row s
          if (cur_ok) flush(!cur_here);
          acc.reset();
          rows = 0;
          ++slot;
          cur_ok = true;
          cur_here = true;
          cur_key = __shfl_sync(0xffffffffu, k, s);
        }
        const unsigned rest = s < 31 ? (H & ~((2u << s) - 1u)) : 0u;
        const int e = rest ? __ffs(rest) - 1 : nv;
        const int len = e - s;
        const unsigned long long* base = (s & 1) ? B + s + 1 : A + s;
        const long long* iv = (const long long*)(base + kSrtS);
        const double* fv = (const double*)(base + (1 + NI) * kSrtS);
        if (len == 32 && small && fin)
          run_body<NI, NF, 0, false>(acc, base, iv, kSrtS, fv, kSrtS, nullptr, 32, xc, lane);
        else
          run_body<NI, NF, 0, true>(acc, base, iv, kSrtS, fv, kSrtS, nullptr, len, xc, lane, small, fin);
        rows += (unsigned long long)len;
        s = e;
      }
      __syncwarp();
    }
    if (cur_ok) flush(!cur_here || end_cont);
  }
  if (NI > 0) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, maxabs, d);
      maxabs = o > maxabs ? o : maxabs;
    }
    if (lane == 0 && maxabs) atomicMax(p.gmaxabs, maxabs);
  }
}

// ------------------------------------------------------------------ host
static size_t srt_al(size_t x) { return (x + 255) & ~(size_t)255; }
// CTAs of the passes: as many as fit resident (k_srt_scatter: 3 per SM for rows of <= 1 value
// column, 2 above -- registers), one chunk each
static int srt_grid(int sms, int nv) { return std::min((nv <= 1 ? PAC_SRT_MINB : 2) * sms, kScanMaxGrid); }

size_t srt_ws_bytes(int64_t n_rows, int nv, int sms) {
  const size_t rows = (size_t)std::max<int64_t>(n_rows, 1);
  size_t b = 0;
  for (int k = 0; k < 2; ++k) {
    b += srt_al(rows * 4) + srt_al(rows * 8);
    for (int c = 0; c < nv; ++c) b += srt_al(rows * 8);
  }
  b += srt_al((size_t)256 * kScanMaxGrid * 8) + srt_al(64) + srt_al(4 * 256 * 8);
  b += srt_al(4 * (size_t)((n_rows + kSrtCH - 1) / kSrtCH + 1));
  b += srt_al(4 * (size_t)((n_rows + kSrtCH - 1) / kSrtCH / 8 + 2));
  return b;
}

// staging (mask, values, key) + warp counters + digit starts + cursors
static size_t srt_smem(int nv, bool) {
  return (size_t)kSrtThreads * srt_rpt(nv) * (8 + 8 * nv + 4) + 256 * kSrtW * 4 + 256 * 4 + 256 * 8;
}

template <int NV>
static cudaError_t srt_pass(const SrtPlan& q, int b, cudaStream_t st) {
  const size_t sm = srt_smem(NV, b == 0);
  auto ks = b == 0 ? k_srt_scatter<NV, true> : k_srt_scatter<NV, false>;
  cudaError_t e = cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  if (b == 0) k_srt_hist<true><<<q.grid, kHistThreads, 0, st>>>(q, b);
  else k_srt_hist<false><<<q.grid, kHistThreads, 0, st>>>(q, b);
  k_srt_scan<<<256, 32, 0, st>>>(q, b);
  ks<<<q.grid, kSrtThreads, sm, st>>>(q, b);
  for (int i = 0; i < 3; ++i) note_launch();
  return cudaGetLastError();
}

using SrtAggFn = void (*)(const SrtPlan&, const AggPlan&, const SrtOut&, int, cudaStream_t);
template <int NI, int NF>
static void srt_agg_launch(const SrtPlan& q, const AggPlan& p, const SrtOut& o, int grid, cudaStream_t st) {
  k_srt_agg<NI, NF><<<grid, 256, 0, st>>>(q, p, o);
}
static const SrtAggFn kSrtAgg[3][3] = {
    {srt_agg_launch<0, 0>, srt_agg_launch<0, 1>, srt_agg_launch<0, 2>},
    {srt_agg_launch<1, 0>, srt_agg_launch<1, 1>, srt_agg_launch<1, 2>},
    {srt_agg_launch<2, 0>, srt_agg_launch<2, 1>, srt_agg_launch<2, 2>}};

// Runs the whole sort-first aggregation into the provisional table of `p` (slots in canonical
// order, *p.gcounter = number of groups).  ws: srt_ws_bytes(n_rows, ni + nf, sms) bytes.
int srt_run(const AggPlan& p, const int64_t* d_pu_key, const uint64_t* d_mask, const pac_key_col* keys, int n_keys,
            int width, int64_t n_rows, int sms, char* ws, const pac_table* out, int n_aggs, const int* kinds,
            const int* idx, cudaStream_t st) {
  SrtOut o{};
  o.t = *out;
  o.n_aggs = n_aggs;
  for (int a = 0; a < n_aggs; ++a) {
    o.kind[a] = kinds[a];
    o.idx[a] = idx[a];
  }
  SrtPlan q{};
  q.n = n_rows;
  q.pu = (const long long*)d_pu_key;
  q.mask_in = (const unsigned long long*)d_mask;
  q.salt = p.salt;
  q.n_keys = n_keys;
  q.width = width;
  for (int c = 0; c < n_keys; ++c) {
    q.key_col[c] = keys[c].d_col;
    q.key_bytes[c] = keys[c].elem_bytes;
  }
  q.nv = p.ni + p.nf;
  q.hash0 = (d_pu_key && q.nv >= 1 && !getenv("PAC_SRT_HASH_KERNEL")) ? 1 : 0;  // the queue lives in the value staging
  for (int c = 0; c < p.ni; ++c) q.val_in[c] = (const unsigned long long*)p.icol[c];
  for (int c = 0; c < p.nf; ++c) q.val_in[p.ni + c] = (const unsigned long long*)p.fcol[c];
  const size_t rows = (size_t)std::max<int64_t>(n_rows, 1);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* x = ws + off;
    off += srt_al(bytes);
    return x;
  };
  for (int k = 0; k < 2; ++k) {
    q.key[k] = (uint32_t*)take(rows * 4);
    q.msk[k] = (unsigned long long*)take(rows * 8);
    for (int c = 0; c < q.nv; ++c) q.val[k][c] = (unsigned long long*)take(rows * 8);
  }
  q.grid = srt_grid(sms, q.nv);
  q.hist = (long long*)take((size_t)256 * q.grid * 8);
  q.ctr = (unsigned long long*)take(64);
  q.dtot = (unsigned long long*)take(4 * 256 * 8);
  if (cudaMemsetAsync(q.dtot, 0, 4 * 256 * 8, st) != cudaSuccess) return PAC_E_CUDA;
  q.nch = (int)((n_rows + kSrtCH - 1) / kSrtCH);
  q.hcnt = (int*)take(4 * (size_t)(q.nch + 1));
  q.hblk = (int*)take(4 * (size_t)(q.nch / 8 + 2));
  const unsigned long long init[3] = {0ull, 0ull, ~0ull};
  if (cudaMemcpyAsync(q.ctr, init, sizeof(init), cudaMemcpyHostToDevice, st) != cudaSuccess) return PAC_E_CUDA;
  for (int b = 0; b < width; ++b) {
    cudaError_t e;
    switch (q.nv) {
      case 0: e = srt_pass<0>(q, b, st); break;
      case 1: e = srt_pass<1>(q, b, st); break;
      case 2: e = srt_pass<2>(q, b, st); break;
      case 3: e = srt_pass<3>(q, b, st); break;
      default: e = srt_pass<4>(q, b, st); break;
    }
    if (e != cudaSuccess) return PAC_E_CUDA;
  }
  if (q.nch > 0) {
    const int hb = (q.nch + 7) / 8;
    if (d_pu_key && !q.hash0) {
      k_srt_hash<<<sms * 8, 256, 0, st>>>(q);
      note_launch();
    }
    k_srt_heads<<<hb, 256, 0, st>>>(q);
    k_srt_hscan<<<1, 1024, 0, st>>>(q, p.gcounter);
    k_srt_bzero<<<hb, 256, 0, st>>>(q, o, p.G_cap);
    kSrtAgg[p.ni][p.nf](q, p, o, std::min(hb, sms * 8), st);
    k_srt_bpresence<<<hb, 256, 0, st>>>(q, o, p.G_cap);
    for (int i = 0; i < 5; ++i) note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

// after k_finish_count: the R15 overflow bound (k_gather's check, which this path skips)
void srt_finish(const AggPlan& p, const pac_table* out, int sms, cudaStream_t st) {
  if (p.ni > 0) {
    k_srt_overflow<<<sms * 4, 256, 0, st>>>(p.gmaxabs, *out, p.G_cap);
    note_launch();
  }
}

}  // namespace pac
