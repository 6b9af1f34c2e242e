// libpac: flat merge buffers for the cross-GPU combine (§8 a5/e; the paper's analogue is
// DuckDB's thread-local partial aggregates + state.combine).
//
// A partial table laid out on the common group dictionary is packed into three flat buffers,
// one per NCCL reduction, so the whole merge is three all_reduce calls with no host
// synchronisation:
//   i64_sum  SUM   rows [G], count [G][64] (if any), per SUM_I64 aggregate [G][64]
//   f64_sum  SUM   per SUM_F64 / AVG_F64 aggregate [G][64]
//   i64_min  MIN   [0] fingerprint f, [1] ~f, [2] ~status, then per MIN aggregate [G][64]
//                  enc_f64 extremes and per MAX aggregate [G][64] ~enc_f64 (bitwise NOT
//                  reverses the int64 order, so one MIN reduction serves both); a world not
//                  in K packs the empty sentinel
// G = G_cap (fixed sizes; groups past num_groups pack the empty state).  The MIN/MAX merge
// runs on the order-preserving encoding, so it follows R31 exactly (NaN largest) whatever
// NCCL's floating-point min/max does with NaN, and presence survives: after the merge a world
// of a MIN/MAX-only table is present iff its merged extreme is not the sentinel -- the OR of
// the ranks' presence bits that NCCL has no operator for.
// Fingerprint: a wrapping sum of a mix of (rank-independent) group keys and their positions
// plus num_groups.  After the MIN reduction min(f) = i64_min[0] and max(f) = ~i64_min[1]; if
// they differ, the ranks did not share one dictionary and unpack marks the table
// PAC_E_MERGE (nothing is released from it, pac_finalize).
#include <algorithm>

#include "common.cuh"

namespace pac {

void note_launch();

struct MergeLayout {
  int n_i64, n_f64, n_min;     // elements
  int has_count;
  int A;
  int kind[PAC_MAX_AGGS];
  int off[PAC_MAX_AGGS];       // element offset of aggregate a's [G][64] block in its buffer
};

static int merge_layout(const pac_agg_spec* aggs, int n_aggs, int64_t G, MergeLayout* m) {
  if (!aggs || n_aggs < 1 || n_aggs > PAC_MAX_AGGS || G < 1 || G > (1 << 24)) return PAC_E_INVAL;
  bool only_mm = true;
  for (int a = 0; a < n_aggs; ++a) {
    const int k = aggs[a].kind;
    if (k < PAC_COUNT || k > PAC_MAX_F64) return PAC_E_INVAL;
    if (k != PAC_MIN_F64 && k != PAC_MAX_F64) only_mm = false;
  }
  *m = MergeLayout{};
  m->A = n_aggs;
  m->has_count = only_mm ? 0 : 1;
  int64_t i64 = G + (m->has_count ? G * kM : 0), f64 = 0, mn = 3;
  for (int a = 0; a < n_aggs; ++a) {
    const int k = aggs[a].kind;
    m->kind[a] = k;
    if (k == PAC_SUM_I64) { m->off[a] = (int)i64; i64 += G * kM; }
    else if (k == PAC_SUM_F64 || k == PAC_AVG_F64) { m->off[a] = (int)f64; f64 += G * kM; }
    else if (k == PAC_MIN_F64 || k == PAC_MAX_F64) { m->off[a] = (int)mn; mn += G * kM; }
    else m->off[a] = -1;
  }
  if (i64 > INT32_MAX || f64 > INT32_MAX || mn > INT32_MAX) return PAC_E_INVAL;
  m->n_i64 = (int)i64;
  m->n_f64 = (int)f64;
  m->n_min = (int)mn;
  return PAC_OK;
}

__device__ __forceinline__ unsigned long long fp_term(uint64_t key, int64_t g) {
  return fmix64(key ^ (0x9E3779B97F4A7C15ull * (uint64_t)(g + 1)));
}

// one warp per group (lane j: worlds j, j+32); block 0 also seeds the fingerprint words
__global__ void k_merge_pack(pac_table t, int64_t G_cap, MergeLayout m, long long* i64, double* f64,
                             long long* mn, unsigned long long* fp) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int64_t G = min(*t.d_num_groups, G_cap);
  for (int64_t g = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); g < G_cap; g += (int64_t)gridDim.x * wpb) {
    const bool live = g < G;
    const uint64_t K = live ? t.d_presence[g] : 0ull;
    if (lane == 0) {
      i64[g] = live ? t.d_rows[g] : 0;
      if (live) atomicAdd(fp, fp_term(t.d_group_key[g], g));
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      const size_t e = (size_t)g * kM + j;
      const bool in = (K >> j) & 1ull;
      if (m.has_count) i64[G_cap + e] = live ? t.d_count[e] : 0;
      for (int a = 0; a < m.A; ++a) {
        const int k = m.kind[a];
        if (k == PAC_SUM_I64) i64[m.off[a] + e] = live ? ((const long long*)t.d_world[a])[e] : 0;
        else if (k == PAC_SUM_F64 || k == PAC_AVG_F64) f64[m.off[a] + e] = live ? ((const double*)t.d_world[a])[e] : 0.0;
        else if (k == PAC_MIN_F64) mn[m.off[a] + e] = in ? enc_f64(((const double*)t.d_world[a])[e]) : kMinEmpty;
        else if (k == PAC_MAX_F64) mn[m.off[a] + e] = ~(in ? enc_f64(((const double*)t.d_world[a])[e]) : kMaxEmpty);
      }
    }
  }
}

__global__ void k_merge_pack_head(pac_table t, int64_t G_cap, long long* mn, unsigned long long* fp) {
  // after k_merge_pack: f = sum of the key terms + num_groups
  const unsigned long long f = *fp + fmix64((uint64_t)min(*t.d_num_groups, G_cap) + 0xD6E8FEB86659FD93ull);
  mn[0] = (long long)f;
  mn[1] = ~(long long)f;
  mn[2] = ~(long long)*t.d_status;
}

__global__ void k_merge_unpack(pac_table t, int64_t G_cap, MergeLayout m, const long long* i64, const double* f64,
                               const long long* mn) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int64_t G = min(*t.d_num_groups, G_cap);
  for (int64_t g = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); g < G; g += (int64_t)gridDim.x * wpb) {
    bool pa = false, pb = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      const size_t e = (size_t)g * kM + j;
      bool present = false;
      if (m.has_count) {
        const long long c = i64[G_cap + e];
        t.d_count[e] = c;
        present = c > 0;  // R5: K == {j : count_j > 0}
      }
      for (int a = 0; a < m.A; ++a) {
        const int k = m.kind[a];
        if (k == PAC_SUM_I64) {
          ((long long*)t.d_world[a])[e] = i64[m.off[a] + e];
        } else if (k == PAC_SUM_F64 || k == PAC_AVG_F64) {
          ((double*)t.d_world[a])[e] = f64[m.off[a] + e];
        } else if (k == PAC_MIN_F64) {
          const long long x = mn[m.off[a] + e];
          ((double*)t.d_world[a])[e] = dec_min(x);
          if (!m.has_count) present |= x != kMinEmpty;
        } else if (k == PAC_MAX_F64) {
          const long long x = ~mn[m.off[a] + e];
          ((double*)t.d_world[a])[e] = dec_max(x);
          if (!m.has_count) present |= x != kMaxEmpty;
        }
      }
      if (h == 0) pa = present; else pb = present;
    }
    const uint64_t K = (uint64_t)__ballot_sync(0xffffffffu, pa) | ((uint64_t)__ballot_sync(0xffffffffu, pb) << 32);
    if (lane == 0) {
      t.d_presence[g] = K;
      t.d_rows[g] = i64[g];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long fmin = mn[0], fmax = ~mn[1];
    const int st = (int)~mn[2];  // the largest status of any rank
    *t.d_status = fmin != fmax ? PAC_E_MERGE : st;
  }
}

}  // namespace pac

using namespace pac;

extern "C" int pac_merge_sizes(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, int64_t* n_i64_sum,
                               int64_t* n_f64_sum, int64_t* n_i64_min) {
  MergeLayout m;
  const int rc = merge_layout(aggs, n_aggs, G_cap, &m);
  if (rc) return rc;
  if (n_i64_sum) *n_i64_sum = m.n_i64;
  if (n_f64_sum) *n_f64_sum = m.n_f64;
  if (n_i64_min) *n_i64_min = m.n_min;
  return PAC_OK;
}

static int table_ok(const pac_table* t, const MergeLayout& m, const pac_agg_spec* aggs) {
  if (!t || (t->m != 0 && t->m != 64) || !t->d_num_groups || !t->d_status || !t->d_rows || !t->d_presence ||
      !t->d_group_key)
    return PAC_E_INVAL;
  if (m.has_count && !t->d_count) return PAC_E_INVAL;
  for (int a = 0; a < m.A; ++a)
    if (aggs[a].kind != PAC_COUNT && !t->d_world[a]) return PAC_E_INVAL;
  return PAC_OK;
}

extern "C" int pac_merge_pack(const pac_table* t, const pac_agg_spec* aggs, int n_aggs, int64_t G_cap,
                              int64_t* d_i64_sum, double* d_f64_sum, int64_t* d_i64_min, pac_stream_t stream) {
  MergeLayout m;
  int rc = merge_layout(aggs, n_aggs, G_cap, &m);
  if (rc) return rc;
  if ((rc = table_ok(t, m, aggs))) return rc;
  if (!d_i64_sum || !d_i64_min || (m.n_f64 > 0 && !d_f64_sum)) return PAC_E_INVAL;
  cudaStream_t st = (cudaStream_t)stream;
  // the fingerprint accumulates in i64_min[0] (seeded 0), then the head kernel finishes it
  unsigned long long* fp = (unsigned long long*)d_i64_min;
  if (cudaMemsetAsync(fp, 0, 8, st) != cudaSuccess) return PAC_E_CUDA;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((G_cap + 7) / 8, 148 * 16));
  k_merge_pack<<<blocks, 256, 0, st>>>(*t, G_cap, m, (long long*)d_i64_sum, d_f64_sum, (long long*)d_i64_min, fp);
  k_merge_pack_head<<<1, 1, 0, st>>>(*t, G_cap, (long long*)d_i64_min, fp);
  note_launch();
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_merge_unpack(const pac_table* t, const pac_agg_spec* aggs, int n_aggs, int64_t G_cap,
                                const int64_t* d_i64_sum, const double* d_f64_sum, const int64_t* d_i64_min,
                                pac_stream_t stream) {
  MergeLayout m;
  int rc = merge_layout(aggs, n_aggs, G_cap, &m);
  if (rc) return rc;
  if ((rc = table_ok(t, m, aggs))) return rc;
  if (!d_i64_sum || !d_i64_min || (m.n_f64 > 0 && !d_f64_sum)) return PAC_E_INVAL;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((G_cap + 7) / 8, 148 * 16));
  k_merge_unpack<<<blocks, 256, 0, (cudaStream_t)stream>>>(*t, G_cap, m, (const long long*)d_i64_sum, d_f64_sum,
                                                           (const long long*)d_i64_min);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
