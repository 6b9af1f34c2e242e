// libpac: the categorical path after the aggregate (§8 f1; §3, §4,
// P:L1643-1647; readings DESIGN.md R22-R26).
//
//  * k_world_vector   table cell -> world vector (y in the released scale, presence K), R22
//  * k_lift           pointwise binary op over world vectors / broadcast scalars, R23
//  * k_lift_cmp       pointwise comparison -> 64 world booleans (one ballot pair per vector)
//  * k_cmp_index      per group: the 64 world values sorted (absent / NaN worlds excluded) and
//                     the 65 suffix masks S[p] = {worlds at sorted positions >= p}
//  * k_select_cmp,    row-parallel pac_select_<cmp> / pac_filter_<cmp>: the 64 comparisons of a
//    k_filter_cmp     row's value v against its group's world vector reduce to two 7-step
//                     binary searches in the sorted values (lb = #{c < v}, ub = #{c <= v}) and
//                     one or two suffix-mask loads -- O(log m) loads per row instead of m
//                     compares (R26)
//  * k_select,        pac_select / pac_filter of world booleans given per group (Eq. pac-select,
//    k_filter         Eq. pac-filter; R25)
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace pac {

uint64_t session_seed(const pac_session* s);  // session.cu

constexpr int kIdxWords = PAC_CMP_INDEX_WORDS;  // 64 sorted values, 65 suffix masks, nv

// ------------------------------------------------------------------ world vectors (R22)
__global__ void k_world_vector(const int64_t* __restrict__ num_groups, int64_t G_cap, int kind,
                               const int64_t* __restrict__ count, const void* __restrict__ world,
                               const uint64_t* __restrict__ K, double* __restrict__ y,
                               uint64_t* __restrict__ pres) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int64_t G = min(*num_groups, G_cap);
  for (int64_t g = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); g < G_cap; g += (int64_t)gridDim.x * wpb) {
    const uint64_t Kg = g < G ? K[g] : 0ull;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      const size_t c = (size_t)g * kM + j;
      double v = 0.0;
      if ((Kg >> j) & 1ull) {  // R9: an absent world reads 0
        switch (kind) {
          case PAC_COUNT: v = 2.0 * (double)count[c]; break;
          case PAC_SUM_I64: v = 2.0 * (double)((const int64_t*)world)[c]; break;
          case PAC_SUM_F64: v = 2.0 * ((const double*)world)[c]; break;
          case PAC_AVG_F64: v = __ddiv_rn(((const double*)world)[c], (double)count[c]); break;
          default: v = ((const double*)world)[c]; break;
        }
      }
      y[c] = v;
    }
    if (lane == 0) pres[g] = Kg;
  }
}

// ------------------------------------------------------------------ lifting (R23)
__device__ __forceinline__ double lift_op(int op, double a, double b) {
  switch (op) {
    case PAC_OP_ADD: return __dadd_rn(a, b);
    case PAC_OP_SUB: return __dsub_rn(a, b);
    case PAC_OP_MUL: return __dmul_rn(a, b);
    case PAC_OP_DIV: return __ddiv_rn(a, b);
    case PAC_OP_MIN: return fmin(a, b);
    default: return fmax(a, b);
  }
}

__device__ __forceinline__ bool cmp_holds(int cmp, double v, double c) {
  switch (cmp) {
    case PAC_CMP_LT: return v < c;
    case PAC_CMP_LE: return v <= c;
    case PAC_CMP_GT: return v > c;
    case PAC_CMP_GE: return v >= c;
    default: return v == c;
  }
}

struct WV {
  const double* y;
  const uint64_t* p;
  double s;
  __device__ __forceinline__ uint64_t pres(int64_t i) const { return y ? p[i] : ~0ull; }
  __device__ __forceinline__ double at(int64_t i, int j) const { return y ? y[i * kM + j] : s; }
};

// one thread per (vector, world) element, vectors in 64-element rows: coalesced
__global__ void k_lift(int op, WV a, WV b, int64_t n, double* __restrict__ out, uint64_t* __restrict__ pout) {
  const int64_t total = n * kM;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e >> 6;
    const int j = (int)(e & 63);
    const uint64_t pr = a.pres(i) & b.pres(i);
    out[e] = ((pr >> j) & 1ull) ? lift_op(op, a.at(i, j), b.at(i, j)) : 0.0;
    if (j == 0) pout[i] = pr;
  }
}

// one warp per vector: lane j compares worlds j and j+32, two ballots give the 64 booleans
__global__ void k_lift_cmp(int cmp, WV a, WV b, int64_t n, uint64_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += (int64_t)gridDim.x * wpb) {
    const uint64_t pr = a.pres(i) & b.pres(i);
    const bool t0 = ((pr >> lane) & 1ull) && cmp_holds(cmp, a.at(i, lane), b.at(i, lane));
    const bool t1 = ((pr >> (lane + 32)) & 1ull) && cmp_holds(cmp, a.at(i, lane + 32), b.at(i, lane + 32));
    const unsigned lo = __ballot_sync(0xffffffffu, t0), hi = __ballot_sync(0xffffffffu, t1);
    if (lane == 0) bits[i] = (uint64_t)lo | ((uint64_t)hi << 32);
  }
}

// ------------------------------------------------------------------ comparison index
// One warp per group.  Valid worlds: present and not NaN (a NaN never compares true, an
// absent world compares false, R26).  rank_j = #{valid i : c_i < c_j or (c_i == c_j and i < j)}
// places the valid values in ascending order; positions >= nv hold +inf (never read).
__global__ void k_cmp_index(const double* __restrict__ c, const uint64_t* __restrict__ pres, int64_t G,
                            uint64_t* __restrict__ index) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int64_t g = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); g < G; g += (int64_t)gridDim.x * wpb) {
    const uint64_t pr = pres[g];
    const double v0 = c[g * kM + lane], v1 = c[g * kM + lane + 32];
    const bool ok0 = ((pr >> lane) & 1ull) && !isnan(v0);
    const bool ok1 = ((pr >> (lane + 32)) & 1ull) && !isnan(v1);
    int r0 = 0, r1 = 0;
#pragma unroll 4
    for (int i = 0; i < 64; ++i) {
      const double ci = __shfl_sync(0xffffffffu, i < 32 ? v0 : v1, i & 31);
      const int oki = __shfl_sync(0xffffffffu, (int)(i < 32 ? ok0 : ok1), i & 31);
      if (oki) {
        r0 += (ci < v0 || (ci == v0 && i < lane)) ? 1 : 0;
        r1 += (ci < v1 || (ci == v1 && i < lane + 32)) ? 1 : 0;
      }
    }
    const int nv = __popc(__ballot_sync(0xffffffffu, ok0)) + __popc(__ballot_sync(0xffffffffu, ok1));
    uint64_t* ix = index + g * kIdxWords;
    double* val = reinterpret_cast<double*>(ix);
    if (lane >= nv) val[lane] = INFINITY;
    if (lane + 32 >= nv) val[lane + 32] = INFINITY;
    __syncwarp();
    if (ok0) val[r0] = v0;
    if (ok1) val[r1] = v1;
    // S[p] = {valid worlds j : rank_j >= p}, p = 0..64
    for (int p = 0; p <= 64; ++p) {
      const unsigned lo = __ballot_sync(0xffffffffu, ok0 && r0 >= p);
      const unsigned hi = __ballot_sync(0xffffffffu, ok1 && r1 >= p);
      if (lane == (p & 31)) ix[64 + p] = (uint64_t)lo | ((uint64_t)hi << 32);
    }
    if (lane == 0) ix[129] = (uint64_t)nv;
  }
}

// b_j = [valid_j and (v cmp c_j)] from the index: lb = #{c < v}, ub = #{c <= v} over the sorted
// valid values; LT -> S[ub], LE -> S[lb], GT -> S[0] \ S[lb], GE -> S[0] \ S[ub], EQ -> S[lb] \ S[ub].
__device__ __forceinline__ uint64_t index_bits(const uint64_t* __restrict__ ix, double v, int cmp) {
  if (isnan(v)) return 0ull;
  const double* val = reinterpret_cast<const double*>(ix);
  const int nv = (int)__ldg(ix + 129);
  int lb = 0, ub = 0;
#pragma unroll
  for (int step = 64; step > 0; step >>= 1) {
    const int tl = lb + step, tu = ub + step;
    if (tl <= nv && __ldg(val + tl - 1) < v) lb = tl;
    if (tu <= nv && __ldg(val + tu - 1) <= v) ub = tu;
  }
  const uint64_t* S = ix + 64;
  switch (cmp) {
    case PAC_CMP_LT: return __ldg(S + ub);
    case PAC_CMP_LE: return __ldg(S + lb);
    case PAC_CMP_GT: return __ldg(S) & ~__ldg(S + lb);
    case PAC_CMP_GE: return __ldg(S) & ~__ldg(S + ub);
    default: return __ldg(S + lb) & ~__ldg(S + ub);
  }
}

__device__ __forceinline__ bool filter_draw(uint64_t seed, uint32_t round, int64_t i, uint64_t b) {
  const u32x4 x = philox4x32_10({(uint32_t)i, (uint32_t)((uint64_t)i >> 32), round, kTagFilter},
                                (uint32_t)seed, (uint32_t)(seed >> 32));
  return (int)(x.x >> 26) < __popcll(b);  // R25: probability popcount(b)/64 exactly
}

__global__ void __launch_bounds__(256) k_select_cmp(int cmp, int64_t n, const uint64_t* __restrict__ h,
                                                    const double* __restrict__ v, const int32_t* __restrict__ gidx,
                                                    const uint64_t* __restrict__ index, uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldcs((const unsigned long long*)h + i) &
             index_bits(index + (int64_t)__ldcs(gidx + i) * kIdxWords, __ldcs(v + i), cmp);
}

__global__ void __launch_bounds__(256) k_filter_cmp(int cmp, int64_t n, const double* __restrict__ v,
                                                    const int32_t* __restrict__ gidx,
                                                    const uint64_t* __restrict__ index, uint64_t seed,
                                                    uint32_t round, uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = filter_draw(seed, round, i, index_bits(index + (int64_t)__ldcs(gidx + i) * kIdxWords, __ldcs(v + i), cmp))
                 ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_select(int64_t n, const uint64_t* __restrict__ h,
                                                const int32_t* __restrict__ gidx, const uint64_t* __restrict__ bits,
                                                uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldcs((const unsigned long long*)h + i) & __ldg(bits + __ldcs(gidx + i));
}

__global__ void __launch_bounds__(256) k_filter(int64_t n, const uint64_t* __restrict__ bits, uint64_t seed,
                                                uint32_t round, uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = filter_draw(seed, round, i, __ldcs((const unsigned long long*)bits + i)) ? 1 : 0;
}

static int grid_for(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + per_block - 1) / per_block, (int64_t)sms * 16));
}

static bool wvec_ok(const pac_wvec* w, int64_t n) {
  return w && (n == 0 || !w->d_y || w->d_presence);
}

}  // namespace pac

using namespace pac;

static int launched() {
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_world_vector(const pac_table* t, const pac_agg_spec* aggs, int n_aggs, int a, int64_t G_cap,
                                double* d_y, uint64_t* d_presence, pac_stream_t stream) {
  if (!t || !aggs || a < 0 || a >= n_aggs || n_aggs > PAC_MAX_AGGS || G_cap < 1 || !d_y || !d_presence ||
      (t->m != 0 && t->m != 64))  // world vectors are m = 64 (R22)
    return PAC_E_INVAL;
  const int kind = aggs[a].kind;
  if (kind < PAC_COUNT || kind > PAC_MAX_F64 || !t->d_num_groups || !t->d_presence) return PAC_E_INVAL;
  if ((kind == PAC_COUNT || kind == PAC_AVG_F64) && !t->d_count) return PAC_E_INVAL;
  if (kind != PAC_COUNT && !t->d_world[a]) return PAC_E_INVAL;
  k_world_vector<<<grid_for(G_cap, 8), 256, 0, (cudaStream_t)stream>>>(
      t->d_num_groups, G_cap, kind, t->d_count, t->d_world[a], t->d_presence, d_y, d_presence);
  return launched();
}

extern "C" int pac_lift(int op, const pac_wvec* a, const pac_wvec* b, int64_t n, double* d_out,
                        uint64_t* d_presence_out, pac_stream_t stream) {
  if (op < PAC_OP_ADD || op > PAC_OP_MAX || n < 0 || !wvec_ok(a, n) || !wvec_ok(b, n)) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  if (!d_out || !d_presence_out) return PAC_E_INVAL;
  WV A{a->d_y, a->d_presence, a->scalar}, B{b->d_y, b->d_presence, b->scalar};
  k_lift<<<grid_for(n * kM, 256), 256, 0, (cudaStream_t)stream>>>(op, A, B, n, d_out, d_presence_out);
  return launched();
}

extern "C" int pac_lift_cmp(int cmp, const pac_wvec* a, const pac_wvec* b, int64_t n, uint64_t* d_bits,
                            pac_stream_t stream) {
  if (cmp < PAC_CMP_LT || cmp > PAC_CMP_EQ || n < 0 || !wvec_ok(a, n) || !wvec_ok(b, n)) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  if (!d_bits) return PAC_E_INVAL;
  WV A{a->d_y, a->d_presence, a->scalar}, B{b->d_y, b->d_presence, b->scalar};
  k_lift_cmp<<<grid_for(n, 8), 256, 0, (cudaStream_t)stream>>>(cmp, A, B, n, d_bits);
  return launched();
}

extern "C" int pac_cmp_index(const double* d_c, const uint64_t* d_presence, int64_t G, uint64_t* d_index,
                             pac_stream_t stream) {
  if (G < 0 || (G > 0 && (!d_c || !d_presence || !d_index))) return PAC_E_INVAL;
  if (G == 0) return PAC_OK;
  k_cmp_index<<<grid_for(G, 8), 256, 0, (cudaStream_t)stream>>>(d_c, d_presence, G, d_index);
  return launched();
}

extern "C" int pac_select(const uint64_t* d_h, const int32_t* d_gidx, const uint64_t* d_bits, int64_t n,
                          uint64_t* d_out, pac_stream_t stream) {
  if (n < 0 || (n > 0 && (!d_h || !d_gidx || !d_bits || !d_out))) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  k_select<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, d_h, d_gidx, d_bits, d_out);
  return launched();
}

extern "C" int pac_select_cmp(int cmp, const uint64_t* d_h, const double* d_v, const int32_t* d_gidx,
                              const uint64_t* d_index, int64_t n, uint64_t* d_out, pac_stream_t stream) {
  if (cmp < PAC_CMP_LT || cmp > PAC_CMP_EQ || n < 0) return PAC_E_INVAL;
  if (n > 0 && (!d_h || !d_v || !d_gidx || !d_index || !d_out)) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  k_select_cmp<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(cmp, n, d_h, d_v, d_gidx, d_index, d_out);
  return launched();
}

extern "C" int pac_filter(pac_session* s, const uint64_t* d_bits, int64_t n, uint32_t round, uint8_t* d_out,
                          pac_stream_t stream) {
  if (!s || n < 0 || (n > 0 && (!d_bits || !d_out))) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  k_filter<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, d_bits, session_seed(s), round, d_out);
  return launched();
}

extern "C" int pac_filter_cmp(pac_session* s, int cmp, const double* d_v, const int32_t* d_gidx,
                              const uint64_t* d_index, int64_t n, uint32_t round, uint8_t* d_out,
                              pac_stream_t stream) {
  if (!s || cmp < PAC_CMP_LT || cmp > PAC_CMP_EQ || n < 0) return PAC_E_INVAL;
  if (n > 0 && (!d_v || !d_gidx || !d_index || !d_out)) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  k_filter_cmp<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(cmp, n, d_v, d_gidx, d_index, session_seed(s),
                                                                   round, d_out);
  return launched();
}
