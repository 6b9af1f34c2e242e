// libpac: session (§8 a1), finalize = fused pac_noised (a6) and posterior update (a7).
//
// Finalize is a parallel prep kernel (one warp per cell: Philox block, NULL decision,
// normal draw, 64-entry y-vector) followed by one warp that walks the cells in canonical
// order (R12) -- the posterior P makes the release chain inherently sequential
// (each cell's variance is taken under the posterior left by the previous).
#include <algorithm>
#include <cmath>
#include <new>

#include "common.cuh"

struct pac_session {
  uint64_t seed;
  double B;
  int32_t jstar;
  uint64_t salt;
  double* d_P;                  // [64]
  unsigned long long* d_count;  // releases counter
};

namespace pac {

__global__ void k_session_init(double* P, unsigned long long* cnt) {
  if (threadIdx.x < kM) P[threadIdx.x] = 1.0 / kM;
  if (threadIdx.x == 0) *cnt = 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

// Box-Muller normal from one Philox block (R13).
__device__ __forceinline__ double normal_from(u32x4 x) {
  const uint64_t m53 = ((uint64_t)x.y << 21) ^ (uint64_t)(x.z >> 11);
  const double u1 = __dmul_rn(__dadd_rn((double)m53, 0.5), 0x1.0p-53);
  const double u2 = __dmul_rn(__dadd_rn((double)x.w, 0.5), 0x1.0p-32);
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(2.0 * 3.141592653589793, u2)));
}

struct FinPrep {
  const int64_t* num_groups;
  int64_t G_cap;
  int A;
  int kinds[PAC_MAX_AGGS];
  const void* world[PAC_MAX_AGGS];
  const int64_t* count;
  const uint64_t* K;
  const int64_t* rows;
  uint64_t seed;
  uint32_t round;
  double* ybuf;     // [cells][64]
  double* zbuf;     // [cells]
  uint8_t* is_null; // [cells]
  uint8_t* flags;   // [G]
};

// one warp per cell
__global__ void k_finalize_prep(FinPrep f) {
  const int64_t G = min(*f.num_groups, f.G_cap);
  const int64_t cells = G * f.A;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int64_t cell = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); cell < cells;
       cell += (int64_t)gridDim.x * wpb) {
    const int64_t g = cell / f.A;
    const int a = (int)(cell % f.A);
    const uint64_t Kg = f.K[g];
    const int pc = __popcll(Kg);
    const u32x4 x = philox4x32_10({(uint32_t)cell, (uint32_t)((uint64_t)cell >> 32), f.round, kTagCell},
                                  (uint32_t)f.seed, (uint32_t)(f.seed >> 32));
    const bool null = (int)(x.x >> 26) >= pc;  // R10
    const int kind = f.kinds[a];
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      const size_t c = (size_t)g * kM + j;
      double y = 0.0;
      if ((Kg >> j) & 1ull) {  // R9: unset worlds read 0
        switch (kind) {
          case PAC_COUNT: y = 2.0 * (double)f.count[c]; break;
          case PAC_SUM_I64: y = 2.0 * (double)((const int64_t*)f.world[a])[c]; break;
          case PAC_SUM_F64: y = 2.0 * ((const double*)f.world[a])[c]; break;
          case PAC_AVG_F64: y = __ddiv_rn(((const double*)f.world[a])[c], (double)f.count[c]); break;
          default: y = ((const double*)f.world[a])[c]; break;
        }
      }
      f.ybuf[cell * kM + j] = y;
    }
    if (lane == 0) {
      f.is_null[cell] = null ? 1 : 0;
      f.zbuf[cell] = null ? 0.0 : normal_from(x);
      if (a == 0 && f.flags) f.flags[g] = (f.rows[g] >= 64 && pc <= 34) ? 1 : 0;  // R18
    }
  }
}

// pac_noised_y prep (R24): one warp per given world vector -- Philox block with TAG_LIFT,
// NULL decision from popcount(presence) (R10), normal draw, y copied with absent worlds 0 (R9).
__global__ void k_noised_prep_y(const double* __restrict__ y, const uint64_t* __restrict__ presence, int64_t n,
                                uint64_t seed, uint32_t round, double* ybuf, double* zbuf, uint8_t* is_null) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += (int64_t)gridDim.x * wpb) {
    const uint64_t pr = presence[i];
    const u32x4 x = philox4x32_10({(uint32_t)i, (uint32_t)((uint64_t)i >> 32), round, kTagLift},
                                  (uint32_t)seed, (uint32_t)(seed >> 32));
    const bool null = (int)(x.x >> 26) >= __popcll(pr);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      ybuf[i * kM + j] = ((pr >> j) & 1ull) ? y[i * kM + j] : 0.0;
    }
    if (lane == 0) {
      is_null[i] = null ? 1 : 0;
      zbuf[i] = null ? 0.0 : normal_from(x);
    }
  }
}

// P <- P*W / sum(P*W) over worlds with P_j > 0 (R14); lane owns j, j+32
__device__ __forceinline__ void bayes_update(double& p0, double& p1, double y0, double y1, double yt,
                                             double delta) {
  const double d0 = __dmul_rn(__dsub_rn(yt, y0), __dsub_rn(yt, y0));
  const double d1 = __dmul_rn(__dsub_rn(yt, y1), __dsub_rn(yt, y1));
  const double dmin = warp_min(fmin(p0 > 0.0 ? d0 : INFINITY, p1 > 0.0 ? d1 : INFINITY));
  const double two_delta = 2.0 * delta;
  if (p0 > 0.0) p0 = __dmul_rn(p0, exp(-__ddiv_rn(__dsub_rn(d0, dmin), two_delta)));
  if (p1 > 0.0) p1 = __dmul_rn(p1, exp(-__ddiv_rn(__dsub_rn(d1, dmin), two_delta)));
  const double tot = warp_sum(p0 + p1);
  p0 = __ddiv_rn(p0, tot);
  p1 = __ddiv_rn(p1, tot);
}

// one warp: the sequential release chain
// num_groups == nullptr: G_cap cells-per-aggregate rows are all valid (pac_noised_y)
__global__ void __launch_bounds__(32) k_finalize_chain(const int64_t* num_groups, int64_t G_cap, int A,
                                                       const double* __restrict__ ybuf,
                                                       const double* __restrict__ zbuf,
                                                       const uint8_t* __restrict__ is_null, double* P,
                                                       unsigned long long* releases, int jstar, double B,
                                                       double* release, double* delta_out) {
  const int lane = threadIdx.x;
  const int64_t G = num_groups ? min(*num_groups, G_cap) : G_cap;
  const int64_t cells = G * A;
  double p0 = P[lane], p1 = P[lane + 32];
  unsigned long long nrel = 0;
  const int jl = jstar & 31;
  const bool jhi = jstar >= 32;
  double ny0 = 0, ny1 = 0;
  if (cells > 0) {
    ny0 = ybuf[lane];
    ny1 = ybuf[lane + 32];
  }
  for (int64_t cell = 0; cell < cells; ++cell) {
    const double y0 = ny0, y1 = ny1;
    if (cell + 1 < cells) {  // prefetch the next cell's y-vector
      ny0 = ybuf[(cell + 1) * kM + lane];
      ny1 = ybuf[(cell + 1) * kM + lane + 32];
    }
    if (is_null[cell]) {
      if (lane == 0) {
        release[cell] = NAN;
        if (delta_out) delta_out[cell] = NAN;
      }
      continue;
    }
    // R11: zero variance iff every y_j with P_j > 0 is equal
    const double lo = warp_min(fmin(p0 > 0.0 ? y0 : INFINITY, p1 > 0.0 ? y1 : INFINITY));
    const double hi = warp_max(fmax(p0 > 0.0 ? y0 : -INFINITY, p1 > 0.0 ? y1 : -INFINITY));
    const double yj = __shfl_sync(0xffffffffu, jhi ? y1 : y0, jl);
    if (lo == hi) {
      if (lane == 0) {
        release[cell] = yj;
        if (delta_out) delta_out[cell] = 0.0;
      }
      continue;
    }
    // R8: population variance under P, two-pass
    const double mu = warp_sum(__dmul_rn(p0, y0) + __dmul_rn(p1, y1));
    const double e0 = __dsub_rn(y0, mu), e1 = __dsub_rn(y1, mu);
    const double s2 = warp_sum(__dmul_rn(__dmul_rn(p0, e0), e0) + __dmul_rn(__dmul_rn(p1, e1), e1));
    const double delta = __ddiv_rn(s2, 2.0 * B);
    if (s2 == 0.0) {  // all weight on worlds equal up to rounding
      if (lane == 0) {
        release[cell] = yj;
        if (delta_out) delta_out[cell] = delta;
      }
      continue;
    }
    const double yt = __dadd_rn(yj, __dmul_rn(sqrt(delta), zbuf[cell]));
    bayes_update(p0, p1, y0, y1, yt, delta);
    ++nrel;
    if (lane == 0) {
      release[cell] = yt;
      if (delta_out) delta_out[cell] = delta;
    }
  }
  P[lane] = p0;
  P[lane + 32] = p1;
  if (lane == 0) *releases += nrel;
}

__global__ void __launch_bounds__(32) k_posterior_update(double* P, const double* y, double yt, double delta) {
  const int lane = threadIdx.x;
  double p0 = P[lane], p1 = P[lane + 32];
  bayes_update(p0, p1, y[lane], y[lane + 32], yt, delta);
  P[lane] = p0;
  P[lane + 32] = p1;
}

static size_t fin_ws(int64_t G_cap, int A, size_t* o_z, size_t* o_n) {
  const size_t cells = (size_t)G_cap * A;
  size_t y = cells * kM * 8;
  *o_z = (y + 255) & ~(size_t)255;
  size_t z = cells * 8;
  *o_n = (*o_z + z + 255) & ~(size_t)255;
  return *o_n + cells + 256;
}

uint64_t session_seed(const pac_session* s) { return s->seed; }

}  // namespace pac

using namespace pac;

extern "C" int pac_session_create(uint64_t seed, double budget_B, pac_session** out) {
  if (!out || !(budget_B > 0.0) || !std::isfinite(budget_B)) return PAC_E_INVAL;
  pac_session* s = new (std::nothrow) pac_session();
  if (!s) return PAC_E_INVAL;
  s->seed = seed;
  s->B = budget_B;
  // R13: j* and salt from Philox(seed; 0,0,0,tag)
  u32x4 a = philox4x32_10({0, 0, 0, kTagJstar}, (uint32_t)seed, (uint32_t)(seed >> 32));
  s->jstar = (int32_t)(a.x & 63u);
  u32x4 b = philox4x32_10({0, 0, 0, kTagSalt}, (uint32_t)seed, (uint32_t)(seed >> 32));
  s->salt = (uint64_t)b.x | ((uint64_t)b.y << 32);
  if (cudaMalloc(&s->d_P, kM * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&s->d_count, sizeof(unsigned long long)) != cudaSuccess) {
    delete s;
    return PAC_E_CUDA;
  }
  k_session_init<<<1, 64>>>(s->d_P, s->d_count);
  note_launch();
  if (cudaDeviceSynchronize() != cudaSuccess) return PAC_E_CUDA;
  *out = s;
  return PAC_OK;
}

extern "C" int pac_session_destroy(pac_session* s) {
  if (!s) return PAC_OK;
  cudaDeviceSynchronize();
  cudaFree(s->d_P);
  cudaFree(s->d_count);
  delete s;
  return PAC_OK;
}

extern "C" int pac_session_query(const pac_session* s, uint64_t* salt, int32_t* jstar, double* h_P64,
                                 uint64_t* releases, uint64_t* seed, double* budget_B) {
  if (!s) return PAC_E_INVAL;
  if (cudaDeviceSynchronize() != cudaSuccess) return PAC_E_CUDA;
  if (salt) *salt = s->salt;
  if (jstar) *jstar = s->jstar;
  if (seed) *seed = s->seed;
  if (budget_B) *budget_B = s->B;
  if (h_P64 && cudaMemcpy(h_P64, s->d_P, kM * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return PAC_E_CUDA;
  if (releases) {
    unsigned long long c = 0;
    if (cudaMemcpy(&c, s->d_count, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return PAC_E_CUDA;
    *releases = c;
  }
  return PAC_OK;
}

extern "C" int pac_session_set_posterior(pac_session* s, const double* h_P64) {
  if (!s || !h_P64) return PAC_E_INVAL;
  if (cudaMemcpy(s->d_P, h_P64, kM * 8, cudaMemcpyHostToDevice) != cudaSuccess) return PAC_E_CUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" double* pac_session_posterior_device(pac_session* s) { return s ? s->d_P : nullptr; }

extern "C" int pac_finalize_workspace_size(int64_t G_cap, int n_aggs, size_t* bytes) {
  if (!bytes || G_cap < 1 || n_aggs < 1 || n_aggs > PAC_MAX_AGGS) return PAC_E_INVAL;
  size_t oz, on;
  *bytes = fin_ws(G_cap, n_aggs, &oz, &on);
  return PAC_OK;
}

extern "C" int pac_finalize(pac_session* s, const pac_table* t, const pac_agg_spec* aggs, int n_aggs,
                            int64_t G_cap, uint32_t round, double* d_release, uint8_t* d_is_null,
                            uint8_t* d_flags, double* d_delta, void* d_ws, size_t ws_bytes,
                            pac_stream_t stream) {
  if (!s || !t || !aggs || n_aggs < 1 || n_aggs > PAC_MAX_AGGS || G_cap < 1 || !d_release || !d_is_null)
    return PAC_E_INVAL;
  if (!t->d_num_groups || !t->d_presence || !t->d_rows) return PAC_E_INVAL;
  bool need_count = false;
  for (int a = 0; a < n_aggs; ++a) {
    const int k = aggs[a].kind;
    if (k < PAC_COUNT || k > PAC_MAX_F64) return PAC_E_INVAL;
    if (k == PAC_COUNT || k == PAC_AVG_F64) need_count = true;
    if (k != PAC_COUNT && !t->d_world[a]) return PAC_E_INVAL;
  }
  if (need_count && !t->d_count) return PAC_E_INVAL;
  size_t oz, on;
  const size_t need = fin_ws(G_cap, n_aggs, &oz, &on);
  if (!d_ws || ws_bytes < need) return PAC_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;
  FinPrep f{};
  f.num_groups = t->d_num_groups;
  f.G_cap = G_cap;
  f.A = n_aggs;
  for (int a = 0; a < n_aggs; ++a) {
    f.kinds[a] = aggs[a].kind;
    f.world[a] = t->d_world[a];
  }
  f.count = t->d_count;
  f.K = t->d_presence;
  f.rows = t->d_rows;
  f.seed = s->seed;
  f.round = round;
  f.ybuf = (double*)ws;
  f.zbuf = (double*)(ws + oz);
  f.is_null = d_is_null;
  f.flags = d_flags;
  const int64_t cells = G_cap * n_aggs;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((cells + 7) / 8, 148 * 32));
  k_finalize_prep<<<blocks, 256, 0, st>>>(f);
  note_launch();
  k_finalize_chain<<<1, 32, 0, st>>>(t->d_num_groups, G_cap, n_aggs, f.ybuf, f.zbuf, d_is_null, s->d_P,
                                     s->d_count, s->jstar, s->B, d_release, d_delta);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_posterior_update(pac_session* s, const double* d_y64, double y_tilde, double delta,
                                    pac_stream_t stream) {
  if (!s || !d_y64 || !(delta > 0.0) || !std::isfinite(delta) || !std::isfinite(y_tilde)) return PAC_E_INVAL;
  k_posterior_update<<<1, 32, 0, (cudaStream_t)stream>>>(s->d_P, d_y64, y_tilde, delta);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_noised_y_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return PAC_E_INVAL;
  size_t oz, on;
  *bytes = fin_ws(n > 0 ? n : 1, 1, &oz, &on);
  return PAC_OK;
}

extern "C" int pac_noised_y(pac_session* s, const double* d_y, const uint64_t* d_presence, int64_t n, uint32_t round,
                            double* d_release, uint8_t* d_is_null, double* d_delta, void* d_ws, size_t ws_bytes,
                            pac_stream_t stream) {
  if (!s || n < 0 || (n > 0 && (!d_y || !d_presence || !d_release || !d_is_null))) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  size_t oz, on;
  const size_t need = fin_ws(n, 1, &oz, &on);
  if (!d_ws || ws_bytes < need) return PAC_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;
  double* ybuf = (double*)ws;
  double* zbuf = (double*)(ws + oz);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, 148 * 32));
  k_noised_prep_y<<<blocks, 256, 0, st>>>(d_y, d_presence, n, s->seed, round, ybuf, zbuf, d_is_null);
  note_launch();
  k_finalize_chain<<<1, 32, 0, st>>>(nullptr, n, 1, ybuf, zbuf, d_is_null, s->d_P, s->d_count, s->jstar, s->B,
                                     d_release, d_delta);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
