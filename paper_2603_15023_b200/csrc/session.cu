// libpac: session (§8 a1), finalize = fused pac_noised (a6) and posterior update (a7).
//
// Finalize is a parallel prep kernel (one warp per cell: Philox block, NULL decision,
// normal draw, 64-entry y-vector) followed by one warp that walks the cells in canonical
// order (R12) -- the posterior P makes the release chain inherently sequential
// (each cell's variance is taken under the posterior left by the previous).
#include <algorithm>
#include <climits>
#include <cmath>
#include <new>

#include "common.cuh"

struct pac_session {
  uint64_t seed;
  double B;
  int32_t jstar;
  uint64_t salt;
  double* d_P;                  // [m]
  unsigned long long* d_count;  // releases counter
  int32_t m;                    // worlds: 64, or 128 (§8 f4, R29)
};

namespace pac {

__global__ void k_session_init(double* P, unsigned long long* cnt, int m) {
  if (threadIdx.x < m) P[threadIdx.x] = 1.0 / m;
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

constexpr int kChainChunk = 16;  // cells per staged chunk of k_finalize_chain
// chain control block (workspace, 64 B): [0] = first cell of the cell-parallel tail
constexpr int kCtlTail = 0;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
// 16-byte async copy of `bytes` (<= 16) source bytes, the rest of the 16 zero-filled
__device__ __forceinline__ void cp_async16z(void* smem_dst, const void* gsrc, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
// 8-byte async copy of `bytes` (<= 8) source bytes, the rest zero-filled
__device__ __forceinline__ void cp_async8z(void* smem_dst, const void* gsrc, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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
  const uint64_t* K;  // [G][M/64] words
  const int64_t* rows;
  uint64_t seed;
  uint32_t round;
  double* zbuf;     // [cells]
  uint8_t* is_null; // [cells]
  uint8_t* flags;   // [G]
  const int32_t* status;  // the table's status (pac_finalize) or NULL
};

// one thread per cell: Philox block, NULL decision, normal draw, diversity flag (the y-vectors are
// derived from the table by the chain itself, YSrc)
template <int M>
__global__ void k_finalize_prep(FinPrep f) {
  constexpr int W = M / 64;
  const int64_t G = min(*f.num_groups, f.G_cap);
  const int64_t cells = G * f.A;
  for (int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; cell < cells;
       cell += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = cell / f.A;
    const int a = (int)(cell % f.A);
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) pc += __popcll(f.K[g * W + w]);
    const u32x4 x = philox4x32_10({(uint32_t)cell, (uint32_t)((uint64_t)cell >> 32), f.round, kTagCell},
                                  (uint32_t)f.seed, (uint32_t)(f.seed >> 32));
    // a table with a nonzero status (CAPACITY: groups missing; OVERFLOW: a wrapped int64 sum)
    // releases nothing: every cell NULL, flags bit 1, the posterior untouched
    const bool bad = f.status && *f.status != 0;
    const bool null = bad || (int)(x.x >> (M == 64 ? 26 : 25)) >= pc;  // R10 / R29
    f.is_null[cell] = null ? 1 : 0;
    f.zbuf[cell] = null ? 0.0 : normal_from(x);
    if (a == 0 && f.flags)
      f.flags[g] = (uint8_t)(((f.rows[g] >= M && pc <= (M == 64 ? 34 : 68)) ? 1 : 0) | (bad ? 2 : 0));  // R18 / R29
  }
}

// Where the chain reads a cell's y-vector: the given vectors of pac_noised_y (ybuf[cells][M], absent
// worlds already 0), or the aggregate table itself for pac_finalize, y derived per world in the
// released scale (R7: 2x for COUNT/SUM, AVG = sum / count; R9: unset worlds read 0) -- no
// [cells][M] y buffer is written and read back.
struct YSrc {
  const double* ybuf;
  int kinds[PAC_MAX_AGGS];
  const void* world[PAC_MAX_AGGS];
  const int64_t* count;
  const uint64_t* K;  // [G][M/64]
};

// y of one world from its staged table words: a = the world's COUNT (COUNT) or value, b = its count
__device__ __forceinline__ double y_of(int kind, unsigned long long a, unsigned long long b, bool set) {
  if (!set) return 0.0;
  switch (kind) {
    case PAC_COUNT:
    case PAC_SUM_I64: return 2.0 * (double)(long long)a;
    case PAC_SUM_F64: return 2.0 * __longlong_as_double((long long)a);
    case PAC_AVG_F64: return __ddiv_rn(__longlong_as_double((long long)a), (double)(long long)b);
    default: return __longlong_as_double((long long)a);
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

// P <- P*W / sum(P*W) over worlds with P_j > 0 (R14); lane owns worlds lane + 32h
template <int H>
__device__ __forceinline__ void bayes_update(double (&p)[H], const double (&y)[H], double yt, double delta) {
  double d[H];
  double lmin = INFINITY;
#pragma unroll
  for (int h = 0; h < H; ++h) {
    d[h] = __dmul_rn(__dsub_rn(yt, y[h]), __dsub_rn(yt, y[h]));
    lmin = fmin(lmin, p[h] > 0.0 ? d[h] : INFINITY);
  }
  const double dmin = warp_min(lmin);
  const double two_delta = 2.0 * delta;
  double lsum = 0.0;
#pragma unroll
  for (int h = 0; h < H; ++h) {
    if (p[h] > 0.0) p[h] = __dmul_rn(p[h], exp(-__ddiv_rn(__dsub_rn(d[h], dmin), two_delta)));
    lsum += p[h];
  }
  const double tot = warp_sum(lsum);
#pragma unroll
  for (int h = 0; h < H; ++h) p[h] = __ddiv_rn(p[h], tot);
}

// one warp: the sequential release chain over M worlds (H = M/32 per lane).
// Latency-bound (each cell's variance is taken under the posterior the previous cell left), so
// the chain keeps two dependent warp reductions per released cell:
//   pass 1: sum P and sum P*y (R11's equality test beside them: ballot, broadcast, vote)
//   pass 2: sum P*(y - mu)^2
// and no reduction in the update: the posterior is normalised at the next released cell with the
// mass pass 1 sums anyway (and when the chain ends), and the likelihood
// is shifted by d_{j*} = (y~ - y_{j*})^2 = Delta*z^2 instead of min_j d_j -- both shifts cancel
// in the normalisation (R14), and W_j = exp((d_{j*} - d_j)/(2 Delta)) <= exp(z^2/2) cannot
// overflow while W_{j*} = 1 keeps the weights from vanishing together.  Equal to the oracle's
// per-cell normalised update up to rounding (R16).
// num_groups == nullptr: G_cap cells-per-aggregate rows are all valid (pac_noised_y)
template <int M>
__global__ void __launch_bounds__(32) k_finalize_chain(const int64_t* num_groups, int64_t G_cap, int A,
                                                       const YSrc ys,
                                                       const double* __restrict__ zbuf,
                                                       const uint8_t* __restrict__ is_null, double* P,
                                                       unsigned long long* releases, int jstar, double B,
                                                       double* release, double* delta_out, long long* ctl) {
  constexpr int H = M / 32;
  constexpr int W = M / 64;
  constexpr int CH = kChainChunk * 64 / M;
  // cells are streamed through shared memory in chunks of CH (double-buffered cp.async), so
  // the chain never waits on HBM latency: the table rows (or y-vectors), normals and NULL flags
  // of chunk c+1 are in flight while chunk c is released
  __shared__ __align__(16) unsigned long long sa[2][CH * M];  // y, or the value / COUNT row
  __shared__ __align__(16) unsigned long long sb[2][CH * M];  // the count row (AVG)
  __shared__ __align__(16) unsigned long long sk[2][CH * 2];  // K words
  __shared__ __align__(16) double sz[2][CH];
  __shared__ __align__(16) uint8_t sn[2][CH];
  const int lane = threadIdx.x;
  const int64_t G = num_groups ? min(*num_groups, G_cap) : G_cap;
  const int64_t cells = G * A;
  const int64_t nchunks = (cells + CH - 1) / CH;
  auto stage = [&](int64_t c) {
    const int b = (int)(c & 1);
    const int64_t c0 = c * CH;
    const int nc = (int)min((int64_t)CH, cells - c0);
    if (ys.ybuf) {
      const char* gy = (const char*)(ys.ybuf + c0 * M);
      char* dy = (char*)sa[b];
      for (int i = lane; i < nc * M / 2; i += 32) cp_async16(dy + 16 * i, gy + 16 * i);
    } else {
      int64_t g = c0 / A;
      int a = (int)(c0 - g * A);
      for (int ci = 0; ci < nc; ++ci) {
        const int kind = ys.kinds[a];
        const char* ra = (const char*)((kind == PAC_COUNT ? (const void*)ys.count : ys.world[a])) + g * M * 8;
#pragma unroll
        for (int i = lane; i < M / 2; i += 32) cp_async16((char*)(sa[b] + ci * M) + 16 * i, ra + 16 * i);
        if (kind == PAC_AVG_F64) {
          const char* rb = (const char*)(ys.count + g * M);
#pragma unroll
          for (int i = lane; i < M / 2; i += 32) cp_async16((char*)(sb[b] + ci * M) + 16 * i, rb + 16 * i);
        }
        if (lane == 0) {
          if (W == 1) cp_async8(sk[b] + 2 * ci, ys.K + g);
          else cp_async16(sk[b] + 2 * ci, ys.K + g * W);
        }
        if (++a == A) {
          a = 0;
          ++g;
        }
      }
    }
    // normals: nc doubles in 16-byte pieces; NULL flags: nc bytes in one piece (zero-filled tails)
    if (lane < (nc + 1) / 2) {
      const int bytes = min(16, 8 * (nc - 2 * lane));
      cp_async16z((char*)sz[b] + 16 * lane, (const char*)(zbuf + c0) + 16 * lane, bytes);
    }
    if (CH == 16) {
      if (lane == 31) cp_async16z(sn[b], is_null + c0, nc);
    } else {  // CH = 8: chunk starts are only 8-byte aligned
      if (lane == 31) cp_async8z(sn[b], is_null + c0, nc);
    }
    cp_async_commit();
  };
  double p[H];
#pragma unroll
  for (int h = 0; h < H; ++h) p[h] = P[lane + 32 * h];
  // exactly one world left in the posterior's support (from then on every cell is R11)
  auto lone_world = [&]() {
    int n = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) n += __popc(__ballot_sync(0xffffffffu, p[h] > 0.0));
    return n == 1;
  };
  unsigned long long nrel = 0;
  const int jl = jstar & 31, jh = jstar >> 5;
  int64_t tail = lone_world() ? 0 : cells;  // first cell left to k_finalize_tail
  if (tail > 0 && nchunks > 0) stage(0);
  int acur = 0;  // aggregate of the current cell
  for (int64_t cell = 0; cell < tail; ++cell, acur = (acur + 1 == A) ? 0 : acur + 1) {
    const int ci = (int)(cell % CH);
    const int b = (int)((cell / CH) & 1);
    if (ci == 0) {
      __syncwarp();  // every lane is done with the buffer chunk c+1 overwrites
      if (cell / CH + 1 < nchunks) {
        stage(cell / CH + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
    }
    double y[H];
    if (ys.ybuf) {
#pragma unroll
      for (int h = 0; h < H; ++h) y[h] = __longlong_as_double((long long)sa[b][ci * M + lane + 32 * h]);
    } else {
      const int kind = ys.kinds[acur];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int j = lane + 32 * h;
        y[h] = y_of(kind, sa[b][ci * M + j], sb[b][ci * M + j], (sk[b][2 * ci + (j >> 6)] >> (j & 63)) & 1ull);
      }
    }
    if (sn[b][ci]) {
      if (lane == 0) {
        release[cell] = NAN;
        if (delta_out) delta_out[cell] = NAN;
      }
      continue;
    }
    // pass 1: the P-mass and the P-weighted sum; R11 zero-variance test as the oracle states it:
    // every y_j with P_j > 0 equals y of the first such world (a NaN there is unequal)
    double lsp = 0.0, lspy = 0.0, yjl = 0.0;
    int first = -1;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      lsp += p[h];
      lspy += __dmul_rn(p[h], y[h]);
      if (h == jh) yjl = y[h];
      const unsigned bal = __ballot_sync(0xffffffffu, p[h] > 0.0);
      if (first < 0 && bal) first = 32 * h + __ffs(bal) - 1;
    }
    double y0 = 0.0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const double t = __shfl_sync(0xffffffffu, y[h], first & 31);
      if (h == (first >> 5)) y0 = t;
    }
    bool eq = true;
#pragma unroll
    for (int h = 0; h < H; ++h) eq &= !(p[h] > 0.0) || lane + 32 * h == first || y[h] == y0;
    const bool all_equal = __all_sync(0xffffffffu, eq);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      lsp += __shfl_xor_sync(0xffffffffu, lsp, d);
      lspy += __shfl_xor_sync(0xffffffffu, lspy, d);
    }
    const double yj = __shfl_sync(0xffffffffu, yjl, jl);
    if (all_equal) {
      if (lane == 0) {
        release[cell] = yj;
        if (delta_out) delta_out[cell] = 0.0;
      }
      continue;
    }
    // the previous update's normalisation, with the mass pass 1 just summed (no extra reduction)
#pragma unroll
    for (int h = 0; h < H; ++h) p[h] = __ddiv_rn(p[h], lsp);
    // pass 2: R8 population variance under P, two-pass
    const double mu = __ddiv_rn(lspy, lsp);
    double ls2 = 0.0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const double e = __dsub_rn(y[h], mu);
      ls2 += __dmul_rn(__dmul_rn(p[h], e), e);
    }
    const double s2 = warp_sum(ls2);
    const double delta = __ddiv_rn(s2, 2.0 * B);
    if (s2 == 0.0) {  // all weight on worlds equal up to rounding
      if (lane == 0) {
        release[cell] = yj;
        if (delta_out) delta_out[cell] = delta;
      }
      continue;
    }
    const double z = sz[b][ci];
    const double yt = __dadd_rn(yj, __dmul_rn(sqrt(delta), z));
    // Bayesian update, shifted by d_{j*} (see above), no normalisation
    const double dj = __dmul_rn(__dsub_rn(yt, yj), __dsub_rn(yt, yj));
    const double inv2d = __drcp_rn(2.0 * delta);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const double d = __dmul_rn(__dsub_rn(yt, y[h]), __dsub_rn(yt, y[h]));
      if (p[h] > 0.0) p[h] = __dmul_rn(p[h], exp(__dmul_rn(__dsub_rn(dj, d), inv2d)));
    }
    ++nrel;
    if (lane == 0) {
      release[cell] = yt;
      if (delta_out) delta_out[cell] = delta;
    }
    // R11 makes every later non-NULL cell a zero-variance release once one world is left
    if (lone_world()) tail = cell + 1;
  }
  cp_async_wait<0>();
  if (lane == 0) ctl[kCtlTail] = tail;
  const double tot = warp_sum([&] {
    double t = 0.0;
#pragma unroll
    for (int h = 0; h < H; ++h) t += p[h];
    return t;
  }());
#pragma unroll
  for (int h = 0; h < H; ++h) P[lane + 32 * h] = __ddiv_rn(p[h], tot);
  if (lane == 0) *releases += nrel;
}

// The chain after the posterior's support has shrunk to one world (P_w = 1): every NULL cell
// is NaN, every other cell is a zero-variance release of y_{j*} (R11: with one world there is
// nothing to compare), and P no longer changes -- so the rest of the chain is cell-parallel.
template <int M>
__global__ void k_finalize_tail(const int64_t* num_groups, int64_t G_cap, int A, const YSrc ys,
                                const uint8_t* __restrict__ is_null, int jstar, double* release, double* delta_out,
                                const long long* ctl) {
  const int64_t G = num_groups ? min(*num_groups, G_cap) : G_cap;
  const int64_t cells = G * A;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t cell = ctl[kCtlTail] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; cell < cells;
       cell += stride) {
    const bool null = is_null[cell] != 0;
    double yj = 0.0;
    if (!null) {
      if (ys.ybuf) {
        yj = ys.ybuf[cell * M + jstar];
      } else {
        const int64_t g = cell / A;
        const int a = (int)(cell - g * A);
        const int kind = ys.kinds[a];
        const size_t c = (size_t)g * M + jstar;
        const unsigned long long va = kind == PAC_COUNT ? (unsigned long long)ys.count[c]
                                                        : ((const unsigned long long*)ys.world[a])[c];
        const unsigned long long vb = kind == PAC_AVG_F64 ? (unsigned long long)ys.count[c] : 0ull;
        yj = y_of(kind, va, vb, (ys.K[g * (M / 64) + (jstar >> 6)] >> (jstar & 63)) & 1ull);
      }
    }
    release[cell] = null ? NAN : yj;
    if (delta_out) delta_out[cell] = null ? NAN : 0.0;
  }
}

__global__ void __launch_bounds__(32) k_posterior_update(double* P, const double* y, double yt, double delta) {
  const int lane = threadIdx.x;
  double p[2] = {P[lane], P[lane + 32]};
  const double yy[2] = {y[lane], y[lane + 32]};
  bayes_update<2>(p, yy, yt, delta);
  P[lane] = p[0];
  P[lane + 32] = p[1];
}

// workspace: [y-vectors [cells][M], pac_noised_y only], normals [cells], chain control block (64 B)
static size_t fin_ws(int64_t G_cap, int A, bool with_y, size_t* o_z, size_t* o_c, int M = kM) {
  const size_t cells = (size_t)G_cap * A;
  const size_t y = with_y ? cells * M * 8 : 0;
  *o_z = (y + 255) & ~(size_t)255;
  size_t z = cells * 8;
  *o_c = (*o_z + z + 255) & ~(size_t)255;
  return *o_c + 64;
}

// the release chain: the sequential part, then the cell-parallel tail (empty unless the
// posterior's support shrank to one world)
template <int M>
static void launch_chain(const int64_t* num_groups, int64_t G_cap, int A, const YSrc& ys, const double* zbuf,
                         const uint8_t* is_null, pac_session* s, double* release, double* delta_out, long long* ctl,
                         cudaStream_t st) {
  k_finalize_chain<M><<<1, 32, 0, st>>>(num_groups, G_cap, A, ys, zbuf, is_null, s->d_P, s->d_count, s->jstar,
                                        s->B, release, delta_out, ctl);
  note_launch();
  const int64_t cells = G_cap * A;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((cells + 255) / 256, 148 * 8));
  k_finalize_tail<M><<<blocks, 256, 0, st>>>(num_groups, G_cap, A, ys, is_null, s->jstar, release, delta_out, ctl);
  note_launch();
}

uint64_t session_seed(const pac_session* s) { return s->seed; }

}  // namespace pac

using namespace pac;

extern "C" int pac_session_create_m(uint64_t seed, double budget_B, int32_t m, pac_session** out) {
  if (!out || !(budget_B > 0.0) || !std::isfinite(budget_B) || (m != 64 && m != 128)) return PAC_E_INVAL;
  pac_session* s = new (std::nothrow) pac_session();
  if (!s) return PAC_E_INVAL;
  s->seed = seed;
  s->B = budget_B;
  s->m = m;
  // R13 / R29: j* and salt from Philox(seed; 0,0,0,tag)
  u32x4 a = philox4x32_10({0, 0, 0, kTagJstar}, (uint32_t)seed, (uint32_t)(seed >> 32));
  s->jstar = (int32_t)(a.x & (uint32_t)(m - 1));
  u32x4 b = philox4x32_10({0, 0, 0, kTagSalt}, (uint32_t)seed, (uint32_t)(seed >> 32));
  s->salt = (uint64_t)b.x | ((uint64_t)b.y << 32);
  if (cudaMalloc(&s->d_P, m * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&s->d_count, sizeof(unsigned long long)) != cudaSuccess) {
    delete s;
    return PAC_E_CUDA;
  }
  k_session_init<<<1, 128>>>(s->d_P, s->d_count, m);
  note_launch();
  if (cudaDeviceSynchronize() != cudaSuccess) return PAC_E_CUDA;
  *out = s;
  return PAC_OK;
}

extern "C" int pac_session_create(uint64_t seed, double budget_B, pac_session** out) {
  return pac_session_create_m(seed, budget_B, 64, out);
}

extern "C" int32_t pac_session_worlds(const pac_session* s) { return s ? s->m : 0; }

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
  if (h_P64 && cudaMemcpy(h_P64, s->d_P, s->m * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return PAC_E_CUDA;
  if (releases) {
    unsigned long long c = 0;
    if (cudaMemcpy(&c, s->d_count, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return PAC_E_CUDA;
    *releases = c;
  }
  return PAC_OK;
}

extern "C" int pac_session_set_posterior(pac_session* s, const double* h_P64) {
  if (!s || !h_P64) return PAC_E_INVAL;
  // a finalize chain still running on a (non-blocking) stream reads and writes d_P: wait for it
  if (cudaDeviceSynchronize() != cudaSuccess) return PAC_E_CUDA;
  if (cudaMemcpy(s->d_P, h_P64, s->m * 8, cudaMemcpyHostToDevice) != cudaSuccess) return PAC_E_CUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" double* pac_session_posterior_device(pac_session* s) { return s ? s->d_P : nullptr; }

extern "C" int pac_finalize_workspace_size(int64_t G_cap, int n_aggs, size_t* bytes) {
  if (!bytes || G_cap < 1 || n_aggs < 1 || n_aggs > PAC_MAX_AGGS) return PAC_E_INVAL;
  size_t oz, oc;
  *bytes = fin_ws(G_cap, n_aggs, false, &oz, &oc, 128);
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
  const int M = t->m ? t->m : 64;
  if (M != s->m) return PAC_E_INVAL;  // the table and the session must agree on m (R29)
  size_t oz, oc;
  const size_t need = fin_ws(G_cap, n_aggs, false, &oz, &oc, M);
  if (!d_ws || ws_bytes < need) return PAC_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;
  FinPrep f{};
  f.num_groups = t->d_num_groups;
  f.G_cap = G_cap;
  f.A = n_aggs;
  f.K = t->d_presence;
  f.rows = t->d_rows;
  f.seed = s->seed;
  f.round = round;
  f.zbuf = (double*)(ws + oz);
  f.is_null = d_is_null;
  f.flags = d_flags;
  f.status = t->d_status;
  YSrc ys{};
  for (int a = 0; a < n_aggs; ++a) {
    ys.kinds[a] = aggs[a].kind;
    ys.world[a] = t->d_world[a];
  }
  ys.count = t->d_count;
  ys.K = t->d_presence;
  const int64_t cells = G_cap * n_aggs;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((cells + 255) / 256, 148 * 8));
  long long* ctl = (long long*)(ws + oc);
  if (M == 64) {
    k_finalize_prep<64><<<blocks, 256, 0, st>>>(f);
    note_launch();
    launch_chain<64>(t->d_num_groups, G_cap, n_aggs, ys, f.zbuf, d_is_null, s, d_release, d_delta, ctl, st);
  } else {
    k_finalize_prep<128><<<blocks, 256, 0, st>>>(f);
    note_launch();
    launch_chain<128>(t->d_num_groups, G_cap, n_aggs, ys, f.zbuf, d_is_null, s, d_release, d_delta, ctl, st);
  }
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_posterior_update(pac_session* s, const double* d_y64, double y_tilde, double delta,
                                    pac_stream_t stream) {
  if (!s || !d_y64 || !(delta > 0.0) || !std::isfinite(delta) || !std::isfinite(y_tilde) || s->m != 64)
    return PAC_E_INVAL;
  k_posterior_update<<<1, 32, 0, (cudaStream_t)stream>>>(s->d_P, d_y64, y_tilde, delta);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_noised_y_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return PAC_E_INVAL;
  size_t oz, oc;
  *bytes = fin_ws(n > 0 ? n : 1, 1, true, &oz, &oc);
  return PAC_OK;
}

extern "C" int pac_noised_y(pac_session* s, const double* d_y, const uint64_t* d_presence, int64_t n, uint32_t round,
                            double* d_release, uint8_t* d_is_null, double* d_delta, void* d_ws, size_t ws_bytes,
                            pac_stream_t stream) {
  if (!s || s->m != 64 || n < 0 || (n > 0 && (!d_y || !d_presence || !d_release || !d_is_null)))
    return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  size_t oz, oc;
  const size_t need = fin_ws(n, 1, true, &oz, &oc);
  if (!d_ws || ws_bytes < need) return PAC_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;
  double* ybuf = (double*)ws;
  double* zbuf = (double*)(ws + oz);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, 148 * 32));
  k_noised_prep_y<<<blocks, 256, 0, st>>>(d_y, d_presence, n, s->seed, round, ybuf, zbuf, d_is_null);
  note_launch();
  YSrc ys{};
  ys.ybuf = ybuf;
  launch_chain<64>(nullptr, n, 1, ys, zbuf, d_is_null, s, d_release, d_delta, (long long*)(ws + oc), st);
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
