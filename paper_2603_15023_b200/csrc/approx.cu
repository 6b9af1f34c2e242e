// libpac: approximate (two-sided) 64-world SUM (§8 f3; §5 "Approximation",
// "Two-sided SUM"; readings DESIGN.md R35, R36).
//
// The paper's approximate state replaces exact (HUGEINT) world sums by 25 levels of 16-bit
// counters per world, level k weighing 2^(4k): a value is routed to level l(v) = (msb(|v|) - 8)/4
// and adds |v| >> 4l; on overflow the counter's upper 12 bits cascade into the next level and its
// low 4 bits are dropped.  The cascades make the result depend on the update order, so R35 fixes
// one: rows in row order inside blocks of block_rows rows (the paper's thread-local states,
// P:L1966), block states combined in block order.  The GPU follows it exactly:
//   k_approx_blocks   one warp per block: the block's rows in order, 32 at a time (lane t hashes
//                     row t's pu key -- pac_hash, R1/R2 -- and loads its value), then row by row
//                     each lane updates its worlds j = lane, lane + 32 (counters in shared memory,
//                     [side][level][world] so a warp's accesses are conflict-free); the block
//                     state is written to the workspace;
//   k_approx_combine  one thread per (side, world): the blocks' states folded in block order with
//                     the same add-and-cascade rule, then decoded into y_j = 2 (dec(pos) - dec(neg)).
// Integer arithmetic throughout: bit-exact with the oracle (orc_approx_sum).
#include <algorithm>
#include <cstdio>

#include "common.cuh"

namespace pac {

void note_launch();

constexpr int kAL = 25;        // levels
constexpr int kAWarps = 4;     // warps per CTA (one block each; 6.4 KB of counters per warp)
constexpr int kAState = 2 * kAL * kM;  // uint16 counters of one block: [side][level][world]

__device__ __forceinline__ int approx_level(uint64_t a) {
  const int msb = 63 - __clzll((long long)a);
  const int l = msb < 8 ? 0 : (msb - 8) >> 2;
  return l > kAL - 1 ? kAL - 1 : l;
}

// add c at level k of one world's unsigned counters (stride kM between levels), cascading on
// overflow: the displaced counter's upper 12 bits carry into the next level, its low 4 bits drop
__device__ __forceinline__ void approx_add_u(uint16_t* C, int k, uint32_t c) {
  while (k < kAL) {
    const uint32_t cur = C[k * kM];
    if (cur + c <= 0xFFFFu) {
      C[k * kM] = (uint16_t)(cur + c);
      return;
    }
    C[k * kM] = (uint16_t)c;
    c = cur >> 4;
    ++k;
  }
}
__global__ void __launch_bounds__(32 * kAWarps) k_approx_blocks(const long long* __restrict__ pu_key,
                                                                const unsigned long long* __restrict__ mask_in,
                                                                uint64_t salt, const long long* __restrict__ values,
                                                                int64_t n, int64_t block_rows, int two_sided,
                                                                uint16_t* __restrict__ blocks) {
  __shared__ uint16_t st[kAWarps][kAState];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint16_t* S = st[w];
  const int64_t nblk = (n + block_rows - 1) / block_rows;
  for (int64_t b = (int64_t)blockIdx.x * kAWarps + w; b < nblk; b += (int64_t)gridDim.x * kAWarps) {
    for (int i = lane; i < kAState; i += 32) S[i] = 0;
    __syncwarp();
    const int64_t r0 = b * block_rows, r1 = min(n, r0 + block_rows);
    for (int64_t g = r0; g < r1; g += 32) {
      const int64_t r = g + lane;
      uint64_t m = 0;
      long long v = 0;
      if (r < r1) {
        v = values[r];
        m = mask_in ? mask_in[r] : pac_hash_dev((uint64_t)pu_key[r], salt);
      }
      const int cnt = (int)min((int64_t)32, r1 - g);
      for (int t = 0; t < cnt; ++t) {  // rows in order
        const long long vt = __shfl_sync(0xffffffffu, v, t);
        const uint64_t mt = __shfl_sync(0xffffffffu, m, t);
        if (vt == 0 || mt == 0) continue;
        // two-sided: |v| into the pos / neg state; single-sided: the two's-complement pattern (R36)
        const uint64_t a = !two_sided ? (uint64_t)vt : (vt > 0 ? (uint64_t)vt : 0ull - (uint64_t)vt);
        const int l = approx_level(a);
        const uint32_t c = (uint32_t)(a >> (4 * l));
        uint16_t* side = S + (two_sided && vt < 0 ? kAL * kM : 0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = lane + 32 * h;
          if ((mt >> j) & 1ull) approx_add_u(side + j, l, c);
        }
      }
    }
    __syncwarp();
    uint16_t* out = blocks + (size_t)b * kAState;
    for (int i = lane; i < kAState; i += 32) out[i] = S[i];
    __syncwarp();
  }
}

// one thread per (side, world): fold the block states in block order, then decode
__global__ void k_approx_combine(const uint16_t* __restrict__ blocks, int64_t nblk, int two_sided,
                                 uint16_t* __restrict__ counters, double* __restrict__ y) {
  __shared__ double dec[2][kM];
  const int t = threadIdx.x;  // side * 64 + world
  const int side = t >> 6, j = t & 63;
  uint16_t run[kAL];
  for (int k = 0; k < kAL; ++k) run[k] = 0;
  if (side == 0 || two_sided) {
    for (int64_t b = 0; b < nblk; ++b) {
      const uint16_t* src = blocks + (size_t)b * kAState + side * kAL * kM + j;
      for (int k = 0; k < kAL; ++k) {
        const uint16_t c = src[k * kM];
        if (c == 0) continue;
        // the same add-with-cascade on the running state (stride 1 here)
        uint32_t cc = c;
        for (int q = k; q < kAL; ++q) {
          const uint32_t cur = run[q];
          if (cur + cc <= 0xFFFFu) {
            run[q] = (uint16_t)(cur + cc);
            break;
          }
          run[q] = (uint16_t)cc;
          cc = cur >> 4;
        }
      }
    }
  }
  double d = 0.0, sc = 1.0;
  uint64_t u = 0;  // single-sided: decoded modulo 2^64 (levels >= 16 vanish), read as int64
  for (int k = 0; k < kAL; ++k, sc *= 16.0) {
    d += (double)run[k] * sc;
    if (k < 16) u += (uint64_t)run[k] << (4 * k);
  }
  for (int k = 0; k < kAL; ++k) counters[((size_t)side * kM + j) * kAL + k] = run[k];
  dec[side][j] = two_sided ? d : (double)(long long)u;
  __syncthreads();
  if (side == 0) y[j] = 2.0 * (two_sided ? dec[0][j] - dec[1][j] : dec[0][j]);
}

}  // namespace pac

using namespace pac;

extern "C" int pac_approx_sum_workspace_size(int64_t n_rows, int64_t block_rows, size_t* bytes) {
  if (!bytes || n_rows < 0 || block_rows < 1) return PAC_E_INVAL;
  const int64_t nblk = std::max<int64_t>(1, (n_rows + block_rows - 1) / block_rows);
  *bytes = (size_t)nblk * kAState * sizeof(uint16_t);
  return PAC_OK;
}

extern "C" int pac_approx_sum(const int64_t* d_pu_key, const uint64_t* d_mask, uint64_t salt, const int64_t* d_values,
                              int64_t n_rows, int32_t two_sided, int64_t block_rows, uint16_t* d_counters, double* d_y,
                              void* d_ws, size_t ws_bytes, pac_stream_t stream) {
  if (n_rows < 0 || block_rows < 1 || !d_counters || !d_y) return PAC_E_INVAL;
  if (n_rows > 0 && (!d_values || (!!d_pu_key == !!d_mask))) return PAC_E_INVAL;
  size_t need = 0;
  pac_approx_sum_workspace_size(n_rows, block_rows, &need);
  if (!d_ws || ws_bytes < need) return PAC_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nblk = (n_rows + block_rows - 1) / block_rows;
  if (nblk > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nblk + kAWarps - 1) / kAWarps, (int64_t)sms * 8));
    k_approx_blocks<<<grid, 32 * kAWarps, 0, st>>>((const long long*)d_pu_key, (const unsigned long long*)d_mask, salt,
                                                   (const long long*)d_values, n_rows, block_rows, two_sided ? 1 : 0,
                                                   (uint16_t*)d_ws);
    note_launch();
  }
  k_approx_combine<<<1, 128, 0, st>>>((const uint16_t*)d_ws, nblk, two_sided ? 1 : 0, d_counters, d_y);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
