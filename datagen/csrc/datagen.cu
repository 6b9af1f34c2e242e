// Device-side counter-based synthetic column generator (sm_100a).
//
// Mirrors datagen/__init__.py bit-for-bit for integers and uniform doubles.
// Holds none of the PAC method's arithmetic (see datagen/__init__.py header).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t fmix_m3(uint64_t z) {
  z ^= z >> 33;
  z *= 0xFF51AFD7ED558CCDull;
  z ^= z >> 33;
  z *= 0xC4CEB9FE1A85EC53ull;
  z ^= z >> 33;
  return z;
}

__host__ __forceinline__ uint64_t fmix_m3_host(uint64_t z) {
  z ^= z >> 33;
  z *= 0xFF51AFD7ED558CCDull;
  z ^= z >> 33;
  z *= 0xC4CEB9FE1A85EC53ull;
  z ^= z >> 33;
  return z;
}

__device__ __forceinline__ uint64_t scramble64(uint64_t rank) {
  return fmix_m3(rank ^ 0x6A09E667F3BCC909ull);
}

__device__ __forceinline__ uint32_t scramble32(uint64_t rank) {
  uint32_t x = (uint32_t)(rank * 0x9E3779B1ull + 0x7F4A7C15ull);
  x ^= x >> 15;
  return x;
}

__device__ __forceinline__ double unit53(uint64_t w) {
  return (double)(w >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ uint64_t zipf_rank(const double* __restrict__ cdf, int64_t n, double u) {
  // first index i with cdf[i] > u (numpy searchsorted side='right'), clamped to n-1
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
  }
  return (uint64_t)(lo < n ? lo : n - 1);
}

__global__ void dg_kernel(int kind, void* __restrict__ out, int elem_bytes, int64_t n, int64_t row0,
                          uint64_t key, uint64_t key2, double lo, double hi, int64_t n_distinct,
                          const double* __restrict__ cdf) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t row = (uint64_t)(row0 + i);
    uint64_t w = fmix_m3(row * 0xE7037ED1A0B428DBull + key);
    switch (kind) {
      case 1: {  // uniform int
        uint64_t span = (uint64_t)((int64_t)hi - (int64_t)lo + 1);
        int64_t v = (int64_t)__umul64hi(w, span) + (int64_t)lo;
        if (elem_bytes == 1) ((int8_t*)out)[i] = (int8_t)v;
        else if (elem_bytes == 2) ((int16_t*)out)[i] = (int16_t)v;
        else if (elem_bytes == 4) ((int32_t*)out)[i] = (int32_t)v;
        else ((int64_t*)out)[i] = v;
        break;
      }
      case 2:
        ((uint64_t*)out)[i] = scramble64(__umul64hi(w, (uint64_t)n_distinct));
        break;
      case 3:
        ((uint32_t*)out)[i] = scramble32(zipf_rank(cdf, n_distinct, unit53(w)));
        break;
      case 4:
        ((uint64_t*)out)[i] = scramble64(zipf_rank(cdf, n_distinct, unit53(w)));
        break;
      case 5:
        ((double*)out)[i] = __dadd_rn(lo, __dmul_rn(unit53(w), __dsub_rn(hi, lo)));
        break;
      case 6: {
        uint64_t w2 = fmix_m3(row * 0xE7037ED1A0B428DBull + key2);
        double u1 = ((double)(w >> 11) + 0.5) * 0x1.0p-53;
        double u2 = ((double)(w2 >> 11) + 0.5) * 0x1.0p-53;
        double z = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
        ((double*)out)[i] = __dadd_rn(lo, __dmul_rn(hi, z));
        break;
      }
      default:
        break;
    }
  }
}

uint64_t column_key(uint64_t seed, uint32_t col) {
  return fmix_m3_host(seed ^ ((uint64_t)col * 0xA0761D6478BD642Full));
}

}  // namespace

extern "C" int dg_fill(int kind, void* out, int elem_bytes, int64_t n, int64_t row0, uint64_t seed,
                       uint32_t col, double lo, double hi, int64_t n_distinct, const double* cdf,
                       void* stream) {
  if (n < 0 || (n > 0 && out == nullptr)) return 1;
  if ((kind == 3 || kind == 4) && cdf == nullptr) return 1;
  if (n == 0) return 0;
  uint64_t key = column_key(seed, col);
  uint64_t key2 = column_key(seed, col + 1);
  int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  dg_kernel<<<(int)blocks, threads, 0, (cudaStream_t)stream>>>(kind, out, elem_bytes, n, row0, key,
                                                                key2, lo, hi, n_distinct, cdf);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
