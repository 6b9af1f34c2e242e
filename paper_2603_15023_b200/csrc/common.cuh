// Device helpers shared by the libpac kernels (product side; independent of oracle/).
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/pac.h"

namespace pac {

constexpr int kM = PAC_M;

// ------------------------------------------------------------------ launch accounting
void note_launch();  // runtime.cu: counts every kernel launch of the library

// ------------------------------------------------------------------ hashing
// SplitMix64 finalizer (R1).
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// pac_hash (§2, §4, R1 + R2 "rejection flips").  `cand` tracks the
// positions that still hold the majority value; a draw that lands on one flips it.
__device__ __forceinline__ uint64_t pac_hash_dev(uint64_t key, uint64_t salt) {
  uint64_t x = fmix64(key ^ salt);
  int c = __popcll(x);
  if (c == 32) return x;
  uint64_t cand = (c > 32) ? x : ~x;
  int k = (c > 32) ? (c - 32) : (32 - c);
  uint64_t w = fmix64(x ^ 0xD1B54A32D192ED03ull);
#pragma unroll 1
  for (int word = 0; word < 64; ++word) {
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      uint32_t p = (uint32_t)(w >> (6 * t)) & 63u;
      uint64_t bit = 1ull << p;
      if (cand & bit) {
        cand ^= bit;
        x ^= bit;
        if (--k == 0) return x;
      }
    }
    w = fmix64(w + 0x9E3779B97F4A7C15ull);
  }
  while (k > 0) {  // safety net of R2 (never reached in practice)
    uint64_t low = cand & (~cand + 1ull);
    cand ^= low;
    x ^= low;
    --k;
  }
  return x;
}

// ------------------------------------------------------------------ Philox4x32-10 (R13)
struct u32x4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    u32x4 n;
    n.x = (uint32_t)(p1 >> 32) ^ c.y ^ k0;
    n.y = (uint32_t)p1;
    n.z = (uint32_t)(p0 >> 32) ^ c.w ^ k1;
    n.w = (uint32_t)p0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

enum { kTagCell = 0, kTagJstar = 1, kTagSalt = 2 };

// ------------------------------------------------------------------ ordered f64 <-> int64
// Monotone map of doubles onto signed int64, so MIN/MAX become atomicMin/atomicMax.
__host__ __device__ __forceinline__ long long enc_f64(double v) {
#ifdef __CUDA_ARCH__
  long long i = __double_as_longlong(v);
#else
  long long i;
  memcpy(&i, &v, 8);
#endif
  return i >= 0 ? i : (i ^ 0x7FFFFFFFFFFFFFFFll);
}
__host__ __device__ __forceinline__ double dec_f64(long long i) {
  long long b = i >= 0 ? i : (i ^ 0x7FFFFFFFFFFFFFFFll);
#ifdef __CUDA_ARCH__
  return __longlong_as_double(b);
#else
  double v;
  memcpy(&v, &b, 8);
  return v;
#endif
}
constexpr long long kEncPosInf = 0x7FF0000000000000ll;                 // enc(+inf)
constexpr long long kEncNegInf = (long long)0x800FFFFFFFFFFFFFull;     // enc(-inf)

// ------------------------------------------------------------------ group keys (R20)
__device__ __forceinline__ uint64_t load_key_part(const void* col, int w, int64_t row) {
  uint64_t v;
  if (w == 1) v = (uint8_t)__ldg((const signed char*)col + row);
  else if (w == 2) v = (uint16_t)__ldg((const short*)col + row);
  else if (w == 4) v = (uint32_t)__ldg((const int*)col + row);
  else v = (uint64_t)__ldg((const long long*)col + row);
  return v ^ (1ull << (8 * w - 1));
}

// hash for dictionary probing (product-side; any good mixer works)
__device__ __forceinline__ uint32_t dict_hash(uint64_t k) {
  return (uint32_t)(fmix64(k ^ 0x9E3779B97F4A7C15ull) >> 32);
}

}  // namespace pac
