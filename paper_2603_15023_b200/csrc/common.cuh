// Device helpers shared by the libpac kernels (product side; independent of oracle/).
#pragma once
#include <cmath>
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

// pac_hash (§2, §4, R1 + R2 "rejection flips").
// `cand` holds the positions that still carry the majority value; a draw that lands on one
// while k > 0 flips it (k--).  The final mask is x ^ (cand_initial ^ cand_final).  Draws are
// processed one 10-draw word at a time, branch-free inside the word (predicated), so a warp
// diverges only at word granularity.
constexpr uint64_t kDrawSeed = 0xD1B54A32D192ED03ull;
constexpr uint64_t kDrawStep = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ void draw_step(uint64_t w, int t, uint64_t& cand, int& k) {
  // t is a compile-time constant (unrolled loops).  Field t = bits [6t, 6t + 6) of w; its bit 5
  // picks the 32-bit half of cand, its low 5 bits the position in that half (the wrapping funnel
  // shift reads only those 5 bits, so the field needs no masking): ~9 SASS per draw.
  const uint32_t wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
  const int o = 6 * t;
  uint32_t fs;
  bool hi;
  if (o + 5 < 32) {
    fs = wl >> o;
    hi = (wl >> (o + 5)) & 1u;
  } else if (o >= 32) {
    fs = wh >> (o - 32);
    hi = (wh >> (o + 5 - 32)) & 1u;
  } else {
    fs = __funnelshift_r(wl, wh, o);
    hi = (wh >> (o + 5 - 32)) & 1u;
  }
  const uint32_t b = __funnelshift_l(0u, 1u, fs);  // 1 << (fs & 31)
  uint32_t c0 = (uint32_t)cand, c1 = (uint32_t)(cand >> 32);
  const uint32_t sel = hi ? c1 : c0;
  if ((sel & b) != 0u && k > 0) {
    const uint32_t nv = sel ^ b;
    c1 = hi ? nv : c1;
    c0 = hi ? c0 : nv;
    --k;
  }
  cand = ((uint64_t)c1 << 32) | c0;
}

__device__ __forceinline__ void draw_word(uint64_t w, uint64_t& cand, int& k) {
#pragma unroll
  for (int t = 0; t < 10; ++t) draw_step(w, t, cand, k);
}

struct HashState {
  uint64_t x;     // fmix64(key ^ salt)
  uint64_t cand;  // current majority positions
  uint64_t w0;    // draw word 0 = fmix64(x ^ kDrawSeed)
  int k;          // flips still needed
};

// mix + popcount + the first draw word.  Returns the state after word 0.
__device__ __forceinline__ HashState pac_hash_begin(uint64_t key, uint64_t salt) {
  HashState h;
  h.x = fmix64(key ^ salt);
  const int c = __popcll(h.x);
  h.k = (c > 32) ? (c - 32) : (32 - c);
  h.cand = (c > 32) ? h.x : ~h.x;
  h.w0 = fmix64(h.x ^ kDrawSeed);
  draw_word(h.w0, h.cand, h.k);
  return h;
}

// Continues from the state after word `word0` (its draw word `w`) until k == 0 (or the R2
// safety net); `m` is the mask after that word.  The majority value is recovered from `m`:
// while k > 0 the mask still has popcount on the majority side.
__device__ __forceinline__ uint64_t pac_hash_continue(uint64_t m, uint64_t w) {
  const bool maj = __popcll(m) > 32;
  uint64_t cand = maj ? m : ~m;
  int k = maj ? (__popcll(m) - 32) : (32 - __popcll(m));
#pragma unroll 1
  for (int word = 1; word < 64 && k > 0; ++word) {
    w = fmix64(w + kDrawStep);
    draw_word(w, cand, k);
  }
  while (k > 0) {  // safety net of R2 (never reached in practice)
    const uint64_t low = cand & (~cand + 1ull);
    cand ^= low;
    --k;
  }
  return maj ? cand : ~cand;
}

// Two independent keys, their draws interleaved so the two dependency chains overlap.
__device__ __forceinline__ void pac_hash_begin2(uint64_t ka, uint64_t kb, uint64_t salt, HashState& a,
                                                HashState& b) {
  a.x = fmix64(ka ^ salt);
  b.x = fmix64(kb ^ salt);
  const int ca = __popcll(a.x), cb = __popcll(b.x);
  a.k = (ca > 32) ? (ca - 32) : (32 - ca);
  b.k = (cb > 32) ? (cb - 32) : (32 - cb);
  a.cand = (ca > 32) ? a.x : ~a.x;
  b.cand = (cb > 32) ? b.x : ~b.x;
  a.w0 = fmix64(a.x ^ kDrawSeed);
  b.w0 = fmix64(b.x ^ kDrawSeed);
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    draw_step(a.w0, t, a.cand, a.k);
    draw_step(b.w0, t, b.cand, b.k);
  }
}

// ---- the same draws with the one-hot position read from a 64-entry shared-memory table
// (entry p = {p < 32 ? 1 << p : 0, p >= 32 ? 1 << (p - 32) : 0}).  draw_step is 10 alu-pipe
// instructions of 11 (shifts, selects and logic ops all issue on the half-rate alu pipe), which
// is what bounds the hash phases.  Here the field becomes a table address with one shift and one
// LOP3 (the table is 512-byte aligned in the shared window, so base | offset needs no add), the
// one-hot pair comes through the otherwise idle LSU, the hit test is two logic ops and two
// compares, and the flip subtracts the one-hot word from each half under the hit predicate (the
// other half's word is 0; the hit bit is set, so c - b clears it) -- adds ptxas may place on the
// fma pipe.  Same arithmetic as draw_step (R2), bit for bit.
constexpr int kBtabBytes = 1024;  // reservation: a 512-byte table at the first 512-aligned address inside

// shared-window address of the table inside the reservation `raw`
__device__ __forceinline__ uint32_t btab_addr(const void* raw) {
  return ((uint32_t)__cvta_generic_to_shared(raw) + 511u) & ~511u;
}
__device__ __forceinline__ void btab_fill(uint32_t bt, int tid) {
  if (tid < 64) {
    const uint32_t lo = tid < 32 ? 1u << tid : 0u, hi = tid >= 32 ? 1u << (tid - 32) : 0u;
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(bt + 8u * tid), "r"(lo), "r"(hi) : "memory");
  }
}

__device__ __forceinline__ uint2 btab_load(uint32_t bt, uint64_t w, int t) {
  const uint32_t wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
  const int o = 6 * t;  // byte offset of the entry = field * 8
  uint32_t off;
  if (o == 0) off = wl << 3;
  else if (o + 6 <= 32) off = wl >> (o - 3);
  else if (o >= 32) off = wh >> (o - 35);  // o = 36, 42, 48, 54
  else off = __funnelshift_r(wl, wh, o - 3);  // o = 30: the field straddles the halves
  uint2 b;
  // not volatile: the table is written once before the first barrier, so the loads may move
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(b.x), "=r"(b.y) : "r"((off & 0x1F8u) | bt));
  return b;
}

__device__ __forceinline__ void draw_apply(uint2 b, uint32_t& c0, uint32_t& c1, int& k) {
#if PAC_DRAW_APPLY_C
  if (((c1 & b.y) | (c0 & b.x)) != 0u && k > 0) {
    c0 -= b.x;
    c1 -= b.y;
    --k;
  }
#else
  asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t"
      "and.b32 t, %0, %3;\n\t"
      "setp.gt.s32 q, %2, 0;\n\t"
      "lop3.and.b32 t|p, %1, %4, t, 0xEA, q;\n\t"  // p = ((c1 & b1) | (c0 & b0)) != 0 && k > 0
      "@p sub.u32 %0, %0, %3;\n\t"
      "@p sub.u32 %1, %1, %4;\n\t"
      "@p add.s32 %2, %2, -1;\n\t}"
      : "+r"(c0), "+r"(c1), "+r"(k)
      : "r"(b.x), "r"(b.y));
#endif
}

__device__ __forceinline__ void draw_word_bt(uint64_t w, uint64_t& cand, int& k, uint32_t bt) {
  uint32_t c0 = (uint32_t)cand, c1 = (uint32_t)(cand >> 32);
#pragma unroll
  for (int t = 0; t < 10; ++t) draw_apply(btab_load(bt, w, t), c0, c1, k);
  cand = ((uint64_t)c1 << 32) | c0;
}

__device__ __forceinline__ uint64_t pac_hash_continue_bt(uint64_t m, uint64_t w, uint32_t bt) {
  const bool maj = __popcll(m) > 32;
  uint64_t cand = maj ? m : ~m;
  int k = maj ? (__popcll(m) - 32) : (32 - __popcll(m));
#pragma unroll 1
  for (int word = 1; word < 64 && k > 0; ++word) {
    w = fmix64(w + kDrawStep);
    draw_word_bt(w, cand, k, bt);
  }
  while (k > 0) {  // safety net of R2 (never reached in practice)
    const uint64_t low = cand & (~cand + 1ull);
    cand ^= low;
    --k;
  }
  return maj ? cand : ~cand;
}

__device__ __forceinline__ void pac_hash_begin2_bt(uint64_t ka, uint64_t kb, uint64_t salt, HashState& a,
                                                   HashState& b, uint32_t bt) {
  a.x = fmix64(ka ^ salt);
  b.x = fmix64(kb ^ salt);
  const int ca = __popcll(a.x), cb = __popcll(b.x);
  a.k = (ca > 32) ? (ca - 32) : (32 - ca);
  b.k = (cb > 32) ? (cb - 32) : (32 - cb);
  a.cand = (ca > 32) ? a.x : ~a.x;
  b.cand = (cb > 32) ? b.x : ~b.x;
  a.w0 = fmix64(a.x ^ kDrawSeed);
  b.w0 = fmix64(b.x ^ kDrawSeed);
  uint32_t a0 = (uint32_t)a.cand, a1 = (uint32_t)(a.cand >> 32);
  uint32_t b0 = (uint32_t)b.cand, b1 = (uint32_t)(b.cand >> 32);
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    draw_apply(btab_load(bt, a.w0, t), a0, a1, a.k);
    draw_apply(btab_load(bt, b.w0, t), b0, b1, b.k);
  }
  a.cand = ((uint64_t)a1 << 32) | a0;
  b.cand = ((uint64_t)b1 << 32) | b0;
}

// mask after the draws so far: x with the flipped majority positions toggled
__device__ __forceinline__ uint64_t hash_mask_now(const HashState& h) {
  return (__popcll(h.x) > 32) ? h.cand : ~h.cand;
}

__device__ __forceinline__ uint64_t pac_hash_dev(uint64_t key, uint64_t salt) {
  const HashState h = pac_hash_begin(key, salt);
  const uint64_t m = hash_mask_now(h);
  if (h.k == 0) return m;
  return pac_hash_continue(m, h.w0);
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

enum { kTagCell = 0, kTagJstar = 1, kTagSalt = 2, kTagLift = 3, kTagFilter = 4 };  // R13, R24, R25

// ------------------------------------------------------------------ ordered f64 <-> int64
// Monotone map of doubles onto signed int64 under the total order of R31 (DuckDB's order on
// DOUBLE: IEEE order, every NaN equal and larger than +inf), so MIN/MAX become integer
// min/max and atomicMin/atomicMax.  Every NaN maps to kEncNaN (just above enc(+inf)).  The
// empty-world sentinels kMinEmpty / kMaxEmpty lie outside the range of every encoded value,
// so "world present" == "extreme != sentinel" holds exactly (a world holding only +inf under
// MIN, or only NaN, is present).
constexpr long long kEncNaN = 0x7FF8000000000000ll;
constexpr long long kMinEmpty = 0x7FFFFFFFFFFFFFFFll;            // empty MIN world
constexpr long long kMaxEmpty = (long long)0x8000000000000000ull;  // empty MAX world
__host__ __device__ __forceinline__ long long enc_f64(double v) {
#ifdef __CUDA_ARCH__
  long long i = __double_as_longlong(v);
#else
  long long i;
  memcpy(&i, &v, 8);
#endif
  if ((i & 0x7FFFFFFFFFFFFFFFll) > 0x7FF0000000000000ll) return kEncNaN;
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
// table value of an encoded extreme: an empty world reads +inf (MIN) / -inf (MAX)
__host__ __device__ __forceinline__ double dec_min(long long e) { return e == kMinEmpty ? INFINITY : dec_f64(e); }
__host__ __device__ __forceinline__ double dec_max(long long e) { return e == kMaxEmpty ? -INFINITY : dec_f64(e); }

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
