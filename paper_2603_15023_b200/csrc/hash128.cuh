// 128-bit balanced pac_hash (R28; §8 f4, P:L92 footnote), shared by m128.cu (k_mask128) and the
// native 128-world tile kernel (agg128.cu).
#pragma once
#include "common.cuh"

namespace pac {

constexpr int kM2 = 128;
constexpr uint64_t kHi128 = 0x6A09E667F3BCC909ull;

// R28: rejection flips over 128 positions with 7-bit draws (9 per word), branch-free per word
__device__ __forceinline__ void draw_word128(uint64_t w, uint64_t& c0, uint64_t& c1, int& k) {
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const uint32_t p = (uint32_t)(w >> (7 * t)) & 127u;
    const uint64_t oh = (uint64_t)(uint32_t)min(k, 1) << (p & 63u);
    const uint64_t o0 = p < 64 ? oh : 0ull, o1 = p < 64 ? 0ull : oh;
    const bool hit = ((c0 & o0) | (c1 & o1)) != 0ull;
    c0 &= ~o0;
    c1 &= ~o1;
    k -= hit ? 1 : 0;
  }
}

__device__ __forceinline__ void pac_hash128_dev(uint64_t key, uint64_t salt, uint64_t& lo, uint64_t& hi) {
  const uint64_t x0 = fmix64(key ^ salt);
  const uint64_t x1 = fmix64(x0 ^ kHi128);
  const int c = __popcll(x0) + __popcll(x1);
  const bool maj = c > 64;
  int k = maj ? c - 64 : 64 - c;
  uint64_t c0 = maj ? x0 : ~x0, c1 = maj ? x1 : ~x1;  // positions carrying the majority value
  uint64_t w = fmix64(x0 ^ x1 ^ kDrawSeed);
  draw_word128(w, c0, c1, k);
#pragma unroll 1
  for (int word = 1; word < 64 && k > 0; ++word) {
    w = fmix64(w + kDrawStep);
    draw_word128(w, c0, c1, k);
  }
  while (k > 0) {  // safety net of R2 / R28 (never reached in practice)
    if (c0) c0 &= c0 - 1; else c1 &= c1 - 1;
    --k;
  }
  lo = maj ? c0 : ~c0;
  hi = maj ? c1 : ~c1;
}


// The same hash as a first draw word plus resumable steps (k_agg_tiles128 finishes the rows that
// need more than one word in full-warp passes, one word per pass):
// word 0: the partial mask, and the state to resume from -- w the last draw word, k the flips
// still owed, maj (the candidates are maj ? mask : ~mask, the majority positions not flipped yet)
__device__ __forceinline__ void pac_hash128_word0(uint64_t key, uint64_t salt, uint64_t& lo, uint64_t& hi,
                                                  uint64_t& w, int& k, bool& maj) {
  const uint64_t x0 = fmix64(key ^ salt);
  const uint64_t x1 = fmix64(x0 ^ kHi128);
  const int c = __popcll(x0) + __popcll(x1);
  maj = c > 64;
  k = maj ? c - 64 : 64 - c;
  uint64_t c0 = maj ? x0 : ~x0, c1 = maj ? x1 : ~x1;
  w = fmix64(x0 ^ x1 ^ kDrawSeed);
  draw_word128(w, c0, c1, k);
  lo = maj ? c0 : ~c0;
  hi = maj ? c1 : ~c1;
}
// draw word `word` (1..63) on a resumed state; after word 63 the safety net of pac_hash128_dev
__device__ __forceinline__ void pac_hash128_step(int word, uint64_t& w, uint64_t& c0, uint64_t& c1, int& k) {
  w = fmix64(w + kDrawStep);
  draw_word128(w, c0, c1, k);
  if (word == 63) {
    while (k > 0) {
      if (c0) c0 &= c0 - 1; else c1 &= c1 - 1;
      --k;
    }
  }
}

}  // namespace pac
