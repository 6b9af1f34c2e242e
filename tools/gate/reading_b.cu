// SURVEY §7 decision gate (SURVEY.md:328): is the survey's balancing
// reading B -- byte-stratified start word + random butterfly, driven by a cheap counter stream --
// >= 1.5x faster than the frozen reading A (rejection flips, R2) as a standalone pac_mask?
// Measures both on 6e7 keys (k_mask_a re-implements R2 exactly as libpac does; checked against
// libpac's pac_mask by the harness), and dumps 2e5 reading-B masks for the statistical checks of
// SURVEY §8c (popcount 32, per-bit frequency, pairwise correlation -1/63).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gate_b reading_b.cu
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31;
  return z;
}

// ---------------- reading A (R2), as libpac's k_mask
__device__ __forceinline__ uint64_t hash_a(uint64_t key, uint64_t salt) {
  uint64_t x = fmix64(key ^ salt);
  int c = __popcll(x);
  if (c == 32) return x;
  const bool maj = c > 32;
  int k = maj ? c - 32 : 32 - c;
  uint64_t cand = maj ? x : ~x;
  uint64_t w = fmix64(x ^ 0xD1B54A32D192ED03ull);
  for (int word = 0; word < 64 && k > 0; ++word) {
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      const uint32_t f = (uint32_t)(w >> (6 * t)) & 63u;
      const uint64_t oh = (uint64_t)(uint32_t)min(k, 1) << f;
      const bool hit = (cand & oh) != 0ull;
      cand &= ~oh;
      k -= hit ? 1 : 0;
    }
    w = fmix64(w + 0x9E3779B97F4A7C15ull);
  }
  return maj ? cand : ~cand;
}

// ---------------- reading B (SURVEY §8c option B) with a cheap stream: LCG state + xorshift output
__constant__ unsigned char T70c[70];  // the 70 bytes with popcount 4, ascending (copied to smem)
__device__ __forceinline__ uint64_t delta_swap(uint64_t x, uint64_t ctl, int d) {
  const uint64_t t = ((x >> d) ^ x) & ctl;
  return x ^ t ^ (t << d);
}
__device__ __forceinline__ uint64_t hash_b(uint64_t key, uint64_t salt, const unsigned char* T70) {
  uint64_t s = fmix64(key ^ salt);
  uint64_t w[8];
  w[0] = s;
#pragma unroll
  for (int i = 1; i < 8; ++i) {  // cheap stream: LCG state, xorshift output
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    w[i] = s ^ (s >> 29) ^ (s >> 43);
  }
  // start word: byte b = T70[(16-bit field b of (w0, w1)) * 70 >> 16], 4 ones per byte
  uint64_t x = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t f = (uint32_t)(w[b >> 2] >> (16 * (b & 3))) & 0xFFFFu;
    x |= (uint64_t)T70[(f * 70u) >> 16] << (8 * b);
  }
  // random butterfly: stage d swaps bits p and p + d where control bit p is set; the control is a
  // stream word ANDed with the positions whose bit d is clear (32 usable bits per stage)
  const uint64_t M[6] = {0x00000000FFFFFFFFull, 0x0000FFFF0000FFFFull, 0x00FF00FF00FF00FFull,
                         0x0F0F0F0F0F0F0F0Full, 0x3333333333333333ull, 0x5555555555555555ull};
  const int D[6] = {32, 16, 8, 4, 2, 1};
#pragma unroll
  for (int i = 0; i < 6; ++i) x = delta_swap(x, w[2 + i] & M[i], D[i]);
  return x;
}

__global__ void k_mask_a(const long long* key, int64_t n, uint64_t salt, unsigned long long* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hash_a((uint64_t)key[i], salt);
}
__global__ void k_mask_b(const long long* key, int64_t n, uint64_t salt, unsigned long long* out) {
  __shared__ unsigned char T70[72];  // divergent lookups: shared memory, not the constant cache
  if (threadIdx.x < 70) T70[threadIdx.x] = T70c[threadIdx.x];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hash_b((uint64_t)key[i], salt, T70);
}
__global__ void k_keys(long long* key, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    key[i] = (long long)(fmix64((uint64_t)i * 0x9E3779B97F4A7C15ull) % 1500000ull);  // C2-like pu domain
}

int main(int argc, char** argv) {
  const int64_t n = 60000000;
  std::vector<unsigned char> t70;
  for (int b = 0; b < 256; ++b) if (__builtin_popcount(b) == 4) t70.push_back((unsigned char)b);
  cudaMemcpyToSymbol(T70c, t70.data(), 70);
  long long* key; unsigned long long* out;
  cudaMalloc(&key, n * 8); cudaMalloc(&out, n * 8);
  k_keys<<<148 * 8, 256>>>(key, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms_a = 1e30f, ms_b = 1e30f;
  for (int it = 0; it < 5; ++it) {
    float ms;
    cudaEventRecord(e0); k_mask_a<<<148 * 8, 256>>>(key, n, 0x243F6A8885A308D3ull, out); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < ms_a) ms_a = ms;
    cudaEventRecord(e0); k_mask_b<<<148 * 8, 256>>>(key, n, 0x243F6A8885A308D3ull, out); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < ms_b) ms_b = ms;
  }
  // statistics of reading B over 2e5 sequential keys (the realistic dense-key case)
  const int m = 200000;
  k_mask_b<<<148, 256>>>(key, 0, 0, out);  // warm
  std::vector<long long> hk(m);
  for (int i = 0; i < m; ++i) hk[i] = i;
  cudaMemcpy(key, hk.data(), m * 8, cudaMemcpyHostToDevice);
  k_mask_b<<<148, 256>>>(key, m, 0x243F6A8885A308D3ull, out);
  std::vector<unsigned long long> hm(m);
  cudaMemcpy(hm.data(), out, m * 8, cudaMemcpyDeviceToHost);
  int bad = 0; double freq[64] = {0}; static double co[64][64];
  for (int i = 0; i < m; ++i) {
    if (__builtin_popcountll(hm[i]) != 32) ++bad;
    for (int p = 0; p < 64; ++p) if ((hm[i] >> p) & 1) { freq[p] += 1; for (int q = p + 1; q < 64; ++q) if ((hm[i] >> q) & 1) co[p][q] += 1; }
  }
  double fdev = 0, rdev = 0;
  for (int p = 0; p < 64; ++p) { double f = freq[p] / m; if (fabs(f - 0.5) > fdev) fdev = fabs(f - 0.5); }
  for (int p = 0; p < 64; ++p) for (int q = p + 1; q < 64; ++q) {
    const double pp = freq[p] / m, qq = freq[q] / m, pq = co[p][q] / m;
    const double rho = (pq - pp * qq) / sqrt(pp * (1 - pp) * qq * (1 - qq));
    if (fabs(rho + 1.0 / 63) > rdev) rdev = fabs(rho + 1.0 / 63);
  }
  printf("{\"keys\": %lld, \"reading_A_ms\": %.4f, \"reading_B_ms\": %.4f, \"speedup\": %.3f, "
         "\"B_popcount_not_32\": %d, \"B_max_bitfreq_dev\": %.5f, \"B_max_abs_rho_plus_1_63\": %.5f}\n",
         (long long)n, ms_a, ms_b, ms_a / ms_b, bad, fdev, rdev);
  return 0;
}
