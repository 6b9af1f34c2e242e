// libpac: host side of k_agg_lean (agg_lean.cuh) -- applicability, raw-tile layout, launch.
// The kernel instances live in agg_lean_ks{0,1,2}.cu (one key spec each, compiled in parallel).
#include "agg_lean.cuh"

namespace pac {

typedef void (*LeanKernel)(AggPlan, int, int);
template <int KS, int OWN> LeanKernel lean_kernel(int ni, int nf);  // agg_lean_ks*.cu
void profile_begin(cudaStream_t st, const char* name);  // runtime.cu

bool lean_applicable(int ni, int nf, int has_min, int has_max, int has_count, int n_keys, int key_width,
                     int64_t G_cap, bool hashed) {
  if (getenv("PAC_NO_LEAN")) return false;
  if (has_min || has_max || !has_count || !hashed) return false;
  if (key_width > 4 || n_keys > PAC_MAX_KEYS) return false;
  if (ni + nf > 3) return false;  // owner mode: 8 slots x wps <= 128 TMEM columns per warp
  return G_cap >= 1 && G_cap <= kLeanLcap;
}

cudaError_t launch_lean(AggPlan& p, int n_keys, int key_width, int sms, cudaStream_t st, char* kname,
                        int kname_len) {
  const int ni = p.ni, nf = p.nf;
  const int wps = 2 + 4 * ni + 4 * nf;
  const bool owner = p.G_cap * wps > 128;
  const int lcap = owner ? kLeanLcap : 128 / wps;
  const int KS = n_keys == 0 ? 0 : (n_keys == 1 && key_width == 4) ? 1 : 2;
  const LeanLayout L = lean_layout(ni, nf);
  int off = 0;
  bool aligned = true;
  p.nraw = 0;
  auto add = [&](const void* col, int eb) {
    p.raw_src[p.nraw] = col;
    p.raw_eb[p.nraw] = eb;
    p.raw_off[p.nraw] = off;
    off += (kLeanT * eb + 15) & ~15;
    aligned = aligned && (((uintptr_t)col) & 15) == 0;
    ++p.nraw;
  };
  add(p.pu_key, 8);
  for (int c = 0; c < ni; ++c) add(p.icol[c], 8);
  for (int c = 0; c < nf; ++c) add(p.fcol[c], 8);
  for (int c = 0; c < n_keys; ++c) add(p.key_col[c], p.key_bytes[c]);
  if (off > L.raw_bytes) return cudaErrorInvalidValue;
  int copied = 0;
  for (int i = 0; i < p.nraw; ++i) copied += kLeanT * p.raw_eb[i];
  p.raw_bytes = copied;
  p.tma_ok = (aligned && !getenv("PAC_NO_TMA")) ? 1 : 0;
  LeanKernel k = KS == 0 ? lean_kernel<0, 0>(ni, nf)
                 : KS == 1 ? (owner ? lean_kernel<1, 1>(ni, nf) : lean_kernel<1, 0>(ni, nf))
                           : (owner ? lean_kernel<2, 1>(ni, nf) : lean_kernel<2, 0>(ni, nf));
  if (!k) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (p.n_rows + kLeanT - 1) / kLeanT;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms));
  snprintf(kname, kname_len, "k_agg_lean<%d,%d,%d,%d>", ni, nf, KS, owner ? 1 : 0);
  if (getenv("PAC_DEBUG"))
    fprintf(stderr, "[libpac] %s %d CTAs x %d threads, mode %s, lcap %d, smem %d B, tma %d\n", kname, grid,
            kLeanThreads, owner ? "owner" : "private", lcap, L.bytes, p.tma_ok);
  profile_begin(st, kname);
  k<<<grid, kLeanThreads, L.bytes, st>>>(p, owner ? 1 : 0, lcap);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pac
