// libpac: m = 128 worlds (§8 f4; P:L92 footnote "Extending to m=128 is possible, and worst-case
// would double the cost of our stochastic-aggregates"; readings DESIGN.md R28, R29).
//
//  * k_mask128     row-parallel 128-bit balanced pac_hash (R28)
//  * pac_agg_grouped128 -- the 128-world aggregation as three passes of the 64-world kernels:
//      k_split128  masks [n][2] -> lo[n] (worlds 0..63), hi[n] (worlds 64..127), nz[n] = [lo|hi != 0]
//      pass N      COUNT over the masks nz: the exact group set and rows (a row is dropped only
//                  when both words are 0, R21)
//      pass L, H   the requested aggregates over the masks lo, and over hi (two full 64-world
//                  aggregations -- the paper's "double the cost")
//      k_merge128  lays L and H out on N's groups: world j < 64 from L, j >= 64 from H; groups
//                  absent from L or H take the empty state (count 0, sums 0, MIN +inf, MAX -inf)
//  * native path (agg.cu agg128_native, kernel k_agg_tiles128 in agg128.cu): for COUNT / SUM / AVG
//    with G_cap <= 32, one pass that hashes both words of a row and updates all 128 worlds
//    (PAC_NO_NATIVE128=1 forces the three passes)
//    The finalize over 128 worlds is pac_finalize with an m = 128 session (session.cu).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "hash128.cuh"

namespace pac {

__global__ void __launch_bounds__(256) k_mask128(const long long* __restrict__ key, int64_t n, uint64_t salt,
                                                 unsigned long long* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t lo, hi;
    pac_hash128_dev((uint64_t)__ldg(key + i), salt, lo, hi);
    out[2 * i] = lo;
    out[2 * i + 1] = hi;
  }
}

__global__ void __launch_bounds__(256) k_split128(const ulonglong2* __restrict__ m, int64_t n,
                                                  unsigned long long* __restrict__ lo,
                                                  unsigned long long* __restrict__ hi,
                                                  unsigned long long* __restrict__ nz) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const ulonglong2 v = __ldcs(m + i);
    lo[i] = v.x;
    hi[i] = v.y;
    nz[i] = (v.x | v.y) ? 1ull : 0ull;
  }
}

__device__ __forceinline__ int64_t find_key(const pac_table& t, uint64_t key) {
  const int64_t G = *t.d_num_groups;
  int64_t lo = 0, hi = G;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t.d_group_key[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < G && t.d_group_key[lo] == key) ? lo : -1;
}

struct MergeKinds {
  int k[PAC_MAX_AGGS];
  int n;
  int has_count;
};

// one warp per union group: lane j copies worlds j, j+32 of L (-> j, j+32) and of H (-> 64+j, 96+j)
__global__ void k_merge128(pac_table N, pac_table L, pac_table H, int64_t G_cap, MergeKinds mk, pac_table out) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int64_t G = min(*N.d_num_groups, G_cap);
  for (int64_t u = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); u < G; u += (int64_t)gridDim.x * wpb) {
    const uint64_t key = N.d_group_key[u];
    const int64_t gl = find_key(L, key), gh = find_key(H, key);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const pac_table& S = half ? H : L;
      const int64_t g = half ? gh : gl;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        const size_t src = (size_t)g * kM + j, dst = (size_t)u * kM2 + 64 * half + j;
        if (mk.has_count) out.d_count[dst] = g >= 0 ? S.d_count[src] : 0;
        for (int a = 0; a < mk.n; ++a) {
          const int k = mk.k[a];
          if (k == PAC_COUNT) continue;
          if (k == PAC_SUM_I64) {
            ((int64_t*)out.d_world[a])[dst] = g >= 0 ? ((const int64_t*)S.d_world[a])[src] : 0;
          } else {
            const double e = k == PAC_MIN_F64 ? INFINITY : (k == PAC_MAX_F64 ? -INFINITY : 0.0);
            ((double*)out.d_world[a])[dst] = g >= 0 ? ((const double*)S.d_world[a])[src] : e;
          }
        }
      }
    }
    if (lane == 0) {
      out.d_group_key[u] = key;
      out.d_rows[u] = N.d_rows[u];
      out.d_presence[2 * u] = gl >= 0 ? L.d_presence[gl] : 0ull;
      out.d_presence[2 * u + 1] = gh >= 0 ? H.d_presence[gh] : 0ull;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *out.d_num_groups = *N.d_num_groups;
    const int sn = *N.d_status, sl = *L.d_status, sh = *H.d_status;
    *out.d_status = sn ? sn : (sl ? sl : sh);
  }
}

// native single-pass path (agg.cu, kernel in agg128.cu)
bool agg128_native_ok(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, const pac_key_col* keys, int n_keys,
                      bool masked);
size_t agg128_native_ws(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap);
int agg128_native(const int64_t* d_pu_key, const uint64_t* d_mask2, uint64_t salt, const pac_key_col* keys,
                  int n_keys, const pac_agg_spec* aggs, int n_aggs, int64_t n_rows, const pac_table* out,
                  int64_t G_cap, void* d_ws, size_t ws_bytes, pac_stream_t stream);

static int grid_for(int64_t work, int per_block, int cap_mult) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + per_block - 1) / per_block, (int64_t)sms * cap_mult));
}

// Workspace carve-up of pac_agg_grouped128 (all pieces 256-byte aligned).
struct Ws128 {
  size_t masks, lo, hi, nz, tabN, tabL, tabH, aggws, bytes;
  size_t tab_bytes_N, tab_bytes_A, aggws_bytes;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// one 64-world table: num_groups, status, keys, rows, presence, count?, worlds
static size_t table64_bytes(int64_t G, bool has_count, int n_world) {
  return al(16) + 3 * al(8 * G) + (has_count ? al(8 * 64 * G) : 0) + (size_t)n_world * al(8 * 64 * G);
}

static pac_table carve_table(char* base, int64_t G, bool has_count, const int* kinds, int n_aggs) {
  pac_table t{};
  size_t off = 0;
  t.d_num_groups = (int64_t*)(base + off);
  t.d_status = (int32_t*)(base + off + 8);
  off += al(16);
  t.d_group_key = (uint64_t*)(base + off);
  off += al(8 * G);
  t.d_rows = (int64_t*)(base + off);
  off += al(8 * G);
  t.d_presence = (uint64_t*)(base + off);
  off += al(8 * G);
  if (has_count) {
    t.d_count = (int64_t*)(base + off);
    off += al(8 * 64 * G);
  }
  for (int a = 0; a < n_aggs; ++a) {
    if (kinds[a] == PAC_COUNT) continue;
    t.d_world[a] = base + off;
    off += al(8 * 64 * G);
  }
  t.m = 64;
  return t;
}

}  // namespace pac

using namespace pac;

extern "C" int pac_mask128(const int64_t* d_pu_key, int64_t n, uint64_t salt, uint64_t* d_mask2,
                           pac_stream_t stream) {
  if (n < 0 || (n > 0 && (!d_pu_key || !d_mask2))) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  k_mask128<<<grid_for(n, 256, 8), 256, 0, (cudaStream_t)stream>>>((const long long*)d_pu_key, n, salt,
                                                                   (unsigned long long*)d_mask2);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

static int ws128(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, int64_t n_rows, bool hashing, Ws128* w) {
  if (G_cap < 1 || n_rows < 0 || n_aggs < 1 || n_aggs > PAC_MAX_AGGS || !aggs) return PAC_E_INVAL;
  bool has_count = false;
  int n_world = 0;
  for (int a = 0; a < n_aggs; ++a) {
    const int k = aggs[a].kind;
    if (k < PAC_COUNT || k > PAC_MAX_F64) return PAC_E_INVAL;
    if (k != PAC_MIN_F64 && k != PAC_MAX_F64) has_count = true;  // as pac_agg_grouped: a count array
    if (k != PAC_COUNT) ++n_world;
  }
  pac_agg_spec cnt{PAC_COUNT, nullptr};
  size_t wsN = 0, wsA = 0;
  int rc = pac_agg_workspace_size(&cnt, 1, G_cap, &wsN);
  if (rc) return rc;
  rc = pac_agg_workspace_size(aggs, n_aggs, G_cap, &wsA);
  if (rc) return rc;
  w->tab_bytes_N = table64_bytes(G_cap, true, 0);
  w->tab_bytes_A = table64_bytes(G_cap, has_count, n_world);
  w->aggws_bytes = al(std::max(wsN, wsA));
  size_t off = 0;
  w->masks = off;
  off += hashing ? al((size_t)16 * n_rows) : 0;
  w->lo = off;
  off += al((size_t)8 * n_rows);
  w->hi = off;
  off += al((size_t)8 * n_rows);
  w->nz = off;
  off += al((size_t)8 * n_rows);
  w->tabN = off;
  off += w->tab_bytes_N;
  w->tabL = off;
  off += w->tab_bytes_A;
  w->tabH = off;
  off += w->tab_bytes_A;
  w->aggws = off;
  off += w->aggws_bytes;
  // room for the native single-pass path too (whichever path the call takes)
  w->bytes = std::max(off, agg128_native_ws(aggs, n_aggs, G_cap));
  return PAC_OK;
}

extern "C" int pac_agg_workspace_size128(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, int64_t n_rows,
                                         int hashing, size_t* bytes) {
  if (!bytes) return PAC_E_INVAL;
  Ws128 w;
  const int rc = ws128(aggs, n_aggs, G_cap, n_rows, hashing != 0, &w);
  if (rc) return rc;
  *bytes = w.bytes;
  return PAC_OK;
}

extern "C" int pac_agg_grouped128(const int64_t* d_pu_key, const uint64_t* d_mask2, uint64_t salt,
                                  const pac_key_col* keys, int n_keys, const pac_agg_spec* aggs, int n_aggs,
                                  int64_t n_rows, const pac_table* out, int64_t G_cap, void* d_ws, size_t ws_bytes,
                                  pac_stream_t stream) {
  if (n_rows < 0 || !out || out->m != 128 || (d_pu_key && d_mask2) || (!d_pu_key && !d_mask2 && n_rows > 0))
    return PAC_E_INVAL;
  Ws128 w;
  int rc = ws128(aggs, n_aggs, G_cap, n_rows, d_pu_key != nullptr, &w);
  if (rc) return rc;
  if (!d_ws || ws_bytes < w.bytes) return PAC_E_WORKSPACE;
  if (!out->d_num_groups || !out->d_status || !out->d_group_key || !out->d_rows || !out->d_presence)
    return PAC_E_INVAL;
  if (agg128_native_ok(aggs, n_aggs, G_cap, keys, n_keys, d_mask2 != nullptr))  // one pass, both mask words per row (agg128.cu)
    return agg128_native(d_pu_key, d_mask2, salt, keys, n_keys, aggs, n_aggs, n_rows, out, G_cap, d_ws, ws_bytes,
                         stream);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;
  int kinds[PAC_MAX_AGGS] = {0};
  bool has_count = false;
  for (int a = 0; a < n_aggs; ++a) {
    kinds[a] = aggs[a].kind;
    if (kinds[a] != PAC_MIN_F64 && kinds[a] != PAC_MAX_F64) has_count = true;
    if (kinds[a] != PAC_COUNT && !out->d_world[a]) return PAC_E_INVAL;
  }
  if (has_count && !out->d_count) return PAC_E_INVAL;
  unsigned long long* lo = (unsigned long long*)(ws + w.lo);
  unsigned long long* hi = (unsigned long long*)(ws + w.hi);
  unsigned long long* nz = (unsigned long long*)(ws + w.nz);
  if (n_rows > 0) {
    const uint64_t* m2 = d_mask2;
    if (d_pu_key) {
      rc = pac_mask128(d_pu_key, n_rows, salt, (uint64_t*)(ws + w.masks), stream);
      if (rc) return rc;
      m2 = (const uint64_t*)(ws + w.masks);
    }
    k_split128<<<grid_for(n_rows, 256, 8), 256, 0, st>>>((const ulonglong2*)m2, n_rows, lo, hi, nz);
    note_launch();
  }
  const int cnt_kind = PAC_COUNT;
  pac_table N = carve_table(ws + w.tabN, G_cap, true, &cnt_kind, 1);
  pac_table L = carve_table(ws + w.tabL, G_cap, has_count, kinds, n_aggs);
  pac_table H = carve_table(ws + w.tabH, G_cap, has_count, kinds, n_aggs);
  pac_agg_spec cnt{PAC_COUNT, nullptr};
  void* aws = ws + w.aggws;
  // pass N: the group set and the rows of nonzero 128-bit masks
  rc = pac_agg_grouped(nullptr, (const uint64_t*)nz, 0, keys, n_keys, &cnt, 1, n_rows, &N, G_cap, aws, w.aggws_bytes,
                       stream);
  if (rc) return rc;
  // passes L and H: worlds 0..63 and 64..127
  rc = pac_agg_grouped(nullptr, (const uint64_t*)lo, 0, keys, n_keys, aggs, n_aggs, n_rows, &L, G_cap, aws,
                       w.aggws_bytes, stream);
  if (rc) return rc;
  rc = pac_agg_grouped(nullptr, (const uint64_t*)hi, 0, keys, n_keys, aggs, n_aggs, n_rows, &H, G_cap, aws,
                       w.aggws_bytes, stream);
  if (rc) return rc;
  MergeKinds mk{};
  for (int a = 0; a < n_aggs; ++a) mk.k[a] = kinds[a];
  mk.n = n_aggs;
  mk.has_count = has_count ? 1 : 0;
  k_merge128<<<grid_for(G_cap, 8, 16), 256, 0, st>>>(N, L, H, G_cap, mk, *out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
