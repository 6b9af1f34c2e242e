// libpac: partition-first grouped aggregation for high-cardinality tables (DESIGN.md §5
// "C3: partition first"; the per-thread partitioned tables of P:L1777 §5, done by group hash).
//
// When a table has far more groups than a CTA holds (G_cap >> Lcap, e.g. BASELINE C3: 1e6 Zipf
// groups), first-touch CTA dictionaries catch about half of the rows and the rest take the HBM
// tier.  Instead the rows are first partitioned by a hash of their group key into P = 2^pbits
// partitions of at most ~128 groups each (by capacity), so one CTA can hold a whole partition:
//   pass 1  k_part_hist + k_part_scan + k_part_scatter on the top 7 bits of the partition id;
//           the pu keys are hashed here (pac_hash, R1/R2) and written as masks
//   pass 2  the same on all pbits bits, over pass 1's output (a CTA's chunk then spans one or two
//           pass-1 buckets, so its write cursors stay few and L2 merges the scattered stores);
//           every partition starts on a 16-row boundary (mask-0 padding rows, dropped by R21) so
//           the aggregation can stage its tiles with TMA
//   units   each partition is cut into units of at most kUnitRows rows; the tile kernels
//           (k_agg_tiles_tm / k_agg_tiles) take units from a global counter and flush and reset
//           their CTA table after each unit
// Within a partition the row order is not preserved (f64 sums: R34).  Integers are exact.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace pac {

void note_launch();

constexpr int kPartCols = 2 + PAC_MAX_KEYS + 5;  // mask/pu, keys, values
constexpr int kPartThreads = 512;

struct PartPlan {
  int64_t n;                // input rows
  int ncol;                 // columns moved (column 0: pu key or mask)
  const void* src[kPartCols];
  void* dst[kPartCols];
  int eb[kPartCols];        // element bytes (1, 2, 4, 8)
  int hash0;                // 1: dst column 0 = pac_hash(src column 0)
  uint64_t salt;
  int n_keys;               // group-key columns: src columns 1 .. n_keys
  int key_bytes[PAC_MAX_KEYS];
  int pbits;                // partition id bits
  int shift;                // digit of this pass = id >> shift
  int nbins;                // 1 << (pbits - shift)
  int64_t chunk;            // rows per CTA
};

__device__ __forceinline__ uint32_t part_id(const PartPlan& q, int64_t r) {
  uint64_t packed = 0;
#pragma unroll
  for (int c = 0; c < PAC_MAX_KEYS; ++c) {
    if (c < q.n_keys) {
      const int w = q.key_bytes[c];
      const uint64_t v = load_key_part(q.src[1 + c], w, r);
      packed = (w == 8) ? v : ((packed << (8 * w)) | v);
    }
  }
  return dict_hash(packed ^ 0xA24BAED4963EE407ull) >> (32 - q.pbits);
}

constexpr int kPR = 8;  // rows per thread and iteration (independent loads in flight)

// hist[b * grid + cta] = rows of the CTA's chunk in bin b
__global__ void __launch_bounds__(kPartThreads) k_part_hist(PartPlan q, int* __restrict__ hist) {
  extern __shared__ int sh[];
  for (int b = threadIdx.x; b < q.nbins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * q.chunk, r1 = min(q.n, r0 + q.chunk);
  for (int64_t rb = r0 + threadIdx.x; rb < r1; rb += (int64_t)blockDim.x * kPR) {
    uint32_t bin[kPR];
#pragma unroll
    for (int k = 0; k < kPR; ++k) {
      const int64_t r = rb + (int64_t)k * blockDim.x;
      bin[k] = r < r1 ? part_id(q, r) >> q.shift : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int k = 0; k < kPR; ++k)
      if (bin[k] != 0xFFFFFFFFu) atomicAdd(&sh[bin[k]], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < q.nbins; b += blockDim.x) hist[(size_t)b * gridDim.x + blockIdx.x] = sh[b];
}

// bin totals (one thread per bin): tot[b] = sum over CTAs
__global__ void k_part_totals(const int* __restrict__ hist, int nbins, int grid, int* __restrict__ tot) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  int s = 0;
  for (int c = 0; c < grid; ++c) s += hist[(size_t)b * grid + c];
  tot[b] = s;
}

// Single CTA: bin starts (each bin padded to `align` rows), unit counts per bin and their starts.
// start[nbins] = padded total rows; ustart[nbins] = units.
__global__ void __launch_bounds__(1024) k_part_scan(const int* __restrict__ tot, int nbins, int align, int unit_rows,
                                                    long long* __restrict__ start, int* __restrict__ ustart) {
  __shared__ long long s_carry;
  __shared__ int s_ucarry;
  __shared__ long long s_w[32];
  __shared__ int s_uw[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_carry = 0;
    s_ucarry = 0;
  }
  __syncthreads();
  for (int b0 = 0; b0 < nbins; b0 += blockDim.x) {
    const int b = b0 + threadIdx.x;
    const long long pad = b < nbins ? ((long long)tot[b] + align - 1) / align * align : 0;
    const int units = (int)((pad + unit_rows - 1) / unit_rows);
    long long x = pad;
    int u = units;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, d);
      const int v = __shfl_up_sync(0xffffffffu, u, d);
      if (lane >= d) {
        x += y;
        u += v;
      }
    }
    if (lane == 31) {
      s_w[wid] = x;
      s_uw[wid] = u;
    }
    __syncthreads();
    if (wid == 0) {
      long long wx = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
      int wu = lane < (int)(blockDim.x >> 5) ? s_uw[lane] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, wx, d);
        const int v = __shfl_up_sync(0xffffffffu, wu, d);
        if (lane >= d) {
          wx += y;
          wu += v;
        }
      }
      s_w[lane] = wx;  // inclusive warp prefix
      s_uw[lane] = wu;
    }
    __syncthreads();
    const long long before = s_carry + (wid > 0 ? s_w[wid - 1] : 0) + x - pad;
    const int ubefore = s_ucarry + (wid > 0 ? s_uw[wid - 1] : 0) + u - units;
    if (b < nbins) {
      start[b] = before;
      ustart[b] = ubefore;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      s_carry = before + pad;
      s_ucarry = ubefore + units;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    start[nbins] = s_carry;
    ustart[nbins] = s_ucarry;
  }
}

// Per bin (one thread): the CTAs' write offsets (in place over hist), the padding rows' masks
// (0: dropped by R21) and, with units, the bin's unit row ranges.
__global__ void k_part_offsets(int* __restrict__ hist, int nbins, int grid, const int* __restrict__ tot,
                               const long long* __restrict__ start, void* mask_dst, int mask_eb,
                               const int* __restrict__ ustart, int unit_rows, longlong2* __restrict__ units) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  long long o = start[b];
  for (int c = 0; c < grid; ++c) {
    const int h = hist[(size_t)b * grid + c];
    hist[(size_t)b * grid + c] = (int)o;  // < 2^31 rows per call (pac_agg_grouped checks)
    o += h;
  }
  const long long end = start[b + 1];
  for (long long r = o; r < end; ++r) ((unsigned long long*)mask_dst)[r] = 0ull;  // 8-byte masks
  if (units) {
    int u = ustart[b];
    for (long long r = start[b]; r < end; r += unit_rows) units[u++] = make_longlong2(r, min(end, r + unit_rows));
  }
}

__device__ __forceinline__ uint64_t load_elem(const void* src, int eb, int64_t i) {
  switch (eb) {
    case 1: return __ldg((const uint8_t*)src + i);
    case 2: return __ldg((const uint16_t*)src + i);
    case 4: return __ldg((const uint32_t*)src + i);
    default: return __ldg((const unsigned long long*)src + i);
  }
}
__device__ __forceinline__ void store_elem(void* dst, int eb, int64_t i, uint64_t v) {
  switch (eb) {
    case 1: ((uint8_t*)dst)[i] = (uint8_t)v; break;
    case 2: ((uint16_t*)dst)[i] = (uint16_t)v; break;
    case 4: ((uint32_t*)dst)[i] = (uint32_t)v; break;
    default: ((unsigned long long*)dst)[i] = v; break;
  }
}

// rows of the CTA's chunk to their bins' next positions (write cursors in shared memory); kPR
// rows per thread: their bins first, then column by column kPR independent loads and stores
__global__ void __launch_bounds__(kPartThreads) k_part_scatter(PartPlan q, const int* __restrict__ offs) {
  extern __shared__ int cur[];
  for (int b = threadIdx.x; b < q.nbins; b += blockDim.x) cur[b] = offs[(size_t)b * gridDim.x + blockIdx.x];
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * q.chunk, r1 = min(q.n, r0 + q.chunk);
  for (int64_t rb = r0 + threadIdx.x; rb < r1; rb += (int64_t)blockDim.x * kPR) {
    uint32_t bin[kPR];
#pragma unroll
    for (int k = 0; k < kPR; ++k) {
      const int64_t r = rb + (int64_t)k * blockDim.x;
      bin[k] = r < r1 ? part_id(q, r) >> q.shift : 0xFFFFFFFFu;
    }
    int pos[kPR];
#pragma unroll
    for (int k = 0; k < kPR; ++k) pos[k] = bin[k] != 0xFFFFFFFFu ? atomicAdd(&cur[bin[k]], 1) : -1;
    for (int c = 0; c < q.ncol; ++c) {
      uint64_t v[kPR];
#pragma unroll
      for (int k = 0; k < kPR; ++k) v[k] = pos[k] >= 0 ? load_elem(q.src[c], q.eb[c], rb + (int64_t)k * blockDim.x) : 0;
      if (c == 0 && q.hash0) {
#pragma unroll
        for (int k = 0; k < kPR; ++k) v[k] = pos[k] >= 0 ? pac_hash_dev(v[k], q.salt) : 0;
      }
#pragma unroll
      for (int k = 0; k < kPR; ++k)
        if (pos[k] >= 0) store_elem(q.dst[c], q.eb[c], pos[k], v[k]);
    }
  }
}

// ------------------------------------------------------------------ host
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// Workspace of part_rows (beyond the aggregation's own): two column sets of n + pad rows, the
// histograms, bin starts and the unit list.
size_t part_ws_bytes(int64_t n_rows, int n_cols_max, int row_bytes, int pbits, int grid, int unit_rows) {
  const int64_t P = (int64_t)1 << pbits;
  const int64_t rows = n_rows + 16 * P;
  size_t b = 2 * (al256((size_t)rows * row_bytes) + (size_t)n_cols_max * 256);
  b += al256(4 * (size_t)P * grid) + al256(4 * (size_t)P) + al256(8 * (size_t)(P + 1)) + al256(4 * (size_t)(P + 1));
  b += al256(16 * (size_t)(P + n_rows / unit_rows + 2)) + 256 + 256;
  return b;
}

struct PartResult {
  const void* col[kPartCols];  // partitioned columns (column 0: masks)
  const longlong2* units;
  const int* n_units;          // device
  int* unit_ctr;               // device, zeroed
  int64_t rows;                // padded rows (upper bound n + 16 P)
};

// Partitions the rows (two passes) into the workspace.  cols: src[0] = pu keys (hash0) or masks,
// then the key columns, then the value columns.  Returns PAC_OK or PAC_E_CUDA.
int part_rows(const void* const* src, const int* eb, int ncol, int hash0, uint64_t salt, int n_keys,
              int64_t n_rows, int pbits, int grid, int unit_rows, char* ws, PartResult* out, cudaStream_t st) {
  const int64_t P = (int64_t)1 << pbits;
  const int64_t rows = n_rows + 16 * P;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = ws + off;
    off += al256(bytes);
    return p;
  };
  void* setA[kPartCols];
  void* setB[kPartCols];
  const int eb0 = hash0 ? 8 : eb[0];
  for (int c = 0; c < ncol; ++c) setA[c] = take((size_t)rows * (c == 0 ? eb0 : eb[c]));
  for (int c = 0; c < ncol; ++c) setB[c] = take((size_t)rows * (c == 0 ? eb0 : eb[c]));
  int* hist = (int*)take(4 * (size_t)P * grid);
  int* tot = (int*)take(4 * (size_t)P);
  long long* start = (long long*)take(8 * (size_t)(P + 1));
  int* ustart = (int*)take(4 * (size_t)(P + 1));
  longlong2* units = (longlong2*)take(16 * (size_t)(P + n_rows / unit_rows + 2));
  int* ctr = (int*)take(4);
  if (cudaMemsetAsync(ctr, 0, 4, st) != cudaSuccess) return PAC_E_CUDA;

  PartPlan q{};
  q.ncol = ncol;
  q.salt = salt;
  q.n_keys = n_keys;
  for (int c = 0; c < n_keys; ++c) q.key_bytes[c] = eb[1 + c];
  q.pbits = pbits;
  const int d1 = std::min(pbits, 7);
  for (int pass = 0; pass < 2; ++pass) {
    q.n = n_rows;  // pass 2 reads pass 1's n_rows rows (pass 1 pads nothing)
    q.hash0 = pass == 0 ? hash0 : 0;
    for (int c = 0; c < ncol; ++c) {
      q.src[c] = pass == 0 ? src[c] : setA[c];
      q.dst[c] = pass == 0 ? setA[c] : setB[c];
      q.eb[c] = (pass == 1 && c == 0) ? eb0 : eb[c];
    }
    q.shift = pass == 0 ? pbits - d1 : 0;
    q.nbins = 1 << (pbits - q.shift);
    q.chunk = (n_rows + grid - 1) / grid;
    const size_t sm = 4 * (size_t)q.nbins;
    if (sm > 48 * 1024) {
      if (cudaFuncSetAttribute(k_part_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
          cudaFuncSetAttribute(k_part_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return PAC_E_CUDA;
    }
    k_part_hist<<<grid, kPartThreads, sm, st>>>(q, hist);
    k_part_totals<<<(q.nbins + 255) / 256, 256, 0, st>>>(hist, q.nbins, grid, tot);
    const int align = pass == 0 ? 1 : 16;
    k_part_scan<<<1, 1024, 0, st>>>(tot, q.nbins, align, unit_rows, start, ustart);
    k_part_offsets<<<(q.nbins + 255) / 256, 256, 0, st>>>(hist, q.nbins, grid, tot, start, q.dst[0], q.eb[0],
                                                          ustart, unit_rows, pass == 0 ? nullptr : units);
    k_part_scatter<<<grid, kPartThreads, sm, st>>>(q, hist);
    for (int k = 0; k < 5; ++k) note_launch();
  }
  for (int c = 0; c < ncol; ++c) out->col[c] = setB[c];
  out->units = units;
  out->n_units = ustart + P;
  out->unit_ctr = ctr;
  out->rows = rows;
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

}  // namespace pac
