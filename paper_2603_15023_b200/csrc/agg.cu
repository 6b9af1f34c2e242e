// libpac: mask hash (§8 a2), grouped 64-world aggregation (a3-a5) and table helpers.
//
// Design:
//  * k_mask: row-parallel pac_hash.
//  * k_agg_tiles<NI,NF,MM>: persistent CTAs over contiguous row ranges, tiles of T rows.
//      phase A (row-parallel): fused pac_hash, group key packing, CTA-local slot lookup
//               (smem dictionary in front of the HBM dictionary), rows staged in smem;
//      phase B: counting sort of the tile's rows by local slot;
//      phase C (world-parallel): each warp takes runs of <= 32 same-slot rows, lane l owns
//               worlds l and l+32, register accumulators, flushed to the CTA's smem table;
//      end:     CTA tables flushed into the provisional HBM table (int64 / f64 atomics).
//  * k_agg_minmax: MIN/MAX-only, pruned: per-CTA cached bounds; rows that
//               cannot improve them are counted and skipped without hashing.
//  * finish: provisional slots sorted by packed key (canonical order R12/R20), gathered
//               into the caller's table; K re-derived from counts / extremes.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "agg_tiles.cuh"
#include "agg_tm.cuh"
#include "agg_ws.cuh"
#include "agg_lean.cuh"

namespace pac {

// ------------------------------------------------------------------ k_mask
// pac_hash (R1, R2) row-parallel.  Each warp takes 256 consecutive keys (8 per lane, coalesced):
// mix, popcount and draw word 0 branch-free for two keys at a time (pac_hash_begin2); the keys that
// still need flips are queued per warp and finished with all 32 lanes busy, so no lane loops alone
// through its later draw words while the other 31 wait.
constexpr int kMaskR = 8;
#ifndef PAC_MASK_BTAB
#define PAC_MASK_BTAB 1  // 1: the draws read their one-hot words from a shared-memory table (common.cuh): 88.8 -> 111.3 Gkeys/s
#endif
__global__ void __launch_bounds__(256) k_mask(const long long* __restrict__ key, int64_t n,
                                              uint64_t salt, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long qm[8][32 * kMaskR], qw[8][32 * kMaskR];
#if PAC_MASK_BTAB
  __shared__ __align__(16) unsigned char s_bt[kBtabBytes];  // one-hot table of the hash draws (common.cuh)
  const uint32_t bt = btab_addr(s_bt);
  btab_fill(bt, threadIdx.x);
  __syncthreads();
#endif
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t step = (int64_t)gridDim.x * 256 * kMaskR;
  for (int64_t b0 = (int64_t)blockIdx.x * 256 * kMaskR + wid * 32 * kMaskR; b0 < n; b0 += step) {
    unsigned long long x[kMaskR];
#pragma unroll
    for (int j = 0; j < kMaskR; ++j) {
      const int64_t r = b0 + 32 * j + lane;
      x[j] = r < n ? (unsigned long long)__ldg(key + r) : 0ull;
    }
    int qn = 0;
#pragma unroll
    for (int j = 0; j < kMaskR; j += 2) {
      HashState ha, hb;
#if PAC_MASK_BTAB
      pac_hash_begin2_bt(x[j], x[j + 1], salt, ha, hb, bt);
#else
      pac_hash_begin2(x[j], x[j + 1], salt, ha, hb);
#endif
      x[j] = hash_mask_now(ha);
      x[j + 1] = hash_mask_now(hb);
      const unsigned ba = __ballot_sync(0xffffffffu, ha.k > 0);
      if (ha.k > 0) {
        const int qi = qn + __popc(ba & lt);
        qm[wid][qi] = x[j];
        qw[wid][qi] = ha.w0;
      }
      qn += __popc(ba);
      const unsigned bb = __ballot_sync(0xffffffffu, hb.k > 0);
      if (hb.k > 0) {
        const int qi = qn + __popc(bb & lt);
        qm[wid][qi] = x[j + 1];
        qw[wid][qi] = hb.w0;
      }
      qn += __popc(bb);
    }
    __syncwarp();
#if PAC_MASK_BTAB
    for (int qi = lane; qi < qn; qi += 32) qm[wid][qi] = pac_hash_continue_bt(qm[wid][qi], qw[wid][qi], bt);
#else
    for (int qi = lane; qi < qn; qi += 32) qm[wid][qi] = pac_hash_continue(qm[wid][qi], qw[wid][qi]);
#endif
    __syncwarp();
    int qp = 0;  // the queue order again: (pair, a before b, lane)
#pragma unroll
    for (int j = 0; j < kMaskR; ++j) {
      const bool st = __popcll(x[j]) != 32;
      const unsigned bq = __ballot_sync(0xffffffffu, st);
      if (st) x[j] = qm[wid][qp + __popc(bq & lt)];
      qp += __popc(bq);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kMaskR; ++j) {
      const int64_t r = b0 + 32 * j + lane;
      if (r < n) out[r] = x[j];
    }
  }
}

// ------------------------------------------------------------------ k_agg_minmax (pruned)
constexpr int kMMQueue = 64;  // k_agg_minmax_v: candidate rows queued per warp
#ifndef PAC_MM_HINT_EVERY
#define PAC_MM_HINT_EVERY 8
#endif
constexpr int kMMHintEvery = PAC_MM_HINT_EVERY;  // tiles between pulls of the per-slot bound hints
struct MMLayout {
  int Lcap, LH;
  int o_lkey, o_lstate, o_lprov, o_lrows, o_bmin, o_bmax, o_dirty, o_misc, o_qr, o_qv, o_qp, o_stage;
  int bytes;
};

// k_agg_minmax_v stages its next tile with cp.async (16-byte LDGSTS per thread: 4 keys + 4 values)
// while it works on the current one, so the global loads are in flight during the dictionary and
// bound work instead of stalling it (long_scoreboard); 0 = plain loads at the top of the tile
#ifndef PAC_MM_STAGE
#define PAC_MM_STAGE 1
#endif
constexpr int kMMStageBytes = 48;  // per thread: int4 keys + 2 x double2 values
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}

#ifndef PAC_MM_LH
#define PAC_MM_LH 4
#endif
__host__ __device__ constexpr MMLayout mm_layout_for(int Lcap, bool vstage = false) {
  // vstage (k_agg_minmax_v with PAC_MM_STAGE): no probe-state array (the packed dictionary does
  // not use it), a per-thread staging area instead -- two CTAs per SM still fit at Lcap = 1024
  MMLayout L{};
  L.Lcap = Lcap;
  L.LH = lay_pow2(PAC_MM_LH * Lcap > 256 ? PAC_MM_LH * Lcap : 256);
  int off = 0;
  L.o_lkey = lay_take(off, L.LH * 8);
  L.o_lrows = lay_take(off, Lcap * 4);
  L.o_bmin = lay_take(off, Lcap * 8);
  L.o_bmax = lay_take(off, Lcap * 8);
  L.o_lstate = vstage ? 0 : lay_take(off, L.LH * 4);
  L.o_lprov = lay_take(off, Lcap * 4);
  L.o_dirty = lay_take(off, (kThreads / 32) * ((Lcap + 31) / 32) * 4);  // per-warp dirty bitmaps
  L.o_misc = lay_take(off, (int)sizeof(Misc));
  L.o_qr = lay_take(off, (kThreads / 32) * kMMQueue * 8);  // candidate queue: row, value, (prov, slot)
  L.o_qv = lay_take(off, (kThreads / 32) * kMMQueue * 8);
  L.o_qp = lay_take(off, (kThreads / 32) * kMMQueue * 8);
  L.o_stage = vstage ? lay_take(off, kThreads * kMMStageBytes) : 0;
  L.bytes = off;
  return L;
}

// Rows per thread per tile: their loads are all issued before any is used, so a thread keeps
// kMMRows independent row loads in flight (the pruned path is memory-latency bound otherwise).
#ifndef PAC_MM_ROWS
#define PAC_MM_ROWS 4
#endif
constexpr int kMMRows = PAC_MM_ROWS;

// candidate mask (rare: rows that can still improve a bound) -- out of line, so the 8-row
// unrolled scan stays small in the instruction cache
__device__ __noinline__ uint64_t mm_candidate_mask(uint64_t key, uint64_t salt) { return pac_hash_dev(key, salt); }

// refresh the cached bounds of slot s from the HBM table (one warp)
__device__ __forceinline__ void mm_refresh(const AggPlan& p, int pv, int s, long long* bmin, long long* bmax,
                                           int lane) {
  const size_t b = (size_t)pv * kM;
  if (p.has_max) {
    long long a = min(*(volatile long long*)&p.prov_max[b + lane], *(volatile long long*)&p.prov_max[b + lane + 32]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) a = min(a, __shfl_xor_sync(0xffffffffu, a, d));
    if (lane == 0) bmax[s] = a;
  }
  if (p.has_min) {
    long long a = max(*(volatile long long*)&p.prov_min[b + lane], *(volatile long long*)&p.prov_min[b + lane + 32]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) a = max(a, __shfl_xor_sync(0xffffffffu, a, d));
    if (lane == 0) bmin[s] = a;
  }
}

// No CTA barrier in the row loop: the cached bounds only have to be some value the HBM table
// held (a stale bound admits extra candidates, never a wrong result), so each warp refreshes
// the slots it updated itself, after its tile, from a per-warp dirty bitmap.
#ifndef PAC_MM_MINB
#define PAC_MM_MINB 2
#endif
__global__ void __launch_bounds__(kThreads, PAC_MM_MINB) k_agg_minmax(AggPlan p, MMLayout L) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* lkey = (unsigned long long*)(smem + L.o_lkey);
  int* lstate = (int*)(smem + L.o_lstate);
  int* lprov = (int*)(smem + L.o_lprov);
  unsigned* lrows = (unsigned*)(smem + L.o_lrows);
  long long* bmin = (long long*)(smem + L.o_bmin);  // max_j MIN_j (enc), cached
  long long* bmax = (long long*)(smem + L.o_bmax);  // min_j MAX_j (enc), cached
  Misc* misc = (Misc*)(smem + L.o_misc);
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int Lcap = L.Lcap, LH = L.LH;
  const int nwords = (Lcap + 31) >> 5;
  unsigned* wdirty = (unsigned*)(smem + L.o_dirty) + wid * nwords;  // this warp's dirty slots

  for (int i = tid; i < LH; i += nth) lstate[i] = 0;
  for (int i = tid; i < Lcap; i += nth) {
    lrows[i] = 0;
    bmin[i] = kMinEmpty;   // nothing can be pruned until every world holds a value
    bmax[i] = kMaxEmpty;
  }
  for (int i = lane; i < nwords; i += 32) wdirty[i] = 0u;
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }
  __syncthreads();

  const int T = nth * kMMRows;
  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * t_per;
  const int64_t t1 = min(ntiles, t0 + t_per);

#pragma unroll 1
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t base = tile * T;
    // all loads of the tile's rows first (kMMRows per thread in flight)
    double vv[kMMRows];
    uint64_t kk[kMMRows], mk[kMMRows];
#pragma unroll
    for (int k = 0; k < kMMRows; ++k) {
      const int64_t r = base + k * nth + tid;
      const bool in = r < p.n_rows;
      vv[k] = in ? __ldcs(p.mcol + r) : 0.0;
      mk[k] = (in && p.mask_in) ? __ldcs((const unsigned long long*)p.mask_in + r) : (in ? ~0ull : 0ull);
      kk[k] = 0ull;
    }
    // group keys column by column (R20), the kMMRows loads of a column issued back to back
    for (int c = 0; c < p.n_keys; ++c) {
      const int w = p.key_bytes[c];
      const void* col = p.key_col[c];
      uint64_t kv[kMMRows];
#pragma unroll
      for (int k = 0; k < kMMRows; ++k) {
        const int64_t r = min(base + k * nth + tid, p.n_rows - 1);
        kv[k] = w == 1 ? (uint64_t)(uint8_t)__ldcs((const signed char*)col + r)
              : w == 2 ? (uint64_t)(uint16_t)__ldcs((const short*)col + r)
              : w == 4 ? (uint64_t)(uint32_t)__ldcs((const int*)col + r)
                       : (uint64_t)__ldcs((const long long*)col + r);
      }
#pragma unroll
      for (int k = 0; k < kMMRows; ++k) {
        const uint64_t v = kv[k] ^ (1ull << (8 * w - 1));
        kk[k] = (w == 8) ? v : ((kk[k] << (8 * w)) | v);
      }
    }
#pragma unroll
    for (int k = 0; k < kMMRows; ++k) {
      const int64_t r = base + k * nth + tid;
      const bool valid = r < p.n_rows && mk[k] != 0;  // R21: a row in no world creates no group
      bool cand = false;
      const double v = vv[k];
      int prov = -1, s = -1;
      if (valid) {
        const long long e = enc_f64(v);
        const int code = local_code(p, kk[k], lkey, lstate, LH, lprov, Lcap, misc);
        if (code < kOvfBase) {
          s = code - 1;
          prov = lprov[s];
          atomicAdd(&lrows[s], 1u);
          cand = (p.has_max && e > bmax[s]) || (p.has_min && e < bmin[s]);
        } else {
          prov = code - kOvfBase - 1;
          if (prov >= 0) atomicAdd(&p.prov_rows[prov], 1ull);
          cand = true;
        }
        if (prov < 0) cand = false;
      }
      // warp-cooperative world update of the candidate rows (lane l: worlds l, l+32)
      unsigned cm = __ballot_sync(0xffffffffu, cand);
      if (cm) {
        uint64_t m = mk[k];
        if (cand && !p.mask_in) m = mm_candidate_mask((uint64_t)__ldg(p.pu_key + r), p.salt);
        while (cm) {
          const int src = __ffs(cm) - 1;
          cm &= cm - 1;
          const uint64_t mm = __shfl_sync(0xffffffffu, m, src);
          const double vs = __shfl_sync(0xffffffffu, v, src);
          const int pv = __shfl_sync(0xffffffffu, prov, src);
          const int ss = __shfl_sync(0xffffffffu, s, src);
          const long long e = enc_f64(vs);
          const size_t b = (size_t)pv * kM;
          if ((mm >> lane) & 1ull) {
            if (p.has_max) atomicMax(&p.prov_max[b + lane], e);
            if (p.has_min) atomicMin(&p.prov_min[b + lane], e);
          }
          if ((mm >> (lane + 32)) & 1ull) {
            if (p.has_max) atomicMax(&p.prov_max[b + lane + 32], e);
            if (p.has_min) atomicMin(&p.prov_min[b + lane + 32], e);
          }
          if (lane == 0 && ss >= 0) wdirty[ss >> 5] |= 1u << (ss & 31);
        }
      }
    }
    __syncwarp();
    // this warp refreshes the bounds of the slots it updated (no CTA barrier)
    for (int wb = 0; wb < nwords; wb += 32) {
      const unsigned bits = wb + lane < nwords ? wdirty[wb + lane] : 0u;
      unsigned have = __ballot_sync(0xffffffffu, bits != 0u);
      while (have) {
        const int src = __ffs(have) - 1;
        have &= have - 1;
        unsigned wbits = __shfl_sync(0xffffffffu, bits, src);
        while (wbits) {
          const int s = ((wb + src) << 5) + __ffs(wbits) - 1;
          wbits &= wbits - 1;
          const int pv = lprov[s];
          if (pv >= 0) mm_refresh(p, pv, s, bmin, bmax, lane);
        }
      }
      if (bits) wdirty[wb + lane] = 0u;
    }
    __syncwarp();
  }
  __syncthreads();
  const int nloc = min(misc->nlocal, Lcap);
  for (int s = tid; s < nloc; s += nth)
    if (lprov[s] >= 0 && lrows[s]) atomicAdd(&p.prov_rows[lprov[s]], (unsigned long long)lrows[s]);
}

// refresh of the double-valued bounds of k_agg_minmax_v: min_j MAX_j and max_j MIN_j decoded, NaN
// when some world is still empty (or the bound is NaN) -- a NaN bound admits every row
__device__ __forceinline__ void mmv_refresh(const AggPlan& p, int pv, int s, double* bmin, double* bmax, int lane) {
  const size_t b = (size_t)pv * kM;
  if (p.has_max) {
    long long a = min(*(volatile long long*)&p.prov_max[b + lane], *(volatile long long*)&p.prov_max[b + lane + 32]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) a = min(a, __shfl_xor_sync(0xffffffffu, a, d));
    if (lane == 0) {
      bmax[s] = a == kMaxEmpty ? __longlong_as_double(kEncNaN) : dec_f64(a);
      if (a != kMaxEmpty) atomicMax(&p.gbmax[pv], a);  // the bound only grows: keep the latest
    }
  }
  if (p.has_min) {
    long long a = max(*(volatile long long*)&p.prov_min[b + lane], *(volatile long long*)&p.prov_min[b + lane + 32]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) a = max(a, __shfl_xor_sync(0xffffffffu, a, d));
    if (lane == 0) {
      bmin[s] = a == kMinEmpty ? __longlong_as_double(kEncNaN) : dec_f64(a);
      if (a != kMinEmpty) atomicMin(&p.gbmin[pv], a);
    }
  }
}

// CTA dictionary for one int32 key column: entry = (code << 32) | packed key in one 64-bit word
// (0 = empty; code 0xFFFFFFFF = being written), so a lookup is one shared load and one compare.
// Codes as local_code's: s + 1 for local slot s, kOvfBase + HBM slot + 1 for a key with none.
// (ld_acquire_cta_shared_u64: agg_lean.cuh)
static __device__ int local_code32(const AggPlan& p, uint32_t key, unsigned long long* dent, int LH, int* lprov,
                                   int Lcap, Misc* misc, double* bmin, double* bmax) {
  uint32_t h = (key * 0x9E3779B1u) >> 16 & (LH - 1);
  for (;;) {
    const unsigned long long e = ld_acquire_cta_shared_u64(&dent[h]);
    if (e != 0ull && (uint32_t)e == key) {
      const uint32_t code = (uint32_t)(e >> 32);
      if (code == 0xFFFFFFFFu) continue;  // being written
      return (int)code;
    }
    if (e == 0ull) {
      if (*(volatile int*)&misc->ndict >= LH / 2) return kOvfBase + global_slot(p, (uint64_t)key) + 1;
      if (atomicCAS(&dent[h], 0ull, 0xFFFFFFFF00000000ull | key) == 0ull) {
        if (atomicAdd(&misc->ndict, 1) >= LH / 2) {  // too full: release, use the HBM tier
          atomicSub(&misc->ndict, 1);
          __threadfence_block();
          atomicExch(&dent[h], 0ull);
          return kOvfBase + global_slot(p, (uint64_t)key) + 1;
        }
        const int sl = atomicAdd(&misc->nlocal, 1);
        const int prov = global_slot(p, (uint64_t)key);
        int code;
        if (sl < Lcap) {
          lprov[sl] = prov;
          code = sl + 1;
          // a slot new to this CTA starts from the group's published bounds (other CTAs' progress)
          if (prov >= 0 && p.gbmax) {
            const long long g = __ldcg(p.gbmax + prov);
            if (g != kMaxEmpty) bmax[sl] = dec_f64(g);
          }
          if (prov >= 0 && p.gbmin) {
            const long long g = __ldcg(p.gbmin + prov);
            if (g != kMinEmpty) bmin[sl] = dec_f64(g);
          }
        } else {
          code = kOvfBase + prov + 1;
        }
        __threadfence_block();
        atomicExch(&dent[h], ((unsigned long long)(uint32_t)code << 32) | key);
        return code;
      }
      continue;
    }
    h = (h + 1) & (LH - 1);
  }
}

// The pruned MIN/MAX kernel for the common layout (one int32 group-key column, pu keys hashed in
// the kernel, 16-byte aligned columns -- BASELINE C4).  Each thread takes ROWS consecutive rows
// per tile with 16-byte loads; MIN / MAX are compile-time; the bounds are cached as doubles (NaN =
// admit every row: some world still empty) so the pruning test is one FP64 compare that is also
// true for a NaN value (!(v <= bound)).  Rows that pass it (candidates) are queued per warp and
// applied 32 at a time -- every lane hashes one candidate's pu key, then the warp applies them one
// by one (lane j: worlds j, j + 32, atomicMax / atomicMin on the order-preserving encodings, R31)
// -- instead of the whole warp hashing whenever one lane has a candidate.  Bounds: after applying,
// the warp refreshes the slots it updated from the HBM table and publishes the result as a per-slot
// hint (gbmin / gbmax, monotone); at every tile each CTA pulls the hints of all its slots, so its
// bounds follow the other CTAs' progress and stale bounds admit few rows.
template <int MM>
__device__ __forceinline__ void mmv_apply(const AggPlan& p, const int64_t* qr, const double* qv, const int2* qp,
                                          int qh, int n, unsigned* wdirty, double* bmin, double* bmax,
                                          const int* lprov, int lane) {
  uint64_t m = 0;
  long long e = 0;
  int pv = -1, sl = -1;
  if (lane == 0) atomicAdd(&p.dbg[0], (unsigned long long)n);  // candidates (PAC_DEBUG statistic)
  if (lane < n) {
    const int i = (qh + lane) & (kMMQueue - 1);
    m = pac_hash_dev((uint64_t)__ldg(p.pu_key + qr[i]), p.salt);
    e = enc_f64(qv[i]);
    pv = qp[i].x;
    sl = qp[i].y;
  }
  for (int src = 0; src < n; ++src) {
    const uint64_t mm = __shfl_sync(0xffffffffu, m, src);
    const long long es = __shfl_sync(0xffffffffu, e, src);
    const int pvs = __shfl_sync(0xffffffffu, pv, src);
    const int ss = __shfl_sync(0xffffffffu, sl, src);
    const size_t b = (size_t)pvs * kM;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if ((mm >> (lane + 32 * h)) & 1ull) {
        if (MM & 2) atomicMax(&p.prov_max[b + lane + 32 * h], es);
        if (MM & 1) atomicMin(&p.prov_min[b + lane + 32 * h], es);
      }
    }
    if (lane == 0 && ss >= 0) wdirty[ss >> 5] |= 1u << (ss & 31);
  }
}

template <int MM, int ROWS, int LC>
__global__ void __launch_bounds__(kThreads, PAC_MM_MINB) k_agg_minmax_v(AggPlan p, MMLayout Lp) {
  // LC > 0: the layout of LC local slots as a compile-time constant (immediate smem offsets)
  constexpr MMLayout Lc = mm_layout_for(LC > 0 ? LC : 1, PAC_MM_STAGE != 0);
  const MMLayout& L = LC > 0 ? Lc : Lp;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* lkey = (unsigned long long*)(smem + L.o_lkey);
  int* lprov = (int*)(smem + L.o_lprov);
  unsigned* lrows = (unsigned*)(smem + L.o_lrows);
  double* bmin = (double*)(smem + L.o_bmin);  // max_j MIN_j, cached (NaN: admit every row)
  double* bmax = (double*)(smem + L.o_bmax);  // min_j MAX_j, cached (NaN: admit every row)
  Misc* misc = (Misc*)(smem + L.o_misc);
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int Lcap = L.Lcap, LH = L.LH;
  const int nwords = (Lcap + 31) >> 5;
  unsigned* wdirty = (unsigned*)(smem + L.o_dirty) + wid * nwords;
  int64_t* qr = (int64_t*)(smem + L.o_qr) + wid * kMMQueue;
  double* qv = (double*)(smem + L.o_qv) + wid * kMMQueue;
  int2* qp = (int2*)(smem + L.o_qp) + wid * kMMQueue;

  for (int i = tid; i < LH; i += nth) lkey[i] = 0ull;  // the packed int32 dictionary (local_code32)
  for (int i = tid; i < Lcap; i += nth) {
    lrows[i] = 0;
    lprov[i] = -1;
    bmin[i] = __longlong_as_double(kEncNaN);  // nothing can be pruned until every world holds a value
    bmax[i] = __longlong_as_double(kEncNaN);
  }
  for (int i = lane; i < nwords; i += 32) wdirty[i] = 0u;
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }
  __syncthreads();

  auto refresh_dirty = [&]() {
    for (int wb = 0; wb < nwords; wb += 32) {
      const unsigned bits = wb + lane < nwords ? wdirty[wb + lane] : 0u;
      unsigned have = __ballot_sync(0xffffffffu, bits != 0u);
      while (have) {
        const int src = __ffs(have) - 1;
        have &= have - 1;
        unsigned wbits = __shfl_sync(0xffffffffu, bits, src);
        while (wbits) {
          const int ss = ((wb + src) << 5) + __ffs(wbits) - 1;
          wbits &= wbits - 1;
          const int pv = lprov[ss];
          if (pv >= 0) mmv_refresh(p, pv, ss, bmin, bmax, lane);
        }
      }
      if (bits) wdirty[wb + lane] = 0u;
    }
    __syncwarp();
  };

  const int T = nth * ROWS;
  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * t_per;
  const int64_t t1 = min(ntiles, t0 + t_per);
  const int* kcol = (const int*)p.key_col[0];
  int qh = 0, qn = 0;
  // staging (PAC_MM_STAGE, ROWS == 4): this thread's 4 keys and 4 values of the next tile
  constexpr bool STAGE = PAC_MM_STAGE != 0 && ROWS == 4;
  int4* stk = (int4*)(smem + L.o_stage);
  double2* stv0 = (double2*)(smem + L.o_stage + kThreads * 16);
  double2* stv1 = stv0 + kThreads;
  // dep is 0 at run time but computed from the values just read out of the staging slots, so the
  // copies that overwrite the slots issue only after those reads completed
  auto prefetch = [&](int64_t tile, int dep) {
    const int64_t r0 = tile * T + ROWS * tid;
    if (tile < t1 && r0 + ROWS <= p.n_rows) {
      cp_async16(stk + tid, (const int4*)kcol + (r0 >> 2) + dep);
      cp_async16(stv0 + tid, (const double2*)p.mcol + (r0 >> 1) + dep);
      cp_async16(stv1 + tid, (const double2*)p.mcol + (r0 >> 1) + 1 + dep);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (STAGE) prefetch(t0, 0);
#pragma unroll 1
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t r0 = tile * T + ROWS * tid;
    int kq[ROWS];
    double vq[ROWS];
    if (STAGE && r0 + ROWS <= p.n_rows) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      const int4 k4 = stk[tid];
      const double2 a = stv0[tid], b = stv1[tid];
      kq[0] = k4.x; kq[1] = k4.y; kq[2] = k4.z; kq[3] = k4.w;
      vq[0] = a.x; vq[1] = a.y; vq[2] = b.x; vq[3] = b.y;
      int dep;
      asm("and.b32 %0, %1, 0;" : "=r"(dep) : "r"(k4.x ^ k4.w ^ __double2loint(a.x) ^ __double2hiint(b.y)));
      prefetch(tile + 1, dep);
    } else if (r0 + ROWS <= p.n_rows) {
#pragma unroll
      for (int g = 0; g < ROWS / 4; ++g) {
        const int4 k4 = __ldcs((const int4*)kcol + (r0 >> 2) + g);
        kq[4 * g] = k4.x; kq[4 * g + 1] = k4.y; kq[4 * g + 2] = k4.z; kq[4 * g + 3] = k4.w;
      }
#pragma unroll
      for (int g = 0; g < ROWS / 2; ++g) {
        const double2 a = __ldcs((const double2*)p.mcol + (r0 >> 1) + g);
        vq[2 * g] = a.x; vq[2 * g + 1] = a.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < ROWS; ++k) {
        const bool in = r0 + k < p.n_rows;
        kq[k] = in ? __ldcs(kcol + r0 + k) : 0;
        vq[k] = in ? __ldcs(p.mcol + r0 + k) : 0.0;
      }
    }
    // the other CTAs' progress: pull the per-slot bound hints
    const int hmask = (p.ablate >> 4) ? (1 << ((p.ablate >> 4) - 1)) - 1 : kMMHintEvery - 1;
    const int nl = (p.ablate & 8) || ((tile - t0) & hmask) ? 0 : min(*(volatile int*)&misc->nlocal, Lcap);
    for (int s2 = tid; s2 < nl; s2 += nth) {
      const int pv = *(volatile int*)&lprov[s2];
      if (pv < 0) continue;
      if (MM & 2) {
        const long long g = __ldcg(p.gbmax + pv);
        if (g != kMaxEmpty) {
          const double d = dec_f64(g);
          if (!(d <= bmax[s2])) bmax[s2] = d;
        }
      }
      if (MM & 1) {
        const long long g = __ldcg(p.gbmin + pv);
        if (g != kMinEmpty) {
          const double d = dec_f64(g);
          if (!(d >= bmin[s2])) bmin[s2] = d;
        }
      }
    }
    const bool full = r0 + ROWS <= p.n_rows;
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int64_t r = r0 + k;
      bool cand = false;
      int prov = -1, s = -1;
      if (full || r < p.n_rows) {
        const uint32_t key = (uint32_t)kq[k] ^ 0x80000000u;  // R20 packing of one int32 column
        const int code = local_code32(p, key, lkey, LH, lprov, Lcap, misc, bmin, bmax);
        if (code < kOvfBase) {
          s = code - 1;
          prov = lprov[s];
          atomicAdd(&lrows[s], 1u);
          // !(v <= b): v beats the bound, or v is NaN, or the bound is NaN (admit all)
          cand = ((MM & 2) && !(vq[k] <= bmax[s])) || ((MM & 1) && !(vq[k] >= bmin[s]));
        } else {
          prov = code - kOvfBase - 1;
          if (prov >= 0) atomicAdd(&p.prov_rows[prov], 1ull);
          cand = true;
        }
        if (prov < 0) cand = false;
      }
      const unsigned cm = __ballot_sync(0xffffffffu, cand);
      if (cand) {
        const int i = (qh + qn + __popc(cm & ((1u << lane) - 1u))) & (kMMQueue - 1);
        qr[i] = r;
        qv[i] = vq[k];
        qp[i] = make_int2(prov, s);
      }
      qn += __popc(cm);
      if (qn >= 32) {
        __syncwarp();
        mmv_apply<MM>(p, qr, qv, qp, qh, 32, wdirty, bmin, bmax, lprov, lane);
        qh = (qh + 32) & (kMMQueue - 1);
        qn -= 32;
        __syncwarp();
        refresh_dirty();
      }
    }
  }
  __syncwarp();
  if (qn > 0) {
    mmv_apply<MM>(p, qr, qv, qp, qh, qn, wdirty, bmin, bmax, lprov, lane);
    __syncwarp();
  }
  __syncthreads();
  const int nloc = min(misc->nlocal, Lcap);
  for (int s = tid; s < nloc; s += nth)
    if (lprov[s] >= 0 && lrows[s]) atomicAdd(&p.prov_rows[lprov[s]], (unsigned long long)lrows[s]);
}

// ------------------------------------------------------------------ deferred HBM tier
// Rows of groups without a CTA-local slot were appended to the spill records by tile_a1
// (AggPlan::sp_*; the pu key is hashed by k_spill_resolve, by full warps, not in the divergent
// tier branch).  Instead of 64 device atomics per row on a table far larger than L2, the
// records are grouped by provisional slot (a counting sort: per-slot counts, slot offsets,
// scatter of (slot, record) pairs) and each warp then folds a chunk of consecutive pairs in
// registers, lane j holding worlds j and j+32, with one coalesced atomic flush per slot run.

// HBM slots of the records the CTA dictionaries could not resolve (full warps, high occupancy:
// the dictionary probes' latency overlaps across warps instead of stalling the tile pipeline),
// then the per-slot record counts
__global__ void __launch_bounds__(256) k_spill_resolve(AggPlan p) {
  const int64_t n = min((int64_t)*p.sp_n, p.sp_cap);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    int prov = i < n ? p.sp_prov[i] : -1;
    if (prov == -2) {
      prov = global_slot(p, p.sp_gkey[i]);
      p.sp_prov[i] = prov;
    }
    // the record's world mask, in place of its pu key (ALU work under the probes' latency)
    if (prov >= 0 && !p.mask_in) p.sp_key[i] = pac_hash_dev(p.sp_key[i], p.salt);
    const unsigned peers = __match_any_sync(0xffffffffu, prov >= 0 ? (unsigned)prov : 0x80000000u | lane);
    if (prov >= 0 && lane == __ffs(peers) - 1) atomicAdd(&p.sp_cnt[prov], __popc(peers));
  }
}

// per-slot offsets of the grouped order (segments in arbitrary order, one atomic per block);
// the slot's row count joins prov_rows
__global__ void __launch_bounds__(256) k_spill_offsets(const int* gcounter, int64_t G_cap, const int* sp_cnt,
                                                       int* sp_off, unsigned long long* prov_rows,
                                                       unsigned long long* sp_tot) {
  __shared__ int wsum[8];
  __shared__ unsigned long long base;
  const int64_t G = min((int64_t)*gcounter, G_cap);
  const int64_t prov = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = prov < G ? sp_cnt[prov] : 0;
  int x = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) {
      const int v = wsum[w];
      wsum[w] = t;
      t += v;
    }
    base = t ? atomicAdd(sp_tot, (unsigned long long)t) : 0ull;
  }
  __syncthreads();
  if (c) {
    sp_off[prov] = (int)(base + wsum[wid] + x - c);
    prov_rows[prov] += (unsigned long long)c;
  }
}

// (slot, record) pairs into the slot's segment; lanes of one warp with the same slot share one
// atomic on the segment cursor
__global__ void __launch_bounds__(256) k_spill_scatter(const unsigned long long* sp_n, int64_t cap,
                                                       const int* sp_prov, int* sp_off, int2* pairs) {
  const int64_t n = min((int64_t)*sp_n, cap);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    const int prov = i < n ? sp_prov[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, prov >= 0 ? (unsigned)prov : 0x80000000u | lane);
    const int leader = __ffs(peers) - 1;
    int b = 0;
    if (prov >= 0 && lane == leader) b = atomicAdd(&sp_off[prov], __popc(peers));
    b = __shfl_sync(0xffffffffu, b, leader);
    if (prov >= 0) pairs[b + __popc(peers & ((1u << lane) - 1u))] = make_int2(prov, (int)i);
  }
}

constexpr int kSpillChunk = 256;  // grouped records per warp work item

__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int src) {
  const unsigned lo = __shfl_sync(0xffffffffu, (unsigned)v, src);
  const unsigned hi = __shfl_sync(0xffffffffu, (unsigned)(v >> 32), src);
  return (unsigned long long)lo | ((unsigned long long)hi << 32);
}

template <int NI, int NF, int MM>
__global__ void __launch_bounds__(256) k_spill_agg(AggPlan p, const unsigned long long* sp_tot,
                                                   const int2* __restrict__ pairs) {
  const int64_t R = (int64_t)*sp_tot;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t nchunks = (R + kSpillChunk - 1) / kSpillChunk;
  constexpr int KF = NI, KM = NI + NF;  // value columns: NI int64, NF f64, then the MIN/MAX column
  for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < nchunks; ch += nwarps) {
    const int64_t c0 = ch * kSpillChunk, c1 = min(R, c0 + kSpillChunk);
    int cur = -1;
    unsigned n0 = 0, n1 = 0;
    long long s0[NI > 0 ? NI : 1], s1[NI > 0 ? NI : 1];
    double f0[NF > 0 ? NF : 1], f1[NF > 0 ? NF : 1];
    long long mn0 = kMinEmpty, mn1 = kMinEmpty, mx0 = kMaxEmpty, mx1 = kMaxEmpty;
    auto reset = [&]() {
      n0 = n1 = 0;
#pragma unroll
      for (int c = 0; c < NI; ++c) s0[c] = s1[c] = 0;
#pragma unroll
      for (int c = 0; c < NF; ++c) f0[c] = f1[c] = 0.0;
      mn0 = mn1 = kMinEmpty;
      mx0 = mx1 = kMaxEmpty;
    };
    auto flush = [&]() {
      if (cur < 0) return;
      const size_t b = (size_t)cur * kM;
      if (p.has_count) {
        if (n0) atomicAdd(&p.prov_count[b + lane], (unsigned long long)n0);
        if (n1) atomicAdd(&p.prov_count[b + lane + 32], (unsigned long long)n1);
      }
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        if (s0[c]) atomicAdd(&p.prov_isum[c][b + lane], (unsigned long long)s0[c]);
        if (s1[c]) atomicAdd(&p.prov_isum[c][b + lane + 32], (unsigned long long)s1[c]);
      }
#pragma unroll
      for (int c = 0; c < NF; ++c) {
        if (n0) atomicAdd(&p.prov_fsum[c][b + lane], f0[c]);
        if (n1) atomicAdd(&p.prov_fsum[c][b + lane + 32], f1[c]);
      }
      if ((MM & 1) && mn0 != kMinEmpty) atomicMin(&p.prov_min[b + lane], mn0);
      if ((MM & 1) && mn1 != kMinEmpty) atomicMin(&p.prov_min[b + lane + 32], mn1);
      if ((MM & 2) && mx0 != kMaxEmpty) atomicMax(&p.prov_max[b + lane], mx0);
      if ((MM & 2) && mx1 != kMaxEmpty) atomicMax(&p.prov_max[b + lane + 32], mx1);
    };
    reset();
    for (int64_t b = c0; b < c1; b += 32) {
      const int64_t k = b + lane;
      const int2 pr = k < c1 ? pairs[k] : make_int2(-1, 0);
      unsigned long long m = 0, v[NI + NF + (MM ? 1 : 0) > 0 ? NI + NF + (MM ? 1 : 0) : 1];
      if (k < c1) {
        m = p.sp_key[pr.y];  // the mask (k_spill_resolve hashed the pu key)
#pragma unroll
        for (int c = 0; c < NI + NF + (MM ? 1 : 0); ++c) v[c] = p.sp_val[(size_t)c * p.sp_cap + pr.y];
      }
      const int nb = (int)min((int64_t)32, c1 - b);
      for (int t = 0; t < nb; ++t) {
        const int prov = __shfl_sync(0xffffffffu, pr.x, t);
        if (prov != cur) {
          flush();
          reset();
          cur = prov;
        }
        const unsigned long long mt = shfl_u64(m, t);
        const bool w0 = (mt >> lane) & 1ull, w1 = (mt >> (lane + 32)) & 1ull;
        n0 += w0;
        n1 += w1;
#pragma unroll
        for (int c = 0; c < NI; ++c) {
          const long long x = (long long)shfl_u64(v[c], t);
          s0[c] += w0 ? x : 0;
          s1[c] += w1 ? x : 0;
        }
#pragma unroll
        for (int c = 0; c < NF; ++c) {
          const double x = __longlong_as_double((long long)shfl_u64(v[KF + c], t));
          if (w0) f0[c] += x;
          if (w1) f1[c] += x;
        }
        if (MM) {
          const long long e = enc_f64(__longlong_as_double((long long)shfl_u64(v[KM], t)));
          if (w0) {
            mn0 = min(mn0, e);
            mx0 = max(mx0, e);
          }
          if (w1) {
            mn1 = min(mn1, e);
            mx1 = max(mx1, e);
          }
        }
      }
    }
    flush();
  }
}

// ------------------------------------------------------------------ finish: count, sort, gather
__global__ void k_finish_count(AggPlan p, int n_keys, int64_t* num_groups, int* status,
                               int* Gdev) {
  int G = *p.gcounter;
  if (n_keys == 0 && G == 0) {  // R21: an ungrouped aggregate always has one group
    init_prov_slot(p, 0, 0ull);
    G = 1;
  }
  int st = 0;
  if (G > p.G_cap) st = PAC_E_CAPACITY;
  *num_groups = G;
  *Gdev = G > p.G_cap ? (int)p.G_cap : G;
  *status = st;
}

// single-CTA bitonic sort of (key, prov) pairs; writes perm[rank] = prov
__global__ void __launch_bounds__(1024) k_sort_small(const unsigned long long* keys, const int* Gdev,
                                                     int* perm) {
  __shared__ unsigned long long sk[kSmallSort];
  __shared__ int si[kSmallSort];
  const int G = *Gdev;
  int n = 1;
  while (n < G) n <<= 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sk[i] = i < G ? keys[i] : ~0ull;
    si[i] = i < G ? i : -1;
  }
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          unsigned long long a = sk[i], b = sk[l];
          bool swap = up ? (a > b || (a == b && si[i] > si[l])) : (a < b || (a == b && si[i] < si[l]));
          if (swap) {
            sk[i] = b;
            sk[l] = a;
            int t = si[i];
            si[i] = si[l];
            si[l] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < G; i += blockDim.x) perm[i] = si[i];
}

// LSD radix sort of (key, idx) for large G: 8 passes of 8 bits.  Each block owns a
// contiguous chunk; per-block digit histograms -> exclusive scan in (digit, block)
// order -> stable scatter (warp-synchronous, chunk processed in order by one warp).
constexpr int kRadixChunk = 2048;

// OR and AND of all keys (rng[0], rng[1], preset to 0 and ~0): a pass whose digit is the same in
// every key is an identity permutation, so its histogram and scan are skipped and its scatter
// is a copy (a packed int32 group key leaves four of the eight passes constant).
__global__ void k_radix_range(const unsigned long long* keys, const int* Gdev, unsigned long long* rng) {
  const int G = *Gdev;
  unsigned long long o = 0, a = ~0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < G; i += gridDim.x * blockDim.x) {
    o |= keys[i];
    a &= keys[i];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    o |= __shfl_xor_sync(0xffffffffu, o, d);
    a &= __shfl_xor_sync(0xffffffffu, a, d);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&rng[0], o);
    atomicAnd(&rng[1], a);
  }
}

__device__ __forceinline__ bool radix_digit_constant(const unsigned long long* rng, int shift) {
  return rng && (((rng[0] ^ rng[1]) >> shift) & 255ull) == 0;
}

__global__ void k_radix_hist(const unsigned long long* keys, const int* Gdev, int shift,
                             int* hist /*[256][nblocks]*/, int nblocks, const unsigned long long* rng) {
  if (radix_digit_constant(rng, shift)) return;
  __shared__ int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int G = *Gdev;
  const int b = blockIdx.x;
  const int lo = b * kRadixChunk, hi = min(G, lo + kRadixChunk);
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
    atomicAdd(&h[(keys[i] >> shift) & 255], 1);
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d * nblocks + b] = h[d];
}

__global__ void __launch_bounds__(1024) k_radix_scan(int* hist, int total, const unsigned long long* rng,
                                                     int shift) {
  if (radix_digit_constant(rng, shift)) return;
  // exclusive scan of `total` ints (a multiple of 256) by one CTA, 16 consecutive ints per
  // thread per round (four 16-byte loads), so a round covers 16K counts
  constexpr int V = 16;
  __shared__ int carry;
  __shared__ int wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < total; base += blockDim.x * V) {
    const int i0 = base + threadIdx.x * V;
    int v[V];
    if (i0 < total) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) {
        const int4 t = reinterpret_cast<const int4*>(hist + i0)[q];
        v[4 * q] = t.x;
        v[4 * q + 1] = t.y;
        v[4 * q + 2] = t.z;
        v[4 * q + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = 0;
    }
    int sum = 0;
#pragma unroll
    for (int k = 0; k < V; ++k) sum += v[k];
    int x = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += a;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      const int y = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
      int yy = y;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, yy, d);
        if (lane >= d) yy += a;
      }
      wsum[lane] = yy - y;
    }
    __syncthreads();
    int run = x - sum + wsum[w] + carry;
    if (i0 < total) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) {
        int4 t;
        t.x = run;
        run += v[4 * q];
        t.y = run;
        run += v[4 * q + 1];
        t.z = run;
        run += v[4 * q + 2];
        t.w = run;
        run += v[4 * q + 3];
        reinterpret_cast<int4*>(hist + i0)[q] = t;
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = run;
    __syncthreads();
  }
}

__global__ void k_radix_scatter(const unsigned long long* kin, const int* iin, unsigned long long* kout,
                                int* iout, const int* Gdev, int shift, const int* hist, int nblocks,
                                const unsigned long long* rng) {
  if (radix_digit_constant(rng, shift)) {  // identity permutation: copy through
    const int G = *Gdev;
    const int lo = blockIdx.x * kRadixChunk, hi = min(G, lo + kRadixChunk);
    for (int i = lo + (int)threadIdx.x; i < hi; i += blockDim.x) {
      kout[i] = kin[i];
      iout[i] = iin ? iin[i] : i;
    }
    return;
  }
  // one warp per block, processes its chunk in order -> stable
  __shared__ int base[256];
  const int b = blockIdx.x, lane = threadIdx.x;
  for (int d = lane; d < 256; d += 32) base[d] = hist[d * nblocks + b];
  __syncwarp();
  const int G = *Gdev;
  const int lo = b * kRadixChunk, hi = min(G, lo + kRadixChunk);
  for (int i0 = lo; i0 < hi; i0 += 32) {
    const int i = i0 + lane;
    const bool ok = i < hi;
    unsigned long long k = ok ? kin[i] : 0ull;
    int d = ok ? (int)((k >> shift) & 255) : 256 + lane;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & ((1u << lane) - 1));
    int leader = __ffs(peers) - 1;
    int pos = 0;
    if (ok) pos = base[d] + rank;
    __syncwarp();
    if (ok && lane == leader) base[d] += __popc(peers);
    __syncwarp();
    if (ok) {
      kout[pos] = k;
      iout[pos] = iin ? iin[i] : i;
    }
  }
}

// one warp per output group (rank)
__global__ void k_gather(AggPlan p, const int* Gdev, const int* perm, pac_table out, int n_aggs,
                         const int* src_kind, const int* src_idx) {
  const int G = *Gdev;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int rank = blockIdx.x * wpb + (threadIdx.x >> 5); rank < G; rank += gridDim.x * wpb) {
    const int prov = perm[rank];
    const size_t pb = (size_t)prov * kM, ob = (size_t)rank * kM;
    uint64_t K = 0;
    if (p.has_count) {
      unsigned long long c0 = p.prov_count[pb + lane], c1 = p.prov_count[pb + lane + 32];
      out.d_count[ob + lane] = (int64_t)c0;
      out.d_count[ob + lane + 32] = (int64_t)c1;
      K = (uint64_t)__ballot_sync(0xffffffffu, c0 != 0) |
          ((uint64_t)__ballot_sync(0xffffffffu, c1 != 0) << 32);
    } else {
      bool a = false, b = false;
      if (p.has_max) {
        a |= p.prov_max[pb + lane] != kMaxEmpty;
        b |= p.prov_max[pb + lane + 32] != kMaxEmpty;
      }
      if (p.has_min) {
        a |= p.prov_min[pb + lane] != kMinEmpty;
        b |= p.prov_min[pb + lane + 32] != kMinEmpty;
      }
      K = (uint64_t)__ballot_sync(0xffffffffu, a) | ((uint64_t)__ballot_sync(0xffffffffu, b) << 32);
    }
    for (int a = 0; a < n_aggs; ++a) {
      void* w = out.d_world[a];
      if (!w) continue;
      const int kd = src_kind[a], ix = src_idx[a];
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (kd == 1) ((int64_t*)w)[ob + j] = (int64_t)p.prov_isum[ix][pb + j];
        else if (kd == 2) ((double*)w)[ob + j] = p.prov_fsum[ix][pb + j];
        else if (kd == 3) ((double*)w)[ob + j] = dec_min(p.prov_min[pb + j]);
        else if (kd == 4) ((double*)w)[ob + j] = dec_max(p.prov_max[pb + j]);
      }
    }
    if (lane == 0) {
      out.d_group_key[rank] = p.prov_key[prov];
      out.d_rows[rank] = (int64_t)p.prov_rows[prov];
      out.d_presence[rank] = K;
      // R15 overflow check: max|v| * rows >= 2^63 may overflow an int64 world sum
      if (p.ni > 0) {
        const unsigned long long ma = *p.gmaxabs, rows = p.prov_rows[prov];
        if (ma && rows > (0x7FFFFFFFFFFFFFFFull / ma)) atomicExch(out.d_status, PAC_E_OVERFLOW);
      }
    }
  }
}

// m = 128 tables (native path, agg128.cu): one warp per output group, lane j -> worlds j + 32 h
__global__ void k_gather128(AggPlan p, const int* Gdev, const int* perm, pac_table out, int n_aggs,
                            const int* src_kind, const int* src_idx) {
  const int G = *Gdev;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int rank = blockIdx.x * wpb + (threadIdx.x >> 5); rank < G; rank += gridDim.x * wpb) {
    const int prov = perm[rank];
    const size_t pb = (size_t)prov * 2 * kM, ob = (size_t)rank * 2 * kM;
    uint64_t K0 = 0, K1 = 0;  // presence of worlds 0..63 and 64..127 (R5)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const unsigned long long c = p.prov_count[pb + lane + 32 * h];
      out.d_count[ob + lane + 32 * h] = (int64_t)c;
      const uint64_t bal = (uint64_t)__ballot_sync(0xffffffffu, c != 0) << (32 * (h & 1));
      if (h < 2) K0 |= bal; else K1 |= bal;
    }
    for (int a = 0; a < n_aggs; ++a) {
      void* w = out.d_world[a];
      if (!w) continue;
      const int kd = src_kind[a], ix = src_idx[a];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int j = lane + 32 * h;
        if (kd == 1) ((int64_t*)w)[ob + j] = (int64_t)p.prov_isum[ix][pb + j];
        else if (kd == 2) ((double*)w)[ob + j] = p.prov_fsum[ix][pb + j];
      }
    }
    if (lane == 0) {
      out.d_group_key[rank] = p.prov_key[prov];
      out.d_rows[rank] = (int64_t)p.prov_rows[prov];
      out.d_presence[2 * rank] = K0;
      out.d_presence[2 * rank + 1] = K1;
      if (p.ni > 0) {  // R15 overflow check, as k_gather
        const unsigned long long ma = *p.gmaxabs, rows = p.prov_rows[prov];
        if (ma && rows > (0x7FFFFFFFFFFFFFFFull / ma)) atomicExch(out.d_status, PAC_E_OVERFLOW);
      }
    }
  }
}

// ------------------------------------------------------------------ host helpers
static int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

struct AccSet {
  int ni = 0, nf = 0, has_min = 0, has_max = 0, has_count = 0;
  const void* icol[2] = {nullptr, nullptr};
  const void* fcol[2] = {nullptr, nullptr};
  const void* mcol = nullptr;
  int src_kind[PAC_MAX_AGGS];  // 0 count, 1 isum, 2 fsum, 3 min, 4 max
  int src_idx[PAC_MAX_AGGS];
};

// Accumulator set of a call.  kinds_only: value pointers are ignored (NULL allowed, no
// column-identity rules) -- for the entry points that only need the aggregate kinds.
static int build_accs(const pac_agg_spec* aggs, int n_aggs, AccSet* A, bool allow_null = false,
                      bool kinds_only = false) {
  if (n_aggs < 1 || n_aggs > PAC_MAX_AGGS || !aggs) return PAC_E_INVAL;
  bool only_mm = true;
  for (int a = 0; a < n_aggs; ++a) {
    const int k = aggs[a].kind;
    const void* v = aggs[a].d_values;
    if (k < PAC_COUNT || k > PAC_MAX_F64) return PAC_E_INVAL;
    if (k != PAC_COUNT && !v && !allow_null) return PAC_E_INVAL;
    if (k != PAC_MIN_F64 && k != PAC_MAX_F64) only_mm = false;
    A->src_idx[a] = 0;
    if (k == PAC_COUNT) {
      A->src_kind[a] = 0;
    } else if (k == PAC_SUM_I64) {
      int f = -1;
      for (int c = 0; c < A->ni; ++c) if (A->icol[c] == v) f = c;
      if (f < 0) {
        if (A->ni == 2) return PAC_E_INVAL;
        A->icol[A->ni] = v;
        f = A->ni++;
      }
      A->src_kind[a] = 1;
      A->src_idx[a] = f;
    } else if (k == PAC_SUM_F64 || k == PAC_AVG_F64) {
      int f = -1;
      for (int c = 0; c < A->nf; ++c) if (A->fcol[c] == v) f = c;
      if (f < 0) {
        if (A->nf == 2) return PAC_E_INVAL;
        A->fcol[A->nf] = v;
        f = A->nf++;
      }
      A->src_kind[a] = 2;
      A->src_idx[a] = f;
    } else {
      if (!kinds_only && A->mcol && A->mcol != v) return PAC_E_INVAL;
      A->mcol = v;
      if (k == PAC_MIN_F64) {
        A->has_min = 1;
        A->src_kind[a] = 3;
      } else {
        A->has_max = 1;
        A->src_kind[a] = 4;
      }
    }
  }
  A->has_count = only_mm ? 0 : 1;
  return PAC_OK;
}

struct WsLayout {
  size_t o_gkey, o_gstate, o_ctr, o_pkey, o_prows, o_pcount, o_pisum[2], o_pfsum[2], o_pmin, o_pmax,
      o_gbmin, o_gbmax, o_perm, o_sk0, o_si0, o_sk1, o_si1, o_hist, o_meta, bytes;
  int64_t Hcap;
  int nblocks;
};

// worlds: words per provisional world row (64; 128 for the native m = 128 path)
static WsLayout ws_layout(const AccSet& A, int64_t G_cap, int worlds = kM) {
  WsLayout w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const int64_t Gc = G_cap < 1 ? 1 : G_cap;
  w.Hcap = next_pow2(std::max<int64_t>(2 * Gc, 64));
  w.o_gkey = take(8 * w.Hcap);
  w.o_gstate = take(4 * w.Hcap);
  w.o_ctr = take(64);  // gcounter, Gdev, gmaxabs, dbg[2], spill records reserved / grouped, key OR / AND
  w.o_pkey = take(8 * Gc);
  w.o_prows = take(8 * Gc);
  w.o_pcount = A.has_count ? take(8 * Gc * worlds) : 0;
  for (int c = 0; c < 2; ++c) w.o_pisum[c] = c < A.ni ? take(8 * Gc * worlds) : 0;
  for (int c = 0; c < 2; ++c) w.o_pfsum[c] = c < A.nf ? take(8 * Gc * worlds) : 0;
  w.o_pmin = A.has_min ? take(8 * Gc * worlds) : 0;
  w.o_pmax = A.has_max ? take(8 * Gc * worlds) : 0;
  const bool mm_only = !A.has_count;  // k_agg_minmax(_v): per-slot bound hints
  w.o_gbmin = mm_only && A.has_min ? take(8 * Gc) : 0;
  w.o_gbmax = mm_only && A.has_max ? take(8 * Gc) : 0;
  w.o_perm = take(4 * Gc);
  w.nblocks = (int)((Gc + kRadixChunk - 1) / kRadixChunk);
  if (Gc > kSmallSort) {
    w.o_sk0 = take(8 * Gc);
    w.o_si0 = take(4 * Gc);
    w.o_sk1 = take(8 * Gc);
    w.o_si1 = take(4 * Gc);
    w.o_hist = take(4 * 256 * (size_t)w.nblocks);
  }
  w.o_meta = take(2 * PAC_MAX_AGGS * 4);
  w.bytes = off;
  return w;
}

// Deferred HBM tier records, appended after the base layout: per-slot counts and offsets,
// then cap records (slot 4 B, mask 8 B, 8 B per value column) and cap (slot, record) pairs.
struct SpillLayout {
  size_t o_cnt, o_off, o_prov, o_gkey, o_mask, o_val, o_pairs, bytes;
  int64_t cap;
};

static int spill_values(const AccSet& A) { return A.ni + A.nf + ((A.has_min || A.has_max) ? 1 : 0); }

static SpillLayout spill_layout(const AccSet& A, int64_t G_cap, size_t base, int64_t cap) {
  SpillLayout s{};
  size_t off = base;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const int64_t Gc = G_cap < 1 ? 1 : G_cap;
  s.cap = cap;
  s.o_cnt = take(4 * Gc);
  s.o_off = take(4 * Gc);
  s.o_prov = take(4 * cap);
  s.o_gkey = take(8 * cap);
  s.o_mask = take(8 * cap);
  s.o_val = take(8 * (size_t)spill_values(A) * cap);
  s.o_pairs = take(8 * cap);
  s.bytes = off;
  return s;
}

// records for n_rows tier rows: each warp may leave up to one partial grab of kSpillGrab unused
static int64_t spill_rows_needed(int64_t n_rows) { return n_rows + (int64_t)4096 * kSpillGrab; }

// the largest record capacity the caller's workspace holds beyond the base layout
static int64_t spill_fit(const AccSet& A, int64_t G_cap, size_t base, size_t ws_bytes, int64_t n_rows) {
  const size_t fixed = spill_layout(A, G_cap, base, 0).bytes + 4 * 256;
  if (ws_bytes <= fixed) return 0;
  const size_t rec = 28 + 8 * (size_t)spill_values(A);
  int64_t cap = std::min<int64_t>((int64_t)((ws_bytes - fixed) / rec),
                                  std::min<int64_t>(spill_rows_needed(n_rows), INT32_MAX - 1));
  while (cap > 0 && spill_layout(A, G_cap, base, cap).bytes > ws_bytes) cap -= 1024;
  return cap < 1024 ? 0 : cap;
}

static int raw_tile_bytes(const AccSet& A, int T, int key_bytes) {
  const int cols8 = 1 + A.ni + A.nf + ((A.has_min || A.has_max) ? 1 : 0);
  return cols8 * T * 8 + ((key_bytes * T + 15) & ~15) + 16 * PAC_MAX_KEYS;
}

static SmemLayout make_layout(const AccSet& A, int T, int Lcap, int key_bytes = 8, bool tm = false) {
  // PAC_NO_TMA: rows read from HBM in A1/A2, no staged raw tile
  const int raw = getenv("PAC_NO_TMA") ? 0 : raw_tile_bytes(A, T, key_bytes);
  return tile_layout(A.ni, A.nf, A.has_min, A.has_max, T, Lcap, raw, tm ? 1 : 0);
}

// Local slot capacity: min(G_cap, 256).  Preference: all wanted slots with three CTAs per SM
// (tile 1024, then 512), then two CTAs per SM, then one CTA per SM with as many slots as
// fit.  PAC_TILE=512|1024 forces the tile size (experiments).
static bool choose_layout(const AccSet& A, int64_t G_cap, int smem_max, int key_bytes, SmemLayout* out) {
  // small tables get kFixedSlots local slots: the compile-time-layout kernel instance
  const int cap = getenv("PAC_LCAP_MAX") ? atoi(getenv("PAC_LCAP_MAX")) : 256;  // experiments
  const int want = (int)std::min<int64_t>(std::max<int64_t>(G_cap, (int64_t)kFixedSlots), cap);
  if (getenv("PAC_FORCE_TM")) {  // experiments: the TMEM-table kernel at any slot count
    const int T = atoi(getenv("PAC_FORCE_TM")) >= 1024 ? atoi(getenv("PAC_FORCE_TM")) : 2048;
    SmemLayout L = make_layout(A, T, want, key_bytes, true);
    if (L.bytes <= smem_max) {
      *out = L;
      return true;
    }
  }
  const char* force = getenv("PAC_TILE");
  const int tiles_fixed[2] = {force ? atoi(force) : 1024, force ? atoi(force) : 512};  // multiples of 512
  for (int per_sm : {PAC_TILE_MINB, 3, 2}) {
    const int budget = smem_max / per_sm - 2048;
    for (int T : tiles_fixed) {
      SmemLayout L = make_layout(A, T, want, key_bytes);
      if (L.bytes <= budget) {
        *out = L;
        return true;
      }
    }
  }
  int best = 0, bestT = 0;
  for (int T : tiles_fixed) {
    int lo = 0, hi = want;
    while (lo < hi) {
      int mid = (lo + hi + 1) / 2;
      if (make_layout(A, T, mid, key_bytes).bytes <= smem_max) lo = mid; else hi = mid - 1;
    }
    if (lo > best) {
      best = lo;
      bestT = T;
    }
  }
  // one CTA per SM: for 33..256 slots whose accumulators fit the 512 TMEM columns, move the CTA
  // table to TMEM (k_agg_tiles_tm) and spend the freed shared memory on 2048-row tiles
  const int wps = 2 + 4 * A.ni + 4 * A.nf + (A.has_min ? 4 : 0) + (A.has_max ? 4 : 0);
  // 65..128 slots are rounded up to the compile-time TMEM instance (kTmFixedSlots, T = 2048)
  const int want_tm = (want > 64 && want <= kTmFixedSlots && 4 * (kTmFixedSlots / 16) * wps <= kTmCols)
                          ? kTmFixedSlots : want;
  if (want > 32 && 4 * ((want_tm + 15) / 16) * wps <= kTmCols && !getenv("PAC_NO_TM")) {
    const int Tx = getenv("PAC_TM_T") ? atoi(getenv("PAC_TM_T")) : 2048;  // experiments
    for (int T : {Tx, 2048, 1024}) {
      SmemLayout L = make_layout(A, T, want_tm, key_bytes, true);
      if (L.bytes <= smem_max) {
        *out = L;
        return true;
      }
    }
  }
  if (best < 1) return false;
  *out = make_layout(A, bestT, best, key_bytes);
  return true;
}

static MMLayout mm_layout(int64_t G_cap, int smem_max, bool vstage = false) {
  int Lcap = (int)std::min<int64_t>(std::max<int64_t>(G_cap, 1), 4096);
  for (;;) {
    const MMLayout L = mm_layout_for(Lcap, vstage);
    if (L.bytes <= smem_max || Lcap == 1) return L;
    Lcap /= 2;
  }
}


// instantiated in agg_inst_ni{0,1,2}.cu

extern template cudaError_t launch_smem<0, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<0, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<1, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_smem<2, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);


typedef cudaError_t (*LaunchFn)(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<0, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<1, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 0, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 0, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 0, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 0, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 1, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 1, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 1, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 1, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 2, 0>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 2, 1>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 2, 2>(const AggPlan&, const SmemLayout&, int, cudaStream_t);
extern template cudaError_t launch_tm<2, 2, 3>(const AggPlan&, const SmemLayout&, int, cudaStream_t);


#define PAC_MM_ROW(NI, NF) {launch_smem<NI, NF, 0>, launch_smem<NI, NF, 1>, launch_smem<NI, NF, 2>, launch_smem<NI, NF, 3>}
static const LaunchFn kLaunch[3][3][4] = {
    {PAC_MM_ROW(0, 0), PAC_MM_ROW(0, 1), PAC_MM_ROW(0, 2)},
    {PAC_MM_ROW(1, 0), PAC_MM_ROW(1, 1), PAC_MM_ROW(1, 2)},
    {PAC_MM_ROW(2, 0), PAC_MM_ROW(2, 1), PAC_MM_ROW(2, 2)},
};


#define PAC_TMM_ROW(NI, NF) {launch_tm<NI, NF, 0>, launch_tm<NI, NF, 1>, launch_tm<NI, NF, 2>, launch_tm<NI, NF, 3>}
static const LaunchFn kLaunchTm[3][3][4] = {
    {PAC_TMM_ROW(0, 0), PAC_TMM_ROW(0, 1), PAC_TMM_ROW(0, 2)},
    {PAC_TMM_ROW(1, 0), PAC_TMM_ROW(1, 1), PAC_TMM_ROW(1, 2)},
    {PAC_TMM_ROW(2, 0), PAC_TMM_ROW(2, 1), PAC_TMM_ROW(2, 2)},
};

typedef cudaError_t (*WsFn)(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<0, 0, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<0, 1, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<0, 2, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<1, 0, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<1, 1, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<1, 2, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<2, 0, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<2, 1, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
extern template cudaError_t launch_ws<2, 2, 0>(const AggPlan&, const WskLayout&, int, cudaStream_t);
static const WsFn kLaunchWs[3][3] = {
    {launch_ws<0, 0, 0>, launch_ws<0, 1, 0>, launch_ws<0, 2, 0>},
    {launch_ws<1, 0, 0>, launch_ws<1, 1, 0>, launch_ws<1, 2, 0>},
    {launch_ws<2, 0, 0>, launch_ws<2, 1, 0>, launch_ws<2, 2, 0>},
};
static bool ws_tmem_ok(const AccSet& A, const WskLayout& L) {
  const int wps = 2 + 4 * A.ni + 4 * A.nf + (A.has_min ? 4 : 0) + (A.has_max ? 4 : 0);
  return ws_tmem_fits(L, wps);
}

typedef void (*SpillFn)(const AggPlan&, const unsigned long long*, const int2*, int, cudaStream_t);
template <int NI, int NF, int MM>
static void launch_spill(const AggPlan& p, const unsigned long long* tot, const int2* pairs, int grid,
                         cudaStream_t st) {
  k_spill_agg<NI, NF, MM><<<grid, 256, 0, st>>>(p, tot, pairs);
}
#define PAC_SP_ROW(NI, NF) {launch_spill<NI, NF, 0>, launch_spill<NI, NF, 1>, launch_spill<NI, NF, 2>, launch_spill<NI, NF, 3>}
static const SpillFn kSpill[3][3][4] = {
    {PAC_SP_ROW(0, 0), PAC_SP_ROW(0, 1), PAC_SP_ROW(0, 2)},
    {PAC_SP_ROW(1, 0), PAC_SP_ROW(1, 1), PAC_SP_ROW(1, 2)},
    {PAC_SP_ROW(2, 0), PAC_SP_ROW(2, 1), PAC_SP_ROW(2, 2)},
};

static int device_info(int* sms, int* smem_optin) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PAC_E_CUDA;
  if (cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return PAC_E_CUDA;
  if (cudaDeviceGetAttribute(smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return PAC_E_CUDA;
  return PAC_OK;
}

// profiling (runtime.cu)
void profile_begin(cudaStream_t st, const char* name);
void profile_end(cudaStream_t st);

}  // namespace pac

using namespace pac;

namespace pac {
// ------------------------------------------------------------------ partition-first (part.cu)
constexpr int kPartCols = 2 + PAC_MAX_KEYS + 5;
struct PartResult {
  const void* col[kPartCols];
  const longlong2* units;
  const int* n_units;
  int* unit_ctr;
  int64_t rows;
};
size_t part_ws_bytes(int64_t n_rows, int n_cols_max, int row_bytes, int pbits, int grid, int unit_rows);
int part_rows(const void* const* src, const int* eb, int ncol, int hash0, uint64_t salt, int n_keys,
              int64_t n_rows, int pbits, int grid, int unit_rows, char* ws, PartResult* out, cudaStream_t st);
constexpr int kPartUnitRows = 32768;    // rows per unit (a multiple of the tile rows)
constexpr int64_t kPartMinRows = 1 << 20;

// Sort-first (sortagg.cu): rows radix-sorted by packed key, then one streaming 64-world fold
size_t srt_ws_bytes(int64_t n_rows, int nv, int sms);
int srt_run(const AggPlan& p, const int64_t* d_pu_key, const uint64_t* d_mask, const pac_key_col* keys, int n_keys,
            int width, int64_t n_rows, int sms, char* ws, const pac_table* out, int n_aggs, const int* kinds,
            const int* idx, cudaStream_t st);
void srt_finish(const AggPlan& p, const pac_table* out, int sms, cudaStream_t st);
constexpr int64_t kSrtMinGroups = 4096;  // below: the tile kernels (CTA-local slots catch most rows)
static bool srt_applicable(const AccSet& A, int n_keys, int width, int64_t G_cap, int64_t n_rows) {
  if (getenv("PAC_NO_SORT") || getenv("PAC_PART") || !A.has_count || A.has_min || A.has_max || n_keys < 1 || width > 4 || n_rows < 1 ||
      n_rows >= ((int64_t)1 << 31))
    return false;
  return G_cap >= kSrtMinGroups || (getenv("PAC_SORT") && G_cap > 128);
}

// Partition-first (opt-in, PAC_PART=1: measured slower than the deferred tier on C3)
// applies to large inputs whose table has many more groups than the TMEM CTA table holds
// (G_cap >= 4 Lcap); P = 2^pbits partitions of <= Lcap / 2 groups by capacity.
static bool want_partition(int64_t G_cap, int64_t n_rows, const SmemLayout& L, int* pbits) {
  if (!getenv("PAC_PART") || !L.tm || G_cap < 4 * (int64_t)L.Lcap || n_rows < kPartMinRows) return false;
  int b = 7;
  while (b < 15 && ((int64_t)1 << b) * (L.Lcap / 2) < G_cap) ++b;
  if (n_rows + (16ll << b) >= INT32_MAX) return false;
  *pbits = b;
  return true;
}
static int part_grid(int sms) { return 2 * sms; }
// worst-case bytes per row of the partitioned columns: mask/pu 8, keys <= 8, values 8 each
static size_t part_ws_for(const AccSet& A, int64_t n_rows, int pbits, int sms) {
  const int nv = A.ni + A.nf + ((A.has_min || A.has_max) ? 1 : 0);
  return part_ws_bytes(n_rows, 1 + PAC_MAX_KEYS + nv, 16 + 8 * nv, pbits, part_grid(sms), kPartUnitRows);
}
}  // namespace pac

extern "C" int pac_mask(const int64_t* d_pu_key, int64_t n, uint64_t salt, uint64_t* d_mask,
                        pac_stream_t stream) {
  if (n < 0 || (n > 0 && (!d_pu_key || !d_mask))) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  int sms = 148, smem = 0;
  if (device_info(&sms, &smem) != PAC_OK) return PAC_E_CUDA;
  int64_t blocks = (n + 256 * kMaskR - 1) / (256 * kMaskR);
  blocks = std::min<int64_t>(blocks, (int64_t)sms * 8);
  k_mask<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>((const long long*)d_pu_key, n, salt,
                                                          (unsigned long long*)d_mask);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_agg_workspace_size(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap,
                                      size_t* bytes) {
  if (!bytes || G_cap < 1) return PAC_E_INVAL;
  AccSet A;
  int rc = build_accs(aggs, n_aggs, &A, true);
  if (rc) return rc;
  *bytes = ws_layout(A, G_cap).bytes;
  return PAC_OK;
}

extern "C" int pac_agg_workspace_size_rows(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, int64_t n_rows,
                                           size_t* bytes) {
  if (!bytes || G_cap < 1 || n_rows < 0) return PAC_E_INVAL;
  AccSet A;
  int rc = build_accs(aggs, n_aggs, &A, true);
  if (rc) return rc;
  const size_t base = ws_layout(A, G_cap).bytes;
  *bytes = base;
  if (!A.has_count || n_rows == 0) return PAC_OK;  // MIN/MAX-only: k_agg_minmax, no deferred tier
  int sms = 148, smem_max = 0;
  if (device_info(&sms, &smem_max) != PAC_OK) return PAC_E_CUDA;
  SmemLayout L{};
  if (!choose_layout(A, G_cap, smem_max, 8, &L)) return PAC_E_INVAL;
  if (G_cap <= L.Lcap) return PAC_OK;  // every group can hold a CTA-local slot: no tier rows
  *bytes = spill_layout(A, G_cap, base, std::min<int64_t>(spill_rows_needed(n_rows), INT32_MAX - 1)).bytes + 4 * 256;
  int pbits = 0;
  if (want_partition(G_cap, n_rows, L, &pbits)) *bytes = std::max(*bytes, base + part_ws_for(A, n_rows, pbits, sms));
  // sort-first (key width unknown here: sized for keys of <= 4 bytes, which are the ones it takes)
  if (srt_applicable(A, 1, 4, G_cap, n_rows)) *bytes = std::max(*bytes, base + srt_ws_bytes(n_rows, A.ni + A.nf, sms));
  return PAC_OK;
}

// group-key columns: at most PAC_MAX_KEYS of 1, 2, 4 or 8 bytes, packed width <= 8 bytes
static int check_keys(const pac_key_col* keys, int n_keys, int64_t n_rows, int* width) {
  if (n_keys < 0 || n_keys > PAC_MAX_KEYS || (n_keys > 0 && !keys)) return PAC_E_INVAL;
  *width = 0;
  for (int c = 0; c < n_keys; ++c) {
    const int w = keys[c].elem_bytes;
    if ((w != 1 && w != 2 && w != 4 && w != 8) || (!keys[c].d_col && n_rows > 0)) return PAC_E_INVAL;
    *width += w;
  }
  return *width > 8 ? PAC_E_INVAL : PAC_OK;
}

// The plan fields every aggregation path shares (inputs, accumulator set, workspace pointers).
static AggPlan make_plan(const int64_t* d_pu_key, const uint64_t* d_mask, uint64_t salt, const pac_key_col* keys,
                         int n_keys, int64_t n_rows, const AccSet& A, const WsLayout& W, char* ws, int64_t G_cap) {
  AggPlan p{};
  p.n_rows = n_rows;
  p.pu_key = (const long long*)d_pu_key;
  p.mask_in = (const unsigned long long*)d_mask;
  p.salt = salt;
  p.n_keys = n_keys;
  for (int c = 0; c < n_keys; ++c) {
    p.key_col[c] = keys[c].d_col;
    p.key_bytes[c] = keys[c].elem_bytes;
  }
  p.ni = A.ni;
  p.nf = A.nf;
  p.has_min = A.has_min;
  p.has_max = A.has_max;
  p.has_count = A.has_count;
  for (int c = 0; c < 2; ++c) {
    p.icol[c] = (const long long*)A.icol[c];
    p.fcol[c] = (const double*)A.fcol[c];
  }
  p.mcol = (const double*)A.mcol;
  p.gkey = (unsigned long long*)(ws + W.o_gkey);
  p.gstate = (int*)(ws + W.o_gstate);
  p.hmask = (uint32_t)(W.Hcap - 1);
  p.gcounter = (int*)(ws + W.o_ctr);
  p.gmaxabs = (unsigned long long*)(ws + W.o_ctr + 8);
  p.dbg = (unsigned long long*)(ws + W.o_ctr + 16);
  p.G_cap = G_cap;
  p.prov_key = (unsigned long long*)(ws + W.o_pkey);
  p.prov_rows = (unsigned long long*)(ws + W.o_prows);
  p.prov_count = A.has_count ? (unsigned long long*)(ws + W.o_pcount) : nullptr;
  for (int c = 0; c < 2; ++c) {
    p.prov_isum[c] = c < A.ni ? (unsigned long long*)(ws + W.o_pisum[c]) : nullptr;
    p.prov_fsum[c] = c < A.nf ? (double*)(ws + W.o_pfsum[c]) : nullptr;
  }
  p.prov_min = A.has_min ? (long long*)(ws + W.o_pmin) : nullptr;
  p.prov_max = A.has_max ? (long long*)(ws + W.o_pmax) : nullptr;
  p.gbmin = W.o_gbmin ? (long long*)(ws + W.o_gbmin) : nullptr;
  p.gbmax = W.o_gbmax ? (long long*)(ws + W.o_gbmax) : nullptr;
  return p;
}

// Clears the workspace dictionary and counters and uploads the output-column map (async on st).
static int plan_reset(const AccSet& A, const WsLayout& W, char* ws, int n_aggs, cudaStream_t st) {
  int* meta = (int*)(ws + W.o_meta);
  if (cudaMemsetAsync(ws + W.o_gstate, 0, 4 * W.Hcap, st) != cudaSuccess) return PAC_E_CUDA;
  if (cudaMemsetAsync(ws + W.o_ctr, 0, 64, st) != cudaSuccess) return PAC_E_CUDA;
  int hmeta[2 * PAC_MAX_AGGS];
  for (int a = 0; a < n_aggs; ++a) {
    hmeta[a] = A.src_kind[a];
    hmeta[PAC_MAX_AGGS + a] = A.src_idx[a];
  }
  if (cudaMemcpyAsync(meta, hmeta, sizeof(hmeta), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return PAC_E_CUDA;
  return PAC_OK;
}

extern "C" int pac_agg_grouped(const int64_t* d_pu_key, const uint64_t* d_mask, uint64_t salt,
                               const pac_key_col* keys, int n_keys, const pac_agg_spec* aggs, int n_aggs,
                               int64_t n_rows, const pac_table* out, int64_t G_cap, void* d_ws,
                               size_t ws_bytes, pac_stream_t stream) {
  if (n_rows < 0 || !out || G_cap < 1 || (out->m != 0 && out->m != 64)) return PAC_E_INVAL;  // m = 128: pac_agg_grouped128
  // exactly one mask source (an empty input may arrive as NULL pointers)
  if (d_pu_key && d_mask) return PAC_E_INVAL;
  if (!d_pu_key && !d_mask && n_rows > 0) return PAC_E_INVAL;
  int width = 0;
  if (check_keys(keys, n_keys, n_rows, &width) != PAC_OK) return PAC_E_INVAL;
  AccSet A;
  int rc = build_accs(aggs, n_aggs, &A, n_rows == 0);
  if (rc) return rc;
  if (!out->d_num_groups || !out->d_status || !out->d_group_key || !out->d_rows || !out->d_presence)
    return PAC_E_INVAL;
  if (A.has_count && !out->d_count) return PAC_E_INVAL;
  for (int a = 0; a < n_aggs; ++a)
    if (aggs[a].kind != PAC_COUNT && !out->d_world[a]) return PAC_E_INVAL;
  WsLayout W = ws_layout(A, G_cap);
  if (!d_ws || ws_bytes < W.bytes) return PAC_E_WORKSPACE;
  int sms = 148, smem_max = 0;
  if (device_info(&sms, &smem_max) != PAC_OK) return PAC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;

  AggPlan p = make_plan(d_pu_key, d_mask, salt, keys, n_keys, n_rows, A, W, ws, G_cap);
  int* Gdev = (int*)(ws + W.o_ctr + 4);
  int* perm = (int*)(ws + W.o_perm);
  int* meta = (int*)(ws + W.o_meta);

  if (int rc2 = plan_reset(A, W, ws, n_aggs, st)) return rc2;
  cudaError_t e = cudaSuccess;
  bool sorted = false;  // sort-first path: provisional slots already in canonical order
  if (n_rows > 0) {
    if (!A.has_count) {
      // one int32 key column, hashed pu keys, 16-byte aligned columns: the vectorized instance
      const bool vec = n_keys == 1 && keys[0].elem_bytes == 4 && d_pu_key && !getenv("PAC_NO_MMV") &&
                       ((uintptr_t)keys[0].d_col & 15) == 0 && ((uintptr_t)A.mcol & 15) == 0;
      MMLayout L = mm_layout(G_cap, smem_max, vec && PAC_MM_STAGE);
      const int mmk = (A.has_min ? 1 : 0) | (A.has_max ? 2 : 0);
      const bool r8 = false;
      p.ablate = (getenv("PAC_MMV_NOHINT") ? 8 : 0) | (getenv("PAC_MM_HINT_LOG") ? (1 + atoi(getenv("PAC_MM_HINT_LOG"))) << 4 : 0);
      const bool fixed = L.Lcap == 1024 && !getenv("PAC_NO_FIXED");  // e.g. BASELINE C4: 1000 groups
      auto kern = !vec ? k_agg_minmax
                  : fixed ? (mmk == 1 ? k_agg_minmax_v<1, 4, 1024>
                                      : (mmk == 2 ? k_agg_minmax_v<2, 4, 1024> : k_agg_minmax_v<3, 4, 1024>))
                          : (mmk == 1 ? k_agg_minmax_v<1, 4, 0> : (mmk == 2 ? k_agg_minmax_v<2, 4, 0> : k_agg_minmax_v<3, 4, 0>));
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
      if (e != cudaSuccess) return PAC_E_CUDA;
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, L.bytes);
      per_sm = std::max(1, per_sm);
      const int rows_per_thread = vec && r8 ? 8 : kMMRows;
      int64_t tiles = (n_rows + kThreads * rows_per_thread - 1) / (kThreads * rows_per_thread);
      int grid = (int)std::min<int64_t>(tiles, (int64_t)sms * per_sm);
      char kname[32];
      snprintf(kname, sizeof(kname), vec ? "k_agg_minmax_v<%d>" : "k_agg_minmax", mmk);
      profile_begin(st, kname);
      kern<<<grid, kThreads, L.bytes, st>>>(p, L);
      note_launch();
      e = cudaGetLastError();
      profile_end(st);
    } else if (A.has_min == 0 && A.has_max == 0 && G_cap <= 128 && getenv("PAC_WS") &&
               ws_tmem_ok(A, wsk_layout(A.ni, A.nf, 0, (int)G_cap)) &&
               wsk_layout(A.ni, A.nf, 0, (int)G_cap).bytes <= smem_max && wsk_layout(A.ni, A.nf, 0, (int)G_cap).mine <= 32) {
      // every group fits a local slot: the warp-specialized kernel (agg_ws.cuh; opt-in with PAC_WS=1 --
      // measured slower than the tile kernels on C2 / C5)
      const WskLayout WL = wsk_layout(A.ni, A.nf, 0, (int)G_cap);
      bool aligned = true;
      p.nraw = 0;
      auto add = [&](const void* col, int eb) {
        p.raw_src[p.nraw] = col;
        p.raw_eb[p.nraw] = eb;
        p.raw_off[p.nraw] = 0;
        aligned = aligned && (((uintptr_t)col) & 15) == 0;
        ++p.nraw;
      };
      add(d_mask ? (const void*)d_mask : (const void*)d_pu_key, 8);
      for (int c = 0; c < A.ni; ++c) add(A.icol[c], 8);
      for (int c = 0; c < A.nf; ++c) add(A.fcol[c], 8);
      for (int c = 0; c < n_keys; ++c) add(keys[c].d_col, keys[c].elem_bytes);
      p.tma_ok = aligned ? 1 : 0;  // 16-byte aligned columns: bulk L2 prefetch of upcoming chunks
      char kname[64];
      snprintf(kname, sizeof(kname), "k_agg_ws<%d,%d,0>", A.ni, A.nf);
      profile_begin(st, kname);
      e = kLaunchWs[A.ni][A.nf](p, WL, sms, st);
      profile_end(st);
    } else if (lean_applicable(A.ni, A.nf, A.has_min, A.has_max, A.has_count, n_keys, width, G_cap,
                               d_pu_key != nullptr)) {
      // every group fits a CTA-local slot and the key packs into 4 bytes: k_agg_lean (agg_lean.cuh)
      char kname[64];
      e = launch_lean(p, n_keys, width, sms, st, kname, (int)sizeof(kname));  // opens the profile region
      profile_end(st);
    } else if (srt_applicable(A, n_keys, width, G_cap, n_rows) &&
               ws_bytes >= W.bytes + srt_ws_bytes(n_rows, A.ni + A.nf, sms)) {
      // high cardinality: rows radix-sorted by key, then a streaming fold (sortagg.cu)
      profile_begin(st, "k_srt_{hist,scan,scatter} x passes + k_srt_{heads,hscan,bzero,agg}");
      const int src = srt_run(p, d_pu_key, d_mask, keys, n_keys, width, n_rows, sms, ws + W.bytes, out, n_aggs,
                              A.src_kind, A.src_idx, st);
      profile_end(st);
      if (src != PAC_OK) return src;
      sorted = true;
    } else {
      SmemLayout L{};
      if (!choose_layout(A, G_cap, smem_max, width, &L)) return PAC_E_INVAL;
      // partition-first (part.cu): the rows reordered by group hash into the workspace, the
      // TMEM kernel then runs unit by unit over them (masks in, no hashing, no deferred tier)
      int pbits = 0;
      bool part = want_partition(G_cap, n_rows, L, &pbits) && ws_bytes >= W.bytes + part_ws_for(A, n_rows, pbits, sms);
      if (part) {
        const void* src[kPartCols];
        int eb[kPartCols];
        int nc = 0;
        src[nc] = d_mask ? (const void*)d_mask : (const void*)d_pu_key;
        eb[nc++] = 8;
        for (int c = 0; c < n_keys; ++c) {
          src[nc] = keys[c].d_col;
          eb[nc++] = keys[c].elem_bytes;
        }
        for (int c = 0; c < A.ni; ++c) {
          src[nc] = A.icol[c];
          eb[nc++] = 8;
        }
        for (int c = 0; c < A.nf; ++c) {
          src[nc] = A.fcol[c];
          eb[nc++] = 8;
        }
        if (A.has_min || A.has_max) {
          src[nc] = A.mcol;
          eb[nc++] = 8;
        }
        PartResult pr{};
        profile_begin(st, "k_part_{hist,totals,scan,offsets,scatter} x2");
        int prc = part_rows(src, eb, nc, d_pu_key ? 1 : 0, salt, n_keys, n_rows, pbits, part_grid(sms), kPartUnitRows,
                            ws + W.bytes, &pr, st);
        profile_end(st);
        if (prc != PAC_OK) return prc;
        int k = 0;
        p.pu_key = nullptr;
        p.mask_in = (const unsigned long long*)pr.col[k++];
        for (int c = 0; c < n_keys; ++c) p.key_col[c] = pr.col[k++];
        for (int c = 0; c < A.ni; ++c) p.icol[c] = (const long long*)pr.col[k++];
        for (int c = 0; c < A.nf; ++c) p.fcol[c] = (const double*)pr.col[k++];
        if (A.has_min || A.has_max) p.mcol = (const double*)pr.col[k++];
        p.n_rows = pr.rows;
        p.units = pr.units;
        p.n_units = pr.n_units;
        p.unit_ctr = pr.unit_ctr;
      }
      // raw columns staged per tile by TMA (k_agg_tiles reads them from smem)
      {
        int off = 0;
        bool aligned = true;
        auto add = [&](const void* col, int eb) {
          p.raw_src[p.nraw] = col;
          p.raw_eb[p.nraw] = eb;
          p.raw_off[p.nraw] = off;
          off += (L.T * eb + 15) & ~15;
          aligned = aligned && (((uintptr_t)col) & 15) == 0;
          ++p.nraw;
        };
        p.nraw = 0;
        add(p.mask_in ? (const void*)p.mask_in : (const void*)p.pu_key, 8);
        for (int c = 0; c < A.ni; ++c) add(p.icol[c], 8);
        for (int c = 0; c < A.nf; ++c) add(p.fcol[c], 8);
        if (A.has_min || A.has_max) add(p.mcol, 8);
        for (int c = 0; c < n_keys; ++c) add(p.key_col[c], keys[c].elem_bytes);
        int copied = 0;
        for (int i = 0; i < p.nraw; ++i) copied += L.T * p.raw_eb[i];
        p.raw_bytes = copied;
        p.tma_ok = (aligned && !getenv("PAC_NO_TMA")) ? 1 : 0;
#ifdef PAC_ABLATE_BUILD
        p.ablate = getenv("PAC_ABLATE") ? atoi(getenv("PAC_ABLATE")) : 0;
#endif
      }
      if (getenv("PAC_DEBUG"))
        fprintf(stderr, "[libpac] k_agg_tiles%s<%d,%d,%d> T=%d Lcap=%d LH=%d smem=%d B (G_cap=%lld)\n",
                L.tm ? "_tm" : "", A.ni, A.nf, (A.has_min ? 1 : 0) | (A.has_max ? 2 : 0), L.T, L.Lcap, L.LH, L.bytes,
                (long long)G_cap);
      const int mm = (A.has_min ? 1 : 0) | (A.has_max ? 2 : 0);
      // deferred HBM tier when groups can miss a CTA-local slot and the workspace has room
      SpillLayout S{};
      if (G_cap > L.Lcap && !part && !getenv("PAC_NO_SPILL")) {
        const int64_t cap = spill_fit(A, G_cap, W.bytes, ws_bytes, n_rows);
        if (cap > 0) S = spill_layout(A, G_cap, W.bytes, cap);
      }
      if (S.cap > 0) {
        p.sp_cap = S.cap;
        p.sp_n = (unsigned long long*)(ws + W.o_ctr + 32);
        p.sp_prov = (int*)(ws + S.o_prov);
        p.sp_gkey = (unsigned long long*)(ws + S.o_gkey);
        p.sp_key = (unsigned long long*)(ws + S.o_mask);
        p.sp_val = (unsigned long long*)(ws + S.o_val);
        p.sp_cnt = (int*)(ws + S.o_cnt);
        if (cudaMemsetAsync(p.sp_cnt, 0, 4 * (size_t)G_cap, st) != cudaSuccess) return PAC_E_CUDA;
      }
      char kname[96];
      snprintf(kname, sizeof(kname), "%s<%d,%d,%d>%s", L.tm ? "k_agg_tiles_tm" : "k_agg_tiles", A.ni, A.nf, mm,
               S.cap > 0 ? " + k_spill_{resolve,offsets,scatter,agg}" : (part ? " (partition units)" : ""));
      profile_begin(st, kname);  // the timed region covers the whole aggregation pass
      e = L.tm ? kLaunchTm[A.ni][A.nf][mm](p, L, sms, st) : kLaunch[A.ni][A.nf][mm](p, L, sms, st);
      if (e == cudaSuccess && S.cap > 0) {
        unsigned long long* sp_tot = (unsigned long long*)(ws + W.o_ctr + 40);
        int* sp_off = (int*)(ws + S.o_off);
        int2* pairs = (int2*)(ws + S.o_pairs);
        k_spill_resolve<<<sms * 16, 256, 0, st>>>(p);
        k_spill_offsets<<<(int)((G_cap + 255) / 256), 256, 0, st>>>(p.gcounter, G_cap, p.sp_cnt, sp_off,
                                                                   p.prov_rows, sp_tot);
        k_spill_scatter<<<sms * 8, 256, 0, st>>>(p.sp_n, S.cap, p.sp_prov, sp_off, pairs);
        kSpill[A.ni][A.nf][mm](p, sp_tot, pairs, sms * 8, st);
        for (int q = 0; q < 4; ++q) note_launch();
        e = cudaGetLastError();
      }
      profile_end(st);
    }
    if (e != cudaSuccess) return PAC_E_CUDA;
  }
  k_finish_count<<<1, 1, 0, st>>>(p, n_keys, out->d_num_groups, out->d_status, Gdev);
  note_launch();
  if (sorted) {  // k_srt_agg wrote the output table in canonical order: no sort, no gather
    srt_finish(p, out, sms, st);
    return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
  }
  if (G_cap <= kSmallSort) {
    k_sort_small<<<1, 1024, 0, st>>>(p.prov_key, Gdev, perm);
    note_launch();
  } else {
    unsigned long long* k0 = (unsigned long long*)(ws + W.o_sk0);
    unsigned long long* k1 = (unsigned long long*)(ws + W.o_sk1);
    int* i0 = (int*)(ws + W.o_si0);
    int* i1 = (int*)(ws + W.o_si1);
    int* hist = (int*)(ws + W.o_hist);
    const unsigned long long* kin = p.prov_key;
    const int* iin = nullptr;
    unsigned long long* rng = (unsigned long long*)(ws + W.o_ctr + 48);  // OR, AND of the keys
    if (cudaMemsetAsync(rng + 1, 0xFF, 8, st) != cudaSuccess) return PAC_E_CUDA;
    k_radix_range<<<(int)std::min<int64_t>((G_cap + 255) / 256, (int64_t)sms * 4), 256, 0, st>>>(p.prov_key, Gdev,
                                                                                                 rng);
    note_launch();
    for (int pass = 0; pass < 8; ++pass) {
      unsigned long long* ko = (pass & 1) ? k1 : k0;
      int* io = (pass & 1) ? i1 : i0;
      if (pass == 7) io = perm;
      k_radix_hist<<<W.nblocks, 256, 0, st>>>(kin, Gdev, 8 * pass, hist, W.nblocks, rng);
      k_radix_scan<<<1, 1024, 0, st>>>(hist, 256 * W.nblocks, rng, 8 * pass);
      k_radix_scatter<<<W.nblocks, 32, 0, st>>>(kin, iin, ko, io, Gdev, 8 * pass, hist, W.nblocks, rng);
      for (int q = 0; q < 3; ++q) note_launch();
      kin = ko;
      iin = io;
    }
  }
  {
    int blocks = (int)std::min<int64_t>((G_cap + 7) / 8, (int64_t)sms * 16);
    k_gather<<<std::max(1, blocks), 256, 0, st>>>(p, Gdev, perm, *out, n_aggs, meta, meta + PAC_MAX_AGGS);
    note_launch();
  }
  if (getenv("PAC_DEBUG")) {
    unsigned long long d[2] = {0, 0};
    cudaMemcpyAsync(d, p.dbg, 16, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[libpac] HBM-tier rows %llu, max local slots used %llu\n", d[0], d[1]);
  }
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

namespace pac {
// ------------------------------------------------------------------ native m = 128 (agg128.cu)
int tiles128_smem(int ni, int nf, int Lcap, int raw_bytes);
int tiles128_rows();
cudaError_t launch_tiles128(const AggPlan& p, int Lcap, int sms, cudaStream_t st);

constexpr int kNative128Slots = 32;  // k_agg_tiles128: one warp scans the slot histogram

// The single-pass m = 128 kernel applies: COUNT / SUM / AVG aggregates, G_cap <= 32 (every group a
// CTA-local slot), and its CTA table fits shared memory.  PAC_NO_NATIVE128=1 forces the 3-pass path.
bool agg128_native_ok(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap, const pac_key_col* keys, int n_keys,
                      bool masked) {
  if (getenv("PAC_NO_NATIVE128") || G_cap < 1 || G_cap > kNative128Slots) return false;
  int width = 0;
  if (check_keys(keys, n_keys, 0, &width) != PAC_OK) return false;
  AccSet A;
  if (build_accs(aggs, n_aggs, &A, true, true) != PAC_OK || A.has_min || A.has_max) return false;
  int sms = 148, smem_max = 0;
  if (device_info(&sms, &smem_max) != PAC_OK) return false;
  return tiles128_smem(A.ni, A.nf, (int)G_cap, 0) <= smem_max;  // staging is dropped when it does not fit
}

// workspace of the native path (0 when the aggregate list is invalid)
size_t agg128_native_ws(const pac_agg_spec* aggs, int n_aggs, int64_t G_cap) {
  AccSet A;
  if (G_cap < 1 || build_accs(aggs, n_aggs, &A, true, true) != PAC_OK) return 0;
  return ws_layout(A, G_cap, 2 * kM).bytes;
}

int agg128_native(const int64_t* d_pu_key, const uint64_t* d_mask2, uint64_t salt, const pac_key_col* keys,
                  int n_keys, const pac_agg_spec* aggs, int n_aggs, int64_t n_rows, const pac_table* out,
                  int64_t G_cap, void* d_ws, size_t ws_bytes, pac_stream_t stream) {
  int width = 0;
  if (check_keys(keys, n_keys, n_rows, &width) != PAC_OK) return PAC_E_INVAL;
  AccSet A;
  int rc = build_accs(aggs, n_aggs, &A, n_rows == 0);
  if (rc) return rc;
  if (A.has_min || A.has_max || !out->d_count) return PAC_E_INVAL;
  for (int a = 0; a < n_aggs; ++a)
    if (aggs[a].kind != PAC_COUNT && !out->d_world[a]) return PAC_E_INVAL;
  const WsLayout W = ws_layout(A, G_cap, 2 * kM);
  if (!d_ws || ws_bytes < W.bytes) return PAC_E_WORKSPACE;
  int sms = 148, smem_max = 0;
  if (device_info(&sms, &smem_max) != PAC_OK) return PAC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;
  AggPlan p = make_plan(d_pu_key, d_mask2, salt, keys, n_keys, n_rows, A, W, ws, G_cap);
  p.m128 = 1;
  {  // raw columns staged per tile by TMA (Cols128 order)
    const int T = tiles128_rows();
    int off = 0;
    bool aligned = true;
    auto add = [&](const void* col, int eb) {
      p.raw_src[p.nraw] = col;
      p.raw_eb[p.nraw] = eb;
      p.raw_off[p.nraw] = off;
      off += (T * eb + 15) & ~15;
      aligned = aligned && (((uintptr_t)col) & 15) == 0;
      ++p.nraw;
    };
    p.nraw = 0;
    add(d_mask2 ? (const void*)d_mask2 : (const void*)d_pu_key, d_mask2 ? 16 : 8);
    for (int c = 0; c < A.ni; ++c) add(A.icol[c], 8);
    for (int c = 0; c < A.nf; ++c) add(A.fcol[c], 8);
    for (int c = 0; c < n_keys; ++c) add(keys[c].d_col, keys[c].elem_bytes);
    p.raw_bytes = off;
    p.tma_ok = (aligned && !getenv("PAC_NO_TMA")) ? 1 : 0;
    if (tiles128_smem(A.ni, A.nf, (int)G_cap, off) > smem_max) {  // large CTA tables: loads, no staging
      p.raw_bytes = 0;
      p.tma_ok = 0;
    }
  }
  int* Gdev = (int*)(ws + W.o_ctr + 4);
  int* perm = (int*)(ws + W.o_perm);
  int* meta = (int*)(ws + W.o_meta);
  if ((rc = plan_reset(A, W, ws, n_aggs, st)) != PAC_OK) return rc;
  if (n_rows > 0) {
    char kname[48];
    snprintf(kname, sizeof(kname), "k_agg_tiles128<%d,%d>", A.ni, A.nf);
    profile_begin(st, kname);
    const cudaError_t e = launch_tiles128(p, (int)G_cap, sms, st);
    profile_end(st);
    if (e != cudaSuccess) return PAC_E_CUDA;
  }
  k_finish_count<<<1, 1, 0, st>>>(p, n_keys, out->d_num_groups, out->d_status, Gdev);
  k_sort_small<<<1, 1024, 0, st>>>(p.prov_key, Gdev, perm);
  k_gather128<<<std::max(1, (int)((G_cap + 7) / 8)), 256, 0, st>>>(p, Gdev, perm, *out, n_aggs, meta,
                                                                   meta + PAC_MAX_AGGS);
  for (int q = 0; q < 3; ++q) note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
}  // namespace pac

extern "C" int pac_table_check(const pac_table* t, int64_t* h_num_groups, pac_stream_t stream) {
  if (!t || !t->d_num_groups || !t->d_status) return PAC_E_INVAL;
  int64_t G = 0;
  int32_t st = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(&G, t->d_num_groups, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return PAC_E_CUDA;
  if (cudaMemcpyAsync(&st, t->d_status, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return PAC_E_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return PAC_E_CUDA;
  if (h_num_groups) *h_num_groups = G;
  return st;
}

// ------------------------------------------------------------------ merge helpers (§8 a5/e)
namespace pac {
// K after a cross-rank merge (NCCL has no OR).  With per-world counts K is exactly {j: count_j > 0}
// (R5).  MIN/MAX-only tables carry no counts, and their double extremes cannot tell an empty world
// from one holding only +inf (MIN) or -inf (MAX); there the caller merges the presence words
// themselves (dist.py: MAX-allreduce of the 64 presence bits) and this kernel only adds the worlds
// whose MIN or MAX is not the empty value -- it never clears a bit.
__global__ void k_rederive(pac_table t, int64_t G_cap, int has_count, int min_a, int max_a) {
  const int64_t G = min(*t.d_num_groups, G_cap);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int64_t g = blockIdx.x * wpb + (threadIdx.x >> 5); g < G; g += (int64_t)gridDim.x * wpb) {
    bool a = false, b = false;
    if (has_count) {
      a = t.d_count[g * kM + lane] > 0;
      b = t.d_count[g * kM + lane + 32] > 0;
    } else {
      const uint64_t K0 = t.d_presence[g];
      a = (K0 >> lane) & 1ull;
      b = (K0 >> (lane + 32)) & 1ull;
      if (min_a >= 0) {
        const double* w = (const double*)t.d_world[min_a];
        a |= w[g * kM + lane] != INFINITY;
        b |= w[g * kM + lane + 32] != INFINITY;
      }
      if (max_a >= 0) {
        const double* w = (const double*)t.d_world[max_a];
        a |= w[g * kM + lane] != -INFINITY;
        b |= w[g * kM + lane + 32] != -INFINITY;
      }
    }
    uint64_t K = (uint64_t)__ballot_sync(0xffffffffu, a) | ((uint64_t)__ballot_sync(0xffffffffu, b) << 32);
    if (lane == 0) t.d_presence[g] = K;
  }
}

struct RemapKinds {  // passed by value in the launch (no device buffer shared between calls)
  int k[PAC_MAX_AGGS];
};

__global__ void k_remap(pac_table in, int64_t G_cap_in, const uint64_t* ukeys, int64_t Gu, pac_table out,
                        int n_aggs, RemapKinds kinds, int has_count) {
  const int64_t Gin = min(*in.d_num_groups, G_cap_in);  // a CAPACITY table holds G_cap_in groups
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int64_t u = blockIdx.x * wpb + (threadIdx.x >> 5); u < Gu; u += (int64_t)gridDim.x * wpb) {
    const uint64_t key = ukeys[u];
    int64_t lo = 0, hi = Gin;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (in.d_group_key[mid] < key) lo = mid + 1; else hi = mid;
    }
    const int64_t g = (lo < Gin && in.d_group_key[lo] == key) ? lo : -1;
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      if (has_count) out.d_count[u * kM + j] = g >= 0 ? in.d_count[g * kM + j] : 0;
      for (int a = 0; a < n_aggs; ++a) {
        const int k = kinds.k[a];
        if (k == PAC_COUNT) continue;
        if (k == PAC_SUM_I64) {
          ((int64_t*)out.d_world[a])[u * kM + j] = g >= 0 ? ((const int64_t*)in.d_world[a])[g * kM + j] : 0;
        } else {
          double e = (k == PAC_MIN_F64) ? INFINITY : (k == PAC_MAX_F64 ? -INFINITY : 0.0);
          ((double*)out.d_world[a])[u * kM + j] = g >= 0 ? ((const double*)in.d_world[a])[g * kM + j] : e;
        }
      }
    }
    if (lane == 0) {
      out.d_group_key[u] = key;
      out.d_rows[u] = g >= 0 ? in.d_rows[g] : 0;
      out.d_presence[u] = g >= 0 ? in.d_presence[g] : 0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *out.d_num_groups = Gu;
    *out.d_status = *in.d_status;
  }
}
}  // namespace pac

extern "C" int pac_table_rederive_presence(const pac_table* t, const pac_agg_spec* aggs, int n_aggs,
                                           int64_t G_cap, pac_stream_t stream) {
  AccSet A;
  if (!t || G_cap < 1 || (t->m != 0 && t->m != 64)) return PAC_E_INVAL;  // m = 64 tables
  int rc = build_accs(aggs, n_aggs, &A, true, true);  // only the kinds matter here
  if (rc) return rc;
  int min_a = -1, max_a = -1;
  for (int a = 0; a < n_aggs; ++a) {
    if (aggs[a].kind == PAC_MIN_F64 && min_a < 0) min_a = a;
    if (aggs[a].kind == PAC_MAX_F64 && max_a < 0) max_a = a;
  }
  if (A.has_count ? !t->d_count : ((min_a < 0 || !t->d_world[min_a]) && (max_a < 0 || !t->d_world[max_a])))
    return PAC_E_INVAL;
  if (min_a >= 0 && !t->d_world[min_a]) min_a = -1;
  if (max_a >= 0 && !t->d_world[max_a]) max_a = -1;
  int blocks = (int)std::min<int64_t>((G_cap + 7) / 8, 148 * 16);
  k_rederive<<<std::max(1, blocks), 256, 0, (cudaStream_t)stream>>>(*t, G_cap, A.has_count, min_a, max_a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_table_remap(const pac_table* in, const uint64_t* d_union_keys, int64_t G_union,
                               const pac_agg_spec* aggs, int n_aggs, int64_t G_cap_in, const pac_table* out,
                               pac_stream_t stream) {
  AccSet A;
  if (!in || !out || !d_union_keys || G_union < 1 || G_cap_in < 1) return PAC_E_INVAL;
  if ((in->m != 0 && in->m != 64) || (out->m != 0 && out->m != 64)) return PAC_E_INVAL;  // m = 64 tables
  int rc = build_accs(aggs, n_aggs, &A, true, true);  // only the kinds matter here
  if (rc) return rc;
  RemapKinds hk{};
  for (int a = 0; a < n_aggs; ++a) hk.k[a] = aggs[a].kind;
  cudaStream_t st = (cudaStream_t)stream;
  int blocks = (int)std::min<int64_t>((G_union + 7) / 8, 148 * 16);
  k_remap<<<std::max(1, blocks), 256, 0, st>>>(*in, G_cap_in, d_union_keys, G_union, *out, n_aggs, hk, A.has_count);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
