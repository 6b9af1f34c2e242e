// libpac: k_agg_lean -- the grouped 64-world aggregation for tables whose groups all fit the CTA
// (G_cap <= 128 local slots, packed group key <= 4 bytes, COUNT / int64 SUM / f64 SUM-AVG, hashed
// pu keys; BASELINE C1, C2, C5).  DESIGN.md §5 "k_agg_lean".
//
// Same arithmetic as k_agg_tiles / k_agg_tiles_tm (R1, R2 hash; 64-world transposed "Four
// Russians" update per 32-row run of one group, P:L249-253 Eq. counter), with the
// generality those kernels carry for high-cardinality tables removed from the per-row path:
//   - no HBM tier, no spill records: every group has a CTA-local slot (a CTA that meets more than
//     128 distinct keys has a table over capacity, which the HBM dictionary reports, R32);
//   - the CTA dictionary packs (key, code) in one 64-bit shared word: one LDS per lookup;
//   - ranks within a slot are per warp (match_any + one leader store, no shared atomics); the
//     slot offsets and per-warp offsets come from one 128-thread scan (phase B);
//   - one compile-time shared-memory layout (T = 2048 rows per tile, 512 threads, 1 CTA per SM);
//   - the CTA accumulator table lives in Tensor Memory in one of two modes:
//       P (private): every warp owns a private copy of the whole table (G_cap * wps <= 128
//         columns), the tile's runs are split evenly across the 16 warps in slot order;
//       O (owner):   slot s belongs to warp s % 16, which runs all runs of its slots (C5).
#pragma once
#include "agg_tm.cuh"

namespace pac {

#ifndef PAC_LEAN_CSFLAT
#define PAC_LEAN_CSFLAT 0  // 1: the carry-slot map written lane-parallel after phase B
#endif
#ifndef PAC_LEAN_QBAL
#define PAC_LEAN_QBAL 0  // (measured slower on C5: 45.8 vs 44.6 ms) owner mode: slot s in TMEM quarter s % 4, its quarter's 4 warps split the slots by runs
#endif
#ifndef PAC_LEAN_BTAB
#define PAC_LEAN_BTAB 1  // 1: mode P's hash draws read their one-hot position from a shared-memory table
                         // (common.cuh; C2 2.070 -> 2.040 ms; mode O measured 0.7 % slower with it: 44.61 -> 44.90 ms)
#endif
#ifndef PAC_LEAN_DYNCOPY
#define PAC_LEAN_DYNCOPY 1  // 1: owner mode claims the copy-out of the leftovers in chunks (warps with fewer runs copy more)
#endif
#ifndef PAC_LEAN_DYNCHUNK
#define PAC_LEAN_DYNCHUNK 32  // carry rows per claim (a multiple of 32)
#endif
#ifndef PAC_LEAN_PREHASH
#define PAC_LEAN_PREHASH 0  // 1: odd warps hash their first row pair before phase B (B is a serial shuffle chain,
                            // replicated per warp: half the warps then do throughput-bound work beside it)
#endif
#ifndef PAC_LEAN_CLK
#define PAC_LEAN_CLK 0  // 1 (profiling builds): per-phase clock64 totals of CTA 0's warps, printed at the end
#endif
#if PAC_LEAN_CLK
// the "memory" clobber keeps the clock read on its side of a barrier
#define LEAN_CLK(i) do { long long c_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_) :: "memory"); clk[i] += c_ - clk_t; clk_t = c_; } while (0)
#else
#define LEAN_CLK(i) do { } while (0)
#endif
#ifndef PAC_LEAN_WORKLIST
#define PAC_LEAN_WORKLIST 0  // 1: owner warps iterate a ballot-built list of their slots with runs
#endif

constexpr int kLeanT = 2048;      // rows per tile
constexpr int kLeanLcap = 128;    // local slots
constexpr int kLeanLH = 256;      // dictionary entries (2 x Lcap)
constexpr int kLeanThreads = 512;
constexpr int kLeanNW = kLeanThreads / 32;
constexpr unsigned long long kLeanLocked = ~0ull;
constexpr uint32_t kLeanDrop = 0x7FFFFFFFu;       // code of a key without a local slot

// Rows carried from one tile to the next (each slot's < 32 leftover rows): CC rows of carry area,
// sized per column count so that sorted buffer + carry area + raw tile fit 227 KB.
__host__ __device__ constexpr int lean_cc(int ni, int nf) {
  const int rb = 8 * (1 + ni + nf);
  const int fit = (195000 - kLeanT * (rb + 4) - kLeanT * rb) / (2 * rb);
  const int cc = fit >= 2048 ? 2048 : (fit / 256) * 256;
  return cc;
}

struct LeanLayout {
  int CC, TS;  // carry rows, sorted-buffer rows (T + CC + Lcap)
  int o_mask, o_ival, o_fval, o_cmask, o_cival, o_cfval, o_raw, o_wpv, o_hist, o_cslot, o_dict, o_lprov,
      o_lrows, o_off, o_tot, o_cpo, o_lfl, o_rdesc, o_queue, o_xcs, o_btab, o_mbar, o_misc, raw_bytes,
      bytes;
};

__host__ __device__ constexpr LeanLayout lean_layout(int ni, int nf) {
  LeanLayout L{};
  L.CC = lean_cc(ni, nf);
  L.TS = kLeanT + L.CC + kLeanLcap;  // + one alignment row per slot
  int off = 0;
  L.o_mask = lay_take(off, L.TS * 8);
  L.o_ival = lay_take(off, ni * L.TS * 8);
  L.o_fval = lay_take(off, nf * L.TS * 8);
  L.o_cmask = lay_take(off, L.CC * 8);
  L.o_cival = lay_take(off, ni * L.CC * 8);
  L.o_cfval = lay_take(off, nf * L.CC * 8);
  // raw tile: 8-byte columns (pu key, int64 sums, f64 sums) then <= 4 key bytes per row
  L.raw_bytes = (1 + ni + nf) * kLeanT * 8 + 4 * kLeanT + 16 * PAC_MAX_KEYS;
  L.o_raw = lay_take(off, L.raw_bytes);
  L.o_wpv = lay_take(off, kLeanNW * kLeanLcap * 4);  // per warp: {sorted base, copy-in offset} per slot (u16)
  L.o_hist = lay_take(off, 2 * kLeanLcap * 4);  // ping-pong by tile parity
  L.o_cslot = lay_take(off, 2 * L.CC);
  L.o_dict = lay_take(off, kLeanLH * 8);
  L.o_lprov = lay_take(off, kLeanLcap * 4);
  L.o_lrows = lay_take(off, kLeanLcap * 8);
  L.o_off = lay_take(off, kLeanLcap * 4);
  L.o_tot = lay_take(off, kLeanLcap * 4);
  L.o_cpo = lay_take(off, kLeanLcap * 4);
  L.o_lfl = lay_take(off, kLeanLcap * 4);
  L.o_rdesc = lay_take(off, (L.TS / 32 + 1) * 4);
  L.o_queue = lay_take(off, kLeanT * 4);
  L.o_xcs = lay_take(off, 32 * 16 + 32 * 8);
  L.o_btab = lay_take(off, kBtabBytes);  // one-hot pairs of the hash draws (btab_fill)
  L.o_mbar = lay_take(off, 16);
  L.o_misc = lay_take(off, (int)sizeof(Misc));
  L.bytes = off;
  return L;
}

__device__ __forceinline__ unsigned long long ld_acquire_cta_shared_u64(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(a))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared_u64(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.cta.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(a)), "l"(v)
               : "memory");
}

// Slow path of the CTA dictionary: insert `key` (or wait for a concurrent insert of it).  The
// entry is claimed with a 64-bit CAS to kLeanLocked, the local slot and the HBM provisional slot
// are taken, then the entry is published as (key << 32 | code) with release semantics.
static __device__ __noinline__ uint32_t lean_insert(const AggPlan& p, uint32_t key, unsigned long long* dict, int* lprov,
                                                    Misc* misc, int lcap) {
  uint32_t h = (key * 0x9E3779B1u) >> 24;
  int probes = 0;
  for (;;) {
    const unsigned long long e = ld_acquire_cta_shared_u64(&dict[h]);
    if (e == 0ull) {
      // over capacity: at most lcap + 16 keys enter the dictionary (lcap <= 128 < kLeanLH, so a free
      // entry always exists); the ones beyond lcap went through global_slot, which counts them, so
      // the table reports CAPACITY (R32) and every further new key is dropped without inserting
      if (*(volatile int*)&misc->nlocal >= lcap + 16) return kLeanDrop;
      if (atomicCAS(&dict[h], 0ull, kLeanLocked) == 0ull) {
        const int s = atomicAdd(&misc->nlocal, 1);
        uint32_t code = kLeanDrop;
        if (s < lcap) {
          lprov[s] = global_slot(p, (uint64_t)key);  // -1: over G_cap (rows dropped, status CAPACITY)
          code = (uint32_t)s + 1u;
        } else {
          global_slot(p, (uint64_t)key);  // more distinct keys than lcap >= G_cap: counted, so CAPACITY
        }
        st_release_cta_shared_u64(&dict[h], ((unsigned long long)key << 32) | code);
        return code;
      }
      continue;
    }
    if (e == kLeanLocked) continue;
    if ((uint32_t)(e >> 32) == key) return (uint32_t)e;
    h = (h + 1) & (kLeanLH - 1);
    if (++probes > kLeanLH) return kLeanDrop;  // full (racing inserts past the cap): over capacity anyway
  }
}

// local slot of `key` (0 .. 127), or -1 (no local slot: dropped, the table is over capacity)
__device__ __forceinline__ int lean_slot(const AggPlan& p, uint32_t key, unsigned long long* dict, int* lprov,
                                         Misc* misc, int lcap) {
  const uint32_t h = (key * 0x9E3779B1u) >> 24;
  const unsigned long long e = ld_acquire_cta_shared_u64(&dict[h]);
  uint32_t code;
  if ((uint32_t)(e >> 32) == key && e != kLeanLocked && (uint32_t)e != 0u) code = (uint32_t)e;
  else code = lean_insert(p, key, dict, lprov, misc, lcap);
  return code == kLeanDrop ? -1 : (int)code - 1;
}

// KS = 0: no key columns (one group, key 0); 1: one 4-byte key column; 2: 1..4 columns, <= 4 bytes
template <int KS>
__device__ __forceinline__ uint32_t lean_key(const AggPlan& p, const unsigned char* raw, int kc0, int li) {
  if (KS == 0) return 0u;
  if (KS == 1) return ((const uint32_t*)(raw + p.raw_off[kc0]))[li] ^ 0x80000000u;
  uint32_t packed = 0;
#pragma unroll
  for (int c = 0; c < PAC_MAX_KEYS; ++c) {
    if (c < p.n_keys) {
      const int w = p.key_bytes[c];
      const unsigned char* col = raw + p.raw_off[kc0 + c];
      uint32_t v;
      if (w == 1) v = col[li];
      else if (w == 2) v = ((const unsigned short*)col)[li];
      else v = ((const uint32_t*)col)[li];
      v ^= 1u << (8 * w - 1);
      packed = w == 4 ? v : ((packed << (8 * w)) | v);
    }
  }
  return packed;
}

// TMEM column of slot s for warp w: mode P = w's private copy; mode O = s's owner (w == s % 16)
__device__ __forceinline__ uint32_t lean_taddr(uint32_t tbase, int w, int s, int wps, bool owner) {
  if (PAC_LEAN_QBAL && owner)  // quarter s % 4, any of its 4 warps (one per slot and tile)
    return tbase + ((uint32_t)(32 * (s & 3)) << 16) + (uint32_t)((s >> 2) * wps);
  const int col = (w >> 2) * 128 + (owner ? (s >> 4) : s) * wps;
  return tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)col;
}
// owner mode: the slots warp w initialises / drains (fixed; mode O's per-tile split is dynamic)
__device__ __forceinline__ bool lean_mine(int w, int s) {
  return PAC_LEAN_QBAL ? ((s & 3) == (w & 3) && ((s >> 2) & 3) == (w >> 2)) : ((s & 15) == w);
}


// whether every int64 value of rows [0, l) of a carried run is below 2^26 (int32 subset tables)
__device__ __forceinline__ bool maxabs_small(const long long* iv, int stride, int l, int lane, int ni) {
  bool ok = true;
  for (int k = 0; k < ni; ++k) {
    const long long v = lane < l ? iv[k * stride + lane] : 0;
    const unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
    ok = ok && a < (1ull << 26);
  }
  return __all_sync(0xffffffffu, ok);
}

// one row (mask + values) from one staging array to another (strides in rows)
template <int NI, int NF>
__device__ __forceinline__ void lean_copy_row(unsigned long long* dm, long long* di, double* df, int dst, int dstride,
                                              const unsigned long long* sm_, const long long* si, const double* sf,
                                              int src, int sstride, unsigned long long& tmax, uint32_t& emax) {
  dm[dst] = sm_[src];
#pragma unroll
  for (int k = 0; k < NI; ++k) {
    const long long v = si[k * sstride + src];
    const unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
    tmax = a > tmax ? a : tmax;
    di[k * dstride + dst] = v;
  }
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const double v = sf[k * sstride + src];
    emax = max(emax, (uint32_t)__double2hiint(v) & 0x7FF00000u);
    df[k * dstride + dst] = v;
  }
}

// Per-warp view of phase B: lane L holds slots 4L .. 4L+3 (v[0..3]).
struct LeanB {
  int cc[4], co[4];  // rows carried into the current tile and their carry-area offsets (slot order)
};

// OWN: 1 = mode O (slot owners), 0 = mode P (private copies) -- separate instances, so each mode
// gets its own register allocation
template <int NI, int NF, int KS, int OWN>
__global__ void __launch_bounds__(kLeanThreads, 1) k_agg_lean(AggPlan p, int owner_mode, int lcap) {
  constexpr LeanLayout L = lean_layout(NI, NF);
  constexpr int T = kLeanT, TS = L.TS, CC = L.CC, Lcap = kLeanLcap, NW = kLeanNW, RPT = T / kLeanThreads;
  using S = TmSlot<NI, NF, 0>;
  constexpr int KC0 = 1 + NI + NF;  // first key column of the raw tile
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t s_tbase;
  unsigned long long* smask = (unsigned long long*)(smem + L.o_mask);
  long long* sival = (long long*)(smem + L.o_ival);
  double* sfval = (double*)(smem + L.o_fval);
  unsigned long long* cmask = (unsigned long long*)(smem + L.o_cmask);
  long long* cival = (long long*)(smem + L.o_cival);
  double* cfval = (double*)(smem + L.o_cfval);
  unsigned char* raw = smem + L.o_raw;
  int* hist = (int*)(smem + L.o_hist);        // [2][Lcap] new rows per slot (A: shared atomics), by parity
  unsigned char* cslot = smem + L.o_cslot;    // [2][CC] slot of each carry row (0xFF: none), by parity
  unsigned long long* dict = (unsigned long long*)(smem + L.o_dict);
  int* lprov = (int*)(smem + L.o_lprov);
  unsigned long long* lrows = (unsigned long long*)(smem + L.o_lrows);
  int* soff = (int*)(smem + L.o_off);   // slot region offset in the sorted buffer (phase C)
  int* stot = (int*)(smem + L.o_tot);   // rows in the region (carried + new)
  int* scpo = (int*)(smem + L.o_cpo);   // copy-out: sorted row of carry row i = scpo[s] + i
  int* slfl = (int*)(smem + L.o_lfl);   // 1: the slot's leftover is run now (carry area full)
  uint32_t* rdesc = (uint32_t*)(smem + L.o_rdesc);
  unsigned short* qpos = (unsigned short*)(smem + L.o_queue);
  unsigned short* qrow = qpos + T;
  uint4* xcs = (uint4*)(smem + L.o_xcs);
  uint2* xcs2 = (uint2*)(smem + L.o_xcs + 32 * 16);
  unsigned long long* mbar = (unsigned long long*)(smem + L.o_mbar);
  const uint32_t btab = btab_addr(smem + L.o_btab);
  Misc* misc = (Misc*)(smem + L.o_misc);
  const unsigned long long* rpu = (const unsigned long long*)raw;  // column 0 of the raw tile

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  constexpr bool owner = OWN != 0;
  (void)owner_mode;
  // this warp's private phase-B results: wpv[s] = sorted base of s's new rows | copy-in offset << 16
  uint32_t* wpv = (uint32_t*)(smem + L.o_wpv) + wid * Lcap;

  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tbase)),
                 "n"(kTmCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < kLeanLH; i += kLeanThreads) dict[i] = 0ull;
  for (int i = tid; i < Lcap; i += kLeanThreads) {
    lrows[i] = 0;
    hist[i] = 0;
    hist[Lcap + i] = 0;
  }
  if (tid == 0) {
    misc->nlocal = 0;
    misc->nruns = misc->big = 0;      // per-parity copy-out chunk counters (PAC_LEAN_DYNCOPY)
    misc->pad[0] = misc->pad[1] = 0;  // per-parity "some value needs the generic run body" flags
    mbar_init(mbar, 1);
  }
  if (tid < 32) store_xpose(xcs, xcs2, tid);
  btab_fill(btab, tid);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = s_tbase;
  if (KS == 0 && tid == 0) {  // ungrouped: the one group (key 0) takes slot 0 up front
    misc->nlocal = 1;
    lprov[0] = global_slot(p, 0ull);
  }
  // zero this warp's table columns: mode P its private copy of every slot, mode O its own slots
  for (int s = 0; s < lcap; ++s) {
    if (owner && !lean_mine(wid, s)) continue;
    tm_init_slot<NI, NF, 0>(lean_taddr(tbase, wid, s, S::wps, owner));
  }
  tm_wait_st();
  __syncthreads();

  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * t_per;
  const int64_t t1 = min(ntiles, t0 + t_per);
  auto staged = [&](int64_t t) { return p.tma_ok && t < t1 && (t + 1) * T <= p.n_rows; };
  uint32_t phase = 0;
  unsigned long long maxabs = 0;
  const XposeConst xc = load_xpose(xcs, xcs2, lane);
  WarpAcc<NI, NF, 0> acc;
  acc.reset();
  if (tid == 0 && staged(t0)) issue_tile(p, raw, mbar, t0 * T, T);

  LeanB cb;  // carried rows (every warp keeps the same copy)
#pragma unroll
  for (int k = 0; k < 4; ++k) cb.cc[k] = cb.co[k] = 0;
  int ncarry = 0;  // rows of the carry area in use (with alignment entries)

#if PAC_LEAN_CLK
  long long clk[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long clk_t = clock64();
#endif
  int par = 0;
  for (int64_t t = t0; t < t1; ++t, par ^= 1) {
    const int64_t base = t * T;
    const int tn = (int)min((int64_t)T, p.n_rows - base);
    int* hp = hist + par * Lcap;
    const unsigned char* cs_in = cslot + par * CC;
    unsigned char* cs_out = cslot + (par ^ 1) * CC;
    int* gflag = misc->pad + par;  // bit 0: some |int64| >= 2^26, bit 1: some f64 non-finite
    int* cpctr = (par ? &misc->big : &misc->nruns);  // copy-out chunk counter of this tile (fields unused here)
    if (tid == 0) {  // their last readers (C of tile t-2) passed two barriers ago
      *gflag = 0;
      *cpctr = 0;
    }
    if (staged(t)) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
    } else {  // ragged or unaligned tile: the threads stage it (zero beyond tn)
      for (int k = 0; k < p.nraw; ++k) {
        const int eb = p.raw_eb[k];
        unsigned char* dst = raw + p.raw_off[k];
        const unsigned char* src = (const unsigned char*)p.raw_src[k] + base * eb;
        for (int i = tid; i < T * eb; i += kLeanThreads) dst[i] = i < tn * eb ? src[i] : 0;
      }
      __syncthreads();
    }

    LEAN_CLK(0);  // wait for the staged tile
    // ---------------- A: slot of every row and its rank within the slot (shared atomic)
    uint32_t sr[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int li = tid + kLeanThreads * j;
      int s = -1;
      if (li < tn) s = KS == 0 ? 0 : lean_slot(p, lean_key<KS>(p, raw, KC0, li), dict, lprov, misc, lcap);
      uint32_t r = 0xFFFFFFFFu;
      if (KS == 0) {  // one slot: one atomic per warp
        const unsigned peers = __ballot_sync(0xffffffffu, s >= 0);
        int b = 0;
        if (lane == 0 && peers) b = atomicAdd(&hp[0], __popc(peers));
        b = __shfl_sync(0xffffffffu, b, 0);
        if (s >= 0) r = (uint32_t)(b + __popc(peers & lt_mask));
      } else if (s >= 0) {
        r = ((uint32_t)s << 16) | (uint32_t)atomicAdd(&hp[s], 1);
      }
      sr[j] = r;
    }
    LEAN_CLK(1);  // A
    __syncthreads();
    LEAN_CLK(2);  // barrier after A

    // ---------------- B, every warp for itself (lane L: slots 4L .. 4L+3): slot totals (carried +
    // new rows), region offsets (even rows: run_body reads 16-byte row pairs), full runs, the
    // leftovers' places in the carry area.  Warp 0 publishes what phase C needs.
    int nruns, ncarry_out;
    unsigned owned_work;  // bit q: owned slot wid + 16 q has runs this tile (mode O)
    HashState pha, phb;
    const bool prehash = PAC_LEAN_PREHASH && (wid & 1);
    if (prehash) {
      if (PAC_LEAN_BTAB && !owner) pac_hash_begin2_bt(rpu[tid], rpu[tid + kLeanThreads], p.salt, pha, phb, btab);
      else pac_hash_begin2(rpu[tid], rpu[tid + kLeanThreads], p.salt, pha, phb);
    }
    {
      const int4 h4 = *(const int4*)(hp + 4 * lane);
      const int n[4] = {h4.x, h4.y, h4.z, h4.w};
      int tot[4], f[4], l[4], tot2[4], l2[4];
      int sx = 0, sy = 0, sz = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tot[k] = cb.cc[k] + n[k];
        f[k] = tot[k] >> 5;
        l[k] = tot[k] & 31;
        tot2[k] = (tot[k] + 1) & ~1;
        l2[k] = (l[k] + 3) & ~3;  // carry ranges 4-aligned: the slot map is written 4 entries per store
        sx += tot2[k];
        sy += l2[k];
        sz += f[k];
      }
      // packed scan of region rows and carry rows (16 bits each); the runs (private mode only)
      const uint32_t v = (uint32_t)sx | ((uint32_t)sy << 16);
      uint32_t incl = v;
      int zin = sz;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t a = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += a;
        if (!owner) {
          const int b = __shfl_up_sync(0xffffffffu, zin, d);
          if (lane >= d) zin += b;
        }
      }
      const uint32_t all = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t ex = incl - v;
      int ox = (int)(ex & 0xFFFFu), oy = (int)(ex >> 16), oz = zin - sz;
      nruns = owner ? 0 : __shfl_sync(0xffffffffu, zin, 31);
      ncarry_out = min((int)(all >> 16), CC);
      LEAN_CLK(8);  // B: totals + scans
      LeanB nb;
      uint32_t wv[4];
      int my_oy = 0, my_valid = 0, my_l4 = 0, my_runs = 0;
      bool my_work = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int s = 4 * lane + k;
        const bool fl = oy + l[k] > CC;  // the carry area is full: this slot's leftover is run now
        // private: new rows' base, copy-in offset of the rows carried in (+ CC keeps it >= 0)
        wv[k] = (uint32_t)(ox + cb.cc[k]) | ((uint32_t)(ox - cb.co[k] + CC) << 16);
        if (wid == 0) {
          soff[s] = ox;
          stot[s] = tot[k];
          slfl[s] = fl ? 1 : 0;
          scpo[s] = ox + (tot[k] & ~31) - oy;
          lrows[s] += (unsigned long long)n[k];
        }
        // the slots of this warp's lane column (s % 16 == wid for the lanes with L % 4 == wid / 4;
        // k == wid % 4 is warp-uniform): carry range, work flag, run descriptors (private mode)
        if (k == (wid & 3)) {
          my_oy = oy;
          my_valid = fl ? 0 : l[k];
          my_l4 = l2[k];
          my_work = tot[k] >= 32 || fl;
          my_runs = f[k] + ((fl && l[k]) ? 1 : 0);
          if (!PAC_LEAN_CSFLAT && (lane & 3) == (wid >> 2)) {
            const uint32_t s4 = (uint32_t)s * 0x01010101u;
            for (int i = 0; i < l2[k] && oy + i < CC; i += 4) {
              const int m = min(max(my_valid - i, 0), 4);
              const uint32_t keep = m == 4 ? 0xFFFFFFFFu : ((1u << (8 * m)) - 1u);
              *(uint32_t*)(cs_out + oy + i) = (s4 & keep) | ~keep;
            }
          }
          if (!owner && (lane & 3) == (wid >> 2))
            for (int i = 0; i < f[k]; ++i) rdesc[oz + i] = pack_run(ox + 32 * i, s, 32);
        }
        nb.cc[k] = fl ? 0 : l[k];
        nb.co[k] = oy;
        ox += tot2[k];
        oy += l2[k];
        oz += f[k];
      }
      *(uint4*)(wpv + 4 * lane) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      // owned slots s = wid + 16 q (q < 8) live in lane (wid / 4) + 4 q: their carry-slot map
      // entries, 4 per store, lane j: slot q = j / 8 (+ 4 in the second pass), word j % 8
      const int col = wid >> 2;
#pragma unroll
      for (int pass = 0; pass < (PAC_LEAN_CSFLAT ? 2 : 0); ++pass) {
        const int q = (lane >> 3) + 4 * pass, e = lane & 7, src = col + 4 * q;
        const int qy = __shfl_sync(0xffffffffu, my_oy, src);
        const int qv = __shfl_sync(0xffffffffu, my_valid, src);
        const int ql = __shfl_sync(0xffffffffu, my_l4, src);
        if (4 * e < ql && qy + 4 * e < CC) {
          const int m = min(max(qv - 4 * e, 0), 4);
          const uint32_t keep = m == 4 ? 0xFFFFFFFFu : ((1u << (8 * m)) - 1u);
          *(uint32_t*)(cs_out + qy + 4 * e) = (((uint32_t)(wid + 16 * q) * 0x01010101u) & keep) | ~keep;
        }
      }
      owned_work = 0;
      if (PAC_LEAN_QBAL && owner) {
        // quarter q = wid % 4 holds slots 4 L + q (this lane's my_*); its 4 warps take contiguous
        // lane ranges of about equal run counts, warp wid / 4 the ((wid / 4))-th
        int incl = my_runs;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int a = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += a;
        }
        if (PAC_LEAN_QBAL == 2) {
          // round robin over the quarter's slots with work (no scan): the j-th such slot goes to the
          // quarter's warp j % 4; a slot mostly has one run per tile, so the warps differ by <= 1 run
          const unsigned wb = __ballot_sync(0xffffffffu, my_work);
          owned_work = __ballot_sync(0xffffffffu, my_work && (__popc(wb & lt_mask) & 3) == (wid >> 2));
        } else {
        const int W = max(__shfl_sync(0xffffffffu, incl, 31), 1);
        const int chunk = min(3, (4 * (incl - my_runs) + 2 * my_runs) / W);  // by the run midpoint
        owned_work = __ballot_sync(0xffffffffu, my_work && chunk == (wid >> 2));
        }
      } else if (PAC_LEAN_WORKLIST) {
        const unsigned wb = __ballot_sync(0xffffffffu, my_work);
#pragma unroll
        for (int q = 0; q < 8; ++q) owned_work |= ((wb >> (col + 4 * q)) & 1u) << q;
      }
      __syncwarp();
      // A2's copy-in reads the offsets of the rows carried INTO this tile (cb.co, set above);
      // the next tile carries nb
      cb = nb;
    }
    const int ncarry_in = ncarry;
    ncarry = ncarry_out;
    LEAN_CLK(3);  // B

    // ---------------- A2: carried rows into their slot regions (flat); hash word 0 of two new
    // rows at a time, straight to the slot-sorted position
    {
      unsigned long long tmax = 0;
      uint32_t emax = 0;
      {
        // copy-in: carry row i of slot s goes to soff[s] + (i - co[s]) = (wpv >> 16) - CC + i; the
        // map of this warp is private, so row i is handled by this warp's lanes only
        const uint32_t* wv = wpv;
        for (int i = lane + 32 * wid; i < ncarry_in; i += kLeanThreads) {
          const int s = cs_in[i];
          if (s != 0xFF)
            lean_copy_row<NI, NF>(smask, sival, sfval, (int)(wv[s] >> 16) - CC + i, TS, cmask, cival, cfval, i, CC,
                                  tmax, emax);
        }
      }
      LEAN_CLK(9);  // A2: copy-in of the carried rows
      unsigned short* wq = qpos + wid * (T / NW);
      unsigned short* wr = qrow + wid * (T / NW);
      int qn = 0;
#pragma unroll
      for (int j = 0; j < RPT; j += 2) {
        const int la = tid + kLeanThreads * j, lb = la + kLeanThreads;
        const uint32_t ra = sr[j], rb = sr[j + 1];
        const bool va = ra != 0xFFFFFFFFu, vb = rb != 0xFFFFFFFFu;
        const int pa = va ? (int)(wpv[ra >> 16] & 0xFFFFu) + (int)(ra & 0xFFFFu) : 0;
        const int pb = vb ? (int)(wpv[rb >> 16] & 0xFFFFu) + (int)(rb & 0xFFFFu) : 0;
        HashState ha, hb;
        if (j == 0 && prehash) {
          ha = pha;
          hb = phb;
        } else if (PAC_LEAN_BTAB && !owner) pac_hash_begin2_bt(rpu[la], rpu[lb], p.salt, ha, hb, btab);
        else pac_hash_begin2(rpu[la], rpu[lb], p.salt, ha, hb);
        const bool qa = va && ha.k > 0, qb = vb && hb.k > 0;
        if (va) {
          smask[pa] = hash_mask_now(ha);
#pragma unroll
          for (int k = 0; k < NI; ++k) {
            const long long v = ((const long long*)(raw + p.raw_off[1 + k]))[la];
            const unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
            tmax = a > tmax ? a : tmax;
            sival[k * TS + pa] = v;
          }
#pragma unroll
          for (int k = 0; k < NF; ++k) {
            const double v = ((const double*)(raw + p.raw_off[1 + NI + k]))[la];
            emax = max(emax, (uint32_t)__double2hiint(v) & 0x7FF00000u);
            sfval[k * TS + pa] = v;
          }
        }
        if (vb) {
          smask[pb] = hash_mask_now(hb);
#pragma unroll
          for (int k = 0; k < NI; ++k) {
            const long long v = ((const long long*)(raw + p.raw_off[1 + k]))[lb];
            const unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
            tmax = a > tmax ? a : tmax;
            sival[k * TS + pb] = v;
          }
#pragma unroll
          for (int k = 0; k < NF; ++k) {
            const double v = ((const double*)(raw + p.raw_off[1 + NI + k]))[lb];
            emax = max(emax, (uint32_t)__double2hiint(v) & 0x7FF00000u);
            sfval[k * TS + pb] = v;
          }
        }
        // a queued row keeps draw word 0 in its (consumed) pu-key slot of the raw tile
        if (qa) ((unsigned long long*)raw)[la] = ha.w0;
        if (qb) ((unsigned long long*)raw)[lb] = hb.w0;
        const unsigned ma = __ballot_sync(0xffffffffu, qa);
        if (qa) {
          const int q = qn + __popc(ma & lt_mask);
          wq[q] = (unsigned short)pa;
          wr[q] = (unsigned short)la;
        }
        qn += __popc(ma);
        const unsigned mb = __ballot_sync(0xffffffffu, qb);
        if (qb) {
          const int q = qn + __popc(mb & lt_mask);
          wq[q] = (unsigned short)pb;
          wr[q] = (unsigned short)lb;
        }
        qn += __popc(mb);
      }
      maxabs = tmax > maxabs ? tmax : maxabs;
      const int fb = (NI > 0 && __any_sync(0xffffffffu, tmax >= (1ull << 26)) ? 1 : 0) |
                     (NF > 0 && __any_sync(0xffffffffu, emax == 0x7FF00000u) ? 2 : 0);
      if (fb && lane == 0) atomicOr(gflag, fb);
      __syncwarp();
      // A3: the warp finishes its queued masks from draw word 1 on (R2)
      for (int qi = lane; qi < qn; qi += 32) {
        const int pos = wq[qi];
        smask[pos] = (PAC_LEAN_BTAB && !owner) ? pac_hash_continue_bt(smask[pos], ((const unsigned long long*)raw)[wr[qi]], btab)
                                   : pac_hash_continue(smask[pos], ((const unsigned long long*)raw)[wr[qi]]);
      }
    }
    LEAN_CLK(4);  // A2 + A3
    __syncthreads();
    LEAN_CLK(5);  // barrier after A2
    if (tid == 0 && staged(t + 1)) issue_tile(p, raw, mbar, base + T, T);  // the raw tile is consumed

    // ---------------- C: full 32-row runs into the TMEM table; leftovers to the carry area
    {
      if (tid < Lcap) hp[tid] = 0;  // every warp read this tile's counts in B, before the last barrier
      const int fl = *gflag;
      const bool small = (NI == 0) || !(fl & 1);
      const bool fin = (NF == 0) || !(fl & 2);
      if (owner && PAC_LEAN_QBAL) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");  // slots change warps between tiles
        for (unsigned wk = owned_work; wk; wk &= wk - 1) {
          const int s = 4 * (__ffs(wk) - 1) + (wid & 3);
          const int tot = stot[s];
          const int lf = slfl[s];
          const int o = soff[s], f = tot >> 5;
          for (int i = 0; i < f; ++i) {
            const int b = o + 32 * i;
            if (small && fin)
              run_body<NI, NF, 0, false>(acc, smask + b, sival + b, TS, sfval + b, TS, nullptr, 32, xc, lane);
            else
              run_body<NI, NF, 0, true>(acc, smask + b, sival + b, TS, sfval + b, TS, nullptr, 32, xc, lane, small,
                                        fin);
          }
          const int l = tot & 31;
          if (l && lf)
            run_body<NI, NF, 0, true>(acc, smask + o + 32 * f, sival + o + 32 * f, TS, sfval + o + 32 * f, TS, nullptr,
                                      l, xc, lane, small, false);
          tm_flush<NI, NF, 0>(acc, lean_taddr(tbase, wid, s, S::wps, true));
          acc.reset();
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      } else if (owner) {
#if PAC_LEAN_WORKLIST
        for (unsigned wk = owned_work; wk; wk &= wk - 1) {
          const int s = wid + 16 * (__ffs(wk) - 1);
          const int tot = stot[s];
          const int lf = slfl[s];
#else
        for (int s = wid; s < Lcap; s += NW) {
          const int tot = stot[s];
          const int lf = slfl[s];
          if (tot < 32 && !lf) continue;  // nothing to run: the rows wait in the carry area
#endif
          const int o = soff[s], f = tot >> 5;
          for (int i = 0; i < f; ++i) {
            const int b = o + 32 * i;
            if (small && fin)
              run_body<NI, NF, 0, false>(acc, smask + b, sival + b, TS, sfval + b, TS, nullptr, 32, xc, lane);
            else
              run_body<NI, NF, 0, true>(acc, smask + b, sival + b, TS, sfval + b, TS, nullptr, 32, xc, lane, small,
                                        fin);
          }
          const int l = tot & 31;
          if (l && lf)
            run_body<NI, NF, 0, true>(acc, smask + o + 32 * f, sival + o + 32 * f, TS, sfval + o + 32 * f, TS, nullptr,
                                      l, xc, lane, small, false);
          tm_flush<NI, NF, 0>(acc, lean_taddr(tbase, wid, s, S::wps, true));
          acc.reset();
        }
      } else {
        const int R = nruns;
        const int r0 = (R * wid) / NW, r1 = (R * (wid + 1)) / NW;
        int cur = -1;
        for (int r = r0; r < r1; ++r) {
          const uint32_t d = rdesc[r];
          const int beg = (int)(d & 0xFFFFu);
          const int s = (int)((d >> 16) & 0x3FFu);
          if (s != cur) {
            if (cur >= 0) {
              tm_flush<NI, NF, 0>(acc, lean_taddr(tbase, wid, cur, S::wps, false));
              acc.reset();
            }
            cur = s;
          }
          if (small && fin)
            run_body<NI, NF, 0, false>(acc, smask + beg, sival + beg, TS, sfval + beg, TS, nullptr, 32, xc, lane);
          else
            run_body<NI, NF, 0, true>(acc, smask + beg, sival + beg, TS, sfval + beg, TS, nullptr, 32, xc, lane,
                                      small, fin);
        }
        if (cur >= 0) {
          tm_flush<NI, NF, 0>(acc, lean_taddr(tbase, wid, cur, S::wps, false));
          acc.reset();
        }
        // leftovers that do not fit the carry area: run now by warp s % 16
        for (int s = wid; s < Lcap; s += NW) {
          const int tot = stot[s], l = tot & 31;
          if (!l || !slfl[s]) continue;
          const int b = soff[s] + (tot & ~31);
          run_body<NI, NF, 0, true>(acc, smask + b, sival + b, TS, sfval + b, TS, nullptr, l, xc, lane, small, false);
          tm_flush<NI, NF, 0>(acc, lean_taddr(tbase, wid, s, S::wps, false));
          acc.reset();
        }
      }
      LEAN_CLK(6);  // C: runs
      // leftovers to the carry area (flat over its rows, every warp a share)
      if (PAC_LEAN_DYNCOPY && owner) {
        // the runs of a tile are split unevenly (a warp owns ~6 slots, each with a run in ~2 of 3
        // tiles), and the next barrier waits for the slowest warp: the warps that finish their runs
        // early take more of the copy-out, 32 carry rows per claim
        for (;;) {
          int c = 0;
          if (lane == 0) c = atomicAdd(cpctr, PAC_LEAN_DYNCHUNK);
          c = __shfl_sync(0xffffffffu, c, 0);
          if (c >= ncarry) break;
#pragma unroll
          for (int h = 0; h < PAC_LEAN_DYNCHUNK / 32; ++h) {
            const int i = c + 32 * h + lane;
            const int s = i < ncarry ? cs_out[i] : 0xFF;
            if (s != 0xFF) {
              unsigned long long tm = 0;
              uint32_t em = 0;
              lean_copy_row<NI, NF>(cmask, cival, cfval, i, CC, smask, sival, sfval, scpo[s] + i, TS, tm, em);
            }
          }
        }
      } else
      for (int i = tid; i < ncarry; i += kLeanThreads) {
        const int s = cs_out[i];
        if (s == 0xFF) continue;
        unsigned long long tm = 0;
        uint32_t em = 0;
        lean_copy_row<NI, NF>(cmask, cival, cfval, i, CC, smask, sival, sfval, scpo[s] + i, TS, tm, em);
      }
    }
    LEAN_CLK(7);  // C: copy-out
    // no barrier: A of the next tile touches only the other parity's counts and the dictionary;
    // B's shared outputs (read by C) are rewritten only after the barrier that follows A
  }
  __syncthreads();  // every leftover is in the carry area
#if PAC_LEAN_CLK
  if (blockIdx.x == 0 && lane == 0)
    printf("LEANCLK w%02d wait %lld A %lld barA %lld Bscan %lld Brest %lld copyin %lld A2 %lld barA2 %lld Cruns %lld Ccopy %lld tiles %lld\n",
           wid, clk[0], clk[1], clk[2], clk[8], clk[3], clk[9], clk[4], clk[5], clk[6], clk[7], (long long)(t1 - t0));
#endif

  // ---------------- the rows still in the carry area: one partial run per slot (owner / s % 16)
  for (int s = wid; s < Lcap; s += NW) {
    if (PAC_LEAN_QBAL && owner && !lean_mine(wid, s)) continue;
    const int src = (s >> 2), k = s & 3;
    const int c0 = __shfl_sync(0xffffffffu, k == 0 ? cb.cc[0] : k == 1 ? cb.cc[1] : k == 2 ? cb.cc[2] : cb.cc[3], src);
    const int o0 = __shfl_sync(0xffffffffu, k == 0 ? cb.co[0] : k == 1 ? cb.co[1] : k == 2 ? cb.co[2] : cb.co[3], src);
    if (!c0) continue;
    run_body<NI, NF, 0, true>(acc, cmask + o0, cival + o0, CC, cfval + o0, CC, nullptr, c0, xc, lane,
                              NI == 0 || maxabs_small(cival + o0, CC, c0, lane, NI), false);
    tm_flush<NI, NF, 0>(acc, lean_taddr(tbase, wid, s, S::wps, owner));
    acc.reset();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---------------- TMEM -> provisional HBM table, rows, the overflow bound
  const int nloc = min(misc->nlocal, lcap);
  for (int s = 0; s < nloc; ++s) {
    if (owner && !lean_mine(wid, s)) continue;
    tm_to_hbm<NI, NF, 0>(p, lean_taddr(tbase, wid, s, S::wps, owner), lprov[s], lane);
  }
  for (int s = tid; s < nloc; s += kLeanThreads)
    if (lprov[s] >= 0 && lrows[s]) atomicAdd(&p.prov_rows[lprov[s]], lrows[s]);
  if (tid == 0) atomicMax(&p.dbg[1], (unsigned long long)misc->nlocal);
  if (NI > 0) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, maxabs, d);
      maxabs = o > maxabs ? o : maxabs;
    }
    if (lane == 0 && maxabs) atomicMax(p.gmaxabs, maxabs);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmCols)
                             : "memory");
}

// Host side: whether the lean kernel applies, and its launch (agg_lean.cu).
bool lean_applicable(int ni, int nf, int has_min, int has_max, int has_count, int n_keys, int key_width,
                     int64_t G_cap, bool hashed);
cudaError_t launch_lean(AggPlan& p, int n_keys, int key_width, int sms, cudaStream_t st, char* kname, int kname_len);

}  // namespace pac
