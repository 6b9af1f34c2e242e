// libpac: k_agg_tiles_tm -- the tile kernel with its CTA accumulator table in Tensor Memory
// (DESIGN.md §5).  For tables of 33..256 groups (e.g. BASELINE C5, 100 groups) the CTA table
// (groups x 64 worlds x count/sums/extremes) is what fills shared memory and forces 1024-row
// tiles, i.e. ~10-row runs per group.  TMEM (256 KB per SM, 512 columns x 128 lanes x 32 bit) is
// idle in this ALU kernel, so the table lives there instead:
//   - warp w owns the slots s with s % 4 == w % 4 (its TMEM lane quarter) and
//     (s / 4) % 4 == w / 4; only the owner ever touches a slot's columns (no atomics);
//   - lane L of the owner holds worlds L and L+32 of a slot in `wps` consecutive columns
//     (count x2, then per int64 SUM lo/hi x2, per f64 SUM lo/hi x2, MIN / MAX encodings);
//   - phase C: the owner runs every run of its slots (register accumulators) and adds them into
//     the slot's columns (tcgen05.ld -> add -> tcgen05.st), once per slot and tile;
//   - the end: owners move their slots from TMEM to the provisional HBM table.
// The freed shared memory holds 2048-row tiles (TMA-staged), doubling the run length.
#pragma once
#include "agg_tiles.cuh"

namespace pac {

constexpr int kTmThreads = 512;  // 16 warps: 4 per TMEM lane quarter
constexpr int kTmCols = 512;

__device__ __forceinline__ void tm_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr));
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(taddr));
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tm_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b),
               "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint64_t u64of(uint32_t lo, uint32_t hi) { return (uint64_t)lo | ((uint64_t)hi << 32); }

template <int NI, int NF, int MM>
struct TmSlot {
  static constexpr int wps = 2 + 4 * NI + 4 * NF + ((MM & 1) ? 4 : 0) + ((MM & 2) ? 4 : 0);
  static constexpr int o_isum = 2;
  static constexpr int o_fsum = 2 + 4 * NI;
  static constexpr int o_min = 2 + 4 * NI + 4 * NF;
  static constexpr int o_max = o_min + ((MM & 1) ? 4 : 0);
};

// Column of slot s = q + 4 i + 16 k (q = TMEM quarter, i = owner index in the quarter).
__device__ __forceinline__ uint32_t tm_slot_addr(uint32_t tbase, int s, int K, int wps) {
  const int q = s & 3, i = (s >> 2) & 3, k = s >> 4;
  return tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)((i * K + k) * wps);
}

template <int NI, int NF, int MM>
__device__ __forceinline__ void tm_init_slot(uint32_t a) {
  using S = TmSlot<NI, NF, MM>;
  tm_st2(a, 0u, 0u);
#pragma unroll
  for (int c = 0; c < NI; ++c) tm_st4(a + S::o_isum + 4 * c, 0u, 0u, 0u, 0u);
#pragma unroll
  for (int c = 0; c < NF; ++c) tm_st4(a + S::o_fsum + 4 * c, 0u, 0u, 0u, 0u);
  if (MM & 1) {
    const uint64_t e = (uint64_t)kMinEmpty;
    tm_st4(a + S::o_min, (uint32_t)e, (uint32_t)(e >> 32), (uint32_t)e, (uint32_t)(e >> 32));
  }
  if (MM & 2) {
    const uint64_t e = (uint64_t)kMaxEmpty;
    tm_st4(a + S::o_max, (uint32_t)e, (uint32_t)(e >> 32), (uint32_t)e, (uint32_t)(e >> 32));
  }
}

// slot's TMEM columns += the warp's register accumulators (owner warp only)
template <int NI, int NF, int MM>
__device__ __forceinline__ void tm_flush(const WarpAcc<NI, NF, MM>& acc, uint32_t a) {
  using S = TmSlot<NI, NF, MM>;
  uint32_t c0, c1, iv[NI > 0 ? NI : 1][4], fv[NF > 0 ? NF : 1][4], mn[4], mx[4];
  tm_ld2(a, c0, c1);
#pragma unroll
  for (int c = 0; c < NI; ++c) tm_ld4(a + S::o_isum + 4 * c, iv[c][0], iv[c][1], iv[c][2], iv[c][3]);
#pragma unroll
  for (int c = 0; c < NF; ++c) tm_ld4(a + S::o_fsum + 4 * c, fv[c][0], fv[c][1], fv[c][2], fv[c][3]);
  if (MM & 1) tm_ld4(a + S::o_min, mn[0], mn[1], mn[2], mn[3]);
  if (MM & 2) tm_ld4(a + S::o_max, mx[0], mx[1], mx[2], mx[3]);
  tm_wait_ld();
  tm_st2(a, c0 + acc.c0, c1 + acc.c1);
#pragma unroll
  for (int c = 0; c < NI; ++c) {
    const uint64_t s0 = u64of(iv[c][0], iv[c][1]) + (uint64_t)acc.ia0[c];
    const uint64_t s1 = u64of(iv[c][2], iv[c][3]) + (uint64_t)acc.ia1[c];
    tm_st4(a + S::o_isum + 4 * c, (uint32_t)s0, (uint32_t)(s0 >> 32), (uint32_t)s1, (uint32_t)(s1 >> 32));
  }
#pragma unroll
  for (int c = 0; c < NF; ++c) {
    const double f0 = __longlong_as_double((long long)u64of(fv[c][0], fv[c][1])) + acc.fa0[c];
    const double f1 = __longlong_as_double((long long)u64of(fv[c][2], fv[c][3])) + acc.fa1[c];
    const uint64_t b0 = (uint64_t)__double_as_longlong(f0), b1 = (uint64_t)__double_as_longlong(f1);
    tm_st4(a + S::o_fsum + 4 * c, (uint32_t)b0, (uint32_t)(b0 >> 32), (uint32_t)b1, (uint32_t)(b1 >> 32));
  }
  if (MM & 1) {
    const long long e0 = min((long long)u64of(mn[0], mn[1]), acc.mn0);
    const long long e1 = min((long long)u64of(mn[2], mn[3]), acc.mn1);
    tm_st4(a + S::o_min, (uint32_t)e0, (uint32_t)((uint64_t)e0 >> 32), (uint32_t)e1, (uint32_t)((uint64_t)e1 >> 32));
  }
  if (MM & 2) {
    const long long e0 = max((long long)u64of(mx[0], mx[1]), acc.mx0);
    const long long e1 = max((long long)u64of(mx[2], mx[3]), acc.mx1);
    tm_st4(a + S::o_max, (uint32_t)e0, (uint32_t)((uint64_t)e0 >> 32), (uint32_t)e1, (uint32_t)((uint64_t)e1 >> 32));
  }
  tm_wait_st();
}

// the owner moves a slot from TMEM to the provisional HBM table
template <int NI, int NF, int MM>
__device__ __forceinline__ void tm_to_hbm(const AggPlan& p, uint32_t a, int prov, int lane) {
  using S = TmSlot<NI, NF, MM>;
  uint32_t c0, c1, iv[NI > 0 ? NI : 1][4], fv[NF > 0 ? NF : 1][4], mn[4], mx[4];
  tm_ld2(a, c0, c1);
#pragma unroll
  for (int c = 0; c < NI; ++c) tm_ld4(a + S::o_isum + 4 * c, iv[c][0], iv[c][1], iv[c][2], iv[c][3]);
#pragma unroll
  for (int c = 0; c < NF; ++c) tm_ld4(a + S::o_fsum + 4 * c, fv[c][0], fv[c][1], fv[c][2], fv[c][3]);
  if (MM & 1) tm_ld4(a + S::o_min, mn[0], mn[1], mn[2], mn[3]);
  if (MM & 2) tm_ld4(a + S::o_max, mx[0], mx[1], mx[2], mx[3]);
  tm_wait_ld();
  if (prov < 0) return;
  const size_t g0 = (size_t)prov * kM + lane, g1 = g0 + 32;
  if (c0) atomicAdd(&p.prov_count[g0], (unsigned long long)c0);
  if (c1) atomicAdd(&p.prov_count[g1], (unsigned long long)c1);
#pragma unroll
  for (int c = 0; c < NI; ++c) {
    const unsigned long long s0 = u64of(iv[c][0], iv[c][1]), s1 = u64of(iv[c][2], iv[c][3]);
    if (s0) atomicAdd(&p.prov_isum[c][g0], s0);
    if (s1) atomicAdd(&p.prov_isum[c][g1], s1);
  }
#pragma unroll
  for (int c = 0; c < NF; ++c) {
    const double f0 = __longlong_as_double((long long)u64of(fv[c][0], fv[c][1]));
    const double f1 = __longlong_as_double((long long)u64of(fv[c][2], fv[c][3]));
    if (f0 != 0.0) atomicAdd(&p.prov_fsum[c][g0], f0);
    if (f1 != 0.0) atomicAdd(&p.prov_fsum[c][g1], f1);
  }
  if (MM & 1) {
    atomicMin(&p.prov_min[g0], (long long)u64of(mn[0], mn[1]));
    atomicMin(&p.prov_min[g1], (long long)u64of(mn[2], mn[3]));
  }
  if (MM & 2) {
    atomicMax(&p.prov_max[g0], (long long)u64of(mx[0], mx[1]));
    atomicMax(&p.prov_max[g1], (long long)u64of(mx[2], mx[3]));
  }
}

// LC = 0: runtime layout; LC > 0: T = 2048 with LC local slots as a compile-time layout (as
// k_agg_tiles' small-table instance: immediate smem offsets, folded index arithmetic).
constexpr int kTmFixedSlots = 128;

template <int NI, int NF, int MM, int LC>
__global__ void __launch_bounds__(kTmThreads, 1) k_agg_tiles_tm(AggPlan p, SmemLayout Lp) {
  constexpr SmemLayout Lc = tile_layout(NI, NF, MM & 1, (MM >> 1) & 1, 2048, LC > 0 ? LC : 1, 0, 1);
  const SmemLayout& L = LC > 0 ? Lc : Lp;
  using S = TmSlot<NI, NF, MM>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t s_tbase;
  TileSmem sm{};
  sm.lkey = (unsigned long long*)(smem + L.o_lkey);
  sm.lstate = (int*)(smem + L.o_lstate);
  sm.lprov = (int*)(smem + L.o_lprov);
  sm.lrows = (unsigned long long*)(smem + L.o_lrows);
  sm.smask = (unsigned long long*)(smem + L.o_mask);
  sm.sival = (long long*)(smem + L.o_ival);
  sm.rdesc = (uint32_t*)(smem + L.o_rdesc);
  sm.sfval = (double*)(smem + L.o_fval);
  sm.smval = (long long*)(smem + L.o_mval);
  sm.sslot = (unsigned short*)(smem + L.o_slot);
  sm.srank = (unsigned char*)(smem + L.o_rank);
  sm.ucnt = (unsigned short*)(smem + L.o_ucnt);
  sm.qpos = (unsigned short*)(smem + L.o_queue);
  sm.qrow = sm.qpos + L.T;
  sm.hist = (int*)(smem + L.o_hist);
  sm.offs = (int*)(smem + L.o_offs);
  sm.runoffs = (int*)(smem + L.o_runoffs);
  sm.xcs = (uint4*)(smem + L.o_xcs);
  sm.xcs2 = (uint2*)(smem + L.o_xcs + 32 * 16);
  sm.misc = (Misc*)(smem + L.o_misc);
  unsigned char* raw = smem + L.o_raw;
  sm.raw = raw;
  unsigned long long* mbar = (unsigned long long*)(smem + L.o_mbar);
  Misc* misc = sm.misc;

  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int T = L.T, Lcap = L.Lcap, LH = L.LH;
  const int K = (Lcap + 15) >> 4;  // slots per owner warp (upper bound)

  // TMEM: warp 0 allocates all 512 columns (one CTA per SM)
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tbase)),
                 "n"(kTmCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < LH; i += nth) sm.lstate[i] = 0;
  for (int i = tid; i < Lcap; i += nth) {
    sm.lrows[i] = 0;
    sm.hist[i] = 0;
  }
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }
  if (tid < 32) store_xpose(sm.xcs, sm.xcs2, tid);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = s_tbase;
  // owners initialise their slots (zeros; MIN/MAX sentinels)
  const int q = wid & 3, oi = (wid >> 2) & 3;
  for (int k = 0; k < K; ++k) {
    const int s = q + 4 * oi + 16 * k;
    if (s < Lcap) tm_init_slot<NI, NF, MM>(tm_slot_addr(tbase, s, K, S::wps));
  }
  tm_wait_st();
  unsigned long long maxabs = 0;

  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  __shared__ long long s_unit[2];
  uint32_t phase = 0;
  if (tid == 0) mbar_init(mbar, 1);
  __syncthreads();

  SpillCur sc;
  sc.init();
  // Row ranges: without units, the CTA's contiguous share of the tiles; with units (partitioned
  // input), units taken from the global counter, the CTA table flushed and reset after each.
  for (int it = 0;; ++it) {
    int64_t r0, r1;
    if (p.units) {
      if (tid == 0) {
        const int u = atomicAdd(p.unit_ctr, 1);
        const bool ok = u < *p.n_units;
        s_unit[0] = ok ? p.units[u].x : 0;
        s_unit[1] = ok ? p.units[u].y : -1;
      }
      __syncthreads();
      r0 = s_unit[0];
      r1 = s_unit[1];
      if (r1 < 0) break;
    } else {
      if (it > 0) break;
      const int64_t t0 = (int64_t)blockIdx.x * t_per;
      r0 = t0 * T;
      r1 = min(p.n_rows, (t0 + t_per) * T);
    }
    const int64_t nt = r1 > r0 ? (r1 - r0 + T - 1) / T : 0;
    auto staged_tile = [&](int64_t i) { return p.tma_ok && i < nt && r0 + (i + 1) * T <= r1; };
    auto tile_rows = [&](int64_t i) { return (int)min((int64_t)T, r1 - (r0 + i * T)); };
    if (tid == 0 && staged_tile(0)) issue_tile(p, raw, mbar, r0, T);
    if (nt > 0) {
      if (staged_tile(0)) {
        mbar_wait(mbar, phase);
        phase ^= 1u;
        tile_a1<NI, NF, MM, true>(p, sm, L, r0, T, sc);
      } else {
        tile_a1<NI, NF, MM, false>(p, sm, L, r0, tile_rows(0), sc);
      }
    }
    for (int64_t i = 0; i < nt; ++i) {
      const int64_t base = r0 + i * T;
      const bool staged = staged_tile(i);
      __syncthreads();  // A1(tile) and C(tile-1) complete
      if (staged) tile_mid<NI, NF, MM, true>(p, sm, L, base, maxabs);
      else tile_mid<NI, NF, MM, false>(p, sm, L, base, maxabs);
      const bool next_staged = staged_tile(i + 1);
      if (tid == 0 && next_staged) issue_tile(p, raw, mbar, base + T, T);

      // ---------------- C: each owner warp runs the runs of its slots, then adds them to TMEM
      {
        const bool small = (NI == 0) || misc->big == 0;
        const bool fin = (NF == 0) || misc->nonfinite == 0;
        const XposeConst xc = load_xpose(sm.xcs, sm.xcs2, lane);
        for (int k = 0; k < K; ++k) {
          const int s = q + 4 * oi + 16 * k;
          if (s >= Lcap) break;
          const int rb = sm.runoffs[s], re = sm.runoffs[s + 1];
          if (rb == re) continue;
          WarpAcc<NI, NF, MM> acc;
          acc.cur = s;
          acc.reset();
          for (int r = rb; r < re; ++r) {
            const uint32_t d = sm.rdesc[r];
            const int beg = (int)(d & 0xFFFFu);
            const int len = (int)(d >> 26) + 1;
            if (small && fin)
              run_body<NI, NF, MM, false>(acc, sm.smask + beg, sm.sival + beg, L.TS, sm.sfval + beg, L.TS,
                                          sm.smval + beg, len, xc, lane);
            else
              run_body<NI, NF, MM, true>(acc, sm.smask + beg, sm.sival + beg, L.TS, sm.sfval + beg, L.TS,
                                         sm.smval + beg, len, xc, lane, small, fin);
          }
          tm_flush<NI, NF, MM>(acc, tm_slot_addr(tbase, s, K, S::wps));
        }
      }
      if (i + 1 < nt) {
        if (next_staged) {
          mbar_wait(mbar, phase);
          phase ^= 1u;
          tile_a1<NI, NF, MM, true>(p, sm, L, base + T, T, sc);
        } else {
          tile_a1<NI, NF, MM, false>(p, sm, L, base + T, tile_rows(i + 1), sc);
        }
      }
    }
    if (p.units) {
      // ---------------- end of a unit: its slots to the provisional HBM table, then a fresh table
      __syncthreads();
      const int nl = min(misc->nlocal, Lcap);
      for (int k = 0; k < K; ++k) {
        const int s = q + 4 * oi + 16 * k;
        if (s >= nl) break;
        const uint32_t a = tm_slot_addr(tbase, s, K, S::wps);
        tm_to_hbm<NI, NF, MM>(p, a, sm.lprov[s], lane);
        tm_init_slot<NI, NF, MM>(a);
      }
      tm_wait_st();
      for (int s = tid; s < nl; s += nth) {
        if (sm.lprov[s] >= 0 && sm.lrows[s]) atomicAdd(&p.prov_rows[sm.lprov[s]], sm.lrows[s]);
        sm.lrows[s] = 0;
      }
      for (int i = tid; i < LH; i += nth) sm.lstate[i] = 0;
      __syncthreads();  // every thread has read nlocal
      if (tid == 0) {
        atomicMax(&p.dbg[1], (unsigned long long)misc->nlocal);
        misc->nlocal = 0;
        misc->ndict = 0;
      }
    }
  }
  __syncthreads();

  sc.finish(p, lane);
  // ---------------- TMEM -> provisional HBM table (owners), rows and the overflow bound
  const int nloc = min(misc->nlocal, Lcap);
  if (tid == 0) atomicMax(&p.dbg[1], (unsigned long long)misc->nlocal);
  for (int k = 0; k < K; ++k) {
    const int s = q + 4 * oi + 16 * k;
    if (s >= nloc) break;
    tm_to_hbm<NI, NF, MM>(p, tm_slot_addr(tbase, s, K, S::wps), sm.lprov[s], lane);
  }
  for (int s = tid; s < nloc; s += nth)
    if (sm.lprov[s] >= 0 && sm.lrows[s]) atomicAdd(&p.prov_rows[sm.lprov[s]], sm.lrows[s]);
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

// TMEM columns one owner warp needs in its lane quarter: 4 owners x K slots x wps words
template <int NI, int NF, int MM>
constexpr int tm_cols_needed(int Lcap) {
  return 4 * ((Lcap + 15) / 16) * TmSlot<NI, NF, MM>::wps;
}

template <int NI, int NF, int MM>
cudaError_t launch_tm(const AggPlan& p, const SmemLayout& L, int sms, cudaStream_t st) {
  const bool fixed = L.T == 2048 && L.Lcap == kTmFixedSlots && !getenv("PAC_NO_FIXED");
  auto k = fixed ? k_agg_tiles_tm<NI, NF, MM, kTmFixedSlots> : k_agg_tiles_tm<NI, NF, MM, 0>;
  if (tm_cols_needed<NI, NF, MM>(L.Lcap) > kTmCols) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (p.n_rows + L.T - 1) / L.T;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms));  // one CTA per SM
  if (getenv("PAC_DEBUG"))
    fprintf(stderr, "[libpac] k_agg_tiles_tm<%d,%d,%d> %d CTAs x %d threads, T=%d Lcap=%d smem=%d B\n", NI, NF, MM,
            grid, kTmThreads, L.T, L.Lcap, L.bytes);
  k<<<grid, kTmThreads, L.bytes, st>>>(p, L);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pac
