// libpac: native 128-world grouped aggregation (§8 f4; P:L92 footnote "Extending to m=128 is
// possible, and worst-case would double the cost of our stochastic-aggregates"; R28, R29).
//
// k_agg_tiles128 is the single-pass counterpart of the three-pass path in m128.cu for tables that
// fit one CTA (every group a CTA-local slot: G_cap <= 32) and COUNT / SUM / AVG aggregates.
// Per 1024-row tile, 256 threads:
//   A1  group slot of every row (CTA dictionary local_code -> HBM dictionary global_slot); the
//       warp's rows of one slot are counted with one shared atomic (match_any)
//   B   one warp: 8-row padded slot offsets, run descriptors, zero padding rows
//   A2  the 128-bit mask of every row (R28: draw word 0 of pac_hash128; or the caller's [n][2]
//       masks) and its values, written to the row's slot-sorted position (warp-aggregated cursor
//       atomics); rows still owing flips queue per warp
//   A3  the warp finishes its queued masks one draw word per pass (pac_hash128_step on the queued
//       state), each pass compacting the queue to the rows still owing flips, so a draw word costs
//       a warp pass per 32 rows that need it rather than per 32 rows
// Full tiles with 16-byte aligned columns are staged by 1-D TMA bulk copies (p.raw_*), issued
// when A2 of the previous tile has consumed the buffer, so they land while phase C runs.
//   C   world-parallel runs: run_body128 -- the transposed Four Russians tables of run_body
//       (agg_tiles.cuh), built once per run and looked up with the nibbles of both mask words,
//       into two warp accumulators (worlds 0..63, 64..127)
// The CTA table is [slot][128] = [2 * slot + half][64]: "virtual" 64-world slots 2s (worlds
// 0..63) and 2s + 1 (64..127), so WarpAcc::flush serves both halves unchanged.  At the end the
// CTA table is added into the provisional HBM table [G_cap][128] (AggPlan::m128 = 1).
// A group with no CTA-local slot exists only when the input has more than G_cap distinct groups:
// its rows are dropped and the finish kernel reports PAC_E_CAPACITY (the table is then invalid).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "agg_tiles.cuh"
#include "hash128.cuh"

namespace pac {

struct Lay128 {
  int T, TS, Lcap, LH;
  int o_cnt, o_isum, o_fsum, o_lrows, o_lkey, o_lstate, o_lprov, o_mask, o_ival, o_fval, o_rdesc, o_slot, o_hist,
      o_cur, o_queue, o_xcs, o_mbar, o_misc, o_raw, bytes;
};

__host__ __device__ constexpr Lay128 lay128(int ni, int nf, int T, int Lcap, int raw_bytes) {
  Lay128 L{};
  L.T = T;
  L.TS = T + 8 * Lcap;
  L.Lcap = Lcap;
  L.LH = lay_pow2(4 * Lcap > 256 ? 4 * Lcap : 256);
  const int V = 2 * Lcap * kM;  // entries of one CTA table: [2 * Lcap virtual slots][64]
  int off = 0;
  L.o_isum = lay_take(off, ni * V * 8);
  L.o_fsum = lay_take(off, nf * V * 8);
  L.o_lrows = lay_take(off, Lcap * 8);
  L.o_lkey = lay_take(off, L.LH * 8);
  L.o_mask = lay_take(off, 2 * L.TS * 8);  // [lo: TS][hi: TS]
  L.o_ival = lay_take(off, ni * L.TS * 8);
  L.o_fval = lay_take(off, nf * L.TS * 8);
  L.o_cnt = lay_take(off, V * 4);
  L.o_lstate = lay_take(off, L.LH * 4);
  L.o_lprov = lay_take(off, Lcap * 4);
  L.o_rdesc = lay_take(off, (T / 32 + Lcap + 1) * 4);
  L.o_hist = lay_take(off, Lcap * 4);
  L.o_cur = lay_take(off, Lcap * 4);
  L.o_slot = lay_take(off, T);
  L.o_queue = lay_take(off, T * 8 + 2 * T * 2);  // per-warp queues of rows owing draw words: w, pos, k|maj
  L.o_xcs = lay_take(off, 32 * 16 + 32 * 8);
  L.o_mbar = lay_take(off, 16);
  L.o_misc = lay_take(off, (int)sizeof(Misc));
  L.o_raw = lay_take(off, raw_bytes);  // the staged tile (1-D TMA bulk copies, p.raw_*)
  L.bytes = off;
  return L;
}

constexpr int kT128 = 1024;
constexpr int kThreads128 = 256;
constexpr unsigned char kNoSlot = 0xFF;

// Columns of one tile: raw column 0 = pu keys (8 B) or masks (16 B), then the int64 and f64 sum
// columns, then the group-key columns.  S: read from the TMA-staged copy in shared memory.
template <bool S, int NI, int NF>
struct Cols128 {
  const AggPlan* p;
  const unsigned char* raw;
  int64_t base;
  int T;
  __device__ __forceinline__ uint64_t key(int li) const {
    return S ? ((const unsigned long long*)(raw + p->raw_off[0]))[li]
             : (uint64_t)__ldg(p->pu_key + base + li);
  }
  __device__ __forceinline__ ulonglong2 mask(int li) const {
    return S ? ((const ulonglong2*)(raw + p->raw_off[0]))[li] : __ldg((const ulonglong2*)p->mask_in + base + li);
  }
  __device__ __forceinline__ long long ival(int c, int li) const {
    return S ? ((const long long*)(raw + p->raw_off[1 + c]))[li] : __ldg(p->icol[c] + base + li);
  }
  __device__ __forceinline__ double fval(int c, int li) const {
    return S ? ((const double*)(raw + p->raw_off[1 + NI + c]))[li] : __ldg(p->fcol[c] + base + li);
  }
  __device__ __forceinline__ uint64_t group_key(int li) const {
    return TileCols<S>{p, raw, base, T}.group_key(1 + NI + NF, li);
  }
};

// run_body (agg_tiles.cuh) over both mask words of a run at once.  The per-lane subset sums of 4
// rows' values (the "Four Russians" tables) do not depend on the masks, so each table is built
// once and looked up with the nibbles of both words: worlds 0..63 into alo, 64..127 into ahi.
// Padding rows as in run_body (zero masks, finite values).
template <int NI, int NF, bool GENERIC>
__device__ __forceinline__ void run_body128(WarpAcc<NI, NF, 0>& alo, WarpAcc<NI, NF, 0>& ahi,
                                            const unsigned long long* __restrict__ smlo,
                                            const unsigned long long* __restrict__ smhi,
                                            const long long* __restrict__ sival, int istride,
                                            const double* __restrict__ sfval, int fstride, int len,
                                            const XposeConst& xc, int lane, bool small_rt = true, bool fin_rt = true) {
  const bool SMALL = GENERIC ? small_rt : true;
  const bool FIN = GENERIC ? fin_rt : true;
  const int tsrc = (lane >> 4) << 2;
  const int ib0 = lane & 1, ib1 = (lane >> 1) & 1, ib2 = (lane >> 2) & 1, ib3 = (lane >> 3) & 1;
  const double db0 = ib0, db1 = ib1, db2 = ib2, db3 = ib3;
  const uint64_t m0 = lane < len ? smlo[lane] : 0ull;
  const uint64_t m1 = lane < len ? smhi[lane] : 0ull;
  uint32_t P0 = (uint32_t)m0, Q0 = (uint32_t)(m0 >> 32), P1 = (uint32_t)m1, Q1 = (uint32_t)(m1 >> 32);
  transpose2x32(P0, Q0, xc);
  transpose2x32(P1, Q1, xc);
  alo.c0 += __popc(P0);
  alo.c1 += __popc(Q0);
  ahi.c0 += __popc(P1);
  ahi.c1 += __popc(Q1);
  // words v = 0..3: worlds 0-31, 32-63 (alo), 64-95, 96-127 (ahi)
  const uint32_t IA0 = P0 & 0x0F0F0F0Fu, IB0 = ((P0 >> 4) & 0x0F0F0F0Fu) | 0x10101010u;
  const uint32_t IA1 = Q0 & 0x0F0F0F0Fu, IB1 = ((Q0 >> 4) & 0x0F0F0F0Fu) | 0x10101010u;
  const uint32_t IA2 = P1 & 0x0F0F0F0Fu, IB2 = ((P1 >> 4) & 0x0F0F0F0Fu) | 0x10101010u;
  const uint32_t IA3 = Q1 & 0x0F0F0F0Fu, IB3 = ((Q1 >> 4) & 0x0F0F0F0Fu) | 0x10101010u;
  const int nq = (len + 7) >> 3;
  int rs0[NI > 0 ? NI : 1], rs1[NI > 0 ? NI : 1], rs2[NI > 0 ? NI : 1], rs3[NI > 0 ? NI : 1];
#pragma unroll
  for (int c = 0; c < NI; ++c) rs0[c] = rs1[c] = rs2[c] = rs3[c] = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q >= nq) break;
    const int a0 = (int)(IA0 >> (8 * q)), b0 = (int)(IB0 >> (8 * q));
    const int a1 = (int)(IA1 >> (8 * q)), b1 = (int)(IB1 >> (8 * q));
    const int a2 = (int)(IA2 >> (8 * q)), b2 = (int)(IB2 >> (8 * q));
    const int a3 = (int)(IA3 >> (8 * q)), b3 = (int)(IB3 >> (8 * q));
    const int row = 8 * q + tsrc;
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      const longlong2 u = *(const longlong2*)(sival + c * istride + row);
      const longlong2 w = *(const longlong2*)(sival + c * istride + row + 2);
      if (SMALL) {
        const int t = (int)u.x * ib0 + (int)u.y * ib1 + (int)w.x * ib2 + (int)w.y * ib3;
        rs0[c] += __shfl_sync(0xffffffffu, t, a0) + __shfl_sync(0xffffffffu, t, b0);
        rs1[c] += __shfl_sync(0xffffffffu, t, a1) + __shfl_sync(0xffffffffu, t, b1);
        rs2[c] += __shfl_sync(0xffffffffu, t, a2) + __shfl_sync(0xffffffffu, t, b2);
        rs3[c] += __shfl_sync(0xffffffffu, t, a3) + __shfl_sync(0xffffffffu, t, b3);
      } else {
        const long long t = u.x * ib0 + u.y * ib1 + w.x * ib2 + w.y * ib3;
        alo.ia0[c] += __shfl_sync(0xffffffffu, t, a0) + __shfl_sync(0xffffffffu, t, b0);
        alo.ia1[c] += __shfl_sync(0xffffffffu, t, a1) + __shfl_sync(0xffffffffu, t, b1);
        ahi.ia0[c] += __shfl_sync(0xffffffffu, t, a2) + __shfl_sync(0xffffffffu, t, b2);
        ahi.ia1[c] += __shfl_sync(0xffffffffu, t, a3) + __shfl_sync(0xffffffffu, t, b3);
      }
    }
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      const double2 u = *(const double2*)(sfval + c * fstride + row);
      const double2 w = *(const double2*)(sfval + c * fstride + row + 2);
      double t;
      if (FIN) {  // exact: 0*v + t == t and 1*v + t == v + t for finite v
        t = fma(db3, w.y, fma(db2, w.x, fma(db1, u.y, db0 * u.x)));
      } else {
        t = ib0 ? u.x : 0.0;
        if (ib1) t += u.y;
        if (ib2) t += w.x;
        if (ib3) t += w.y;
      }
      alo.fa0[c] += shfl_d(t, a0);
      alo.fa0[c] += shfl_d(t, b0);
      alo.fa1[c] += shfl_d(t, a1);
      alo.fa1[c] += shfl_d(t, b1);
      ahi.fa0[c] += shfl_d(t, a2);
      ahi.fa0[c] += shfl_d(t, b2);
      ahi.fa1[c] += shfl_d(t, a3);
      ahi.fa1[c] += shfl_d(t, b3);
    }
  }
  if (SMALL) {
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      alo.ia0[c] += rs0[c];
      alo.ia1[c] += rs1[c];
      ahi.ia0[c] += rs2[c];
      ahi.ia1[c] += rs3[c];
    }
  }
}

template <bool V>
using BoolTag = std::integral_constant<bool, V>;

template <int NI, int NF>
__global__ void __launch_bounds__(kThreads128, 2) k_agg_tiles128(AggPlan p, Lay128 L) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* cnt = (unsigned*)(smem + L.o_cnt);
  unsigned long long* isum = (unsigned long long*)(smem + L.o_isum);
  double* fsum = (double*)(smem + L.o_fsum);
  unsigned long long* lrows = (unsigned long long*)(smem + L.o_lrows);
  unsigned long long* lkey = (unsigned long long*)(smem + L.o_lkey);
  int* lstate = (int*)(smem + L.o_lstate);
  int* lprov = (int*)(smem + L.o_lprov);
  unsigned long long* smask = (unsigned long long*)(smem + L.o_mask);
  long long* sival = (long long*)(smem + L.o_ival);
  double* sfval = (double*)(smem + L.o_fval);
  uint32_t* rdesc = (uint32_t*)(smem + L.o_rdesc);
  unsigned char* sslot = smem + L.o_slot;
  int* hist = (int*)(smem + L.o_hist);
  int* cursor = (int*)(smem + L.o_cur);
  uint4* xcs = (uint4*)(smem + L.o_xcs);
  uint2* xcs2 = (uint2*)(smem + L.o_xcs + 32 * 16);
  Misc* misc = (Misc*)(smem + L.o_misc);
  unsigned char* squeue = smem + L.o_queue;
  unsigned long long* mbar = (unsigned long long*)(smem + L.o_mbar);
  unsigned char* raw = smem + L.o_raw;

  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int T = L.T, TS = L.TS, Lcap = L.Lcap, LH = L.LH;
  const int V = 2 * Lcap;  // virtual 64-world slots

  for (int i = tid; i < LH; i += nth) lstate[i] = 0;
  for (int i = tid; i < Lcap; i += nth) {
    lrows[i] = 0;
    hist[i] = 0;
  }
  for (int i = tid; i < V * kM; i += nth) {
    cnt[i] = 0;
#pragma unroll
    for (int c = 0; c < NI; ++c) isum[(size_t)c * V * kM + i] = 0;
#pragma unroll
    for (int c = 0; c < NF; ++c) fsum[(size_t)c * V * kM + i] = 0.0;
  }
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }
  if (tid < 32) store_xpose(xcs, xcs2, tid);
  unsigned long long maxabs = 0;

  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * t_per;
  const int64_t t1 = min(ntiles, t0 + t_per);
  auto tile_rows = [&](int64_t t) { return (int)min((int64_t)T, p.n_rows - t * T); };
  const bool masked = p.mask_in != nullptr;
  // a tile is staged by TMA when it is full and every column is 16-byte aligned
  auto staged_tile = [&](int64_t t) { return p.tma_ok && t < t1 && (t + 1) * T <= p.n_rows; };
  uint32_t phase = 0;

  // A1: slot of every row; per-slot row counts of the tile
  auto a1 = [&](auto stg, int64_t base, int tn) {
    const Cols128<decltype(stg)::value, NI, NF> cl{&p, raw, base, T};
    for (int li = tid; li < T; li += nth) {
      int s = -1;
      if (li < tn) {
        bool keep = true;
        if (masked) {
          const ulonglong2 m = cl.mask(li);
          keep = (m.x | m.y) != 0ull;  // R21: a row in no world is dropped
        }
        if (keep) {
          const int code = local_code(p, cl.group_key(li), lkey, lstate, LH, lprov, Lcap, misc);
          if (code < kOvfBase) s = code - 1;  // else: more than G_cap groups (CAPACITY), dropped
        }
      }
      const unsigned peers = __match_any_sync(0xffffffffu, s >= 0 ? (unsigned)s : 0x100u + lane);
      if (s >= 0 && (peers & lt_mask) == 0) atomicAdd(&hist[s], __popc(peers));
      sslot[li] = s >= 0 ? (unsigned char)s : kNoSlot;
    }
  };
  // A2: masks (word 0 of the hash; rows owing more draws queued per warp) and values to the
  // slot-sorted positions; A3: the warp finishes its queued rows 32 at a time
  auto a2 = [&](auto stg, int64_t base) {
    const Cols128<decltype(stg)::value, NI, NF> cl{&p, raw, base, T};
    unsigned long long tmax = 0;
    uint32_t emax = 0;
    unsigned long long* qw = (unsigned long long*)squeue + wid * (T / nw);
    unsigned short* qpos = (unsigned short*)(squeue + T * 8) + wid * (T / nw);
    unsigned short* qk = (unsigned short*)(squeue + T * 8) + T + wid * (T / nw);
    int qn = 0;
    for (int li = tid; li < T; li += nth) {
      const int s = sslot[li];
      const unsigned peers = __match_any_sync(0xffffffffu, s != kNoSlot ? (unsigned)s : 0x100u + lane);
      int b = 0;
      if (s != kNoSlot && (peers & lt_mask) == 0) b = atomicAdd(&cursor[s], __popc(peers));
      b = __shfl_sync(0xffffffffu, b, __ffs(peers) - 1);
      const int pos = b + __popc(peers & lt_mask);
      bool pend = false;
      uint64_t w = 0;
      int k = 0;
      bool maj = false;
      if (s != kNoSlot) {
        uint64_t lo, hi;
        if (masked) {
          const ulonglong2 m = cl.mask(li);
          lo = m.x;
          hi = m.y;
        } else {
          pac_hash128_word0(cl.key(li), p.salt, lo, hi, w, k, maj);
          pend = k > 0;
        }
        smask[pos] = lo;
        smask[TS + pos] = hi;
#pragma unroll
        for (int c = 0; c < NI; ++c) {
          const long long v = cl.ival(c, li);
          const unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
          tmax = a > tmax ? a : tmax;
          sival[c * TS + pos] = v;
        }
#pragma unroll
        for (int c = 0; c < NF; ++c) {
          const double v = cl.fval(c, li);
          emax = max(emax, (uint32_t)__double2hiint(v) & 0x7FF00000u);
          sfval[c * TS + pos] = v;
        }
      }
      const unsigned pm = __ballot_sync(0xffffffffu, pend);
      if (pend) {
        const int q = qn + __popc(pm & lt_mask);
        qw[q] = w;
        qpos[q] = (unsigned short)pos;
        qk[q] = (unsigned short)(k | (maj ? 128 : 0));
      }
      qn += __popc(pm);
    }
    maxabs = tmax > maxabs ? tmax : maxabs;
    if (NI > 0 && __any_sync(0xffffffffu, tmax >= (1ull << 26)) && lane == 0) misc->big = 1;
    if (NF > 0 && __any_sync(0xffffffffu, emax == 0x7FF00000u) && lane == 0) misc->nonfinite = 1;
    __syncwarp();
    // A3: one draw word per pass over the warp's queue, compacted in place to the rows still owing
    for (int word = 1; qn > 0; ++word) {
      int nq = 0;
      for (int qb = 0; qb < qn; qb += 32) {
        const int qi = qb + lane;
        bool pend = false;
        int pos = 0, km = 0;
        uint64_t w = 0;
        if (qi < qn) {
          w = qw[qi];
          pos = qpos[qi];
          km = qk[qi];
          const bool maj = (km & 128) != 0;
          int k = km & 127;
          const uint64_t lo = smask[pos], hi = smask[TS + pos];
          uint64_t c0 = maj ? lo : ~lo, c1 = maj ? hi : ~hi;
          pac_hash128_step(word, w, c0, c1, k);
          smask[pos] = maj ? c0 : ~c0;
          smask[TS + pos] = maj ? c1 : ~c1;
          pend = k > 0;
          km = k | (km & 128);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, pend);  // entries of this pass all read
        if (pend) {
          const int q = nq + __popc(pm & lt_mask);  // q <= qi: never an entry not yet read
          qw[q] = w;
          qpos[q] = (unsigned short)pos;
          qk[q] = (unsigned short)km;
        }
        nq += __popc(pm);
      }
      qn = nq;
      __syncwarp();
    }
  };

  if (tid == 0) {
    mbar_init(mbar, 1);
    if (staged_tile(t0)) issue_tile(p, raw, mbar, t0 * T, T);
  }
  __syncthreads();
  WarpAcc<NI, NF, 0> alo, ahi;
  alo.cur = ahi.cur = -1;
  alo.reset();
  ahi.reset();
  if (t0 < t1) {
    if (staged_tile(t0)) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
      a1(BoolTag<true>{}, t0 * T, T);
    } else {
      a1(BoolTag<false>{}, t0 * T, tile_rows(t0));
    }
  }
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t base = tile * T;
    __syncthreads();  // A1(tile) and C(tile - 1) complete
    // ---------------- B: slot offsets (8-row padded), runs, padding rows; lane = slot
    if (wid == 0) {
      const int h = lane < Lcap ? hist[lane] : 0;
      const int h8 = (h + 7) & ~7, hr = (h + 31) >> 5;
      int hx = h8, rx = hr;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, hx, d);
        const int b = __shfl_up_sync(0xffffffffu, rx, d);
        if (lane >= d) {
          hx += a;
          rx += b;
        }
      }
      if (lane == 31) {
        misc->nruns = rx;
        misc->big = 0;
        misc->nonfinite = 0;
      }
      hx -= h8;
      rx -= hr;
      if (lane < Lcap) {
        cursor[lane] = hx;
        lrows[lane] += (unsigned long long)h;
        hist[lane] = 0;
        for (int q = hx + h; q < hx + h8; ++q) {  // zero padding rows (mask 0, finite values)
          smask[q] = 0;
          smask[TS + q] = 0;
#pragma unroll
          for (int c = 0; c < NI; ++c) sival[c * TS + q] = 0;
#pragma unroll
          for (int c = 0; c < NF; ++c) sfval[c * TS + q] = 0.0;
        }
        for (int i = 0; 32 * i < h; ++i) rdesc[rx + i] = pack_run(hx + 32 * i, lane, min(32, h - 32 * i));
      }
    }
    __syncthreads();
    // ---------------- A2 + A3
    const bool staged = staged_tile(tile);
    if (staged) a2(BoolTag<true>{}, base);
    else a2(BoolTag<false>{}, base);
    __syncthreads();
    // the raw tile buffer is free: stage the next tile while phase C runs
    const bool next_staged = staged_tile(tile + 1);
    if (tid == 0 && next_staged) issue_tile(p, raw, mbar, (tile + 1) * T, T);
    // ---------------- C: runs of the low and of the high mask words
    {
      const int R = misc->nruns;
      const bool small = (NI == 0) || misc->big == 0;
      const bool fin = (NF == 0) || misc->nonfinite == 0;
      const int r0 = (R * wid) / nw, r1 = (R * (wid + 1)) / nw;
#pragma unroll 1
      for (int r = r0; r < r1; ++r) {
        const uint32_t d = rdesc[r];
        const int beg = (int)(d & 0xFFFFu);
        const int s = (int)((d >> 16) & 0x3FFu);
        const int len = (int)(d >> 26) + 1;
        if (2 * s != alo.cur) {
          alo.flush(cnt, isum, fsum, nullptr, nullptr, V, lane);
          ahi.flush(cnt, isum, fsum, nullptr, nullptr, V, lane);
          alo.cur = 2 * s;
          ahi.cur = 2 * s + 1;
        }
        const XposeConst xc = load_xpose(xcs, xcs2, lane);
        if (small && fin)
          run_body128<NI, NF, false>(alo, ahi, smask + beg, smask + TS + beg, sival + beg, TS, sfval + beg, TS, len,
                                     xc, lane);
        else
          run_body128<NI, NF, true>(alo, ahi, smask + beg, smask + TS + beg, sival + beg, TS, sfval + beg, TS, len,
                                    xc, lane, small, fin);
      }
    }
    // ---------------- A1 of the next tile (touches only the dictionary, sslot and hist)
    if (tile + 1 < t1) {
      if (next_staged) {
        mbar_wait(mbar, phase);
        phase ^= 1u;
        a1(BoolTag<true>{}, base + T, T);
      } else {
        a1(BoolTag<false>{}, base + T, tile_rows(tile + 1));
      }
    }
  }
  __syncthreads();
  alo.flush(cnt, isum, fsum, nullptr, nullptr, V, lane);
  ahi.flush(cnt, isum, fsum, nullptr, nullptr, V, lane);
  __syncthreads();

  // ---------------- CTA table -> provisional HBM table [G_cap][128] (entry i = slot i / 128)
  const int nloc = min(misc->nlocal, Lcap);
  for (int i = tid; i < nloc * 2 * kM; i += nth) {
    const int prov = lprov[i / (2 * kM)];
    if (prov < 0) continue;
    const size_t g = (size_t)prov * 2 * kM + (i % (2 * kM));
    if (cnt[i]) atomicAdd(&p.prov_count[g], (unsigned long long)cnt[i]);
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      const unsigned long long v = isum[(size_t)c * V * kM + i];
      if (v) atomicAdd(&p.prov_isum[c][g], v);
    }
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      const double v = fsum[(size_t)c * V * kM + i];
      if (v != 0.0) atomicAdd(&p.prov_fsum[c][g], v);
    }
  }
  for (int s = tid; s < nloc; s += nth)
    if (lprov[s] >= 0 && lrows[s]) atomicAdd(&p.prov_rows[lprov[s]], lrows[s]);
  if (NI > 0) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, maxabs, d);
      maxabs = o > maxabs ? o : maxabs;
    }
    if (lane == 0 && maxabs) atomicMax(p.gmaxabs, maxabs);
  }
}

template <int NI, int NF>
static cudaError_t launch128(const AggPlan& p, const Lay128& L, int sms, cudaStream_t st) {
  auto k = k_agg_tiles128<NI, NF>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads128, L.bytes);
  per_sm = std::max(1, per_sm);
  const int64_t tiles = (p.n_rows + L.T - 1) / L.T;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * per_sm));
  if (getenv("PAC_DEBUG"))
    fprintf(stderr, "[libpac] k_agg_tiles128<%d,%d> Lcap=%d smem=%d B, %d CTAs (%d per SM)\n", NI, NF, L.Lcap, L.bytes,
            grid, per_sm);
  k<<<grid, kThreads128, L.bytes, st>>>(p, L);
  note_launch();
  return cudaGetLastError();
}

using Launch128 = cudaError_t (*)(const AggPlan&, const Lay128&, int, cudaStream_t);
static const Launch128 kLaunch128[3][3] = {
    {launch128<0, 0>, launch128<0, 1>, launch128<0, 2>},
    {launch128<1, 0>, launch128<1, 1>, launch128<1, 2>},
    {launch128<2, 0>, launch128<2, 1>, launch128<2, 2>},
};

// shared-memory bytes of the kernel for ni int64 and nf f64 sum columns and Lcap = G_cap slots
// (raw_bytes: the staged tile, raw_tile128_bytes)
int tiles128_smem(int ni, int nf, int Lcap, int raw_bytes) { return lay128(ni, nf, kT128, Lcap, raw_bytes).bytes; }
int tiles128_rows() { return kT128; }

cudaError_t launch_tiles128(const AggPlan& p, int Lcap, int sms, cudaStream_t st) {
  const Lay128 L = lay128(p.ni, p.nf, kT128, Lcap, p.raw_bytes);
  return kLaunch128[p.ni][p.nf](p, L, sms, st);
}

}  // namespace pac
