// libpac: k_agg_warp -- the low-cardinality grouped 64-world aggregation.
//
// For tables of at most kWarpSlots groups (the paper's Q01-shaped queries; BASELINE
// configs C1/C2) every warp runs the whole path on its own contiguous row range, with no
// CTA-wide barrier after the prologue:
//   chunk of 32 rows (lane = row, loads of the next chunk in flight):
//     group key -> CTA-local slot (lock-free smem dictionary in front of the HBM dictionary),
//     pac_hash word 0 (R1, R2); rows that need more draws go to the warp's straggler queue,
//     finished rows are appended to the warp's per-slot buffer (16 lanes at a time);
//   a slot buffer holding 32 rows is one full run: world-parallel update (run_body: bit
//     transpose, popc COUNT, "Four Russians" subset-sum tables for SUM/AVG, MIN/MAX) into
//     the warp's register accumulators, flushed into the CTA's smem table on slot change;
//   the straggler queue is finished 32 rows at a time (draw words 1.., R2) and appended;
//   the end: queue and partial runs drained, CTA table -> provisional HBM table.
// Compared with k_agg_tiles this removes the tile-wide counting sort and its eight barriers
// per tile, and every run is a full 32-row run except one partial run per slot and warp.
#pragma once
#include "agg_tiles.cuh"

namespace pac {

constexpr int kWarpSlots = 8;     // max local slots of k_agg_warp
constexpr int kWarpCap = 48;      // rows per slot buffer: <= 31 left + 16 appended
constexpr int kWarpQueue = 64;    // straggler queue: <= 31 left + 32 appended
constexpr int kWarpThreads = 256;

struct WarpLayout {
  int Lw, LH, nw;
  // CTA-shared
  int o_lkey, o_lstate, o_lprov, o_lrows, o_cnt, o_isum, o_fsum, o_min, o_max, o_misc;
  // per warp (offset of warp 0; warp w at + w * warp_bytes)
  int o_warp, warp_bytes;
  int w_mask, w_ival, w_fval, w_mval, w_cnt, w_qw0, w_qm, w_qslot, w_qival, w_qfval, w_qmval;
  int bytes;
};

template <int NI, int NF, int MM>
struct WarpBufs {
  unsigned long long* mask;  // [Lw][kWarpCap]
  long long* ival;           // [NI][Lw][kWarpCap]
  double* fval;              // [NF][Lw][kWarpCap]
  double* mval;              // [Lw][kWarpCap]
  int* cnt;                  // [Lw]
  unsigned long long* qw0;   // [kWarpQueue] draw word 0 of a queued row
  unsigned long long* qm;    // [kWarpQueue] its mask after word 0
  int* qslot;                // [kWarpQueue]
  long long* qival;          // [NI][kWarpQueue]
  double* qfval;             // [NF][kWarpQueue]
  double* qmval;             // [kWarpQueue]
};

// One row's inputs (lane = row), loaded a chunk ahead.
template <int NI, int NF, int MM>
struct RowIn {
  uint64_t key;  // pu_key or explicit mask
  uint64_t gkey;
  long long iv[NI > 0 ? NI : 1];
  double fv[NF > 0 ? NF : 1];
  double mv;
};

template <int NI, int NF, int MM>
__device__ __forceinline__ void load_row(const AggPlan& p, int64_t r, RowIn<NI, NF, MM>& x) {
  if (r < p.n_rows) {
    x.key = (uint64_t)__ldcs((const long long*)p.raw_src[0] + r);
    x.gkey = row_group_key(p, r);
#pragma unroll
    for (int c = 0; c < NI; ++c) x.iv[c] = __ldcs(p.icol[c] + r);
#pragma unroll
    for (int c = 0; c < NF; ++c) x.fv[c] = __ldcs(p.fcol[c] + r);
    x.mv = MM ? __ldcs(p.mcol + r) : 0.0;
  } else {
    x.key = 0;
    x.gkey = 0;
#pragma unroll
    for (int c = 0; c < NI; ++c) x.iv[c] = 0;
#pragma unroll
    for (int c = 0; c < NF; ++c) x.fv[c] = 0.0;
    x.mv = 0.0;
  }
}

template <int NI, int NF, int MM>
struct WarpCtx {
  const AggPlan* p;
  WarpBufs<NI, NF, MM> b;
  WarpAcc<NI, NF, MM> acc;
  XposeConst xc;
  unsigned* cnt;
  unsigned long long* isum;
  double* fsum;
  long long* emin;
  long long* emax;
  unsigned* lrows;
  int Lw, lane;

  // World-parallel update of the first `len` rows of slot s's buffer.
  __device__ __noinline__ void run(int s, int len) {
    if (s != acc.cur) {
      acc.flush(cnt, isum, fsum, emin, emax, Lw, lane);
      acc.cur = s;
    }
    bool big = false, nonfin = false;
    if (lane < len) {
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        const long long v = b.ival[(c * Lw + s) * kWarpCap + lane];
        big |= (unsigned long long)(v + (1ll << 26)) >= (1ull << 27);
      }
#pragma unroll
      for (int c = 0; c < NF; ++c) nonfin |= !finite_bits(b.fval[(c * Lw + s) * kWarpCap + lane]);
    }
    const bool small = NI == 0 || !__any_sync(0xffffffffu, big);
    const bool fin = NF == 0 || !__any_sync(0xffffffffu, nonfin);
    const unsigned long long* m = b.mask + s * kWarpCap;
    const long long* iv = b.ival + s * kWarpCap;
    const double* fv = b.fval + s * kWarpCap;
    const double* mv = b.mval + s * kWarpCap;
    const int is = Lw * kWarpCap;
    if (small && fin) run_body<NI, NF, MM, false>(acc, m, iv, is, fv, is, mv, len, xc, lane);
    else run_body<NI, NF, MM, true>(acc, m, iv, is, fv, is, mv, len, xc, lane, small, fin);
  }

  // Every slot buffer holding >= 32 rows: run its first 32 rows, move the rest to the front.
  __device__ __forceinline__ void drain_full() {
    const int c = lane < Lw ? b.cnt[lane] : 0;
    unsigned full = __ballot_sync(0xffffffffu, c >= 32);
    while (full) {
      const int s = __ffs(full) - 1;
      full &= full - 1;
      run(s, 32);
      const int rest = __shfl_sync(0xffffffffu, c, s) - 32;
      unsigned long long mk = 0;
      long long iv[NI > 0 ? NI : 1];
      double fv[NF > 0 ? NF : 1];
      double mv = 0.0;
      if (lane < rest) {
        mk = b.mask[s * kWarpCap + 32 + lane];
#pragma unroll
        for (int k = 0; k < NI; ++k) iv[k] = b.ival[(k * Lw + s) * kWarpCap + 32 + lane];
#pragma unroll
        for (int k = 0; k < NF; ++k) fv[k] = b.fval[(k * Lw + s) * kWarpCap + 32 + lane];
        if (MM) mv = b.mval[s * kWarpCap + 32 + lane];
      }
      __syncwarp();
      if (lane < rest) {
        b.mask[s * kWarpCap + lane] = mk;
#pragma unroll
        for (int k = 0; k < NI; ++k) b.ival[(k * Lw + s) * kWarpCap + lane] = iv[k];
#pragma unroll
        for (int k = 0; k < NF; ++k) b.fval[(k * Lw + s) * kWarpCap + lane] = fv[k];
        if (MM) b.mval[s * kWarpCap + lane] = mv;
      }
      if (lane == 0) b.cnt[s] = rest;
      __syncwarp();
    }
  }

  // Append the rows of the lanes with `v` (slot s, mask m, values) to the slot buffers, 16
  // lanes at a time so a buffer never holds more than 31 + 16 rows.
  __device__ __forceinline__ void append(bool v, int s, uint64_t m, const long long (&iv)[NI > 0 ? NI : 1],
                                         const double (&fv)[NF > 0 ? NF : 1], double mv) {
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool on = v && (lane >> 4) == h;
      if (!__any_sync(0xffffffffu, on)) continue;
      const unsigned peers = __match_any_sync(0xffffffffu, on ? (unsigned)s : 0x10000u + lane);
      int base = 0, rank = 0;
      if (on) {
        rank = __popc(peers & lt);
        base = b.cnt[s];
        const int pos = s * kWarpCap + base + rank;
        b.mask[pos] = m;
#pragma unroll
        for (int k = 0; k < NI; ++k) b.ival[k * Lw * kWarpCap + pos] = iv[k];
#pragma unroll
        for (int k = 0; k < NF; ++k) b.fval[k * Lw * kWarpCap + pos] = fv[k];
        if (MM) b.mval[pos] = mv;
      }
      __syncwarp();
      if (on && rank == 0) {
        b.cnt[s] = base + __popc(peers);
        atomicAdd(&lrows[s], (unsigned)__popc(peers));
      }
      __syncwarp();
      drain_full();
    }
  }

  // Finish the first `n` (<= 32) queued masks (draw words 1.., R2) and append those rows.
  __device__ __forceinline__ void finish_queue(int& qn, int n) {
    const bool on = lane < n;
    uint64_t m = 0;
    int s = 0;
    long long iv[NI > 0 ? NI : 1];
    double fv[NF > 0 ? NF : 1];
    double mv = 0.0;
#pragma unroll
    for (int k = 0; k < NI; ++k) iv[k] = 0;
#pragma unroll
    for (int k = 0; k < NF; ++k) fv[k] = 0.0;
    if (on) {
      m = pac_hash_continue(b.qm[lane], b.qw0[lane]);
      s = b.qslot[lane];
#pragma unroll
      for (int k = 0; k < NI; ++k) iv[k] = b.qival[k * kWarpQueue + lane];
#pragma unroll
      for (int k = 0; k < NF; ++k) fv[k] = b.qfval[k * kWarpQueue + lane];
      if (MM) mv = b.qmval[lane];
    }
    // move the entries behind them to the front of the queue
    const int rest = qn - n;
    const bool mv_on = lane < rest;
    unsigned long long w0 = 0, qm = 0;
    int qs = 0;
    long long qiv[NI > 0 ? NI : 1];
    double qfv[NF > 0 ? NF : 1];
    double qmv = 0.0;
    if (mv_on) {
      w0 = b.qw0[n + lane];
      qm = b.qm[n + lane];
      qs = b.qslot[n + lane];
#pragma unroll
      for (int k = 0; k < NI; ++k) qiv[k] = b.qival[k * kWarpQueue + n + lane];
#pragma unroll
      for (int k = 0; k < NF; ++k) qfv[k] = b.qfval[k * kWarpQueue + n + lane];
      if (MM) qmv = b.qmval[n + lane];
    }
    __syncwarp();
    if (mv_on) {
      b.qw0[lane] = w0;
      b.qm[lane] = qm;
      b.qslot[lane] = qs;
#pragma unroll
      for (int k = 0; k < NI; ++k) b.qival[k * kWarpQueue + lane] = qiv[k];
#pragma unroll
      for (int k = 0; k < NF; ++k) b.qfval[k * kWarpQueue + lane] = qfv[k];
      if (MM) b.qmval[lane] = qmv;
    }
    __syncwarp();
    qn = rest;
    append(on, s, m, iv, fv, mv);
  }
};

template <int NI, int NF, int MM>
__global__ void __launch_bounds__(kWarpThreads, 2) k_agg_warp(AggPlan p, WarpLayout L) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  const int Lw = L.Lw, LH = L.LH;
  unsigned long long* lkey = (unsigned long long*)(smem + L.o_lkey);
  int* lstate = (int*)(smem + L.o_lstate);
  int* lprov = (int*)(smem + L.o_lprov);
  unsigned* lrows = (unsigned*)(smem + L.o_lrows);
  unsigned* cnt = (unsigned*)(smem + L.o_cnt);
  unsigned long long* isum = (unsigned long long*)(smem + L.o_isum);
  double* fsum = (double*)(smem + L.o_fsum);
  long long* emin = (long long*)(smem + L.o_min);
  long long* emax = (long long*)(smem + L.o_max);
  Misc* misc = (Misc*)(smem + L.o_misc);

  for (int i = tid; i < LH; i += nth) lstate[i] = 0;
  for (int i = tid; i < Lw; i += nth) lrows[i] = 0;
  for (int i = tid; i < Lw * kM; i += nth) {
    cnt[i] = 0;
#pragma unroll
    for (int c = 0; c < NI; ++c) isum[c * Lw * kM + i] = 0;
#pragma unroll
    for (int c = 0; c < NF; ++c) fsum[c * Lw * kM + i] = 0.0;
    if (MM & 1) emin[i] = kEncPosInf;
    if (MM & 2) emax[i] = kEncNegInf;
  }
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }

  WarpCtx<NI, NF, MM> w;
  {
    unsigned char* wb = smem + L.o_warp + wid * L.warp_bytes;
    w.b.mask = (unsigned long long*)(wb + L.w_mask);
    w.b.ival = (long long*)(wb + L.w_ival);
    w.b.fval = (double*)(wb + L.w_fval);
    w.b.mval = (double*)(wb + L.w_mval);
    w.b.cnt = (int*)(wb + L.w_cnt);
    w.b.qw0 = (unsigned long long*)(wb + L.w_qw0);
    w.b.qm = (unsigned long long*)(wb + L.w_qm);
    w.b.qslot = (int*)(wb + L.w_qslot);
    w.b.qival = (long long*)(wb + L.w_qival);
    w.b.qfval = (double*)(wb + L.w_qfval);
    w.b.qmval = (double*)(wb + L.w_qmval);
    if (lane < Lw) w.b.cnt[lane] = 0;
  }
  w.p = &p;
  w.cnt = cnt;
  w.isum = isum;
  w.fsum = fsum;
  w.emin = emin;
  w.emax = emax;
  w.lrows = lrows;
  w.Lw = Lw;
  w.lane = lane;
  w.acc.cur = -1;
  w.acc.reset();
  w.xc = make_xpose(lane);
  __syncthreads();

  // contiguous chunk range of this warp
  const int64_t nchunks = (p.n_rows + 31) >> 5;
  const int64_t gw = (int64_t)blockIdx.x * nw + wid, GW = (int64_t)gridDim.x * nw;
  const int64_t per = (nchunks + GW - 1) / GW;
  const int64_t c0 = gw * per, c1 = min(nchunks, c0 + per);
  unsigned long long maxabs = 0;
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;

  RowIn<NI, NF, MM> cur, nxt;
  if (c0 < c1) load_row(p, c0 * 32 + lane, cur);
#pragma unroll 1
  for (int64_t ch = c0; ch < c1; ++ch) {
    const int64_t row = ch * 32 + lane;
    if (ch + 1 < c1) load_row(p, row + 32, nxt);
    const bool valid = row < p.n_rows;
    // ---- mask: word 0 of pac_hash for every lane (uniform), or the explicit mask
    uint64_t m;
    HashState h;
    if (p.mask_in) {
      m = cur.key;
      h.k = 0;
      h.w0 = 0;
    } else {
      h = pac_hash_begin(cur.key, p.salt);
      m = hash_mask_now(h);
    }
    // ---- group slot (R21: a row in no world is dropped)
    int s = -1;
    if (valid && m != 0ull) {
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        const unsigned long long a = cur.iv[c] < 0 ? 0ull - (unsigned long long)cur.iv[c] : (unsigned long long)cur.iv[c];
        maxabs = a > maxabs ? a : maxabs;
      }
      const int code = local_code(p, cur.gkey, lkey, lstate, LH, lprov, Lw, misc);
      if (code < kOvfBase) {
        s = code - 1;
      } else {  // no local slot: straight to the HBM table (rare)
        const uint64_t mf = h.k > 0 ? pac_hash_continue(m, h.w0) : m;
        global_row_update<NI, NF, MM>(p, code - kOvfBase - 1, mf, cur.iv, cur.fv, cur.mv);
      }
    }
    // ---- rows that need more draws -> straggler queue
    const bool pend = s >= 0 && h.k > 0;
    const unsigned pm = __ballot_sync(0xffffffffu, pend);
    if (pm) {
      if (pend) {
        const int q = qn + __popc(pm & lt);
        w.b.qw0[q] = h.w0;
        w.b.qm[q] = m;
        w.b.qslot[q] = s;
#pragma unroll
        for (int k = 0; k < NI; ++k) w.b.qival[k * kWarpQueue + q] = cur.iv[k];
#pragma unroll
        for (int k = 0; k < NF; ++k) w.b.qfval[k * kWarpQueue + q] = cur.fv[k];
        if (MM) w.b.qmval[q] = cur.mv;
      }
      qn += __popc(pm);
      __syncwarp();
    }
    // ---- finished rows -> slot buffers (full runs are processed as they fill)
    w.append(s >= 0 && !pend, s, m, cur.iv, cur.fv, cur.mv);
    if (qn >= 32) w.finish_queue(qn, 32);
    cur = nxt;
  }
  // ---- drain: the straggler queue, then one partial run per non-empty slot buffer
  while (qn > 0) w.finish_queue(qn, min(qn, 32));
  for (int s = 0; s < Lw; ++s) {
    const int c = w.b.cnt[s];
    if (c == 0) continue;
    // zero padding up to the next multiple of 8 rows (finite table entries, R16)
    if (lane >= c && lane < ((c + 7) & ~7)) {
      w.b.mask[s * kWarpCap + lane] = 0;
#pragma unroll
      for (int k = 0; k < NI; ++k) w.b.ival[(k * Lw + s) * kWarpCap + lane] = 0;
#pragma unroll
      for (int k = 0; k < NF; ++k) w.b.fval[(k * Lw + s) * kWarpCap + lane] = 0.0;
      if (MM) w.b.mval[s * kWarpCap + lane] = 0.0;
    }
    __syncwarp();
    w.run(s, c);
  }
  w.acc.flush(cnt, isum, fsum, emin, emax, Lw, lane);
  __syncthreads();

  // ---------------- CTA table -> provisional HBM table
  const int nloc = min(misc->nlocal, Lw);
  if (tid == 0) atomicMax(&p.dbg[1], (unsigned long long)misc->nlocal);
  for (int i = tid; i < nloc * kM; i += nth) {
    const int s = i / kM;
    const int prov = lprov[s];
    if (prov < 0) continue;
    const size_t g = (size_t)prov * kM + (i % kM);
    if (cnt[i]) atomicAdd(&p.prov_count[g], (unsigned long long)cnt[i]);
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      const unsigned long long v = isum[c * Lw * kM + i];
      if (v) atomicAdd(&p.prov_isum[c][g], v);
    }
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      const double v = fsum[c * Lw * kM + i];
      if (v != 0.0) atomicAdd(&p.prov_fsum[c][g], v);
    }
    if (MM & 1) atomicMin(&p.prov_min[g], emin[i]);
    if (MM & 2) atomicMax(&p.prov_max[g], emax[i]);
  }
  for (int s = tid; s < nloc; s += nth)
    if (lprov[s] >= 0 && lrows[s]) atomicAdd(&p.prov_rows[lprov[s]], (unsigned long long)lrows[s]);
  if (NI > 0) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, maxabs, d);
      maxabs = o > maxabs ? o : maxabs;
    }
    if (lane == 0 && maxabs) atomicMax(p.gmaxabs, maxabs);
  }
}

template <int NI, int NF, int MM>
cudaError_t launch_warp(const AggPlan& p, const WarpLayout& L, int sms, cudaStream_t st) {
  auto k = k_agg_warp<NI, NF, MM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kWarpThreads, L.bytes);
  per_sm = std::max(1, per_sm);
  const int64_t chunks = (p.n_rows + 31) / 32;
  const int64_t want = (chunks + (kWarpThreads / 32) * 4 - 1) / ((kWarpThreads / 32) * 4);  // >= 4 chunks per warp
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * per_sm));
  if (getenv("PAC_DEBUG"))
    fprintf(stderr, "[libpac] k_agg_warp<%d,%d,%d> %d CTAs x %d threads (%d per SM), Lw=%d smem=%d B\n", NI, NF,
            MM, grid, kWarpThreads, per_sm, L.Lw, L.bytes);
  k<<<grid, kWarpThreads, L.bytes, st>>>(p, L);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pac
