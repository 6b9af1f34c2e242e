// libpac: k_agg_ws -- the warp-specialized grouped aggregation kernel for tables
// whose groups all fit the CTA's local slots (BASELINE C1, C2, C5).  One CTA of kWsWarps warps per
// SM and no CTA-wide barrier in the steady state.  Every warp plays both roles:
//
//   hashing   its own 64-row chunks (two rows per lane, read from HBM with the chunk kWsAhead
//             rounds ahead prefetched into L2 by a bulk prefetch): group key -> local slot (CTA
//             dictionary), pac_hash word 0 (R1, R2; two interleaved chains per lane); a finished
//             row is appended to its slot's run buffer; rows still needing draw words (~16 %) wait
//             in the warp's queue and are finished 32 at a time with every lane busy;
//   consuming the run buffers it owns: a buffer holding a full 32-row run is bit-transposed and
//             aggregated with the "Four Russians" tables of run_body, added into the buffer's
//             accumulators in Tensor Memory (the owner's lane quarter, tcgen05.ld/st) and
//             released.  Between chunks a warp services its buffers.
//
// Run buffers: slot s has NB buffers of 32 rows (mask, then the value columns, each 32 x 8 B).
// Row position pos = atomicAdd(fill[s]) goes to buffer (pos/32) % NB, generation (pos/32)/NB.
// A row is written once its buffer's generation counter shows the previous run in that buffer was
// consumed (else the reserved position is kept in the warp's short pending list and retried when
// the warp next services -- no lane ever waits, so no warp can wait on another that waits on it);
// the writer then bumps the buffer's row count, and the owner processes the buffer when the count
// reaches 32, resets it and advances the generation.  Rows reach a run in any order (integer sums
// are exact in any order, f64 sums within R16).  Every run but the last one per buffer is a full
// 32-row run: the per-run fixed costs (transpose, TMEM add) are paid once per 32 rows whatever the
// number of groups, and no tile-wide sort exists.
#pragma once
#include "agg_tiles.cuh"
#include "agg_tm.cuh"

namespace pac {

constexpr int kWsChunk = 64;                    // rows per chunk (two rows per lane)
constexpr int kWsWarps = 16;                    // 4 per TMEM lane quarter
constexpr int kWsThreads = 32 * kWsWarps;
constexpr int kWsQueue = 64;                    // straggler entries per warp
constexpr int kWsPend = 8;                      // deferred writes per warp
constexpr int kWsCols = kTmCols / (kWsWarps / 4);  // TMEM columns per warp (128)
constexpr int kWsAhead = 2;                     // L2 prefetch distance, in rounds of kWsWarps chunks

struct WskLayout {
  int Lcap, LH, NB, lognb;
  int logr;    // accumulator units: buffer b of slot s adds into unit s * R + (b % R), R = 2^logr <= NB
  int mine;    // buffers per warp: warp w owns units w, w + kWsWarps, ... and each unit's NB / R buffers
  int nv;      // staged 8-byte value columns (NI + NF + (MM ? 1 : 0))
  int npairs;  // Lcap * NB run buffers
  int o_buf, o_qm, o_qw, o_qs, o_qv, o_pm, o_pp, o_ps, o_pf, o_pv, o_fill, o_cnt, o_gen, o_flag, o_ready, o_lkey,
      o_lstate, o_lprov, o_misc, o_xcs;
  int bytes;
};

struct WsMisc {
  Misc m;            // nlocal / ndict of the dictionary (local_code)
  int done;          // warps finished with their chunks
  int pending;       // deferred writes outstanding in the CTA
  int next;          // next chunk (dynamic assignment)
  int pad;
};

__device__ __forceinline__ int ld_vol(const int* a) { return *(const volatile int*)a; }

struct WsSmem {
  unsigned char* buf;      // [npairs][32 * 8 * (1 + nv)]
  unsigned long long* qm;  // [warps][kWsQueue] straggler partial masks
  unsigned long long* qw;  // draw word 0
  int* qs;                 // slot
  unsigned long long* qv;  // [warps][nv][kWsQueue] value words
  unsigned long long* pm;  // [warps][kWsPend] deferred: final mask
  int* pp;                 // reserved position
  int* ps;                 // slot
  int* pf;                 // value flags
  unsigned long long* pv;  // [warps][nv][kWsPend]
  int* fill;               // [Lcap]
  int* cnt;                // [npairs]
  int* gen;                // [npairs]
  int* flag;               // [npairs] bit 0: some |int64| >= 2^26, bit 1: some f64 non-finite
  unsigned* ready;         // [warps] bit i: the warp's i-th buffer holds a full run
  unsigned long long* lkey;
  int* lstate;
  int* lprov;
  WsMisc* misc;
  uint4* xcs;
  uint2* xcs2;
};

__device__ __forceinline__ WsSmem ws_smem(unsigned char* smem, const WskLayout& L) {
  WsSmem s;
  s.buf = smem + L.o_buf;
  s.qm = (unsigned long long*)(smem + L.o_qm);
  s.qw = (unsigned long long*)(smem + L.o_qw);
  s.qs = (int*)(smem + L.o_qs);
  s.qv = (unsigned long long*)(smem + L.o_qv);
  s.pm = (unsigned long long*)(smem + L.o_pm);
  s.pp = (int*)(smem + L.o_pp);
  s.ps = (int*)(smem + L.o_ps);
  s.pf = (int*)(smem + L.o_pf);
  s.pv = (unsigned long long*)(smem + L.o_pv);
  s.fill = (int*)(smem + L.o_fill);
  s.cnt = (int*)(smem + L.o_cnt);
  s.gen = (int*)(smem + L.o_gen);
  s.flag = (int*)(smem + L.o_flag);
  s.ready = (unsigned*)(smem + L.o_ready);
  s.lkey = (unsigned long long*)(smem + L.o_lkey);
  s.lstate = (int*)(smem + L.o_lstate);
  s.lprov = (int*)(smem + L.o_lprov);
  s.misc = (WsMisc*)(smem + L.o_misc);
  s.xcs = (uint4*)(smem + L.o_xcs);
  s.xcs2 = (uint2*)(smem + L.o_xcs + 32 * 16);
  return s;
}

// flags of a row's staged value words (int64 / f64 bits) and the running max |int64|
template <int NI, int NF>
__device__ __forceinline__ int ws_row_flags(const unsigned long long* v, unsigned long long& maxabs) {
  int f = 0;
#pragma unroll
  for (int c = 0; c < NI; ++c) {
    const long long x = (long long)v[c];
    const unsigned long long a = x < 0 ? 0ull - (unsigned long long)x : (unsigned long long)x;
    maxabs = a > maxabs ? a : maxabs;
    if (a >= (1ull << 26)) f |= 1;
  }
#pragma unroll
  for (int c = 0; c < NF; ++c)
    if ((__double2hiint(__longlong_as_double((long long)v[NI + c])) & 0x7FF00000) == 0x7FF00000) f |= 2;
  return f;
}

// Ownership.  Unit u = s * R + r (r < R) accumulates buffers s * NB + r + R * j (j < NB / R); warp w
// owns units w, w + kWsWarps, ..., the k-th of them at TMEM column (w / 4) * kWsCols + k * wps of lane
// quarter w % 4.  The warp's i-th buffer: k = i / (NB / R), j = i % (NB / R).
__device__ __forceinline__ uint32_t ws_tmine(uint32_t tbase, int wid) {
  return tbase + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((wid >> 2) * kWsCols);
}
__device__ __forceinline__ int ws_my_pair(const WskLayout& L, int wid, int i, int& k) {
  const int per = L.lognb - L.logr;  // log2(NB / R)
  k = i >> per;
  const int j = i & ((1 << per) - 1);
  const int u = wid + kWsWarps * k;
  return ((u >> L.logr) << L.lognb) + (u & ((1 << L.logr) - 1)) + (j << L.logr);
}
// owner warp of a buffer and the buffer's index i in the owner's enumeration
__device__ __forceinline__ int ws_owner(const WskLayout& L, int pair, int& i) {
  const int b = pair & (L.NB - 1);
  const int u = ((pair >> L.lognb) << L.logr) + (b & ((1 << L.logr) - 1));
  i = ((u / kWsWarps) << (L.lognb - L.logr)) + (b >> L.logr);
  return u % kWsWarps;
}

// Writes a row at its reserved position `pos` of slot s if the buffer is free for that generation;
// false (nothing written) otherwise.  The calling lane alone.
template <int NI, int NF, int MM>
__device__ __forceinline__ bool ws_try_write(const WsSmem& sm, const WskLayout& L, int s, int pos, uint64_t mask,
                                             const unsigned long long* v, int f) {
  constexpr int NV = NI + NF + (MM ? 1 : 0);
  const int run = pos >> 5;
  const int pair = s * L.NB + (run & (L.NB - 1));
  // the owner released the buffer (generation) after its reads: these writes depend on that load
  if (ld_vol(&sm.gen[pair]) != (run >> L.lognb)) return false;
  unsigned long long* b = (unsigned long long*)(sm.buf + (size_t)pair * (32 * 8 * (1 + NV)));
  const int i = pos & 31;
  b[i] = mask;
#pragma unroll
  for (int c = 0; c < NV; ++c) b[32 * (1 + c) + i] = v[c];
  if (f) atomicOr(&sm.flag[pair], f);
  asm volatile("fence.acq_rel.cta;" ::: "memory");
  if (atomicAdd(&sm.cnt[pair], 1) == 31) {  // the run is full: tell its owner
    int idx;
    const int owner = ws_owner(L, pair, idx);
    atomicOr(&sm.ready[owner], 1u << idx);
  }
  return true;
}

template <int NI, int NF, int MM>
__device__ void ws_service(const WsSmem& sm, const WskLayout& L, uint32_t tmine, const XposeConst& xc,
                                        int wid, int lane, int& pn);

// Appends the rows of the lanes with `want` (slot s, mask, values): reserve a position (lanes with
// the same slot share one atomic), write it, or keep it in the warp's pending list.  Warp-collective.
template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_append(const WsSmem& sm, const WskLayout& L, bool want, int s, uint64_t mask,
                                          const unsigned long long* v, int f, uint32_t tmine, const XposeConst& xc,
                                          int wid, int lane, int& pn) {
  constexpr int NV = NI + NF + (MM ? 1 : 0);
  int pos = 0;
  if (L.Lcap >= 32) {  // many slots: lanes rarely share one, one atomic per lane
    if (want) pos = atomicAdd(&sm.fill[s], 1);
  } else {  // few slots: lanes with the same slot share one atomic (consecutive positions)
    const unsigned peers = __match_any_sync(0xffffffffu, want ? s : -1);
    if (want) {
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(&sm.fill[s], __popc(peers));
      base = __shfl_sync(peers, base, leader);
      pos = base + __popc(peers & ((1u << lane) - 1u));
    }
  }
  bool def = want && !ws_try_write<NI, NF, MM>(sm, L, s, pos, mask, v, f);
  unsigned dm = __ballot_sync(0xffffffffu, def);
  if (!dm) return;
  // no room in the pending list: service (which may free the buffers) and retry these rows too --
  // their reserved positions may be what the pending entries are waiting for
  while (pn + __popc(dm) > kWsPend) {
    ws_service<NI, NF, MM>(sm, L, tmine, xc, wid, lane, pn);
    if (def) def = !ws_try_write<NI, NF, MM>(sm, L, s, pos, mask, v, f);
    dm = __ballot_sync(0xffffffffu, def);
  }
  if (!dm) return;
  if (def) {
    const int k = pn + __popc(dm & ((1u << lane) - 1u));
    const int e = wid * kWsPend + k;
    sm.pm[e] = mask;
    sm.pp[e] = pos;
    sm.ps[e] = s;
    sm.pf[e] = f;
#pragma unroll
    for (int c = 0; c < NV; ++c) sm.pv[((size_t)wid * NV + c) * kWsPend + k] = v[c];
  }
  pn += __popc(dm);
  if (lane == 0) atomicAdd(&sm.misc->pending, __popc(dm));
  __syncwarp();
}

// runs holding |int64| >= 2^26 or non-finite f64 values (rare): out of line, keeps the hot code small
template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_run_generic(WarpAcc<NI, NF, MM>& acc, const unsigned long long* b, const long long* iv,
                                            const double* fv, const long long* mv, int len, const XposeConst& xc,
                                            int lane, int f) {
  run_body<NI, NF, MM, true>(acc, b, iv, 32, fv, 32, mv, len, xc, lane, (f & 1) == 0, (f & 2) == 0);
}

// consume one run (len rows) of buffer `pair` into the TMEM columns at taddr, release the buffer
template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_consume(const WsSmem& sm, const WskLayout& L, int pair, int len, uint32_t taddr,
                                           const XposeConst& xc, int lane) {
  constexpr int NV = NI + NF + (MM ? 1 : 0);
  asm volatile("fence.acq_rel.cta;" ::: "memory");  // acquire: the count was read; now the rows
  const unsigned long long* b = (const unsigned long long*)(sm.buf + (size_t)pair * (32 * 8 * (1 + NV)));
  const int f = ld_vol(&sm.flag[pair]);
  WarpAcc<NI, NF, MM> acc;
  acc.cur = 0;
  acc.reset();
  const long long* iv = (const long long*)(b + 32);
  const double* fv = (const double*)(b + 32 * (1 + NI));
  const long long* mv = (const long long*)(b + 32 * (1 + NI + NF));
  if (f == 0)
    run_body<NI, NF, MM, false>(acc, b, iv, 32, fv, 32, mv, len, xc, lane);
  else
    ws_run_generic<NI, NF, MM>(acc, b, iv, fv, mv, len, xc, lane, f);
  tm_flush<NI, NF, MM>(acc, taddr);
  __syncwarp();
  if (lane == 0) {
    sm.flag[pair] = 0;
    sm.cnt[pair] = 0;
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    atomicAdd(&sm.gen[pair], 1);  // release: the next run may be written
  }
  __syncwarp();
}

// Retry the pending writes, then consume every full run of this warp's buffers (the writers that
// complete a run set its bit in the owner's ready word).
template <int NI, int NF, int MM>
__device__ void ws_service(const WsSmem& sm, const WskLayout& L, uint32_t tmine, const XposeConst& xc,
                                        int wid, int lane, int& pn) {
  constexpr int NV = NI + NF + (MM ? 1 : 0);
  using S = TmSlot<NI, NF, MM>;
  if (pn > 0) {
    bool ok = false;
    const int e = wid * kWsPend + lane;
    unsigned long long v[NV > 0 ? NV : 1];
    unsigned long long m = 0;
    int pp = 0, ps = 0, pf = 0;
    if (lane < pn) {
#pragma unroll
      for (int c = 0; c < NV; ++c) v[c] = sm.pv[((size_t)wid * NV + c) * kWsPend + lane];
      m = sm.pm[e];
      pp = sm.pp[e];
      ps = sm.ps[e];
      pf = sm.pf[e];
      ok = ws_try_write<NI, NF, MM>(sm, L, ps, pp, m, v, pf);
    }
    const unsigned okm = __ballot_sync(0xffffffffu, ok);
    // compact the entries still pending to the front
    const bool keep = lane < pn && !ok;
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      const int k = __popc(km & ((1u << lane) - 1u));
      const int d = wid * kWsPend + k;
      sm.pm[d] = m;
      sm.pp[d] = pp;
      sm.ps[d] = ps;
      sm.pf[d] = pf;
#pragma unroll
      for (int c = 0; c < NV; ++c) sm.pv[((size_t)wid * NV + c) * kWsPend + k] = v[c];
    }
    __syncwarp();
    pn = __popc(km);
    if (lane == 0 && okm) {
      asm volatile("fence.acq_rel.cta;" ::: "memory");
      atomicSub(&sm.misc->pending, __popc(okm));
    }
  }
  unsigned bal = 0u;
  if (lane == 0 && ld_vol((const int*)&sm.ready[wid]) != 0) bal = atomicExch(&sm.ready[wid], 0u);
  bal = __shfl_sync(0xffffffffu, bal, 0);
  while (bal) {
    const int i = __ffs(bal) - 1;
    bal &= bal - 1;
    int k;
    const int pr = ws_my_pair(L, wid, i, k);
    ws_consume<NI, NF, MM>(sm, L, pr, 32, tmine + (uint32_t)(k * S::wps), xc, lane);
  }
}

template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_tier_rows(const AggPlan& p, int64_t row, uint64_t key, int gprov, SpillCur& sc,
                                          int lane, unsigned gp);

// HBM tier for rows whose group has no local slot (gprov: HBM slot, -2 when the dictionary
// lookup was deferred): recorded for the k_spill_* kernels, or applied with device atomics when
// the records are full (as k_agg_tiles' tile_a1).  Reads the row's words from HBM.
template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_tier(const AggPlan& p, int64_t row, uint64_t key, int gprov, SpillCur& sc,
                                        int lane) {
  constexpr int kNoProv = INT_MIN;
  const unsigned gp = __ballot_sync(0xffffffffu, gprov != kNoProv);
  if (!gp) return;
  ws_tier_rows<NI, NF, MM>(p, row, key, gprov, sc, lane, gp);
}

template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_tier_rows(const AggPlan& p, int64_t row, uint64_t key, int gprov, SpillCur& sc,
                                          int lane, unsigned gp) {
  constexpr int kNoProv = INT_MIN;
  constexpr int NVAL = NI + NF + (MM ? 1 : 0);
  const unsigned lt_mask = (1u << lane) - 1u;
  auto w8 = [&](int k, int64_t r) { return (uint64_t)__ldg((const unsigned long long*)p.raw_src[k] + r); };
  sc.ntier += __popc(gp);
  if (p.sp_cap > 0) {
    const bool mine = gprov != kNoProv && gprov != -1;
    const unsigned sb = __ballot_sync(0xffffffffu, mine);
    const unsigned long long b0 = sb ? sc.take(p, __popc(sb), lane) : 0ull;
    const unsigned long long i = b0 + __popc(sb & lt_mask);
    if (b0 != ~0ull) {
      if (mine) {
        p.sp_prov[i] = gprov;
        p.sp_gkey[i] = key;
        p.sp_key[i] = w8(0, row);
#pragma unroll
        for (int c = 0; c < NVAL; ++c) p.sp_val[(size_t)c * p.sp_cap + i] = w8(1 + c, row);
      }
      gp = 0;
    }
  }
  uint64_t gm = 0;
  if (gp && gprov == -2) gprov = global_slot(p, key);
  if (gp && gprov != kNoProv) gm = p.mask_in ? w8(0, row) : pac_hash_dev(w8(0, row), p.salt);
  while (gp) {
    const int src = __ffs(gp) - 1;
    gp &= gp - 1;
    const int prov = __shfl_sync(0xffffffffu, gprov, src);
    const uint64_t m = __shfl_sync(0xffffffffu, gm, src);
    const int64_t rs = __shfl_sync(0xffffffffu, row, src);
    if (prov < 0) continue;  // capacity exhausted: reported by the finish kernel
    if (lane == 0) atomicAdd(&p.prov_rows[prov], 1ull);
    const size_t b = (size_t)prov * kM;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      if (!((m >> j) & 1ull)) continue;
      if (p.has_count) atomicAdd(&p.prov_count[b + j], 1ull);
#pragma unroll
      for (int c = 0; c < NI; ++c) atomicAdd(&p.prov_isum[c][b + j], (unsigned long long)w8(1 + c, rs));
#pragma unroll
      for (int c = 0; c < NF; ++c) atomicAdd(&p.prov_fsum[c][b + j], __longlong_as_double((long long)w8(1 + NI + c, rs)));
      if (MM & 1) atomicMin(&p.prov_min[b + j], enc_f64(__longlong_as_double((long long)w8(1 + NI + NF, rs))));
      if (MM & 2) atomicMax(&p.prov_max[b + j], enc_f64(__longlong_as_double((long long)w8(1 + NI + NF, rs))));
    }
  }
}

// finish up to 32 queued stragglers (lane j: entry (qh + j) % kWsQueue, j < take) and append them
template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_drain(const WsSmem& sm, const WskLayout& L, int wid, int& qh, int& qn, int take,
                                         uint32_t tmine, const XposeConst& xc, int lane, int& pn) {
  constexpr int NV = NI + NF + (MM ? 1 : 0);
  uint64_t m = 0;
  int s = 0;
  unsigned long long v[NV > 0 ? NV : 1];
  const bool on = lane < take;
  if (on) {
    const int e = wid * kWsQueue + ((qh + lane) & (kWsQueue - 1));
    m = pac_hash_continue(sm.qm[e], sm.qw[e]);
    s = sm.qs[e];
#pragma unroll
    for (int c = 0; c < NV; ++c) v[c] = sm.qv[((size_t)wid * NV + c) * kWsQueue + ((qh + lane) & (kWsQueue - 1))];
  }
  __syncwarp();
  qh = (qh + take) & (kWsQueue - 1);
  qn -= take;
  unsigned long long dummy = 0;
  const int f = on ? ws_row_flags<NI, NF>(v, dummy) : 0;
  ws_append<NI, NF, MM>(sm, L, on, s, m, v, f, tmine, xc, wid, lane, pn);
}

// one 64-row chunk starting at global row `base` (nrows valid), two rows per lane
template <int NI, int NF, int MM>
__device__ __forceinline__ void ws_hash_chunk(const AggPlan& p, const WsSmem& sm, const WskLayout& L, int64_t base,
                                              int nrows, int wid, int& qh, int& qn, int& pn, SpillCur& sc,
                                              unsigned long long& maxabs, uint32_t tmine, const XposeConst& xc,
                                              int lane) {
  constexpr int NV = NI + NF + (MM ? 1 : 0);
  constexpr int kNoProv = INT_MIN;
  const unsigned lt_mask = (1u << lane) - 1u;
  const bool defer = p.sp_cap > 0;
  // every load of the chunk first (both rows of the lane, all columns)
  uint64_t w[2], key[2];
  unsigned long long v[2][NV > 0 ? NV : 1];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = lane + 32 * h;
    const bool in = r < nrows;
    const int64_t row = in ? base + r : base;
    w[h] = in ? (uint64_t)__ldg((const unsigned long long*)p.raw_src[0] + row) : 0ull;
#pragma unroll
    for (int c = 0; c < NV; ++c) v[h][c] = (uint64_t)__ldg((const unsigned long long*)p.raw_src[1 + c] + row);
    uint64_t packed = 0;
#pragma unroll
    for (int c = 0; c < PAC_MAX_KEYS; ++c) {
      if (c < p.n_keys) {
        const int wb = p.key_bytes[c];
        const uint64_t kv = load_key_part(p.key_col[c], wb, row);
        packed = (wb == 8) ? kv : ((packed << (8 * wb)) | kv);
      }
    }
    key[h] = packed;
  }
  int s[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = lane + 32 * h;
    const bool keep = r < nrows && (!p.mask_in || w[h] != 0ull);  // R21: a row in no world is dropped
    s[h] = -1;
    int gprov = kNoProv;
    if (keep) {
      const int code = local_code(p, key[h], sm.lkey, sm.lstate, L.LH, sm.lprov, L.Lcap, &sm.misc->m, defer);
      if (code == kUnresolved) gprov = -2;
      else if (code < kOvfBase) s[h] = code - 1;
      else gprov = code - kOvfBase - 1;
    }
    ws_tier<NI, NF, MM>(p, base + r, key[h], gprov, sc, lane);
  }
  uint64_t m[2] = {w[0], w[1]};
  bool pend[2] = {false, false};
  uint64_t w0[2] = {0, 0};
  if (!p.mask_in) {
    HashState ha, hb;
    pac_hash_begin2(w[0], w[1], p.salt, ha, hb);
    m[0] = hash_mask_now(ha);
    m[1] = hash_mask_now(hb);
    pend[0] = s[0] >= 0 && ha.k > 0;
    pend[1] = s[1] >= 0 && hb.k > 0;
    w0[0] = ha.w0;
    w0[1] = hb.w0;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (MM) v[h][NV - 1] = (unsigned long long)enc_f64(__longlong_as_double((long long)v[h][NV - 1]));
    const int f = s[h] >= 0 ? ws_row_flags<NI, NF>(v[h], maxabs) : 0;
    ws_append<NI, NF, MM>(sm, L, s[h] >= 0 && !pend[h], s[h], m[h], v[h], f, tmine, xc, wid, lane, pn);
    // stragglers: into the warp's queue (partial mask, draw word 0, slot, values)
    const unsigned pm = __ballot_sync(0xffffffffu, pend[h]);
    if (pend[h]) {
      const int slot = (qh + qn + __popc(pm & lt_mask)) & (kWsQueue - 1);
      const int e = wid * kWsQueue + slot;
      sm.qm[e] = m[h];
      sm.qw[e] = w0[h];
      sm.qs[e] = s[h];
#pragma unroll
      for (int c = 0; c < NV; ++c) sm.qv[((size_t)wid * NV + c) * kWsQueue + slot] = v[h][c];
    }
    qn += __popc(pm);
    __syncwarp();
    if (qn >= 32) ws_drain<NI, NF, MM>(sm, L, wid, qh, qn, 32, tmine, xc, lane, pn);
  }
}

template <int NI, int NF, int MM>
__global__ void __launch_bounds__(kWsThreads, 1) k_agg_ws(AggPlan p, WskLayout L) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t s_tbase;
  constexpr int NV = NI + NF + (MM ? 1 : 0);
  using S = TmSlot<NI, NF, MM>;
  const WsSmem sm = ws_smem(smem, L);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  // ---- init
  for (int i = tid; i < L.LH; i += blockDim.x) sm.lstate[i] = 0;
  for (int i = tid; i < L.Lcap; i += blockDim.x) sm.fill[i] = 0;
  for (int i = tid; i < L.npairs; i += blockDim.x) {
    sm.cnt[i] = 0;
    sm.gen[i] = 0;
    sm.flag[i] = 0;
  }
  for (int i = tid; i < kWsWarps; i += blockDim.x) sm.ready[i] = 0u;
  if (tid == 0) {
    sm.misc->m.nlocal = 0;
    sm.misc->m.ndict = 0;
    sm.misc->done = 0;
    sm.misc->pending = 0;
    sm.misc->next = kWsWarps;  // chunk w is warp w's first; the rest are taken dynamically
  }
  if (tid < 32) store_xpose(sm.xcs, sm.xcs2, tid);
  if (wid == 0) {  // one CTA per SM: warp 0 allocates all of TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tbase)),
                 "n"(kTmCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmine = ws_tmine(s_tbase, wid);
  const int units = (((L.Lcap << L.logr) - wid) + kWsWarps - 1) / kWsWarps;  // units this warp owns
  for (int i = 0; i < units; ++i) tm_init_slot<NI, NF, MM>(tmine + (uint32_t)(i * S::wps));
  tm_wait_st();
  const XposeConst xc = load_xpose(sm.xcs, sm.xcs2, lane);

  // this CTA's chunks: a contiguous range; warp w takes chunks c0 + w, c0 + w + kWsWarps, ...
  const int64_t nch = (p.n_rows + kWsChunk - 1) / kWsChunk;
  const int64_t per = (nch + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = (int64_t)blockIdx.x * per;
  const int64_t c1 = min(nch, c0 + per);
  auto prefetch = [&](int64_t c) {  // lane i < nraw: bulk L2 prefetch of column i of chunk c
    if (c < c1 && lane < p.nraw && p.tma_ok && (c + 1) * kWsChunk <= p.n_rows) {
      const char* src = (const char*)p.raw_src[lane] + c * kWsChunk * p.raw_eb[lane];
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"((uint32_t)(kWsChunk * p.raw_eb[lane]))
                   : "memory");
    }
  };
  for (int a = 0; a < kWsAhead; ++a) prefetch(c0 + wid + (int64_t)a * kWsWarps);

  int qh = 0, qn = 0, pn = 0;
  unsigned long long maxabs = 0;
  SpillCur sc;
  sc.init();
  for (int64_t c = c0 + wid; c < c1;) {
    prefetch(c + (int64_t)kWsAhead * kWsWarps);
    const int nrows = (int)min((int64_t)kWsChunk, p.n_rows - c * kWsChunk);
    ws_hash_chunk<NI, NF, MM>(p, sm, L, c * kWsChunk, nrows, wid, qh, qn, pn, sc, maxabs, tmine, xc, lane);
    ws_service<NI, NF, MM>(sm, L, tmine, xc, wid, lane, pn);
    int nx = 0;  // the next chunk: dynamic, so the warps finish together
    if (lane == 0) nx = atomicAdd(&sm.misc->next, 1);
    c = c0 + __shfl_sync(0xffffffffu, nx, 0);
  }
  if (qn > 0) ws_drain<NI, NF, MM>(sm, L, wid, qh, qn, qn, tmine, xc, lane, pn);
  sc.finish(p, lane);
  if (NI > 0) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, maxabs, d);
      maxabs = o > maxabs ? o : maxabs;
    }
    if (lane == 0 && maxabs) atomicMax(p.gmaxabs, maxabs);
  }
  __syncwarp();
  if (lane == 0) {
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    atomicAdd(&sm.misc->done, 1);
  }
  // keep servicing until every warp is done and no write is pending anywhere: after that no row
  // can arrive, so a final sweep consumes the full runs and then the last partial run per buffer
  unsigned nap = 32;
  for (;;) {
    ws_service<NI, NF, MM>(sm, L, tmine, xc, wid, lane, pn);
    const bool fin = ld_vol(&sm.misc->done) == kWsWarps && ld_vol(&sm.misc->pending) == 0;
    if (__shfl_sync(0xffffffffu, fin ? 1 : 0, 0)) break;
    __nanosleep(nap);
    nap = nap < 1024 ? 2 * nap : 1024;
  }
  asm volatile("fence.acq_rel.cta;" ::: "memory");
  ws_service<NI, NF, MM>(sm, L, tmine, xc, wid, lane, pn);
  for (int i = 0; i < L.mine; ++i) {
    int k;
    const int pair = ws_my_pair(L, wid, i, k);
    if (pair >= L.npairs) continue;
    const int len = ld_vol(&sm.cnt[pair]);
    if (len == 0) continue;
    unsigned long long* b = (unsigned long long*)(sm.buf + (size_t)pair * (32 * 8 * (1 + NV)));
    const int pad = ((len + 7) & ~7);  // run_body reads whole 8-row groups: zero rows up to the boundary
    if (lane >= len && lane < pad) {
      b[lane] = 0ull;
#pragma unroll
      for (int cc = 0; cc < NV; ++cc) b[32 * (1 + cc) + lane] = 0ull;
    }
    __syncwarp();
    ws_consume<NI, NF, MM>(sm, L, pair, len, tmine + (uint32_t)(k * S::wps), xc, lane);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ---- TMEM -> provisional HBM table (owners), rows per slot
  const int nloc = min(sm.misc->m.nlocal, L.Lcap);
  for (int i = 0; i < units; ++i) {
    const int s = (wid + kWsWarps * i) >> L.logr;
    tm_to_hbm<NI, NF, MM>(p, tmine + (uint32_t)(i * S::wps), s < nloc ? sm.lprov[s] : -1, lane);
  }
  for (int s = tid; s < nloc; s += blockDim.x)
    if (sm.lprov[s] >= 0 && sm.fill[s]) atomicAdd(&p.prov_rows[sm.lprov[s]], (unsigned long long)sm.fill[s]);
  if (tid == 0) atomicMax(&p.dbg[1], (unsigned long long)sm.misc->m.nlocal);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (wid == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tbase), "n"(kTmCols) : "memory");
}

// ------------------------------------------------------------------ host side
__host__ inline WskLayout wsk_layout(int ni, int nf, int mm, int Lcap) {
  WskLayout L{};
  const int wps = 2 + 4 * ni + 4 * nf + ((mm & 1) ? 4 : 0) + ((mm & 2) ? 4 : 0);
  L.Lcap = Lcap;
  L.LH = lay_pow2(4 * Lcap > 256 ? 4 * Lcap : 256);
  // few slots: more buffers per slot, so that >= ~128 buffers spread over the warps' services
  L.lognb = 1;
  while (L.lognb < 6 && (Lcap << L.lognb) < 128) ++L.lognb;
  L.NB = 1 << L.lognb;
  L.nv = ni + nf + (mm ? 1 : 0);
  L.npairs = Lcap * L.NB;
  // as many accumulator units per slot as the TMEM columns allow (more owners for few slots)
  L.logr = L.lognb;
  while (L.logr > 0 && (((Lcap << L.logr) + kWsWarps - 1) / kWsWarps) * wps > kWsCols) --L.logr;
  L.mine = (((Lcap << L.logr) + kWsWarps - 1) / kWsWarps) << (L.lognb - L.logr);
  const int nv1 = L.nv > 0 ? L.nv : 1;
  int off = 0;
  L.o_buf = lay_take(off, L.npairs * 32 * 8 * (1 + L.nv));
  L.o_qm = lay_take(off, kWsWarps * kWsQueue * 8);
  L.o_qw = lay_take(off, kWsWarps * kWsQueue * 8);
  L.o_qv = lay_take(off, kWsWarps * kWsQueue * 8 * nv1);
  L.o_qs = lay_take(off, kWsWarps * kWsQueue * 4);
  L.o_pm = lay_take(off, kWsWarps * kWsPend * 8);
  L.o_pv = lay_take(off, kWsWarps * kWsPend * 8 * nv1);
  L.o_pp = lay_take(off, kWsWarps * kWsPend * 4);
  L.o_ps = lay_take(off, kWsWarps * kWsPend * 4);
  L.o_pf = lay_take(off, kWsWarps * kWsPend * 4);
  L.o_fill = lay_take(off, Lcap * 4);
  L.o_cnt = lay_take(off, L.npairs * 4);
  L.o_gen = lay_take(off, L.npairs * 4);
  L.o_flag = lay_take(off, L.npairs * 4);
  L.o_ready = lay_take(off, kWsWarps * 4);
  L.o_lkey = lay_take(off, L.LH * 8);
  L.o_lstate = lay_take(off, L.LH * 4);
  L.o_lprov = lay_take(off, Lcap * 4);
  L.o_misc = lay_take(off, (int)sizeof(WsMisc));
  L.o_xcs = lay_take(off, 32 * 16 + 32 * 8);
  L.bytes = off;
  return L;
}

// TMEM columns: a warp holds the accumulators of ceil(units / kWsWarps) units
__host__ inline bool ws_tmem_fits(const WskLayout& L, int wps) {
  return (((L.Lcap << L.logr) + kWsWarps - 1) / kWsWarps) * wps <= kWsCols;
}

template <int NI, int NF, int MM>
cudaError_t launch_ws(const AggPlan& p, const WskLayout& L, int sms, cudaStream_t st) {
  if (!ws_tmem_fits(L, TmSlot<NI, NF, MM>::wps)) return cudaErrorInvalidValue;
  auto k = k_agg_ws<NI, NF, MM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  const int64_t chunks = (p.n_rows + kWsChunk - 1) / kWsChunk;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((chunks + 7) / 8, (int64_t)sms));
  if (getenv("PAC_DEBUG"))
    fprintf(stderr, "[libpac] k_agg_ws<%d,%d,%d> %d CTAs x %d threads, Lcap=%d NB=%d smem=%d B\n", NI, NF, MM, grid,
            kWsThreads, L.Lcap, L.NB, L.bytes);
  k<<<grid, kWsThreads, L.bytes, st>>>(p, L);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pac
