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

#include "common.cuh"

namespace pac {

constexpr int kThreads = 512;      // k_agg_minmax
constexpr int kTileThreads = 256;  // k_agg_tiles: 128-register budget (2 CTAs / SM)
constexpr int kOvfBase = 0x20000000;  // local-dict code for keys without a local slot
constexpr int kSmallSort = 4096;      // single-CTA bitonic sort up to this many groups

struct AggPlan {
  int64_t n_rows;
  const long long* pu_key;
  const unsigned long long* mask_in;
  uint64_t salt;
  int n_keys;
  const void* key_col[PAC_MAX_KEYS];
  int key_bytes[PAC_MAX_KEYS];
  int ni, nf, has_min, has_max, has_count;
  const long long* icol[2];
  const double* fcol[2];
  const double* mcol;
  // HBM dictionary + provisional table (workspace)
  unsigned long long* gkey;
  int* gstate;
  uint32_t hmask;
  int* gcounter;
  unsigned long long* gmaxabs;  // max |v| over int64 sum columns (overflow check)
  unsigned long long* dbg;      // [0] rows sent to the HBM tier, [1] max local slots used
  // raw input columns staged per tile by 1-D TMA bulk copies (k_agg_tiles):
  // 0 = pu_key or mask, 1..n_keys = key columns, then int64 sums, f64 sums, min/max column
  int nraw, tma_ok;
  int ablate;  // profiling only (PAC_ABLATE): 1 = no draws, 2 = no A3, 4 = no phase C
  const void* raw_src[1 + PAC_MAX_KEYS + 5];
  int raw_eb[1 + PAC_MAX_KEYS + 5];
  int raw_off[1 + PAC_MAX_KEYS + 5];  // byte offset of the column inside the raw tile buffer
  int raw_bytes;                       // bytes of one staged tile
  int64_t G_cap;
  unsigned long long* prov_key;
  unsigned long long* prov_rows;
  unsigned long long* prov_count;
  unsigned long long* prov_isum[2];
  double* prov_fsum[2];
  long long* prov_min;
  long long* prov_max;
};

struct SmemLayout {
  int T, TS, Lcap, LH;
  int o_lkey, o_lstate, o_lprov, o_lrows, o_cnt, o_isum, o_fsum, o_min, o_max;
  int o_mask, o_slot, o_rank, o_ucnt, o_queue, o_ival, o_i32, o_fval, o_mval, o_hist, o_offs,
      o_runoffs, o_tcs, o_raw, o_mbar, o_misc;
  int bytes;
};

struct Misc {
  int nlocal;   // local slots handed out
  int ndict;    // local dictionary reservations
  int nruns;    // runs in the current tile
  int big;        // some int64 value of the tile has |v| >= 2^26 (no int32 tables)
  int nqueue;     // rows whose mask needs more than one draw word
  int nonfinite;  // some f64 value of the tile is inf/nan (no 0/1-FMA tables)
  int pad[2];
};

// ------------------------------------------------------------------ dictionaries
__device__ __forceinline__ void init_prov_slot(const AggPlan& p, int prov, uint64_t key) {
  p.prov_key[prov] = key;
  p.prov_rows[prov] = 0;
  size_t b = (size_t)prov * kM;
  for (int j = 0; j < kM; ++j) {
    if (p.has_count) p.prov_count[b + j] = 0;
    for (int c = 0; c < p.ni; ++c) p.prov_isum[c][b + j] = 0;
    for (int c = 0; c < p.nf; ++c) p.prov_fsum[c][b + j] = 0.0;
    if (p.has_min) p.prov_min[b + j] = kEncPosInf;
    if (p.has_max) p.prov_max[b + j] = kEncNegInf;
  }
}

// Insert-or-find `key` in the HBM dictionary; returns the provisional slot, or -1 when
// the capacity G_cap is exhausted (the table is then flagged by the finish kernel).
__device__ int global_slot(const AggPlan& p, uint64_t key) {
  uint32_t h = dict_hash(key) & p.hmask;
  for (;;) {
    int st = *(volatile int*)&p.gstate[h];
    if (st == 0) {
      if (atomicCAS(&p.gstate[h], 0, -1) == 0) {
        int prov = atomicAdd(p.gcounter, 1);
        if (prov >= p.G_cap) {  // out of capacity: release the claim, report via counter
          __threadfence();
          atomicExch(&p.gstate[h], 0);
          return -1;
        }
        *(volatile unsigned long long*)&p.gkey[h] = key;
        init_prov_slot(p, prov, key);
        __threadfence();
        atomicExch(&p.gstate[h], prov + 1);
        return prov;
      }
      continue;
    }
    if (st < 0) continue;  // being written
    __threadfence();
    if (*(volatile unsigned long long*)&p.gkey[h] == key) return st - 1;
    h = (h + 1) & p.hmask;
  }
}

// CTA-local dictionary: code = s+1 for local slot s (< Lcap); kOvfBase + prov + 1 for a
// key that has no local slot (its rows go straight to the HBM table; prov -1 = dropped).
// An empty entry is claimed with CAS first; only then is the entry counted, so concurrent
// contenders for one key never inflate the fill count.  At half full no more keys are
// inserted (their rows use the HBM dictionary directly).
__device__ int local_code(const AggPlan& p, uint64_t key, unsigned long long* lkey, int* lstate,
                          int LH, int* lprov, int Lcap, Misc* misc) {
  uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 40) & (LH - 1);
  for (;;) {
    int st = *(volatile int*)&lstate[h];
    if (st == 0) {
      if (atomicCAS(&lstate[h], 0, -1) == 0) {
        if (atomicAdd(&misc->ndict, 1) >= LH / 2) {  // too full: release, use the HBM tier
          atomicSub(&misc->ndict, 1);
          __threadfence_block();
          atomicExch(&lstate[h], 0);
          return kOvfBase + global_slot(p, key) + 1;
        }
        lkey[h] = key;
        int s = atomicAdd(&misc->nlocal, 1);
        int prov = global_slot(p, key);
        int code;
        if (s < Lcap) {
          lprov[s] = prov;
          code = s + 1;
        } else {
          code = kOvfBase + prov + 1;
        }
        __threadfence_block();
        atomicExch(&lstate[h], code);
        return code;
      }
      continue;
    }
    if (st < 0) continue;
    __threadfence_block();
    if (*(volatile unsigned long long*)&lkey[h] == key) return st;
    h = (h + 1) & (LH - 1);
  }
}

__device__ __forceinline__ uint64_t row_group_key(const AggPlan& p, int64_t r) {
  uint64_t packed = 0;
#pragma unroll
  for (int c = 0; c < PAC_MAX_KEYS; ++c) {
    if (c < p.n_keys) {
      int w = p.key_bytes[c];
      uint64_t v = load_key_part(p.key_col[c], w, r);
      packed = (w == 8) ? v : ((packed << (8 * w)) | v);
    }
  }
  return packed;
}

// Direct HBM update for a row whose group has no CTA-local slot.
template <int NI, int NF, int MM>
__device__ __forceinline__ void global_row_update(const AggPlan& p, int prov, uint64_t m,
                                                  const long long (&iv)[NI > 0 ? NI : 1],
                                                  const double (&fv)[NF > 0 ? NF : 1], double mv) {
  atomicAdd(&p.dbg[0], 1ull);
  if (prov < 0) return;
  atomicAdd(&p.prov_rows[prov], 1ull);
  const size_t b = (size_t)prov * kM;
#pragma unroll 1
  for (int j = 0; j < kM; ++j) {
    if (!((m >> j) & 1ull)) continue;
    atomicAdd(&p.prov_count[b + j], 1ull);
#pragma unroll
    for (int c = 0; c < NI; ++c) atomicAdd(&p.prov_isum[c][b + j], (unsigned long long)iv[c]);
#pragma unroll
    for (int c = 0; c < NF; ++c) atomicAdd(&p.prov_fsum[c][b + j], fv[c]);
    if (MM & 1) atomicMin(&p.prov_min[b + j], enc_f64(mv));
    if (MM & 2) atomicMax(&p.prov_max[b + j], enc_f64(mv));
  }
}

// ------------------------------------------------------------------ k_mask
__global__ void __launch_bounds__(256) k_mask(const long long* __restrict__ key, int64_t n,
                                              uint64_t salt, unsigned long long* __restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = pac_hash_dev((uint64_t)__ldg(key + i), salt);
}

// ------------------------------------------------------------------ TMA bulk staging
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(m)), "r"(parity) : "memory");
}
// one thread: stage the raw columns of the full tile starting at row `base`
__device__ __forceinline__ void issue_tile(const AggPlan& p, unsigned char* raw, unsigned long long* mbar,
                                           int64_t base, int T) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(mbar, (uint32_t)p.raw_bytes);
  for (int i = 0; i < p.nraw; ++i)
    bulk_g2s(raw + p.raw_off[i], (const char*)p.raw_src[i] + base * p.raw_eb[i], (uint32_t)(T * p.raw_eb[i]), mbar);
}

// ------------------------------------------------------------------ k_agg_tiles (v3)
// Bit-matrix transpose of a 32-row run: on input lane r holds row r's
// 32-bit mask word; on output lane c holds the pattern of world c over the run.  Stage s
// swaps the off-diagonal s x s blocks: the partner's word is rotated by s (low lane) or
// 32-s (high lane) with one funnel shift and merged with one LOP3 under a per-lane mask.
// Per-lane constants of the 5 stages live in shared memory (tcs[stage*32 + lane] =
// {keep mask, rotate amount}), loaded once per run: cheaper than rematerialising them.
__device__ __forceinline__ uint2 transpose_const(int lane, int i) {
  const int s = 16 >> i;
  const uint32_t M = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu
                   : s == 2 ? 0x33333333u : 0x55555555u;
  const bool up = (lane & s) != 0;
  return make_uint2(up ? ~M : M, (uint32_t)(up ? 32 - s : s));
}

__device__ __forceinline__ void transpose2x32(uint32_t& a, uint32_t& b, const uint2* __restrict__ tcs,
                                              int lane) {
  uint2 c[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) c[i] = tcs[i * 32 + lane];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int s = 16 >> i;
    const uint32_t ya = __shfl_xor_sync(0xffffffffu, a, s);
    const uint32_t yb = __shfl_xor_sync(0xffffffffu, b, s);
    a = (a & c[i].x) | (__funnelshift_l(ya, ya, c[i].y) & ~c[i].x);
    b = (b & c[i].x) | (__funnelshift_l(yb, yb, c[i].y) & ~c[i].x);
  }
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  const int lo = __shfl_sync(0xffffffffu, __double2loint(v), src);
  const int hi = __shfl_sync(0xffffffffu, __double2hiint(v), src);
  return __hiloint2double(hi, lo);
}

__device__ __forceinline__ bool finite_bits(double v) {
  return (__double2hiint(v) & 0x7FF00000) != 0x7FF00000;
}

// Register accumulators of the slot a warp is currently working on (lane: worlds lane, lane+32).
template <int NI, int NF, int MM>
struct WarpAcc {
  int cur;
  unsigned c0, c1;
  long long ia0[NI > 0 ? NI : 1], ia1[NI > 0 ? NI : 1];
  double fa0[NF > 0 ? NF : 1], fa1[NF > 0 ? NF : 1];
  double mn0, mn1, mx0, mx1;

  __device__ __forceinline__ void reset() {
    c0 = c1 = 0;
#pragma unroll
    for (int c = 0; c < NI; ++c) ia0[c] = ia1[c] = 0;
#pragma unroll
    for (int c = 0; c < NF; ++c) fa0[c] = fa1[c] = 0.0;
    mn0 = mn1 = INFINITY;
    mx0 = mx1 = -INFINITY;
  }
  // add into the CTA's smem table (shared by the warps working on the same slot)
  __device__ __forceinline__ void flush(unsigned* cnt, unsigned long long* isum, double* fsum, long long* emin,
                                        long long* emax, int Lcap, int lane) {
    if (cur < 0) return;
    const size_t b = (size_t)cur * kM;
    if (c0) atomicAdd(&cnt[b + lane], c0);
    if (c1) atomicAdd(&cnt[b + lane + 32], c1);
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      atomicAdd(&isum[(size_t)c * Lcap * kM + b + lane], (unsigned long long)ia0[c]);
      atomicAdd(&isum[(size_t)c * Lcap * kM + b + lane + 32], (unsigned long long)ia1[c]);
    }
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      atomicAdd(&fsum[(size_t)c * Lcap * kM + b + lane], fa0[c]);
      atomicAdd(&fsum[(size_t)c * Lcap * kM + b + lane + 32], fa1[c]);
    }
    if (MM & 1) {
      atomicMin(&emin[b + lane], enc_f64(mn0));
      atomicMin(&emin[b + lane + 32], enc_f64(mn1));
    }
    if (MM & 2) {
      atomicMax(&emax[b + lane], enc_f64(mx0));
      atomicMax(&emax[b + lane + 32], enc_f64(mx1));
    }
    reset();
  }
};

struct RunCtx {  // read-only per-tile state of phase C
  const unsigned long long* smask;
  const long long* sival;
  const int* si32;
  const double* sfval;
  const double* smval;
  const int* hist;
  const int* offs;
  const int* runoffs;
  const uint2* tcs;
  int TS, Lcap, R;
};

// Phase C of one tile for one warp: runs [r0, r1) of the tile's slot-sorted rows.
// SMALL: int64 values of the tile fit int32 nibble tables; FIN: f64 values are finite, so
// the f64 nibble tables are built with exact 0/1 FMAs.
template <int NI, int NF, int MM, bool SMALL, bool FIN>
__device__ __forceinline__ void run_tiles(WarpAcc<NI, NF, MM>& acc, const RunCtx& x, unsigned* cnt,
                                          unsigned long long* isum, double* fsum, long long* emin,
                                          long long* emax, int wid, int nw, int lane) {
  const int R = x.R, TS = x.TS;
  const int r0 = (int)(((long long)R * wid) / nw);
  const int r1 = (int)(((long long)R * (wid + 1)) / nw);
  if (r0 >= r1) return;
  const int sub = lane & 15;
  const int tsrc = (lane >> 4) << 2;
  const int ib0 = sub & 1, ib1 = (sub >> 1) & 1, ib2 = (sub >> 2) & 1, ib3 = (sub >> 3) & 1;
  const double db0 = ib0, db1 = ib1, db2 = ib2, db3 = ib3;
  int s;
  {
    int lo = 0, hi = x.Lcap;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (x.runoffs[mid] <= r0) lo = mid; else hi = mid - 1;
    }
    s = lo;
  }
  int rs_end = x.runoffs[s + 1];
  int k0 = 32 * (r0 - x.runoffs[s]);
  int slot_beg = x.offs[s], slot_len = x.hist[s];
  for (int r = r0; r < r1; ++r) {
    if (r >= rs_end) {  // next non-empty slot
      do {
        ++s;
        rs_end = x.runoffs[s + 1];
      } while (rs_end <= r);
      k0 = 0;
      slot_beg = x.offs[s];
      slot_len = x.hist[s];
    }
    if (s != acc.cur) {
      acc.flush(cnt, isum, fsum, emin, emax, x.Lcap, lane);
      acc.cur = s;
    }
    const int beg = slot_beg + k0;
    const int len = min(32, slot_len - k0);
    k0 += 32;
    const uint64_t m = lane < len ? x.smask[beg + lane] : 0ull;
    uint32_t P = (uint32_t)m, Q = (uint32_t)(m >> 32);
    transpose2x32(P, Q, x.tcs, lane);
    acc.c0 += __popc(P);
    acc.c1 += __popc(Q);
    // nibble indices: table A (lanes 0-15) covers rows 8q..8q+3, B (16-31) rows 8q+4..8q+7;
    // shfl uses only the low 5 bits of the source lane.
    const uint32_t PA = P & 0x0F0F0F0Fu, PB = ((P >> 4) & 0x0F0F0F0Fu) | 0x10101010u;
    const uint32_t QA = Q & 0x0F0F0F0Fu, QB = ((Q >> 4) & 0x0F0F0F0Fu) | 0x10101010u;
    const int nq = (len + 7) >> 3;
    int rs0[NI > 0 ? NI : 1], rs1[NI > 0 ? NI : 1];
#pragma unroll
    for (int c = 0; c < NI; ++c) rs0[c] = rs1[c] = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q >= nq) break;
      const int a0 = (int)(PA >> (8 * q)), b0 = (int)(PB >> (8 * q));
      const int a1 = (int)(QA >> (8 * q)), b1 = (int)(QB >> (8 * q));
      const int row = beg + 8 * q + tsrc;
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        if (SMALL) {
          const int4 v = *(const int4*)(x.si32 + c * TS + row);
          const int t = v.x * ib0 + v.y * ib1 + v.z * ib2 + v.w * ib3;
          rs0[c] += __shfl_sync(0xffffffffu, t, a0) + __shfl_sync(0xffffffffu, t, b0);
          rs1[c] += __shfl_sync(0xffffffffu, t, a1) + __shfl_sync(0xffffffffu, t, b1);
        } else {
          const longlong2 u = *(const longlong2*)(x.sival + c * TS + row);
          const longlong2 w = *(const longlong2*)(x.sival + c * TS + row + 2);
          const long long t = u.x * ib0 + u.y * ib1 + w.x * ib2 + w.y * ib3;
          acc.ia0[c] += __shfl_sync(0xffffffffu, t, a0) + __shfl_sync(0xffffffffu, t, b0);
          acc.ia1[c] += __shfl_sync(0xffffffffu, t, a1) + __shfl_sync(0xffffffffu, t, b1);
        }
      }
#pragma unroll
      for (int c = 0; c < NF; ++c) {
        const double2 u = *(const double2*)(x.sfval + c * TS + row);
        const double2 w = *(const double2*)(x.sfval + c * TS + row + 2);
        double t;
        if (FIN) {  // exact: 0*v + t == t and 1*v + t == v + t for finite v
          t = fma(db3, w.y, fma(db2, w.x, fma(db1, u.y, db0 * u.x)));
        } else {
          t = ib0 ? u.x : 0.0;
          if (ib1) t += u.y;
          if (ib2) t += w.x;
          if (ib3) t += w.y;
        }
        acc.fa0[c] += shfl_d(t, a0);
        acc.fa0[c] += shfl_d(t, b0);
        acc.fa1[c] += shfl_d(t, a1);
        acc.fa1[c] += shfl_d(t, b1);
      }
      if (MM) {
        const double2 u = *(const double2*)(x.smval + row);
        const double2 w = *(const double2*)(x.smval + row + 2);
        if (MM & 1) {
          double t = ib0 ? u.x : INFINITY;
          if (ib1) t = fmin(t, u.y);
          if (ib2) t = fmin(t, w.x);
          if (ib3) t = fmin(t, w.y);
          acc.mn0 = fmin(acc.mn0, fmin(shfl_d(t, a0), shfl_d(t, b0)));
          acc.mn1 = fmin(acc.mn1, fmin(shfl_d(t, a1), shfl_d(t, b1)));
        }
        if (MM & 2) {
          double t = ib0 ? u.x : -INFINITY;
          if (ib1) t = fmax(t, u.y);
          if (ib2) t = fmax(t, w.x);
          if (ib3) t = fmax(t, w.y);
          acc.mx0 = fmax(acc.mx0, fmax(shfl_d(t, a0), shfl_d(t, b0)));
          acc.mx1 = fmax(acc.mx1, fmax(shfl_d(t, a1), shfl_d(t, b1)));
        }
      }
    }
    if (SMALL) {
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        acc.ia0[c] += rs0[c];
        acc.ia1[c] += rs1[c];
      }
    }
  }
}

struct TileSmem {
  unsigned long long* lkey;
  int* lstate;
  int* lprov;
  unsigned long long* lrows;
  unsigned* cnt;
  unsigned long long* isum;
  double* fsum;
  long long* emin;
  long long* emax;
  unsigned long long* smask;  // [TS] slot-sorted masks
  long long* sival;           // [NI][TS]
  int* si32;                  // [NI][TS]
  double* sfval;              // [NF][TS]
  double* smval;              // [TS]
  unsigned short* sslot;      // [T]
  unsigned char* srank;       // [T]
  unsigned short* ucnt;       // [units][Lcap]
  unsigned short* qpos;       // [T]
  unsigned short* qrow;       // [T]
  int* hist;
  int* offs;
  int* runoffs;
  uint2* tcs;
  Misc* misc;
  const unsigned char* raw;   // staged raw tile: 8-byte columns k at k*T*8, then key columns
};

// Column k of the tile: 0 = pu_key/mask, 1..NI int64 sums, NI+1..NI+NF f64 sums, then the
// MIN/MAX column; group-key columns after them.  Staged tiles read the TMA copy in smem.
template <bool STAGED>
struct TileCols {
  const AggPlan* p;
  const unsigned char* raw;
  int64_t base;
  int T;
  __device__ __forceinline__ uint64_t w8(int k, int li) const {
    if (STAGED) return ((const unsigned long long*)raw)[(size_t)k * T + li];
    return (uint64_t)__ldg((const unsigned long long*)p->raw_src[k] + base + li);
  }
  __device__ __forceinline__ uint64_t group_key(int k0, int li) const {
    uint64_t packed = 0;
#pragma unroll
    for (int c = 0; c < PAC_MAX_KEYS; ++c) {
      if (c < p->n_keys) {
        const int w = p->key_bytes[c];
        uint64_t v;
        if (STAGED) {
          const unsigned char* col = raw + p->raw_off[k0 + c];
          if (w == 1) v = col[li];
          else if (w == 2) v = ((const unsigned short*)col)[li];
          else if (w == 4) v = ((const unsigned*)col)[li];
          else v = ((const unsigned long long*)col)[li];
          v ^= 1ull << (8 * w - 1);
        } else {
          v = load_key_part(p->key_col[c], w, base + li);
        }
        packed = (w == 8) ? v : ((packed << (8 * w)) | v);
      }
    }
    return packed;
  }
};

// A1 (slots + ranks), B (offsets), A2 (hash word 0 + sorted staging), A3 (stragglers) of one
// tile.  Leaves the slot-sorted tile in smem and the run table for phase C.
template <int NI, int NF, int MM, bool STAGED>
__device__ __forceinline__ void tile_front(const AggPlan& p, const TileSmem& sm, const SmemLayout& L, int64_t base,
                                           int tn, unsigned long long& maxabs) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int T = L.T, TS = L.TS, Lcap = L.Lcap, LH = L.LH;
  const int units = T >> 5;
  const unsigned short kNone = 0xFFFF;
  const unsigned lt_mask = (1u << lane) - 1u;
  constexpr int KF = 1 + NI;             // first f64 sum column
  constexpr int KM = 1 + NI + NF;        // min/max column
  constexpr int KK = 1 + NI + NF + (MM ? 1 : 0);  // first group-key column
  TileCols<STAGED> tc{&p, sm.raw, base, T};
  Misc* misc = sm.misc;

  // ---------------- A1: group slot of every row + rank within its 32-row unit
  for (int li = tid; li < T; li += nth) {
    int s = -1;
    if (li < tn) {
      bool keep = true;
      if (p.mask_in) keep = tc.w8(0, li) != 0ull;  // R21: a row in no world is dropped
      if (keep) {
        const uint64_t key = tc.group_key(KK, li);
        const int code = local_code(p, key, sm.lkey, sm.lstate, LH, sm.lprov, Lcap, misc);
        if (code < kOvfBase) {
          s = code - 1;
        } else {  // no local slot: straight to the HBM table (rare)
          long long iv[NI > 0 ? NI : 1];
          double fv[NF > 0 ? NF : 1];
#pragma unroll
          for (int c = 0; c < NI; ++c) iv[c] = (long long)tc.w8(1 + c, li);
#pragma unroll
          for (int c = 0; c < NF; ++c) fv[c] = __longlong_as_double((long long)tc.w8(KF + c, li));
          const double mv = MM ? __longlong_as_double((long long)tc.w8(KM, li)) : 0.0;
          const uint64_t m = p.mask_in ? tc.w8(0, li) : pac_hash_dev(tc.w8(0, li), p.salt);
          global_row_update<NI, NF, MM>(p, code - kOvfBase - 1, m, iv, fv, mv);
        }
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, s >= 0 ? (unsigned)s : 0x10000u + lane);
    if (s >= 0) {
      sm.srank[li] = (unsigned char)__popc(peers & lt_mask);
      if ((peers & lt_mask) == 0) sm.ucnt[(li >> 5) * Lcap + s] = (unsigned short)__popc(peers);
    }
    sm.sslot[li] = s >= 0 ? (unsigned short)s : kNone;
  }
  __syncthreads();

  // ---------------- B: slot totals, 8-row padded offsets, run offsets, unit positions
  for (int s = tid; s < Lcap; s += nth) {
    int tot = 0;
    for (int u = 0; u < units; ++u) tot += sm.ucnt[u * Lcap + s];
    sm.hist[s] = tot;
  }
  __syncthreads();
  if (wid == 0) {
    const int per = (Lcap + 31) / 32;
    const int s0 = lane * per;
    int hsum = 0, rsum = 0;
    for (int s = s0; s < min(Lcap, s0 + per); ++s) {
      hsum += (sm.hist[s] + 7) & ~7;
      rsum += (sm.hist[s] + 31) >> 5;
    }
    int hx = hsum, rx = rsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, hx, d);
      const int b = __shfl_up_sync(0xffffffffu, rx, d);
      if (lane >= d) {
        hx += a;
        rx += b;
      }
    }
    hx -= hsum;
    rx -= rsum;
    for (int s = s0; s < min(Lcap, s0 + per); ++s) {
      sm.offs[s] = hx;
      sm.runoffs[s] = rx;
      sm.lrows[s] += (unsigned long long)sm.hist[s];
      hx += (sm.hist[s] + 7) & ~7;
      rx += (sm.hist[s] + 31) >> 5;
    }
    if (lane == 31) {
      sm.runoffs[Lcap] = rx;
      misc->nruns = rx;
    }
  }
  __syncthreads();
  for (int s = tid; s < Lcap; s += nth) {
    const int o0 = sm.offs[s];
    int o = o0;
    for (int u = 0; u < units; ++u) {
      const int c = sm.ucnt[u * Lcap + s];
      sm.ucnt[u * Lcap + s] = (unsigned short)o;
      o += c;
    }
    for (int q = o; q < o0 + ((sm.hist[s] + 7) & ~7); ++q) {  // zero padding rows (mask 0)
      sm.smask[q] = 0;
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        sm.sival[c * TS + q] = 0;
        sm.si32[c * TS + q] = 0;
      }
#pragma unroll
      for (int c = 0; c < NF; ++c) sm.sfval[c * TS + q] = 0.0;
      if (MM) sm.smval[q] = 0.0;
    }
  }
  __syncthreads();

  // ---------------- A2: hash word 0 (two rows per thread, interleaved) + values, written
  // straight to the slot-sorted position; rows still needing flips are queued for A3.
  bool big = false, nonfin = false;
  for (int la = tid; la < T; la += 2 * nth) {
    const int lb = la + nth;  // T is a multiple of 2 * nth
    const unsigned short sa = sm.sslot[la], sb = sm.sslot[lb];
    const int pa = sa != kNone ? sm.ucnt[(la >> 5) * Lcap + sa] + sm.srank[la] : 0;
    const int pb = sb != kNone ? sm.ucnt[(lb >> 5) * Lcap + sb] + sm.srank[lb] : 0;
    bool qa = false, qb = false;
    const uint64_t ka = sa != kNone ? tc.w8(0, la) : 0ull;
    const uint64_t kb = sb != kNone ? tc.w8(0, lb) : 0ull;
    uint64_t ma = ka, mb = kb;
    if (!p.mask_in) {
      HashState ha, hb;
      if (p.ablate & 1) {
        ha.x = ka; ha.cand = ka; ha.k = 0; hb.x = kb; hb.cand = kb; hb.k = 0;
      } else {
        pac_hash_begin2(ka, kb, p.salt, ha, hb);
      }
      ma = ha.x ^ (((__popcll(ha.x) > 32) ? ha.x : ~ha.x) ^ ha.cand);
      mb = hb.x ^ (((__popcll(hb.x) > 32) ? hb.x : ~hb.x) ^ hb.cand);
      qa = sa != kNone && ha.k > 0;
      qb = sb != kNone && hb.k > 0;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int li = h ? lb : la;
      const int pos = h ? pb : pa;
      if ((h ? sb : sa) == kNone) continue;
      sm.smask[pos] = h ? mb : ma;
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        const long long v = (long long)tc.w8(1 + c, li);
        const unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
        maxabs = a > maxabs ? a : maxabs;
        big |= a >= (1ull << 26);
        sm.sival[c * TS + pos] = v;
        sm.si32[c * TS + pos] = (int)v;
      }
#pragma unroll
      for (int c = 0; c < NF; ++c) {
        const double v = __longlong_as_double((long long)tc.w8(KF + c, li));
        nonfin |= !finite_bits(v);
        sm.sfval[c * TS + pos] = v;
      }
      if (MM) sm.smval[pos] = __longlong_as_double((long long)tc.w8(KM, li));
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool pend = h ? qb : qa;
      const unsigned pm = __ballot_sync(0xffffffffu, pend);
      int qbase = 0;
      if (lane == 0 && pm) qbase = atomicAdd(&misc->nqueue, __popc(pm));
      qbase = __shfl_sync(0xffffffffu, qbase, 0) + __popc(pm & lt_mask);
      if (pend) {
        sm.qpos[qbase] = (unsigned short)(h ? pb : pa);
        sm.qrow[qbase] = (unsigned short)(h ? lb : la);
      }
    }
  }
  if (NI > 0 && __any_sync(0xffffffffu, big) && lane == 0) misc->big = 1;
  if (NF > 0 && __any_sync(0xffffffffu, nonfin) && lane == 0) misc->nonfinite = 1;
  __syncthreads();

  // ---------------- A3: finish the queued masks.  State re-derived from the key and the
  // partial mask: cand = majority positions of the current word, k = |popcount - 32|.
  if (!(p.ablate & 2)) {
    const int qn = misc->nqueue;
    for (int qi = tid; qi < qn; qi += nth) {
      const int pos = sm.qpos[qi];
      const uint64_t x = fmix64(tc.w8(0, sm.qrow[qi]) ^ p.salt);
      const uint64_t m = sm.smask[pos];
      sm.smask[pos] = pac_hash_finish(x, (__popcll(x) > 32) ? m : ~m, abs(__popcll(m) - 32));
    }
  }
  __syncthreads();
}

template <int NI, int NF, int MM>
__global__ void __launch_bounds__(kTileThreads, 3) k_agg_tiles(AggPlan p, SmemLayout L) {
  extern __shared__ __align__(16) unsigned char smem[];
  TileSmem sm;
  sm.lkey = (unsigned long long*)(smem + L.o_lkey);
  sm.lstate = (int*)(smem + L.o_lstate);
  sm.lprov = (int*)(smem + L.o_lprov);
  sm.lrows = (unsigned long long*)(smem + L.o_lrows);
  sm.cnt = (unsigned*)(smem + L.o_cnt);
  sm.isum = (unsigned long long*)(smem + L.o_isum);
  sm.fsum = (double*)(smem + L.o_fsum);
  sm.emin = (long long*)(smem + L.o_min);
  sm.emax = (long long*)(smem + L.o_max);
  sm.smask = (unsigned long long*)(smem + L.o_mask);
  sm.sival = (long long*)(smem + L.o_ival);
  sm.si32 = (int*)(smem + L.o_i32);
  sm.sfval = (double*)(smem + L.o_fval);
  sm.smval = (double*)(smem + L.o_mval);
  sm.sslot = (unsigned short*)(smem + L.o_slot);
  sm.srank = (unsigned char*)(smem + L.o_rank);
  sm.ucnt = (unsigned short*)(smem + L.o_ucnt);
  sm.qpos = (unsigned short*)(smem + L.o_queue);
  sm.qrow = sm.qpos + L.T;
  sm.hist = (int*)(smem + L.o_hist);
  sm.offs = (int*)(smem + L.o_offs);
  sm.runoffs = (int*)(smem + L.o_runoffs);
  sm.tcs = (uint2*)(smem + L.o_tcs);
  sm.misc = (Misc*)(smem + L.o_misc);
  unsigned char* raw = smem + L.o_raw;
  sm.raw = raw;
  unsigned long long* mbar = (unsigned long long*)(smem + L.o_mbar);
  Misc* misc = sm.misc;

  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  const int T = L.T, Lcap = L.Lcap, LH = L.LH;
  const int units = T >> 5;

  for (int i = tid; i < LH; i += nth) sm.lstate[i] = 0;
  for (int i = tid; i < Lcap; i += nth) sm.lrows[i] = 0;
  for (int i = tid; i < Lcap * kM; i += nth) {
    sm.cnt[i] = 0;
#pragma unroll
    for (int c = 0; c < NI; ++c) sm.isum[(size_t)c * Lcap * kM + i] = 0;
#pragma unroll
    for (int c = 0; c < NF; ++c) sm.fsum[(size_t)c * Lcap * kM + i] = 0.0;
    if (MM & 1) sm.emin[i] = kEncPosInf;
    if (MM & 2) sm.emax[i] = kEncNegInf;
  }
  if (tid < 32) {
#pragma unroll
    for (int i = 0; i < 5; ++i) sm.tcs[i * 32 + tid] = transpose_const(tid, i);
  }
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }
  unsigned long long maxabs = 0;

  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * t_per;
  const int64_t t1 = min(ntiles, t0 + t_per);
  // a tile is staged by TMA when it is full and every column is 16-byte aligned
  auto staged_tile = [&](int64_t t) { return p.tma_ok && t < t1 && (t + 1) * T <= p.n_rows; };
  uint32_t phase = 0;
  if (tid == 0) {
    mbar_init(mbar, 1);
    if (staged_tile(t0)) issue_tile(p, raw, mbar, t0 * T, T);
  }
  __syncthreads();

  WarpAcc<NI, NF, MM> acc;
  acc.cur = -1;
  acc.reset();

  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t base = tile * T;
    const int tn = (int)min((int64_t)T, p.n_rows - base);
    for (int i = tid; i < units * Lcap; i += nth) sm.ucnt[i] = 0;
    if (tid == 0) {
      misc->big = 0;
      misc->nonfinite = 0;
      misc->nqueue = 0;
    }
    const bool staged = staged_tile(tile);
    if (staged) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
    }
    __syncthreads();
    if (staged) tile_front<NI, NF, MM, true>(p, sm, L, base, tn, maxabs);
    else tile_front<NI, NF, MM, false>(p, sm, L, base, tn, maxabs);
    // the raw tile buffer is free: stage the next tile while phase C runs
    if (tid == 0 && staged_tile(tile + 1)) issue_tile(p, raw, mbar, (tile + 1) * T, T);

    // ---------------- C: world-parallel runs, transposed "Four Russians" tables
    if (!(p.ablate & 4)) {
      RunCtx x;
      x.smask = sm.smask;
      x.sival = sm.sival;
      x.si32 = sm.si32;
      x.sfval = sm.sfval;
      x.smval = sm.smval;
      x.hist = sm.hist;
      x.offs = sm.offs;
      x.runoffs = sm.runoffs;
      x.tcs = sm.tcs;
      x.TS = L.TS;
      x.Lcap = Lcap;
      x.R = misc->nruns;
      const bool small = (NI == 0) || misc->big == 0;
      const bool fin = (NF == 0) || misc->nonfinite == 0;
      if (small && fin)
        run_tiles<NI, NF, MM, true, true>(acc, x, sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, wid, nw, lane);
      else if (small)
        run_tiles<NI, NF, MM, true, false>(acc, x, sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, wid, nw, lane);
      else if (fin)
        run_tiles<NI, NF, MM, false, true>(acc, x, sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, wid, nw, lane);
      else
        run_tiles<NI, NF, MM, false, false>(acc, x, sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, wid, nw, lane);
    }
    __syncthreads();
  }
  acc.flush(sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, Lcap, lane);
  __syncthreads();

  // ---------------- CTA table -> provisional HBM table
  const int nloc = min(misc->nlocal, Lcap);
  if (tid == 0) atomicMax(&p.dbg[1], (unsigned long long)misc->nlocal);
  for (int i = tid; i < nloc * kM; i += nth) {
    const int s = i / kM;
    const int prov = sm.lprov[s];
    if (prov < 0) continue;
    const size_t g = (size_t)prov * kM + (i % kM);
    if (sm.cnt[i]) atomicAdd(&p.prov_count[g], (unsigned long long)sm.cnt[i]);
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      const unsigned long long v = sm.isum[(size_t)c * Lcap * kM + i];
      if (v) atomicAdd(&p.prov_isum[c][g], v);
    }
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      const double v = sm.fsum[(size_t)c * Lcap * kM + i];
      if (v != 0.0) atomicAdd(&p.prov_fsum[c][g], v);
    }
    if (MM & 1) atomicMin(&p.prov_min[g], sm.emin[i]);
    if (MM & 2) atomicMax(&p.prov_max[g], sm.emax[i]);
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
}

// ------------------------------------------------------------------ k_agg_minmax (pruned)
struct MMLayout {
  int Lcap, LH;
  int o_lkey, o_lstate, o_lprov, o_lrows, o_bmin, o_bmax, o_dirty, o_misc;
  int bytes;
};

__global__ void __launch_bounds__(kThreads) k_agg_minmax(AggPlan p, MMLayout L) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* lkey = (unsigned long long*)(smem + L.o_lkey);
  int* lstate = (int*)(smem + L.o_lstate);
  int* lprov = (int*)(smem + L.o_lprov);
  unsigned long long* lrows = (unsigned long long*)(smem + L.o_lrows);
  long long* bmin = (long long*)(smem + L.o_bmin);  // max_j MIN_j (enc), cached
  long long* bmax = (long long*)(smem + L.o_bmax);  // min_j MAX_j (enc), cached
  int* dirty = (int*)(smem + L.o_dirty);
  Misc* misc = (Misc*)(smem + L.o_misc);
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  const int Lcap = L.Lcap, LH = L.LH;

  for (int i = tid; i < LH; i += nth) lstate[i] = 0;
  for (int i = tid; i < Lcap; i += nth) {
    lrows[i] = 0;
    bmin[i] = kEncPosInf;   // nothing can be pruned until every world holds a value
    bmax[i] = kEncNegInf;
    dirty[i] = 0;
  }
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }
  __syncthreads();

  const int T = nth * 4;
  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * t_per;
  const int64_t t1 = min(ntiles, t0 + t_per);

  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t base = tile * T;
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int64_t r = base + k * nth + tid;
      bool valid = r < p.n_rows;
      bool cand = false;
      uint64_t m = 0;
      double v = 0.0;
      int prov = -1, s = -1;
      if (valid) {
        if (p.mask_in) {
          m = __ldg(p.mask_in + r);
          valid = m != 0;  // R21: a row in no world creates no group
        }
      }
      if (valid) {
        v = __ldg(p.mcol + r);
        const long long e = enc_f64(v);
        const uint64_t key = row_group_key(p, r);
        const int code = local_code(p, key, lkey, lstate, LH, lprov, Lcap, misc);
        if (code < kOvfBase) {
          s = code - 1;
          prov = lprov[s];
          atomicAdd(&lrows[s], 1ull);
          cand = (p.has_max && e > bmax[s]) || (p.has_min && e < bmin[s]);
        } else {
          prov = code - kOvfBase - 1;
          if (prov >= 0) atomicAdd(&p.prov_rows[prov], 1ull);
          cand = true;
        }
        if (prov < 0) cand = false;
        if (cand && !p.mask_in) m = pac_hash_dev((uint64_t)__ldg(p.pu_key + r), p.salt);
      }
      // warp-cooperative world update of the candidate rows (lane l: worlds l, l+32)
      unsigned cm = __ballot_sync(0xffffffffu, cand);
      while (cm) {
        const int src = __ffs(cm) - 1;
        cm &= cm - 1;
        const uint64_t mm = __shfl_sync(0xffffffffu, m, src);
        const double vv = __shfl_sync(0xffffffffu, v, src);
        const int pv = __shfl_sync(0xffffffffu, prov, src);
        const int ss = __shfl_sync(0xffffffffu, s, src);
        const long long e = enc_f64(vv);
        const size_t b = (size_t)pv * kM;
        if ((mm >> lane) & 1ull) {
          if (p.has_max) atomicMax(&p.prov_max[b + lane], e);
          if (p.has_min) atomicMin(&p.prov_min[b + lane], e);
        }
        if ((mm >> (lane + 32)) & 1ull) {
          if (p.has_max) atomicMax(&p.prov_max[b + lane + 32], e);
          if (p.has_min) atomicMin(&p.prov_min[b + lane + 32], e);
        }
        if (lane == 0 && ss >= 0) dirty[ss] = 1;
      }
    }
    __syncthreads();
    // refresh the bounds of the slots that received candidates (warp per slot)
    const int nloc = min(misc->nlocal, Lcap);
    for (int s = wid; s < nloc; s += nw) {
      if (!dirty[s]) continue;
      const int pv = lprov[s];
      if (pv >= 0) {
        const size_t b = (size_t)pv * kM;
        if (p.has_max) {
          long long a = min(*(volatile long long*)&p.prov_max[b + lane],
                            *(volatile long long*)&p.prov_max[b + lane + 32]);
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) a = min(a, __shfl_xor_sync(0xffffffffu, a, d));
          if (lane == 0) bmax[s] = a;
        }
        if (p.has_min) {
          long long a = max(*(volatile long long*)&p.prov_min[b + lane],
                            *(volatile long long*)&p.prov_min[b + lane + 32]);
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) a = max(a, __shfl_xor_sync(0xffffffffu, a, d));
          if (lane == 0) bmin[s] = a;
        }
      }
      if (lane == 0) dirty[s] = 0;
    }
    __syncthreads();
  }
  const int nloc = min(misc->nlocal, Lcap);
  for (int s = tid; s < nloc; s += nth)
    if (lprov[s] >= 0 && lrows[s]) atomicAdd(&p.prov_rows[lprov[s]], lrows[s]);
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

__global__ void k_radix_hist(const unsigned long long* keys, const int* Gdev, int shift,
                             int* hist /*[256][nblocks]*/, int nblocks) {
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

__global__ void __launch_bounds__(1024) k_radix_scan(int* hist, int total) {
  // exclusive scan of `total` ints by one CTA
  __shared__ int carry;
  __shared__ int wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < total; base += blockDim.x) {
    int i = base + threadIdx.x;
    int v = i < total ? hist[i] : 0;
    int x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int a = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += a;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int y = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
      int yy = y;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        int a = __shfl_up_sync(0xffffffffu, yy, d);
        if (lane >= d) yy += a;
      }
      wsum[lane] = yy - y;
    }
    __syncthreads();
    int excl = x - v + wsum[w] + carry;
    if (i < total) hist[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
}

__global__ void k_radix_scatter(const unsigned long long* kin, const int* iin, unsigned long long* kout,
                                int* iout, const int* Gdev, int shift, const int* hist, int nblocks) {
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
        a |= p.prov_max[pb + lane] != kEncNegInf;
        b |= p.prov_max[pb + lane + 32] != kEncNegInf;
      }
      if (p.has_min) {
        a |= p.prov_min[pb + lane] != kEncPosInf;
        b |= p.prov_min[pb + lane + 32] != kEncPosInf;
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
        else if (kd == 3) ((double*)w)[ob + j] = dec_f64(p.prov_min[pb + j]);
        else if (kd == 4) ((double*)w)[ob + j] = dec_f64(p.prov_max[pb + j]);
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
      o_perm, o_sk0, o_si0, o_sk1, o_si1, o_hist, o_meta, bytes;
  int64_t Hcap;
  int nblocks;
};

static WsLayout ws_layout(const AccSet& A, int64_t G_cap) {
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
  w.o_ctr = take(64);  // gcounter, Gdev, gmaxabs
  w.o_pkey = take(8 * Gc);
  w.o_prows = take(8 * Gc);
  w.o_pcount = A.has_count ? take(8 * Gc * kM) : 0;
  for (int c = 0; c < 2; ++c) w.o_pisum[c] = c < A.ni ? take(8 * Gc * kM) : 0;
  for (int c = 0; c < 2; ++c) w.o_pfsum[c] = c < A.nf ? take(8 * Gc * kM) : 0;
  w.o_pmin = A.has_min ? take(8 * Gc * kM) : 0;
  w.o_pmax = A.has_max ? take(8 * Gc * kM) : 0;
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

static int raw_tile_bytes(const AccSet& A, int T, int key_bytes) {
  const int cols8 = 1 + A.ni + A.nf + ((A.has_min || A.has_max) ? 1 : 0);
  return cols8 * T * 8 + ((key_bytes * T + 15) & ~15) + 16 * PAC_MAX_KEYS;
}

static SmemLayout make_layout(const AccSet& A, int T, int Lcap, int key_bytes = 8) {
  SmemLayout L{};
  L.T = T;
  L.TS = T + 8 * Lcap;  // slot-sorted staging, each slot padded to a multiple of 8 rows
  L.Lcap = Lcap;
  L.LH = (int)next_pow2(std::max(4 * Lcap, 256));
  int off = 0;
  auto take = [&](int bytes) {
    int o = off;
    off += (std::max(bytes, 16) + 15) & ~15;
    return o;
  };
  const bool mm = A.has_min || A.has_max;
  const int TS = L.TS;
  L.o_isum = take(A.ni * Lcap * kM * 8);
  L.o_fsum = take(A.nf * Lcap * kM * 8);
  L.o_min = take(A.has_min ? Lcap * kM * 8 : 0);
  L.o_max = take(A.has_max ? Lcap * kM * 8 : 0);
  L.o_lrows = take(Lcap * 8);
  L.o_lkey = take(L.LH * 8);
  L.o_mask = take(TS * 8);
  L.o_ival = take(A.ni * TS * 8);
  L.o_fval = take(A.nf * TS * 8);
  L.o_mval = take(mm ? TS * 8 : 0);
  L.o_i32 = take(A.ni * TS * 4);
  L.o_cnt = take(Lcap * kM * 4);
  L.o_lstate = take(L.LH * 4);
  L.o_lprov = take(Lcap * 4);
  L.o_hist = take(Lcap * 4);
  L.o_offs = take(Lcap * 4);
  L.o_runoffs = take((Lcap + 1) * 4);
  L.o_ucnt = take((T / 32) * Lcap * 2);
  L.o_queue = take(T * 4);
  L.o_slot = take(T * 2);
  L.o_rank = take(T);
  L.o_tcs = take(5 * 32 * 8);
  L.o_raw = take(raw_tile_bytes(A, T, key_bytes));
  L.o_mbar = take(16);
  L.o_misc = take(sizeof(Misc));
  L.bytes = off;
  return L;
}

// Local slot capacity: min(G_cap, 256).  Preference: all wanted slots with three CTAs per SM
// (tile 1024, then 512), then two CTAs per SM, then one CTA per SM with as many slots as
// fit.  PAC_TILE=512|1024 forces the tile size (experiments).
static bool choose_layout(const AccSet& A, int64_t G_cap, int smem_max, int key_bytes, SmemLayout* out) {
  const int want = (int)std::min<int64_t>(std::max<int64_t>(G_cap, 1), 256);
  const char* force = getenv("PAC_TILE");
  const int tiles_fixed[2] = {force ? atoi(force) : 1024, force ? atoi(force) : 512};
  for (int per_sm : {3, 2}) {
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
  if (best < 1) return false;
  *out = make_layout(A, bestT, best, key_bytes);
  return true;
}

static MMLayout mm_layout(int64_t G_cap, int smem_max) {
  MMLayout L{};
  int Lcap = (int)std::min<int64_t>(std::max<int64_t>(G_cap, 1), 4096);
  for (;;) {
    L.Lcap = Lcap;
    L.LH = (int)next_pow2(std::max(4 * Lcap, 256));
    int off = 0;
    auto take = [&](int bytes) {
      int o = off;
      off += (bytes + 15) & ~15;
      return o;
    };
    L.o_lkey = take(L.LH * 8);
    L.o_lrows = take(Lcap * 8);
    L.o_bmin = take(Lcap * 8);
    L.o_bmax = take(Lcap * 8);
    L.o_lstate = take(L.LH * 4);
    L.o_lprov = take(Lcap * 4);
    L.o_dirty = take(Lcap * 4);
    L.o_misc = take(sizeof(Misc));
    L.bytes = off;
    if (L.bytes <= smem_max || Lcap == 1) break;
    Lcap /= 2;
  }
  return L;
}

template <int NI, int NF, int MM>
static cudaError_t launch_smem(const AggPlan& p, const SmemLayout& L, int sms, cudaStream_t st) {
  auto k = k_agg_tiles<NI, NF, MM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kTileThreads, L.bytes);
  per_sm = std::max(1, per_sm);
  const int64_t tiles = (p.n_rows + L.T - 1) / L.T;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * per_sm));
  k<<<grid, kTileThreads, L.bytes, st>>>(p, L);
  note_launch();
  return cudaGetLastError();
}

typedef cudaError_t (*LaunchFn)(const AggPlan&, const SmemLayout&, int, cudaStream_t);

#define PAC_MM_ROW(NI, NF) {launch_smem<NI, NF, 0>, launch_smem<NI, NF, 1>, launch_smem<NI, NF, 2>, launch_smem<NI, NF, 3>}
static const LaunchFn kLaunch[3][3][4] = {
    {PAC_MM_ROW(0, 0), PAC_MM_ROW(0, 1), PAC_MM_ROW(0, 2)},
    {PAC_MM_ROW(1, 0), PAC_MM_ROW(1, 1), PAC_MM_ROW(1, 2)},
    {PAC_MM_ROW(2, 0), PAC_MM_ROW(2, 1), PAC_MM_ROW(2, 2)},
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
void profile_begin(cudaStream_t st);
void profile_end(cudaStream_t st);

}  // namespace pac

using namespace pac;

extern "C" int pac_mask(const int64_t* d_pu_key, int64_t n, uint64_t salt, uint64_t* d_mask,
                        pac_stream_t stream) {
  if (n < 0 || (n > 0 && (!d_pu_key || !d_mask))) return PAC_E_INVAL;
  if (n == 0) return PAC_OK;
  int sms = 148, smem = 0;
  if (device_info(&sms, &smem) != PAC_OK) return PAC_E_CUDA;
  int64_t blocks = (n + 255) / 256;
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

extern "C" int pac_agg_grouped(const int64_t* d_pu_key, const uint64_t* d_mask, uint64_t salt,
                               const pac_key_col* keys, int n_keys, const pac_agg_spec* aggs, int n_aggs,
                               int64_t n_rows, const pac_table* out, int64_t G_cap, void* d_ws,
                               size_t ws_bytes, pac_stream_t stream) {
  if (n_rows < 0 || !out || G_cap < 1) return PAC_E_INVAL;
  // exactly one mask source (an empty input may arrive as NULL pointers)
  if (d_pu_key && d_mask) return PAC_E_INVAL;
  if (!d_pu_key && !d_mask && n_rows > 0) return PAC_E_INVAL;
  if (n_keys < 0 || n_keys > PAC_MAX_KEYS || (n_keys > 0 && !keys)) return PAC_E_INVAL;
  int width = 0;
  for (int c = 0; c < n_keys; ++c) {
    int w = keys[c].elem_bytes;
    if ((w != 1 && w != 2 && w != 4 && w != 8) || (!keys[c].d_col && n_rows > 0)) return PAC_E_INVAL;
    width += w;
  }
  if (width > 8) return PAC_E_INVAL;
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
  int* Gdev = (int*)(ws + W.o_ctr + 4);
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
  int* perm = (int*)(ws + W.o_perm);
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

  cudaError_t e = cudaSuccess;
  if (n_rows > 0) {
    if (!A.has_count) {
      MMLayout L = mm_layout(G_cap, smem_max);
      e = cudaFuncSetAttribute(k_agg_minmax, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
      if (e != cudaSuccess) return PAC_E_CUDA;
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_agg_minmax, kThreads, L.bytes);
      per_sm = std::max(1, per_sm);
      int64_t tiles = (n_rows + kThreads * 4 - 1) / (kThreads * 4);
      int grid = (int)std::min<int64_t>(tiles, (int64_t)sms * per_sm);
      profile_begin(st);
      k_agg_minmax<<<grid, kThreads, L.bytes, st>>>(p, L);
      note_launch();
      e = cudaGetLastError();
      profile_end(st);
    } else {
      SmemLayout L{};
      if (!choose_layout(A, G_cap, smem_max, width, &L)) return PAC_E_INVAL;
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
        add(d_mask ? (const void*)d_mask : (const void*)d_pu_key, 8);
        for (int c = 0; c < A.ni; ++c) add(A.icol[c], 8);
        for (int c = 0; c < A.nf; ++c) add(A.fcol[c], 8);
        if (A.has_min || A.has_max) add(A.mcol, 8);
        for (int c = 0; c < n_keys; ++c) add(keys[c].d_col, keys[c].elem_bytes);
        int copied = 0;
        for (int i = 0; i < p.nraw; ++i) copied += L.T * p.raw_eb[i];
        p.raw_bytes = copied;
        p.tma_ok = (aligned && !getenv("PAC_NO_TMA")) ? 1 : 0;
        p.ablate = getenv("PAC_ABLATE") ? atoi(getenv("PAC_ABLATE")) : 0;
      }
      if (getenv("PAC_DEBUG"))
        fprintf(stderr, "[libpac] k_agg_tiles<%d,%d,%d> T=%d Lcap=%d LH=%d smem=%d B (G_cap=%lld)\n", A.ni,
                A.nf, (A.has_min ? 1 : 0) | (A.has_max ? 2 : 0), L.T, L.Lcap, L.LH, L.bytes, (long long)G_cap);
      const int mm = (A.has_min ? 1 : 0) | (A.has_max ? 2 : 0);
      profile_begin(st);
      e = kLaunch[A.ni][A.nf][mm](p, L, sms, st);
      profile_end(st);
    }
    if (e != cudaSuccess) return PAC_E_CUDA;
  }
  k_finish_count<<<1, 1, 0, st>>>(p, n_keys, out->d_num_groups, out->d_status, Gdev);
  note_launch();
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
    for (int pass = 0; pass < 8; ++pass) {
      unsigned long long* ko = (pass & 1) ? k1 : k0;
      int* io = (pass & 1) ? i1 : i0;
      if (pass == 7) io = perm;
      k_radix_hist<<<W.nblocks, 256, 0, st>>>(kin, Gdev, 8 * pass, hist, W.nblocks);
      k_radix_scan<<<1, 1024, 0, st>>>(hist, 256 * W.nblocks);
      k_radix_scatter<<<W.nblocks, 32, 0, st>>>(kin, iin, ko, io, Gdev, 8 * pass, hist, W.nblocks);
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
__global__ void k_rederive(pac_table t, int64_t G_cap, int has_count, int mm_a, int mm_kind) {
  const int64_t G = min(*t.d_num_groups, G_cap);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int64_t g = blockIdx.x * wpb + (threadIdx.x >> 5); g < G; g += (int64_t)gridDim.x * wpb) {
    bool a, b;
    if (has_count) {
      a = t.d_count[g * kM + lane] > 0;
      b = t.d_count[g * kM + lane + 32] > 0;
    } else {
      const double* w = (const double*)t.d_world[mm_a];
      const double s = mm_kind == PAC_MIN_F64 ? INFINITY : -INFINITY;
      a = w[g * kM + lane] != s;
      b = w[g * kM + lane + 32] != s;
    }
    uint64_t K = (uint64_t)__ballot_sync(0xffffffffu, a) | ((uint64_t)__ballot_sync(0xffffffffu, b) << 32);
    if (lane == 0) t.d_presence[g] = K;
  }
}

__global__ void k_remap(pac_table in, const uint64_t* ukeys, int64_t Gu, pac_table out, int n_aggs,
                        const int* kinds, int has_count) {
  const int64_t Gin = *in.d_num_groups;
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
        const int k = kinds[a];
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
  if (!t || G_cap < 1) return PAC_E_INVAL;
  int rc = build_accs(aggs, n_aggs, &A, true, true);  // only the kinds matter here
  if (rc) return rc;
  int mm_a = -1, mm_kind = 0;
  for (int a = 0; a < n_aggs; ++a)
    if (aggs[a].kind == PAC_MIN_F64 || aggs[a].kind == PAC_MAX_F64) {
      mm_a = a;
      mm_kind = aggs[a].kind;
      break;
    }
  if (A.has_count ? !t->d_count : (mm_a < 0 || !t->d_world[mm_a])) return PAC_E_INVAL;
  int blocks = (int)std::min<int64_t>((G_cap + 7) / 8, 148 * 16);
  k_rederive<<<std::max(1, blocks), 256, 0, (cudaStream_t)stream>>>(*t, G_cap, A.has_count, mm_a, mm_kind);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_table_remap(const pac_table* in, const uint64_t* d_union_keys, int64_t G_union,
                               const pac_agg_spec* aggs, int n_aggs, int64_t G_cap_in, const pac_table* out,
                               pac_stream_t stream) {
  AccSet A;
  if (!in || !out || !d_union_keys || G_union < 1 || G_cap_in < 1) return PAC_E_INVAL;
  int rc = build_accs(aggs, n_aggs, &A, true, true);  // only the kinds matter here
  if (rc) return rc;
  // kinds are passed by value through a small device buffer embedded in the launch
  static int* d_kinds = nullptr;
  if (!d_kinds && cudaMalloc(&d_kinds, sizeof(int) * PAC_MAX_AGGS) != cudaSuccess) return PAC_E_CUDA;
  int hk[PAC_MAX_AGGS] = {0};
  for (int a = 0; a < n_aggs; ++a) hk[a] = aggs[a].kind;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(d_kinds, hk, sizeof(hk), cudaMemcpyHostToDevice, st) != cudaSuccess) return PAC_E_CUDA;
  int blocks = (int)std::min<int64_t>((G_union + 7) / 8, 148 * 16);
  k_remap<<<std::max(1, blocks), 256, 0, st>>>(*in, d_union_keys, G_union, *out, n_aggs, d_kinds, A.has_count);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
