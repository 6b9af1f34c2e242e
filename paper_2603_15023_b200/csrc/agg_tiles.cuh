// libpac: the k_agg_tiles kernel family -- shared by agg.cu and the explicit
// instantiation units agg_inst_ni{0,1,2}.cu (split so the 72 kernels compile in parallel).
#pragma once
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace pac {

constexpr int kThreads = 512;      // k_agg_minmax
constexpr int kTileThreads = 256;  // k_agg_tiles
#ifndef PAC_TILE_FLUSH
#define PAC_TILE_FLUSH 0  // 1: warp accumulators flushed at the end of every tile's phase C
#endif
#ifndef PAC_TILE_MINB
#define PAC_TILE_MINB 3  // min resident CTAs per SM the register allocation targets
#endif
constexpr int kOvfBase = 0x20000000;
constexpr int kUnresolved = 0x7FFFFFFF;  // local_code(defer): not in the CTA dictionary, HBM slot not looked up
#ifdef PAC_ABLATE_BUILD
constexpr bool kAblate = true;   // profiling build: PAC_ABLATE switches phases off
#else
constexpr bool kAblate = false;
#endif  // local-dict code for keys without a local slot
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
  int ablate;  // profiling builds only (-DPAC_ABLATE_BUILD, env PAC_ABLATE): 1 = no draws, 2 = no A3, 4 = no phase C
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
  long long* gbmin;  // per provisional slot: a recent max_j MIN_j (enc), hint for the pruning bounds
  long long* gbmax;  // per provisional slot: a recent min_j MAX_j (enc)
  // deferred HBM tier (agg.cu k_spill_*): rows of groups without a CTA-local slot are appended
  // here (record i: sp_prov[i] = the HBM slot, or -2 when the CTA dictionary did not know it
  // (resolved from the group key sp_gkey[i] after the pass), sp_key[i] = the pu key, or the
  // mask when mask_in, raw 8-byte values sp_val[k * sp_cap + i] in column order) and
  // aggregated after the pass, grouped by slot; sp_cap = 0: direct atomics
  int64_t sp_cap;
  unsigned long long* sp_n;  // records reserved (may exceed sp_cap: the excess took atomics)
  int* sp_prov;
  unsigned long long* sp_gkey;
  unsigned long long* sp_key;
  unsigned long long* sp_val;
  int* sp_cnt;  // [G_cap] records per provisional slot
  int m128;     // 1: provisional world rows are 128 words (k_agg_tiles128, agg128.cu)
  // partition-first input (part.cu): the CTA takes row ranges [x, y) from `units` through the
  // global counter unit_ctr and flushes and resets its table after each (k_agg_tiles_tm)
  const longlong2* units;
  const int* n_units;
  int* unit_ctr;
};

struct SmemLayout {
  int T, TS, Lcap, LH;
  int o_lkey, o_lstate, o_lprov, o_lrows, o_cnt, o_isum, o_fsum, o_min, o_max;
  int o_mask, o_slot, o_rank, o_ucnt, o_queue, o_ival, o_rdesc, o_fval, o_mval, o_hist, o_offs,
      o_runoffs, o_xcs, o_raw, o_mbar, o_misc;
  int bytes;
  int tm;  // 1: the CTA table lives in TMEM (k_agg_tiles_tm), no smem table
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

// Shared-memory layout of k_agg_tiles (host: agg.cu make_layout; also usable at compile time).
__host__ __device__ constexpr int lay_take(int& off, int bytes) {
  const int o = off;
  off += ((bytes > 16 ? bytes : 16) + 15) & ~15;
  return o;
}
__host__ __device__ constexpr int lay_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}
__host__ __device__ constexpr SmemLayout tile_layout(int ni, int nf, int has_min, int has_max, int T, int Lcap,
                                                     int raw_bytes, int tm) {
  SmemLayout L{};
  L.tm = tm;
  const int tl = tm ? 0 : Lcap;  // slots of the smem CTA table (none in TMEM mode)
  L.T = T;
  L.TS = T + 8 * Lcap;  // slot-sorted staging, each slot padded to a multiple of 8 rows
  L.Lcap = Lcap;
  L.LH = lay_pow2(4 * Lcap > 256 ? 4 * Lcap : 256);
  int off = 0;
  const int TS = L.TS;
  const bool mm = has_min || has_max;
  L.o_isum = lay_take(off, ni * tl * kM * 8);
  L.o_fsum = lay_take(off, nf * tl * kM * 8);
  L.o_min = lay_take(off, has_min ? tl * kM * 8 : 0);
  L.o_max = lay_take(off, has_max ? tl * kM * 8 : 0);
  L.o_lrows = lay_take(off, Lcap * 8);
  L.o_lkey = lay_take(off, L.LH * 8);
  L.o_mask = lay_take(off, TS * 8);
  L.o_ival = lay_take(off, ni * TS * 8);
  L.o_fval = lay_take(off, nf * TS * 8);
  L.o_mval = lay_take(off, mm ? TS * 8 : 0);
  L.o_rdesc = lay_take(off, (T / 32 + Lcap + 1) * 4);
  L.o_cnt = lay_take(off, tl * kM * 4);
  L.o_lstate = lay_take(off, L.LH * 4);
  L.o_lprov = lay_take(off, Lcap * 4);
  L.o_hist = lay_take(off, Lcap * 4);
  L.o_offs = lay_take(off, Lcap * 4);
  L.o_runoffs = lay_take(off, (Lcap + 1) * 4);
  L.o_ucnt = lay_take(off, (T / 32) * Lcap * 2);
  L.o_xcs = lay_take(off, 32 * 16 + 32 * 8);
  L.o_queue = lay_take(off, T * 4);
  L.o_slot = lay_take(off, T * 2);
  L.o_rank = lay_take(off, T);
  L.o_mbar = lay_take(off, 16);
  L.o_misc = lay_take(off, (int)sizeof(Misc));
  L.o_raw = lay_take(off, raw_bytes);  // last: every other offset is independent of the columns staged
  L.bytes = off;
  return L;
}

// ------------------------------------------------------------------ dictionaries
// 64 consecutive 8-byte words = v, as 16-byte stores (one thread; slot rows are 512 B aligned)
__device__ __forceinline__ void fill_world_row(void* dst, long long v) {
  longlong2* d = (longlong2*)dst;
  const longlong2 x = make_longlong2(v, v);
#pragma unroll 8
  for (int i = 0; i < kM / 2; ++i) d[i] = x;
}

__device__ __forceinline__ void init_prov_slot(const AggPlan& p, int prov, uint64_t key) {
  p.prov_key[prov] = key;
  p.prov_rows[prov] = 0;
  const int halves = p.m128 ? 2 : 1;
  for (int h = 0; h < halves; ++h) {
    const size_t b = ((size_t)prov * halves + h) * kM;
    if (p.has_count) fill_world_row(p.prov_count + b, 0);
    for (int c = 0; c < p.ni; ++c) fill_world_row(p.prov_isum[c] + b, 0);
    for (int c = 0; c < p.nf; ++c) fill_world_row(p.prov_fsum[c] + b, 0);  // +0.0
    if (p.has_min) fill_world_row(p.prov_min + b, kMinEmpty);
    if (p.has_max) fill_world_row(p.prov_max + b, kMaxEmpty);
  }
  if (p.gbmin) p.gbmin[prov] = kMinEmpty;
  if (p.gbmax) p.gbmax[prov] = kMaxEmpty;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* a) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// Insert-or-find `key` in the HBM dictionary; returns the provisional slot, or -1 when
// the capacity G_cap is exhausted (the table is then flagged by the finish kernel).
static __device__ int global_slot(const AggPlan& p, uint64_t key) {
  uint32_t h = dict_hash(key) & p.hmask;
  for (;;) {
    // acquire: a published state orders the key read after it (the writer releases with a
    // fence before publishing)
    const int st = ld_acquire_gpu(&p.gstate[h]);
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
    if (*(volatile unsigned long long*)&p.gkey[h] == key) return st - 1;
    h = (h + 1) & p.hmask;
  }
}

// CTA-local dictionary: code = s+1 for local slot s (< Lcap); kOvfBase + prov + 1 for a
// key that has no local slot (its rows go straight to the HBM table; prov -1 = dropped).
// An empty entry is claimed with CAS first; only then is the entry counted, so concurrent
// contenders for one key never inflate the fill count.  At half full no more keys are
// inserted (their rows use the HBM dictionary directly).
// defer: a key the full dictionary cannot take returns kUnresolved instead of its HBM slot (the
// deferred tier resolves it after the pass, k_spill_resolve).
// acquire load of a shared-memory word (an LDS: CTA-scope acquire on shared memory needs no fence)
__device__ __forceinline__ int ld_acquire_cta_shared(const int* a) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(a))
               : "memory");
  return v;
}

static __device__ int local_code(const AggPlan& p, uint64_t key, unsigned long long* lkey, int* lstate,
                          int LH, int* lprov, int Lcap, Misc* misc, bool defer = false) {
  uint32_t h = (((uint32_t)key ^ (uint32_t)(key >> 32)) * 0x9E3779B1u) >> 16 & (LH - 1);
  for (;;) {
    // acquire: a published state (the writer fences before publishing) orders the key read after it
    const int st = ld_acquire_cta_shared(&lstate[h]);
    if (st == 0) {
      // a full dictionary stays full: skip the claim-and-release
      if (*(volatile int*)&misc->ndict >= LH / 2) return defer ? kUnresolved : kOvfBase + global_slot(p, key) + 1;
      if (atomicCAS(&lstate[h], 0, -1) == 0) {
        if (atomicAdd(&misc->ndict, 1) >= LH / 2) {  // too full: release, use the HBM tier
          atomicSub(&misc->ndict, 1);
          __threadfence_block();
          atomicExch(&lstate[h], 0);
          return defer ? kUnresolved : kOvfBase + global_slot(p, key) + 1;
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

// ------------------------------------------------------------------ k_agg_tiles (v4)
// Bit-matrix transpose of a 32-row run: on input lane r holds row r's
// 32-bit mask word; on output lane c holds the pattern of world c over the run.  Stage s
// swaps the off-diagonal s x s blocks: the partner's word is rotated by s (low lane) or
// 32-s (high lane) with one funnel shift and merged with one LOP3 under a per-lane mask.
// The per-lane constants live in registers: five keep masks and the five rotate amounts
// packed 6 bits apart (the funnel shift only reads the low 5 bits of its amount).
struct XposeConst {
  uint32_t keep[5];
  uint32_t amt;
};

__device__ __forceinline__ XposeConst make_xpose(int lane) {
  XposeConst c;
  c.amt = 0;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int s = 16 >> i;
    const uint32_t M = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu
                     : s == 2 ? 0x33333333u : 0x55555555u;
    const bool up = (lane & s) != 0;
    c.keep[i] = up ? ~M : M;
    c.amt |= (uint32_t)(up ? 32 - s : s) << (6 * i);
  }
  return c;
}

// The constants of one lane, kept in shared memory (xcs[lane] = keep 0-3, xcs2[lane] = keep 4 and
// the packed amounts) and loaded with two vector loads per run: cheaper than keeping six
// registers live across the whole tile loop.
__device__ __forceinline__ void store_xpose(uint4* xcs, uint2* xcs2, int lane) {
  const XposeConst c = make_xpose(lane);
  xcs[lane] = make_uint4(c.keep[0], c.keep[1], c.keep[2], c.keep[3]);
  xcs2[lane] = make_uint2(c.keep[4], c.amt);
}
__device__ __forceinline__ XposeConst load_xpose(const uint4* xcs, const uint2* xcs2, int lane) {
  XposeConst c;
  const uint4 a = xcs[lane];
  const uint2 b = xcs2[lane];
  c.keep[0] = a.x;
  c.keep[1] = a.y;
  c.keep[2] = a.z;
  c.keep[3] = a.w;
  c.keep[4] = b.x;
  c.amt = b.y;
  return c;
}

__device__ __forceinline__ void transpose2x32(uint32_t& a, uint32_t& b, const XposeConst& c) {
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int s = 16 >> i;
    const uint32_t r = c.amt >> (6 * i);
    const uint32_t ya = __shfl_xor_sync(0xffffffffu, a, s);
    const uint32_t yb = __shfl_xor_sync(0xffffffffu, b, s);
    a = (a & c.keep[i]) | (__funnelshift_l(ya, ya, r) & ~c.keep[i]);
    b = (b & c.keep[i]) | (__funnelshift_l(yb, yb, r) & ~c.keep[i]);
  }
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  double r;
  asm volatile(
      "{\n .reg .b32 lo, hi, rlo, rhi;\n mov.b64 {lo, hi}, %1;\n"
      " shfl.sync.idx.b32 rlo, lo, %2, 0x1f, 0xffffffff;\n"
      " shfl.sync.idx.b32 rhi, hi, %2, 0x1f, 0xffffffff;\n mov.b64 %0, {rlo, rhi};\n}"
      : "=d"(r) : "d"(v), "r"(src));
  return r;
}

__device__ __forceinline__ bool finite_bits(double v) {
  return (__double2hiint(v) & 0x7FF00000) != 0x7FF00000;
}

// 64-bit add into shared memory as two 32-bit atomics (the carry of the low word is the
// carry of this addition, whatever other adds interleave): cheaper than the CAS loop a
// 64-bit shared-memory atomicAdd compiles to.
__device__ __forceinline__ void smem_add_u64(unsigned long long* addr, unsigned long long v) {
  unsigned* w = reinterpret_cast<unsigned*>(addr);
  const unsigned lo = (unsigned)v, hi = (unsigned)(v >> 32);
  const unsigned old = atomicAdd(w, lo);
  const unsigned carry = (old + lo) < old ? 1u : 0u;
  if (hi + carry) atomicAdd(w + 1, hi + carry);
}

// Register accumulators of the slot a warp is currently working on (lane: worlds lane, lane+32).
template <int NI, int NF, int MM>
struct WarpAcc {
  int cur;
  unsigned c0, c1;
  long long ia0[NI > 0 ? NI : 1], ia1[NI > 0 ? NI : 1];
  double fa0[NF > 0 ? NF : 1], fa1[NF > 0 ? NF : 1];
  long long mn0, mn1, mx0, mx1;  // enc_f64 extremes (R31 total order), kMinEmpty / kMaxEmpty when empty

  __device__ __forceinline__ void reset() {
    c0 = c1 = 0;
#pragma unroll
    for (int c = 0; c < NI; ++c) ia0[c] = ia1[c] = 0;
#pragma unroll
    for (int c = 0; c < NF; ++c) fa0[c] = fa1[c] = 0.0;
    mn0 = mn1 = kMinEmpty;
    mx0 = mx1 = kMaxEmpty;
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
      smem_add_u64(&isum[(size_t)c * Lcap * kM + b + lane], (unsigned long long)ia0[c]);
      smem_add_u64(&isum[(size_t)c * Lcap * kM + b + lane + 32], (unsigned long long)ia1[c]);
    }
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      if (fa0[c] != 0.0) atomicAdd(&fsum[(size_t)c * Lcap * kM + b + lane], fa0[c]);
      if (fa1[c] != 0.0) atomicAdd(&fsum[(size_t)c * Lcap * kM + b + lane + 32], fa1[c]);
    }
    if (MM & 1) {
      if (mn0 != kMinEmpty) atomicMin(&emin[b + lane], mn0);
      if (mn1 != kMinEmpty) atomicMin(&emin[b + lane + 32], mn1);
    }
    if (MM & 2) {
      if (mx0 != kMaxEmpty) atomicMax(&emax[b + lane], mx0);
      if (mx1 != kMaxEmpty) atomicMax(&emax[b + lane + 32], mx1);
    }
    reset();
  }
};

// Run descriptor (phase B): one 32-row run of one slot, packed into 32 bits.
__device__ __forceinline__ uint32_t pack_run(int beg, int slot, int len) {
  return (uint32_t)beg | ((uint32_t)slot << 16) | ((uint32_t)(len - 1) << 26);
}

struct RunCtx {  // read-only per-tile state of phase C
  const unsigned long long* smask;
  const long long* sival;
  const double* sfval;
  const long long* smval;
  const uint32_t* rdesc;
  const uint4* xcs;
  const uint2* xcs2;
  int TS, Lcap, R;
};

// World-parallel update of one run of len <= 32 same-slot rows (row 0 at smask[0]; column c
// of the int64 / f64 values at sival[c * istride] / sfval[c * fstride]).  Rows [len, 8*ceil(len/8))
// must hold finite values (zero padding): they enter table entries that are never looked up.
// SMALL: |int64 values| < 2^26, so 4-row subset sums and 32-row partials fit int32; FIN: the
// f64 values are finite, so the f64 nibble tables are built with exact 0/1 FMAs.  Both hold
// for the synthetic workloads; GENERIC instances test them at run time.
template <int NI, int NF, int MM, bool GENERIC>
__device__ __forceinline__ void run_body(WarpAcc<NI, NF, MM>& acc, const unsigned long long* __restrict__ smask,
                                         const long long* __restrict__ sival, int istride,
                                         const double* __restrict__ sfval, int fstride,
                                         const long long* __restrict__ smval, int len, const XposeConst& xc, int lane,
                                         bool small_rt = true, bool fin_rt = true) {
  // GENERIC = false: the common case (SMALL and FIN) with no runtime tests inside the loop
  const bool SMALL = GENERIC ? small_rt : true;
  const bool FIN = GENERIC ? fin_rt : true;
  const int tsrc = (lane >> 4) << 2;
  const int ib0 = lane & 1, ib1 = (lane >> 1) & 1, ib2 = (lane >> 2) & 1, ib3 = (lane >> 3) & 1;
  const double db0 = ib0, db1 = ib1, db2 = ib2, db3 = ib3;
  const uint64_t m = lane < len ? smask[lane] : 0ull;
  uint32_t P = (uint32_t)m, Q = (uint32_t)(m >> 32);
  transpose2x32(P, Q, xc);
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
    const int row = 8 * q + tsrc;
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      const longlong2 u = *(const longlong2*)(sival + c * istride + row);
      const longlong2 w = *(const longlong2*)(sival + c * istride + row + 2);
      if (SMALL) {
        const int t = (int)u.x * ib0 + (int)u.y * ib1 + (int)w.x * ib2 + (int)w.y * ib3;
        rs0[c] += __shfl_sync(0xffffffffu, t, a0) + __shfl_sync(0xffffffffu, t, b0);
        rs1[c] += __shfl_sync(0xffffffffu, t, a1) + __shfl_sync(0xffffffffu, t, b1);
      } else {
        const long long t = u.x * ib0 + u.y * ib1 + w.x * ib2 + w.y * ib3;
        acc.ia0[c] += __shfl_sync(0xffffffffu, t, a0) + __shfl_sync(0xffffffffu, t, b0);
        acc.ia1[c] += __shfl_sync(0xffffffffu, t, a1) + __shfl_sync(0xffffffffu, t, b1);
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
      acc.fa0[c] += shfl_d(t, a0);
      acc.fa0[c] += shfl_d(t, b0);
      acc.fa1[c] += shfl_d(t, a1);
      acc.fa1[c] += shfl_d(t, b1);
    }
    if (MM) {  // extremes on enc_f64 encodings (R31 total order: NaN above +inf); the
               // empty subset is the sentinel, which every encoded value beats
      const longlong2 u = *(const longlong2*)(smval + row);
      const longlong2 w = *(const longlong2*)(smval + row + 2);
      if (MM & 1) {
        long long t = ib0 ? u.x : kMinEmpty;
        if (ib1) t = min(t, u.y);
        if (ib2) t = min(t, w.x);
        if (ib3) t = min(t, w.y);
        acc.mn0 = min(acc.mn0, min(__shfl_sync(0xffffffffu, t, a0), __shfl_sync(0xffffffffu, t, b0)));
        acc.mn1 = min(acc.mn1, min(__shfl_sync(0xffffffffu, t, a1), __shfl_sync(0xffffffffu, t, b1)));
      }
      if (MM & 2) {
        long long t = ib0 ? u.x : kMaxEmpty;
        if (ib1) t = max(t, u.y);
        if (ib2) t = max(t, w.x);
        if (ib3) t = max(t, w.y);
        acc.mx0 = max(acc.mx0, max(__shfl_sync(0xffffffffu, t, a0), __shfl_sync(0xffffffffu, t, b0)));
        acc.mx1 = max(acc.mx1, max(__shfl_sync(0xffffffffu, t, a1), __shfl_sync(0xffffffffu, t, b1)));
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

// Phase C of one tile for one warp: runs [r0, r1) of the tile's slot-sorted rows.
template <int NI, int NF, int MM, bool GENERIC>
__device__ __forceinline__ void run_tiles(WarpAcc<NI, NF, MM>& acc, const RunCtx& x,
                                          unsigned* cnt, unsigned long long* isum, double* fsum, long long* emin,
                                          long long* emax, int wid, int nw, int lane, bool small, bool fin) {
  const int R = x.R, TS = x.TS;
  const int r0 = (R * wid) / nw;
  const int r1 = (R * (wid + 1)) / nw;
#pragma unroll 1
  for (int r = r0; r < r1; ++r) {
    const uint32_t d = x.rdesc[r];
    const int beg = (int)(d & 0xFFFFu);
    const int s = (int)((d >> 16) & 0x3FFu);
    const int len = (int)(d >> 26) + 1;
    if (s != acc.cur) {
      acc.flush(cnt, isum, fsum, emin, emax, x.Lcap, lane);
      acc.cur = s;
    }
    const XposeConst xc = load_xpose(x.xcs, x.xcs2, lane);
    run_body<NI, NF, MM, GENERIC>(acc, x.smask + beg, x.sival + beg, TS, x.sfval + beg, TS, x.smval + beg, len,
                                  xc, lane, small, fin);
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
  uint32_t* rdesc;            // [runs] run descriptors (pack_run)
  double* sfval;              // [NF][TS]
  long long* smval;           // [TS] enc_f64 of the MIN/MAX column
  unsigned short* sslot;      // [T]
  unsigned char* srank;       // [T]
  unsigned short* ucnt;       // [units][Lcap]
  unsigned short* qpos;       // [T]
  unsigned short* qrow;       // [T]
  int* hist;
  int* offs;
  int* runoffs;
  uint4* xcs;                 // [32] transpose constants (store_xpose)
  uint2* xcs2;                // [32]
  Misc* misc;
  unsigned char* raw;         // staged raw tile: 8-byte columns k at k*T*8, then key columns
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

// Per-tile phases.  Pipeline of one CTA, 4 barriers per tile:
//   [C(t-1) | A1(t)]  sync  B2(t)  sync  B3(t)  sync  A2+A3(t)  sync  -> [C(t) | A1(t+1)] ...
// A1 touches only sslot/srank/ucnt/hist and the dictionary, C only the slot-sorted staging
// and the run table, so a warp runs its share of C(t) and then its share of A1(t+1) with no
// barrier in between.

// Per-warp cursor into the deferred-tier records: the warp reserves kSpillGrab records at a time
// (one device atomic per kSpillGrab tier rows, not per 32) and marks what it leaves unused
// (slot -1).  ntier counts the warp's tier rows (debug statistic, one atomic per warp).
constexpr int kSpillGrab = 256;
struct SpillCur {
  unsigned long long cur, end;
  unsigned long long ntier;
  __device__ __forceinline__ void init() { cur = end = 0; ntier = 0; }
  // marks [cur, end) unused; every lane of the warp calls it
  __device__ __forceinline__ void retire(const AggPlan& p, int lane) {
    for (unsigned long long i = cur + lane; i < end; i += 32) p.sp_prov[i] = -1;
    cur = end;
  }
  // n <= 32 records for the calling warp: base index, or ~0 when the records are full
  __device__ __forceinline__ unsigned long long take(const AggPlan& p, int n, int lane) {
    if (cur + n > end) {
      retire(p, lane);
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(p.sp_n, (unsigned long long)kSpillGrab);
      b = __shfl_sync(0xffffffffu, b, 0);
      const unsigned long long cap = (unsigned long long)p.sp_cap;
      cur = b < cap ? b : cap;
      end = b + kSpillGrab < cap ? b + kSpillGrab : cap;
      if (cur + n > end) {  // the records are full: this and every later row takes atomics
        retire(p, lane);
        return ~0ull;
      }
    }
    const unsigned long long b = cur;
    cur += n;
    return b;
  }
  __device__ __forceinline__ void finish(const AggPlan& p, int lane) {
    if (p.sp_cap > 0) retire(p, lane);
    if (lane == 0 && ntier) atomicAdd(&p.dbg[0], ntier);
  }
};

// A1: group slot of every row, rank within its 32-row unit, per-unit and per-tile slot counts.
template <int NI, int NF, int MM, bool STAGED>
__device__ __forceinline__ void tile_a1(const AggPlan& p, const TileSmem& sm, const SmemLayout& L, int64_t base,
                                        int tn, SpillCur& sc) {
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31;
  const int T = L.T, Lcap = L.Lcap, LH = L.LH;
  const unsigned short kNone = 0xFFFF;
  const unsigned lt_mask = (1u << lane) - 1u;
  constexpr int KF = 1 + NI;
  constexpr int KM = 1 + NI + NF;
  constexpr int KK = 1 + NI + NF + (MM ? 1 : 0);
  TileCols<STAGED> tc{&p, sm.raw, base, T};
  constexpr int kNoProv = INT_MIN;
  constexpr int kDeferred = -2;  // HBM slot not looked up yet (deferred tier)
  const bool defer = p.sp_cap > 0;
  for (int li = tid; li < T; li += nth) {
    int s = -1;
    int gprov = kNoProv;  // provisional HBM slot of a row without a local slot (-1: no capacity)
    uint64_t key = 0;
    if (li < tn) {
      bool keep = true;
      if (p.mask_in) keep = tc.w8(0, li) != 0ull;  // R21: a row in no world is dropped
      if (keep) {
        key = tc.group_key(KK, li);
        const int code = local_code(p, key, sm.lkey, sm.lstate, LH, sm.lprov, Lcap, sm.misc, defer);
        if (code == kUnresolved) {
          gprov = kDeferred;
        } else if (code < kOvfBase) {
          s = code - 1;
        } else {  // no local slot: the HBM tier, below
          gprov = code - kOvfBase - 1;
        }
      }
    }
    // HBM tier (groups without a CTA-local slot, e.g. the long tail of C3): the warp applies
    // each such row cooperatively -- lane j updates worlds j and j+32, so the 64 world
    // updates of a row are coalesced device atomics on consecutive addresses
    unsigned gp = __ballot_sync(0xffffffffu, gprov != kNoProv);
    if (gp) {
      sc.ntier += __popc(gp);
      if (p.sp_cap > 0) {  // deferred: append the warp's tier rows to the spill records
        const bool mine = gprov != kNoProv && gprov != -1;
        const unsigned sb = __ballot_sync(0xffffffffu, mine);
        const unsigned long long b0 = sb ? sc.take(p, __popc(sb), lane) : 0ull;
        const unsigned long long i = b0 + __popc(sb & lt_mask);
        if (b0 != ~0ull) {
          if (mine) {
            p.sp_prov[i] = gprov;
            p.sp_gkey[i] = key;
            p.sp_key[i] = tc.w8(0, li);  // hashed by k_spill_resolve with full warps
            unsigned long long* v = p.sp_val + i;
#pragma unroll
            for (int c = 0; c < KK - 1; ++c) v[(size_t)c * p.sp_cap] = tc.w8(1 + c, li);
          }
          gp = 0;
        }
      }
      uint64_t gm = 0;
      if (gp && gprov == kDeferred) gprov = global_slot(p, key);  // records full: resolve now
      if (gp && gprov != kNoProv) gm = p.mask_in ? tc.w8(0, li) : pac_hash_dev(tc.w8(0, li), p.salt);
      while (gp) {
        const int src = __ffs(gp) - 1;
        gp &= gp - 1;
        const int prov = __shfl_sync(0xffffffffu, gprov, src);
        const uint64_t m = __shfl_sync(0xffffffffu, gm, src);
        const int lsrc = (li & ~31) + src;
        if (prov < 0) continue;  // capacity exhausted: reported by the finish kernel
        if (lane == 0) atomicAdd(&p.prov_rows[prov], 1ull);
        const size_t b = (size_t)prov * kM;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = lane + 32 * h;
          if (!((m >> j) & 1ull)) continue;
          if (p.has_count) atomicAdd(&p.prov_count[b + j], 1ull);
#pragma unroll
          for (int c = 0; c < NI; ++c) atomicAdd(&p.prov_isum[c][b + j], (unsigned long long)tc.w8(1 + c, lsrc));
#pragma unroll
          for (int c = 0; c < NF; ++c) atomicAdd(&p.prov_fsum[c][b + j], __longlong_as_double((long long)tc.w8(KF + c, lsrc)));
          if (MM & 1) atomicMin(&p.prov_min[b + j], enc_f64(__longlong_as_double((long long)tc.w8(KM, lsrc))));
          if (MM & 2) atomicMax(&p.prov_max[b + j], enc_f64(__longlong_as_double((long long)tc.w8(KM, lsrc))));
        }
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, s >= 0 ? (unsigned)s : 0x10000u + lane);
    unsigned short* uc = sm.ucnt + (li >> 5) * Lcap;
    if (Lcap <= 32) {  // this unit's counts start at zero
      if (lane < Lcap) uc[lane] = 0;
    } else if ((Lcap & 3) == 0) {  // 8-byte stores (a unit's row is Lcap * 2 bytes, 8-aligned)
      for (int z = lane; z < (Lcap >> 2); z += 32) reinterpret_cast<uint2*>(uc)[z] = make_uint2(0u, 0u);
    } else {
      for (int z = lane; z < Lcap; z += 32) uc[z] = 0;
    }
    __syncwarp();
    if (s >= 0) {
      sm.srank[li] = (unsigned char)__popc(peers & lt_mask);
      if ((peers & lt_mask) == 0) {
        uc[s] = (unsigned short)__popc(peers);
        atomicAdd(&sm.hist[s], __popc(peers));
      }
    }
    sm.sslot[li] = s >= 0 ? (unsigned short)s : kNone;
  }
}

// B2 + B3 + A2 + A3 of one tile (A1 done, hist complete).  Leaves the slot-sorted tile in smem
// and the run table for phase C; ends with a barrier.
template <int NI, int NF, int MM, bool STAGED>
__device__ __forceinline__ void tile_mid(const AggPlan& p, const TileSmem& sm, const SmemLayout& L, int64_t base,
                                         unsigned long long& maxabs) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  const int T = L.T, TS = L.TS, Lcap = L.Lcap;
  const int units = T >> 5;
  const unsigned short kNone = 0xFFFF;
  const unsigned lt_mask = (1u << lane) - 1u;
  constexpr int KF = 1 + NI;             // first f64 sum column
  constexpr int KM = 1 + NI + NF;        // min/max column
  TileCols<STAGED> tc{&p, sm.raw, base, T};
  Misc* misc = sm.misc;

  if (Lcap <= 32) {
    // ---------------- B2 + B3, at most 32 slots: every warp scans the slot histogram itself
    // (lane s = slot s, no barrier between B2 and B3); warp w then owns slots w, w + nw, ...
    // and scans that slot's per-unit counts with lane = unit.
    const int h = lane < Lcap ? sm.hist[lane] : 0;
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
    if (wid == 0 && lane == 31) {
      misc->nruns = rx;
      misc->big = 0;
      misc->nonfinite = 0;
    }
    hx -= h8;
    rx -= hr;
    for (int s = wid; s < Lcap; s += nw) {
      const int o0 = __shfl_sync(0xffffffffu, hx, s);
      const int rb = __shfl_sync(0xffffffffu, rx, s);
      const int hs = __shfl_sync(0xffffffffu, h, s);
      int carry = o0;
      for (int ub = 0; ub < units; ub += 32) {
        const int u = ub + lane;
        const int c = u < units ? sm.ucnt[u * Lcap + s] : 0;
        int inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int a = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += a;
        }
        if (u < units) sm.ucnt[u * Lcap + s] = (unsigned short)(carry + inc - c);
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      const int q = o0 + hs + lane;  // zero padding rows (mask 0) up to the 8-row boundary
      if (q < o0 + ((hs + 7) & ~7)) {
        sm.smask[q] = 0;
#pragma unroll
        for (int c = 0; c < NI; ++c) sm.sival[c * TS + q] = 0;
#pragma unroll
        for (int c = 0; c < NF; ++c) sm.sfval[c * TS + q] = 0.0;
        if (MM) sm.smval[q] = 0;
      }
      for (int i = lane; 32 * i < hs; i += 32) sm.rdesc[rb + i] = pack_run(o0 + 32 * i, s, min(32, hs - 32 * i));
      if (lane == 0) sm.lrows[s] += (unsigned long long)hs;
    }
    __syncthreads();
    if (tid < Lcap) sm.hist[tid] = 0;  // every warp has read it; the next A1 follows a barrier
  } else {
  // ---------------- B2: 8-row padded slot offsets and run offsets (one warp)
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
      misc->big = 0;
      misc->nonfinite = 0;
    }
  }
  // ---------------- B3: unit positions, zero padding rows, run descriptors (thread = slot)
  __syncthreads();
  for (int s = tid; s < Lcap; s += nth) {
    const int o0 = sm.offs[s];
    int o = o0;
    for (int u = 0; u < units; ++u) {
      const int c = sm.ucnt[u * Lcap + s];
      sm.ucnt[u * Lcap + s] = (unsigned short)o;
      o += c;
    }
    const int h = sm.hist[s];
    for (int q = o; q < o0 + ((h + 7) & ~7); ++q) {  // zero padding rows (mask 0)
      sm.smask[q] = 0;
#pragma unroll
      for (int c = 0; c < NI; ++c) sm.sival[c * TS + q] = 0;
#pragma unroll
      for (int c = 0; c < NF; ++c) sm.sfval[c * TS + q] = 0.0;
      if (MM) sm.smval[q] = 0;
    }
    for (int i = 0, rb = sm.runoffs[s]; 32 * i < h; ++i)
      sm.rdesc[rb + i] = pack_run(o0 + 32 * i, s, min(32, h - 32 * i));
    sm.hist[s] = 0;  // ready for the next tile's A1
  }
  __syncthreads();
  }

  // ---------------- A2: hash word 0 (two rows per thread, interleaved) + values, written
  // straight to the slot-sorted position; rows still needing flips go to the warp's queue.
  unsigned long long tmax = 0;  // max |int64 value| of this thread's rows of the tile
  uint32_t emax = 0;            // max f64 exponent field (0x7FF00000 = inf/nan) of its rows
  unsigned short* qpos = sm.qpos + wid * (T / nw);
  unsigned short* qrow = sm.qrow + wid * (T / nw);
  int qn = 0;
  for (int la = tid; la < T; la += 2 * nth) {
    const int lb = la + nth;  // T is a multiple of nth; lb >= T when T < 2 * nth
    const unsigned short sa = sm.sslot[la], sb = lb < T ? sm.sslot[lb] : kNone;
    const int pa = sa != kNone ? sm.ucnt[(la >> 5) * Lcap + sa] + sm.srank[la] : 0;
    const int pb = sb != kNone ? sm.ucnt[(lb >> 5) * Lcap + sb] + sm.srank[lb] : 0;
    bool qa = false, qb = false;
    const uint64_t ka = sa != kNone ? tc.w8(0, la) : 0ull;
    const uint64_t kb = sb != kNone ? tc.w8(0, lb) : 0ull;
    uint64_t ma = ka, mb = kb;
    if (!p.mask_in) {
      HashState ha, hb;
      if (kAblate && (p.ablate & 1)) {
        ha.x = ka; ha.cand = ka; ha.k = 0; hb.x = kb; hb.cand = kb; hb.k = 0;
      } else {
        pac_hash_begin2(ka, kb, p.salt, ha, hb);
      }
      ma = hash_mask_now(ha);
      mb = hash_mask_now(hb);
      qa = sa != kNone && ha.k > 0;
      qb = sb != kNone && hb.k > 0;
      // a queued row keeps its draw word 0 in the (consumed) key slot of the staged tile
      if (STAGED && qa) ((unsigned long long*)sm.raw)[la] = ha.w0;
      if (STAGED && qb) ((unsigned long long*)sm.raw)[lb] = hb.w0;
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
        tmax = a > tmax ? a : tmax;
        sm.sival[c * TS + pos] = v;
      }
#pragma unroll
      for (int c = 0; c < NF; ++c) {
        const double v = __longlong_as_double((long long)tc.w8(KF + c, li));
        emax = max(emax, (uint32_t)__double2hiint(v) & 0x7FF00000u);
        sm.sfval[c * TS + pos] = v;
      }
      if (MM) sm.smval[pos] = enc_f64(__longlong_as_double((long long)tc.w8(KM, li)));
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool pend = h ? qb : qa;
      const unsigned pm = __ballot_sync(0xffffffffu, pend);
      if (pend) {
        const int q = qn + __popc(pm & lt_mask);
        qpos[q] = (unsigned short)(h ? pb : pa);
        qrow[q] = (unsigned short)(h ? lb : la);
      }
      qn += __popc(pm);
    }
  }
  maxabs = tmax > maxabs ? tmax : maxabs;
  if (NI > 0 && __any_sync(0xffffffffu, tmax >= (1ull << 26)) && lane == 0) misc->big = 1;
  if (NF > 0 && __any_sync(0xffffffffu, emax == 0x7FF00000u) && lane == 0) misc->nonfinite = 1;
  __syncwarp();

  // ---------------- A3: the warp finishes its own queued masks from draw word 1 on (state
  // re-derived from the partial mask, R2; word 0 from the staged key slot, or recomputed).
  if (!(kAblate && (p.ablate & 2))) {
    for (int qi = lane; qi < qn; qi += 32) {
      const int pos = qpos[qi];
      const int li = qrow[qi];
      const uint64_t w0 = STAGED ? ((const unsigned long long*)sm.raw)[li]
                                 : fmix64(fmix64(tc.w8(0, li) ^ p.salt) ^ kDrawSeed);
      sm.smask[pos] = pac_hash_continue(sm.smask[pos], w0);
    }
  }
  __syncthreads();
}

// THREADS = 256: three CTAs per SM (small tables); 512: one CTA per SM with 16 warps and a
// 128-register budget (large CTA tables, e.g. 100 groups x 3 aggregates).
// LC = 0: the layout is the runtime parameter.  LC > 0: T = 1024 and LC local slots, the layout is
// a compile-time constant (every smem address an immediate offset, tile/unit/slot index math
// folded) -- the instance for small group counts (<= 8 groups, e.g. the paper's Q01 shapes).
template <int NI, int NF, int MM, int THREADS, int LC>
__global__ void __launch_bounds__(THREADS, THREADS == 256 ? PAC_TILE_MINB : 1) k_agg_tiles(AggPlan p, SmemLayout Lp) {
  constexpr SmemLayout Lc = tile_layout(NI, NF, MM & 1, (MM >> 1) & 1, 1024, LC > 0 ? LC : 1, 0, 0);
  const SmemLayout& L = LC > 0 ? Lc : Lp;
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
  const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  const int T = L.T, Lcap = L.Lcap, LH = L.LH;

  for (int i = tid; i < LH; i += nth) sm.lstate[i] = 0;
  for (int i = tid; i < Lcap; i += nth) {
    sm.lrows[i] = 0;
    sm.hist[i] = 0;
  }
  for (int i = tid; i < Lcap * kM; i += nth) {
    sm.cnt[i] = 0;
#pragma unroll
    for (int c = 0; c < NI; ++c) sm.isum[(size_t)c * Lcap * kM + i] = 0;
#pragma unroll
    for (int c = 0; c < NF; ++c) sm.fsum[(size_t)c * Lcap * kM + i] = 0.0;
    if (MM & 1) sm.emin[i] = kMinEmpty;
    if (MM & 2) sm.emax[i] = kMaxEmpty;
  }
  if (tid == 0) {
    misc->nlocal = 0;
    misc->ndict = 0;
  }
  if (tid < 32) store_xpose(sm.xcs, sm.xcs2, tid);
  unsigned long long maxabs = 0;

  const int64_t ntiles = (p.n_rows + T - 1) / T;
  const int64_t t_per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * t_per;
  const int64_t t1 = min(ntiles, t0 + t_per);
  // a tile is staged by TMA when it is full and every column is 16-byte aligned
  auto staged_tile = [&](int64_t t) { return p.tma_ok && t < t1 && (t + 1) * T <= p.n_rows; };
  auto tile_rows = [&](int64_t t) { return (int)min((int64_t)T, p.n_rows - t * T); };
  uint32_t phase = 0;
  if (tid == 0) {
    mbar_init(mbar, 1);
    if (staged_tile(t0)) issue_tile(p, raw, mbar, t0 * T, T);
  }
  __syncthreads();

#if !PAC_TILE_FLUSH
  WarpAcc<NI, NF, MM> acc;
  acc.cur = -1;
  acc.reset();
#endif

  SpillCur sc;
  sc.init();
  // prologue: A1 of the first tile
  if (t0 < t1) {
    if (staged_tile(t0)) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
      tile_a1<NI, NF, MM, true>(p, sm, L, t0 * T, tile_rows(t0), sc);
    } else {
      tile_a1<NI, NF, MM, false>(p, sm, L, t0 * T, tile_rows(t0), sc);
    }
  }
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t base = tile * T;
    const bool staged = staged_tile(tile);
    __syncthreads();  // A1(tile) and C(tile-1) complete
    if (staged) tile_mid<NI, NF, MM, true>(p, sm, L, base, maxabs);
    else tile_mid<NI, NF, MM, false>(p, sm, L, base, maxabs);
    // the raw tile buffer is free: stage the next tile while phase C runs
    const bool next_staged = staged_tile(tile + 1);
    if (tid == 0 && next_staged) issue_tile(p, raw, mbar, (tile + 1) * T, T);

    // ---------------- C: world-parallel runs, transposed "Four Russians" tables
    if (!(kAblate && (p.ablate & 4))) {
      RunCtx x;
      x.smask = sm.smask;
      x.sival = sm.sival;
      x.sfval = sm.sfval;
      x.smval = sm.smval;
      x.rdesc = sm.rdesc;
      x.xcs = sm.xcs;
      x.xcs2 = sm.xcs2;
      x.TS = L.TS;
      x.Lcap = Lcap;
      x.R = misc->nruns;
      const bool small = (NI == 0) || misc->big == 0;
      const bool fin = (NF == 0) || misc->nonfinite == 0;
#if PAC_TILE_FLUSH
      // accumulators live only inside phase C (not across the register-heavy front phases)
      WarpAcc<NI, NF, MM> acc;
      acc.cur = -1;
      acc.reset();
#endif
      if (small && fin)
        run_tiles<NI, NF, MM, false>(acc, x, sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, wid, nw, lane, true, true);
      else
        run_tiles<NI, NF, MM, true>(acc, x, sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, wid, nw, lane, small, fin);
#if PAC_TILE_FLUSH
      acc.flush(sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, Lcap, lane);
#endif
    }
    // ---------------- A1 of the next tile (disjoint smem; no barrier needed)
    if (tile + 1 < t1) {
      if (next_staged) {
        mbar_wait(mbar, phase);
        phase ^= 1u;
        tile_a1<NI, NF, MM, true>(p, sm, L, base + T, tile_rows(tile + 1), sc);
      } else {
        tile_a1<NI, NF, MM, false>(p, sm, L, base + T, tile_rows(tile + 1), sc);
      }
    }
  }
  __syncthreads();
#if !PAC_TILE_FLUSH
  acc.flush(sm.cnt, sm.isum, sm.fsum, sm.emin, sm.emax, Lcap, lane);
#endif
  __syncthreads();

  sc.finish(p, lane);
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


void note_launch();

constexpr int kFixedSlots = 8;  // LC of the compile-time-layout instance

template <int NI, int NF, int MM>
cudaError_t launch_smem(const AggPlan& p, const SmemLayout& L, int sms, cudaStream_t st) {
  // one CTA per SM -> the 16-warp variant; T = 1024 with 8 slots -> the compile-time layout
  const bool wide = L.bytes > 232448 / 2 - 2048;
  const bool fixed = !wide && L.T == 1024 && L.Lcap == kFixedSlots && !L.tm && !getenv("PAC_NO_FIXED");
  auto k = wide ? k_agg_tiles<NI, NF, MM, 512, 0>
                : (fixed ? k_agg_tiles<NI, NF, MM, 256, kFixedSlots> : k_agg_tiles<NI, NF, MM, 256, 0>);
  const int threads = wide ? 512 : 256;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, L.bytes);
  per_sm = std::max(1, per_sm);
  const int64_t tiles = (p.n_rows + L.T - 1) / L.T;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * per_sm));
  if (getenv("PAC_DEBUG"))
    fprintf(stderr, "[libpac] launch %d CTAs x %d threads (%d per SM)\n", grid, threads, per_sm);
  k<<<grid, threads, L.bytes, st>>>(p, L);
  note_launch();
  return cudaGetLastError();
}


}  // namespace pac
