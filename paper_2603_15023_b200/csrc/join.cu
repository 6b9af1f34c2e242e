// libpac: PU-key join (§8 f2; §3 Eq. join-addition / join-elim, §2;
// reading DESIGN.md R27).
//
// A build table maps a primary key to the tuple's next foreign key along the chain
// T -fk1-> T1 -> ... -> Tk -fkU-> U.  Layout (caller-allocated, pac_join_table_bytes):
//   header 64 B: capacity C (power of two), status (PAC_OK / PAC_E_INVAL on a duplicate PK),
//                the entry for the key INT64_MIN (the empty-slot sentinel) if present;
//   slots [C] x 16 B: {key, next}, open addressing with linear probing, load factor <= 1/2.
// One 16-byte vector load per probe step.  k_join_mask walks the chain per row and hashes
// the final FK in the same thread (pac_hash, R1/R2): the PU table is never joined.
#include <algorithm>
#include <climits>

#include "common.cuh"

namespace pac {

constexpr long long kEmptyKey = LLONG_MIN;

struct JoinHeader {
  long long cap;
  int status;
  int has_min;
  long long min_next;
  long long pad[5];
};
static_assert(sizeof(JoinHeader) == 64, "join header is 64 bytes");

__device__ __forceinline__ uint32_t join_hash(long long k) { return dict_hash((uint64_t)k ^ 0x5851F42D4C957F2Dull); }

__global__ void k_join_init(JoinHeader* hdr, longlong2* slots, long long cap) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += stride)
    slots[i] = make_longlong2(kEmptyKey, 0);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hdr->cap = cap;
    hdr->status = PAC_OK;
    hdr->has_min = 0;
    hdr->min_next = 0;
  }
}

__global__ void k_join_build(JoinHeader* hdr, longlong2* slots, const long long* __restrict__ pk,
                             const long long* __restrict__ nxt, int64_t n) {
  const long long mask = hdr->cap - 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long k = pk[i], v = nxt[i];
    if (k == kEmptyKey) {  // the sentinel key lives in the header
      if (atomicExch(&hdr->has_min, 1)) hdr->status = PAC_E_INVAL;
      hdr->min_next = v;
      continue;
    }
    long long h = join_hash(k) & mask;
    for (;;) {
      const unsigned long long old =
          atomicCAS((unsigned long long*)&slots[h].x, (unsigned long long)kEmptyKey, (unsigned long long)k);
      if (old == (unsigned long long)kEmptyKey) {
        slots[h].y = v;
        break;
      }
      if ((long long)old == k) {  // duplicate primary key (R27)
        hdr->status = PAC_E_INVAL;
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

__device__ __forceinline__ bool join_lookup(const JoinHeader* __restrict__ hdr, const longlong2* __restrict__ slots,
                                            long long mask, long long& x) {
  if (x == kEmptyKey) {
    if (!hdr->has_min) return false;
    x = hdr->min_next;
    return true;
  }
  long long h = join_hash(x) & mask;
  for (;;) {
    const longlong2 s = __ldg(slots + h);
    if (s.x == x) {
      x = s.y;
      return true;
    }
    if (s.x == kEmptyKey) return false;
    h = (h + 1) & mask;
  }
}

struct Chain {
  const JoinHeader* hdr[PAC_JOIN_MAX_CHAIN];
  int k;
};

// per row: follow the chain from fk1, then pac_hash the PU key (join elimination)
__global__ void __launch_bounds__(256) k_join_mask(Chain c, const long long* __restrict__ fk, int64_t n,
                                                   uint64_t salt, unsigned long long* __restrict__ out,
                                                   long long* __restrict__ pu_out) {
  long long masks[PAC_JOIN_MAX_CHAIN];
#pragma unroll
  for (int t = 0; t < PAC_JOIN_MAX_CHAIN; ++t) masks[t] = t < c.k ? c.hdr[t]->cap - 1 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    long long x = __ldcs(fk + i);
    bool ok = true;
#pragma unroll
    for (int t = 0; t < PAC_JOIN_MAX_CHAIN; ++t)
      if (t < c.k && ok) ok = join_lookup(c.hdr[t], (const longlong2*)(c.hdr[t] + 1), masks[t], x);
    if (out) out[i] = ok ? pac_hash_dev((uint64_t)x, salt) : 0ull;  // R27: no PU -> in no world
    if (pu_out) pu_out[i] = ok ? x : 0;
  }
}

static int sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static long long join_cap(int64_t n_build) {
  long long c = 64;
  while (c < 2 * n_build) c <<= 1;
  return c;
}

}  // namespace pac

using namespace pac;

extern "C" int pac_join_table_bytes(int64_t n_build, size_t* bytes) {
  if (!bytes || n_build < 0) return PAC_E_INVAL;
  *bytes = sizeof(JoinHeader) + (size_t)join_cap(n_build) * sizeof(longlong2);
  return PAC_OK;
}

extern "C" int pac_join_build(const int64_t* d_pk, const int64_t* d_next, int64_t n_build, void* d_table,
                              size_t table_bytes, pac_stream_t stream) {
  if (n_build < 0 || !d_table || (n_build > 0 && (!d_pk || !d_next))) return PAC_E_INVAL;
  const long long cap = join_cap(n_build);
  if (table_bytes < sizeof(JoinHeader) + (size_t)cap * sizeof(longlong2)) return PAC_E_WORKSPACE;
  if (((uintptr_t)d_table & 15) != 0) return PAC_E_INVAL;
  cudaStream_t st = (cudaStream_t)stream;
  JoinHeader* hdr = (JoinHeader*)d_table;
  longlong2* slots = (longlong2*)(hdr + 1);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, (int64_t)sms() * 16));
  k_join_init<<<grid, 256, 0, st>>>(hdr, slots, cap);
  note_launch();
  if (n_build > 0) {
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((n_build + 255) / 256, (int64_t)sms() * 16));
    k_join_build<<<g2, 256, 0, st>>>(hdr, slots, (const long long*)d_pk, (const long long*)d_next, n_build);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}

extern "C" int pac_join_table_status(const void* d_table, pac_stream_t stream) {
  if (!d_table) return PAC_E_INVAL;
  int h = PAC_E_CUDA;
  const JoinHeader* hdr = (const JoinHeader*)d_table;
  if (cudaMemcpyAsync(&h, &hdr->status, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
      cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
    return PAC_E_CUDA;
  return h;
}

extern "C" int pac_join_mask(const void* const* d_tables, int k, const int64_t* d_fk, int64_t n, uint64_t salt,
                             uint64_t* d_mask, int64_t* d_pu_key, pac_stream_t stream) {
  if (k < 1 || k > PAC_JOIN_MAX_CHAIN || !d_tables || n < 0) return PAC_E_INVAL;
  if (n > 0 && (!d_fk || (!d_mask && !d_pu_key))) return PAC_E_INVAL;
  Chain c{};
  c.k = k;
  for (int t = 0; t < k; ++t) {
    if (!d_tables[t]) return PAC_E_INVAL;
    c.hdr[t] = (const JoinHeader*)d_tables[t];
  }
  if (n == 0) return PAC_OK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms() * 8));
  k_join_mask<<<grid, 256, 0, (cudaStream_t)stream>>>(c, (const long long*)d_fk, n, salt,
                                                       (unsigned long long*)d_mask, (long long*)d_pu_key);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? PAC_OK : PAC_E_CUDA;
}
