// libpac runtime: launch accounting, kernel timing hooks, version.
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace pac {

static std::atomic<unsigned long long> g_launches{0};
static std::atomic<int> g_profile{0};
static std::mutex g_mu;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
static cudaEvent_t g_pending = nullptr;
static std::string g_name;  // kernel(s) of the last timed region

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void profile_begin(cudaStream_t st, const char* name) {
  if (!g_profile.load()) return;
  std::lock_guard<std::mutex> lk(g_mu);
  g_name = name ? name : "";
  cudaEvent_t a;
  if (cudaEventCreate(&a) != cudaSuccess) return;
  cudaEventRecord(a, st);
  g_pending = a;
}

void profile_end(cudaStream_t st) {
  if (!g_profile.load()) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_pending) return;
  cudaEvent_t b;
  if (cudaEventCreate(&b) != cudaSuccess) return;
  cudaEventRecord(b, st);
  g_events.emplace_back(g_pending, b);
  g_pending = nullptr;
}

}  // namespace pac

extern "C" uint64_t pac_launch_count(void) { return pac::g_launches.load(); }

extern "C" int pac_profile_enable(int on) {
  pac::g_profile.store(on ? 1 : 0);
  return PAC_OK;
}

extern "C" int pac_profile_read(double* h_total_ms, int64_t* h_launches) {
  std::lock_guard<std::mutex> lk(pac::g_mu);
  double tot = 0.0;
  int64_t n = 0;
  int rc = PAC_OK;
  for (auto& e : pac::g_events) {
    float ms = 0.f;
    if (cudaEventSynchronize(e.second) != cudaSuccess || cudaEventElapsedTime(&ms, e.first, e.second) != cudaSuccess)
      rc = PAC_E_CUDA;
    tot += ms;
    ++n;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  pac::g_events.clear();
  if (h_total_ms) *h_total_ms = tot;
  if (h_launches) *h_launches = n;
  return rc;
}

extern "C" const char* pac_profile_last_kernel(void) {
  std::lock_guard<std::mutex> lk(pac::g_mu);
  static thread_local std::string copy;
  copy = pac::g_name;
  return copy.c_str();
}

extern "C" const char* pac_version(void) { return "libpac 0.2.0 (sm_100a)"; }
