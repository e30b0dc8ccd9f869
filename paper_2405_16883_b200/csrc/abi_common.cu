// Error state and version of the C ABI (include/stc.h).
#include <atomic>
#include <string>

#include "abi_util.cuh"

namespace stc {
namespace {
thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
namespace {
std::atomic<size_t> g_persist{0};
std::atomic<size_t> g_max_window{0};
}
size_t l2_persist_bytes() { return g_persist.load(); }
size_t l2_max_window() { return g_max_window.load(); }
void set_error_message(const char* msg) { g_last_error = msg; }
}  // namespace stc

extern "C" int stc_abi_version(void) { return STC_ABI_VERSION; }

extern "C" const char* stc_last_error(void) { return stc::g_last_error.c_str(); }

extern "C" long long stc_launch_count(void) { return stc::g_launches.load(); }

extern "C" long long stc_l2_set_persisting(size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return stc::fail(STC_ELAUNCH, "cudaGetDevice: %s", cudaGetErrorString(e));
  int maxw = 0, maxp = 0;
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  if (bytes > (size_t)maxp) bytes = (size_t)maxp;
  e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes);
  if (e != cudaSuccess) return stc::fail(STC_ELAUNCH, "persisting L2 limit: %s", cudaGetErrorString(e));
  size_t got = 0;
  cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
  if (bytes == 0) cudaCtxResetPersistingL2Cache();
  stc::g_max_window.store((size_t)maxw);
  stc::g_persist.store(got);
  return (long long)got;
}

extern "C" int stc_l2_reset_persisting(void) {
  const cudaError_t e = cudaCtxResetPersistingL2Cache();
  if (e != cudaSuccess) return stc::fail(STC_ELAUNCH, "reset persisting L2: %s", cudaGetErrorString(e));
  return STC_OK;
}
