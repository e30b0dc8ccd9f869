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
void set_error_message(const char* msg) { g_last_error = msg; }
}  // namespace stc

extern "C" int stc_abi_version(void) { return STC_ABI_VERSION; }

extern "C" const char* stc_last_error(void) { return stc::g_last_error.c_str(); }

extern "C" long long stc_launch_count(void) { return stc::g_launches.load(); }

