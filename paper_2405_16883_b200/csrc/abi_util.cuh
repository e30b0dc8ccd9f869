// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "../../include/stc.h"

namespace stc {

// Thread-local last-error message (defined in abi_common.cu).
void set_error_message(const char* msg);
// Process-wide count of successful kernel launches (defined in abi_common.cu).
void count_launch();
inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error_message(buf);
  return code;
}

inline int check_launch(const char* what) {
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(STC_ELAUNCH, "%s: %s", what, cudaGetErrorString(err));
  count_launch();
  set_error_message("");
  return STC_OK;
}

// NVTX range around one C-ABI call (header-only NVTX v3: a no-op unless a profiler injects
// itself), named after the entry point and, for SpMM, the variant -- nsys / ncu --nvtx group
// the launches by the reference operation they replace.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define STC_NVTX(name) ::stc::NvtxRange stc_nvtx_range_(name)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace stc
