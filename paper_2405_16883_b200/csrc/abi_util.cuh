// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <utility>

#include "../../include/stc.h"

namespace stc {

// Thread-local last-error message (defined in abi_common.cu).
void set_error_message(const char* msg);
// Process-wide count of successful kernel launches (defined in abi_common.cu).
void count_launch();
// Persisting-L2 carve-out granted by stc_l2_set_persisting (0 = off) and the
// device's maximum access-policy window.
size_t l2_persist_bytes();
size_t l2_max_window();

// Access-policy window covering a gathered operand, if a carve-out is active.
inline bool l2_window(const void* base, size_t bytes, cudaAccessPolicyWindow* w) {
  const size_t persist = l2_persist_bytes();
  if (!persist || !base || !bytes) return false;
  const size_t n = bytes < l2_max_window() ? bytes : l2_max_window();
  w->base_ptr = const_cast<void*>(base);
  w->num_bytes = n;
  w->hitRatio = persist >= n ? 1.0f : (float)persist / (float)n;
  w->hitProp = cudaAccessPropertyPersisting;
  w->missProp = cudaAccessPropertyStreaming;
  return true;
}

// Launch with an optional access-policy window (cudaLaunchKernelEx).
template <typename... KArgs, typename... Args>
cudaError_t launch_windowed(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            const void* wbase, size_t wbytes, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  if (l2_window(wbase, wbytes, &attr.val.accessPolicyWindow)) {
    attr.id = cudaLaunchAttributeAccessPolicyWindow;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

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

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace stc
