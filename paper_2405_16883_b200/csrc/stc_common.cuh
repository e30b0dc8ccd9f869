// Shared device helpers for the sparse-contraction kernels (sm_100a).
//
// Memory-path conventions used by every kernel in this library:
//   * index/value streams (rowptr, colidx, values, COO coordinates) are read
//     exactly once -> ld.global.nc.L1::no_allocate (do not pollute L1 with them)
//   * the dense operand that is gathered by sparse coordinates is re-read many
//     times -> ld.global.nc (read-only path, L1-allocating)
//   * outputs are written once -> st.global.cs (streaming, evict-first)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define STC_DEVICE __device__ __forceinline__

// Device-side bounds / protocol checks, compiled in only for the checked build
// (libstc_checked.so, `python -m paper_2405_16883_b200._build --checked`; tools/run_checked.sh).
// A failed check prints its site and traps, so the launch reports an error.
#include <cstdio>
#ifdef STC_CHECKED
#define STC_CHECK(cond, what)                                                                        \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("STC_CHECK failed: %s (%s:%d) block (%d,%d,%d) thread %d\n", what, __FILE__, __LINE__,   \
             blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);                                        \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define STC_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

namespace stc {

constexpr int kWarp = 32;

STC_DEVICE int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
STC_DEVICE float ld_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

STC_DEVICE float4 ld_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

STC_DEVICE uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Gather of a dense-operand vector: read-only (non-coherent) path, L1-cached.
// cp.async 16-byte copy (L2 -> SMEM, bypassing L1); pred == false zero-fills
STC_DEVICE void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
STC_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
STC_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

STC_DEVICE float4 ld_gather4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
STC_DEVICE float ld_gather1(const float* p) { return __ldg(p); }

STC_DEVICE void st_stream4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
STC_DEVICE void st_stream1(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// ---- packed fp32 arithmetic (sm_100a: PTX *.f32x2 -> SASS FFMA2 / FMUL2) ---------
// One issue slot for two IEEE fp32 operations on an aligned register pair; each half is
// exactly fma.rn.f32 / mul.rn.f32, so results are bit-identical to the scalar forms. The
// FP32 pipe spends two cycles on a packed op (tools/ffma2_probe.cu: 117.8 against 124.7
// FMA/clk/SM), so this buys issue slots, not flops: it pays in the kernels that are bound by
// instruction issue (COLTILE, the tiled attention kernel, the MTTKRP loop).
// ptxas folds the b64 packing moves into register allocation when the halves already sit in
// an aligned pair (float4 loads, tcgen05.ld quads) and uses the scalar-broadcast form of
// FFMA2 when both halves of a multiplicand are the same register.
#ifndef STC_NO_PACKED_FMA
#define STC_PACKED_FMA 1
#else
#define STC_PACKED_FMA 0
#endif

// (d0, d1) = a * (b0, b1) + (d0, d1)
STC_DEVICE void fma2(float& d0, float& d1, float a, float b0, float b1) {
#if STC_PACKED_FMA
  uint64_t av, bv, dv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(dv) : "f"(d0), "f"(d1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dv) : "l"(av), "l"(bv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(dv));
#else
  d0 = fmaf(a, b0, d0);
  d1 = fmaf(a, b1, d1);
#endif
}
// (d0, d1) = (a0, a1) * (b0, b1) + (d0, d1)
STC_DEVICE void fma2v(float& d0, float& d1, float a0, float a1, float b0, float b1) {
#if STC_PACKED_FMA
  uint64_t av, bv, dv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(dv) : "f"(d0), "f"(d1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dv) : "l"(av), "l"(bv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(dv));
#else
  d0 = fmaf(a0, b0, d0);
  d1 = fmaf(a1, b1, d1);
#endif
}
// (d0, d1) = a * (b0, b1)
STC_DEVICE void mul2(float& d0, float& d1, float a, float b0, float b1) {
#if STC_PACKED_FMA
  uint64_t av, bv, dv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(dv) : "l"(av), "l"(bv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(dv));
#else
  d0 = a * b0;
  d1 = a * b1;
#endif
}

// ---- VEC-wide register fragments ------------------------------------------------

template <int VEC>
struct Frag;

template <>
struct Frag<4> {
  float v[4];
  STC_DEVICE void zero() { v[0] = v[1] = v[2] = v[3] = 0.f; }
  STC_DEVICE void load_gather(const float* p) {
    float4 t = ld_gather4(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  STC_DEVICE void load_plain(const float* p) {
    float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  // L2-coherent read of data published by another CTA in the same launch
  STC_DEVICE void load_l2(const float* p) {
    float4 t = __ldcg(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  STC_DEVICE void store_stream(float* p) const { st_stream4(p, make_float4(v[0], v[1], v[2], v[3])); }
  STC_DEVICE void store_plain(float* p) const {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

template <>
struct Frag<1> {
  float v[1];
  STC_DEVICE void zero() { v[0] = 0.f; }
  STC_DEVICE void load_gather(const float* p) { v[0] = ld_gather1(p); }
  STC_DEVICE void load_plain(const float* p) { v[0] = *p; }
  STC_DEVICE void load_l2(const float* p) { v[0] = __ldcg(p); }
  STC_DEVICE void store_stream(float* p) const { st_stream1(p, v[0]); }
  STC_DEVICE void store_plain(float* p) const { *p = v[0]; }
};

// Epilogues shared by every dense-output kernel: out = act(acc + D).
enum Epilogue : int { EPI_NONE = 0, EPI_RELU = 1 };

template <int EPI>
STC_DEVICE float act(float x) {
  if constexpr (EPI == EPI_RELU) return x > 0.f ? x : 0.f;
  return x;
}

// Mask of the SUBW-lane sub-warp that contains this lane.
template <int SUBW>
STC_DEVICE unsigned subwarp_mask() {
  if constexpr (SUBW == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31u;
    return ((1u << SUBW) - 1u) << (lane & ~(unsigned)(SUBW - 1));
  }
}

}  // namespace stc
