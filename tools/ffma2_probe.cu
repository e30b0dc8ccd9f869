// Probe: issue / pipe throughput of the packed fp32 FMA (PTX fma.rn.f32x2 -> SASS FFMA2) on sm_100a
// against scalar FFMA, alone and interleaved with LDS.128 traffic.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma2_probe tools/ffma2_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ffma2(float& d0, float& d1, float a, float b0, float b1) {
  uint64_t av, bv, dv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(dv) : "f"(d0), "f"(d1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dv) : "l"(av), "l"(bv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(dv));
}

// MODE 0: 32 scalar FFMA per iteration; MODE 1: 16 FFMA2 per iteration (same 32 FMAs);
// LDS > 0: that many LDS.128 per iteration feed the multiplicands.
template <int MODE, int LDS>
__global__ void __launch_bounds__(256) fma_k(float* out, int iters, float seed) {
  __shared__ float4 sh[256];
  sh[threadIdx.x] = make_float4(seed, seed * 0.5f, seed * 0.25f, seed * 0.125f);
  __syncthreads();
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = (float)i;
  float4 b[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) b[u] = sh[(threadIdx.x + u) & 255];
  float a = seed;
  for (int it = 0; it < iters; ++it) {
    if (LDS > 0) {
#pragma unroll
      for (int u = 0; u < LDS; ++u) b[u & 3] = sh[(threadIdx.x + it + u) & 255];
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float4 v = b[g & 3];
      if (MODE == 0) {
        acc[4 * g + 0] = fmaf(a, v.x, acc[4 * g + 0]);
        acc[4 * g + 1] = fmaf(a, v.y, acc[4 * g + 1]);
        acc[4 * g + 2] = fmaf(a, v.z, acc[4 * g + 2]);
        acc[4 * g + 3] = fmaf(a, v.w, acc[4 * g + 3]);
      } else {
        ffma2(acc[4 * g + 0], acc[4 * g + 1], a, v.x, v.y);
        ffma2(acc[4 * g + 2], acc[4 * g + 3], a, v.z, v.w);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <typename F>
float time_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 1 && ms < best) best = ms;
  }
  return best;
}

int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int khz = 0; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, (size_t)nsm * 8 * 256 * 4);
  const int iters = 20000;
  const int ctas = nsm * 8;  // 8 CTAs x 8 warps = 64 warps / SM
  const double fmas = (double)ctas * 256 * iters * 32;
  auto report = [&](const char* name, float ms) {
    printf("%-34s %8.3f ms  %7.2f TFLOP/s  %6.1f FMA/clk/SM (at %d MHz)\n", name, ms, 2 * fmas / ms / 1e9,
           fmas / (ms * 1e-3) / nsm / (khz * 1e3), khz / 1000);
  };
  report("FFMA  x32", time_ms([&] { fma_k<0, 0><<<ctas, 256>>>(out, iters, 1.0001f); }));
  report("FFMA2 x16", time_ms([&] { fma_k<1, 0><<<ctas, 256>>>(out, iters, 1.0001f); }));
  report("FFMA  x32 + 4 LDS.128", time_ms([&] { fma_k<0, 4><<<ctas, 256>>>(out, iters, 1.0001f); }));
  report("FFMA2 x16 + 4 LDS.128", time_ms([&] { fma_k<1, 4><<<ctas, 256>>>(out, iters, 1.0001f); }));
  report("FFMA  x32 + 8 LDS.128", time_ms([&] { fma_k<0, 8><<<ctas, 256>>>(out, iters, 1.0001f); }));
  report("FFMA2 x16 + 8 LDS.128", time_ms([&] { fma_k<1, 8><<<ctas, 256>>>(out, iters, 1.0001f); }));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
