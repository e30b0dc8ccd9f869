// Probe: what bounds 512-byte row gathers on a B200 -- the L2 slices (then L1/SMEM hits
// help in proportion) or the SM's L1TEX pipe (then they do not)?  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_probe tools/l2_probe.cu
// 1. A fraction f of the gathers goes to a 16 KB table (L1-resident) or to a 16 KB
//    shared-memory copy, the rest to an 8 MB table (L2-resident): time vs f.
// 2. Row width: 128 / 256 / 512-byte rows from the 8 MB table (same total bytes).
// 3. Coalesced streaming read of an L2-resident 32 MB buffer (L2 -> SM ceiling).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

// idx < 0 encodes a hot row (-1 - r, r < 32); >= 0 a cold row.  SRC 0: hot rows from global
// (L1 hits), SRC 1: hot rows from shared memory.
template <int SRC, int U>
__global__ void __launch_bounds__(256) mix_k(const float4* __restrict__ cold, const float4* __restrict__ hot,
                                             const int* __restrict__ idx, int per_warp, float* out) {
  __shared__ float4 sh[32 * 32];
  if (SRC == 1) {
    for (int i = threadIdx.x; i < 32 * 32; i += 256) sh[i] = hot[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * 256LL + threadIdx.x) >> 5;
  const int* my_idx = idx + warp * per_warp;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int b = 0; b < per_warp; b += 32) {
    int my = __ldg(my_idx + b + lane);
#pragma unroll 1
    for (int q0 = 0; q0 < 32; q0 += U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int r = __shfl_sync(0xffffffffu, my, q0 + u);
        if (r >= 0) v[u] = __ldg(cold + (size_t)r * 32 + lane);
        else if (SRC == 0) v[u] = __ldg(hot + (size_t)(-1 - r) * 32 + lane);
        else v[u] = sh[(-1 - r) * 32 + lane];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
  out[(blockIdx.x * 256 + threadIdx.x) & ((1 << 20) - 1)] += acc.x + acc.y + acc.z + acc.w;
}

// W-byte rows (W = 128, 256, 512): L = W/16 lanes per row, 32/L rows per warp instruction.
template <int W, int U>
__global__ void __launch_bounds__(256) width_k(const float4* __restrict__ table, const int* __restrict__ idx,
                                               int per_warp, float* out) {
  constexpr int L = W / 16, R = 32 / L;
  const int lane = threadIdx.x & 31, sub = lane % L, slot = lane / L;
  const long long warp = (blockIdx.x * 256LL + threadIdx.x) >> 5;
  const int* my_idx = idx + warp * per_warp;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int b = 0; b < per_warp; b += 32) {
    int my = __ldg(my_idx + b + lane);
#pragma unroll 1
    for (int q0 = 0; q0 < 32; q0 += U * R) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int r = __shfl_sync(0xffffffffu, my, q0 + u * R + slot);
        v[u] = __ldg(table + (size_t)r * (W / 16) + sub);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
  out[(blockIdx.x * 256 + threadIdx.x) & ((1 << 20) - 1)] += acc.x + acc.y + acc.z + acc.w;
}

__global__ void __launch_bounds__(256) stream_k(const float4* __restrict__ buf, size_t n4, int passes, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * 256;
  for (int p = 0; p < passes; ++p) {
    size_t start = ((size_t)blockIdx.x * 256 + threadIdx.x + (size_t)p * 4096 * 256) % stride;
    for (size_t i = start; i < n4; i += stride) {
      float4 v = __ldg(buf + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[(blockIdx.x * 256 + threadIdx.x) & ((1 << 20) - 1)] += acc.x + acc.y + acc.z + acc.w;
}

template <typename F>
float time_us(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) best = std::min(best, ms);
  }
  return best * 1e3f;
}

int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int per_warp = 512;
  const int ctas = nsm * 4 * 4;            // 4 waves of 4 CTAs/SM
  const long long n = (long long)ctas * 8 * per_warp;   // gathers
  size_t cold_bytes = 8ull << 20;
  long long cold_rows = cold_bytes / 512;
  float4 *cold, *hot, *big; float* out;
  cudaMalloc(&cold, cold_bytes); cudaMemset(cold, 0, cold_bytes);
  cudaMalloc(&hot, 16384); cudaMemset(hot, 0, 16384);
  cudaMalloc(&out, 4 << 20); cudaMemset(out, 0, 4 << 20);
  int* idx; cudaMalloc(&idx, n * 4);
  std::vector<int> h(n);
  printf("gathers per launch: %lld (%.1f MB of 512-byte rows)\n", n, n * 512.0 / 1e6);
  for (double f : {0.0, 0.25, 0.5, 0.75, 1.0}) {
    srand(7);
    for (long long i = 0; i < n; ++i) {
      double u = rand() / (RAND_MAX + 1.0);
      h[i] = u < f ? -1 - (rand() & 31) : (int)(((long long)rand() * 7919LL + rand()) % cold_rows);
    }
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    float t0 = time_us([&] { mix_k<0, 8><<<ctas, 256>>>(cold, hot, idx, per_warp, out); });
    float t1 = time_us([&] { mix_k<1, 8><<<ctas, 256>>>(cold, hot, idx, per_warp, out); });
    double gb = n * 512.0 / 1e3;
    printf("hot fraction %.2f: hot from L1 %7.1f us (%6.0f GB/s delivered) | hot from SMEM %7.1f us (%6.0f GB/s)\n",
           f, t0, gb / t0, t1, gb / t1);
  }
  // row width: same total bytes
  srand(9);
  for (long long i = 0; i < n; ++i) h[i] = (int)(((long long)rand() * 7919LL + rand()) % cold_rows);
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  {
    double gb = n * 512.0 / 1e3;
    float t512 = time_us([&] { width_k<512, 8><<<ctas, 256>>>(cold, idx, per_warp, out); });
    printf("512-byte rows: %7.1f us (%6.0f GB/s)\n", t512, gb / t512);
    // 256-byte rows: 2x the rows, rows index a table of 2x rows of 256 B (same 8 MB)
    for (long long i = 0; i < n; ++i) h[i] = (int)(((long long)rand() * 7919LL + rand()) % (cold_rows * 2));
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    float t256 = time_us([&] { width_k<256, 4><<<ctas * 2, 256>>>(cold, idx, per_warp / 2, out); });
    printf("256-byte rows (same bytes): %7.1f us (%6.0f GB/s)\n", t256, gb / t256);
    for (long long i = 0; i < n; ++i) h[i] = (int)(((long long)rand() * 7919LL + rand()) % (cold_rows * 4));
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    float t128 = time_us([&] { width_k<128, 2><<<ctas * 4, 256>>>(cold, idx, per_warp / 4, out); });
    float t128b = time_us([&] { width_k<128, 4><<<ctas * 4, 256>>>(cold, idx, per_warp / 4, out); });
    printf("128-byte rows (same bytes): U2 %7.1f us (%6.0f GB/s)  U4 %7.1f us (%6.0f GB/s)\n", t128, gb / t128, t128b, gb / t128b);
  }
  // streaming reads of L2-resident buffers
  for (int mb : {16, 32, 64}) {
    size_t bytes = (size_t)mb << 20;
    cudaMalloc(&big, bytes); cudaMemset(big, 0, bytes);
    const int passes = 16;
    float t = time_us([&] { stream_k<<<nsm * 8, 256>>>(big, bytes / 16, passes, out); });
    printf("stream %d MB x %d passes: %7.1f us (%6.0f GB/s)\n", mb, passes, t, bytes * (double)passes / 1e3 / t);
    cudaFree(big);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
