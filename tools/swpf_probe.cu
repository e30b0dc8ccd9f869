// Probe: does a software L2 prefetch of the gathered row PD entries ahead (prefetch.global.L2,
// no register or L1 cost) raise the memory-level parallelism of cfg2's DRAM-missing gathers?
// Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/swpf_probe tools/swpf_probe.cu
//   tools/swpf_probe tools/cfg2_colidx.bin
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) gather_k(const float4* __restrict__ table, const int* __restrict__ idx,
                                                long long n, int per_warp, int pd, float* out) {
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * 256LL + threadIdx.x) >> 5;
  long long p0 = gw * per_warp;
  if (p0 >= n) return;
  long long p1 = min(p0 + per_warp, n);
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long b = p0; b < p1; b += 32) {
    const int my = (b + lane < p1) ? __ldg(idx + b + lane) : 0;
    // prefetch distance pd within the warp's own range: lane l prefetches row idx[b + l + pd]
    if (pd > 0 && b + lane + pd < p1) {
      const int r = __ldg(idx + b + lane + pd);
      const char* a = reinterpret_cast<const char*>(table + (size_t)r * 32);
#pragma unroll
      for (int s = 0; s < 4; ++s) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + 128 * s));
    }
    const int cnt = (int)min(32LL, p1 - b);
    for (int q0 = 0; q0 < cnt; q0 += U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = __shfl_sync(0xffffffffu, my, (q0 + u) & 31);
        v[u] = (q0 + u < cnt) ? __ldg(table + (size_t)r * 32 + lane) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
  out[(gw * 32 + lane) & ((1 << 20) - 1)] += acc.x + acc.y + acc.z + acc.w;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  fseek(f, 0, SEEK_END); long long m = ftell(f) / 4; fseek(f, 0, SEEK_SET);
  std::vector<int> hi(m); size_t got = fread(hi.data(), 4, m, f); fclose(f);
  int* di; cudaMalloc(&di, m * 4); cudaMemcpy(di, hi.data(), got * 4, cudaMemcpyHostToDevice);
  size_t tb = 200000ull * 512;
  float4* table; cudaMalloc(&table, tb); cudaMemset(table, 0, tb);
  float* out; cudaMalloc(&out, 4 << 20); cudaMemset(out, 0, 4 << 20);
  char* fl; cudaMalloc(&fl, 512ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int pw : {64, 256, 1024}) {
    const long long warps = (m + pw - 1) / pw;
    const int blocks = (int)((warps * 32 + 255) / 256);
    for (int pd : {0, 32, 64, 128, 256}) {
      if (pd >= pw) continue;
      float best = 1e30f;
      for (int r = 0; r < 10; ++r) {
        cudaMemsetAsync(fl, r, 512ull << 20);
        cudaEventRecord(a);
        gather_k<8><<<blocks, 256>>>(table, di, m, pw, pd, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (r >= 2) best = std::min(best, ms);
      }
      printf("per_warp %4d prefetch distance %3d: %.1f us\n", pw, pd, best * 1e3);
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
