// Probe: does an L2 bulk prefetch of the dense operand at kernel start (cp.async.bulk.prefetch.L2)
// take the cold DRAM misses out of cfg2's gather?  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/prefetch_probe tools/prefetch_probe.cu
//   tools/prefetch_probe tools/cfg2_colidx.bin
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

// PF 0: none; 1: every CTA prefetches its 1/grid slice of the table at start (ascending);
// 2: descending (cold rows of a Chung-Lu order first)
template <int PF, int U>
__global__ void __launch_bounds__(256) gather_k(const float4* __restrict__ table, size_t table_bytes,
                                                const int* __restrict__ idx, long long n, int per_warp,
                                                float* __restrict__ out, int pf_chunk) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (PF && warp == 0) {
    size_t slice = (table_bytes / gridDim.x + 4095) & ~size_t(4095);
    size_t b0 = (size_t)(PF == 1 ? blockIdx.x : gridDim.x - 1 - blockIdx.x) * slice;
    size_t b1 = b0 + slice < table_bytes ? b0 + slice : table_bytes;
    for (size_t b = b0 + (size_t)lane * pf_chunk; b < b1; b += (size_t)32 * pf_chunk) {
      unsigned sz = (unsigned)((size_t)pf_chunk < b1 - b ? (size_t)pf_chunk : b1 - b);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"((const char*)table + b), "r"(sz) : "memory");
    }
  }
  const long long gw = (blockIdx.x * 256LL + threadIdx.x) >> 5;
  long long p0 = gw * per_warp;
  if (p0 >= n) return;
  long long p1 = min(p0 + per_warp, n);
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long b = p0; b < p1; b += 32) {
    int my = (b + lane < p1) ? __ldg(idx + b + lane) : -1;
    int cnt = (int)min(32LL, p1 - b);
    for (int q0 = 0; q0 < cnt; q0 += U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int r = __shfl_sync(0xffffffffu, my, (q0 + u) & 31);
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
  fseek(f, 0, SEEK_END); long long m = ftell(f) / 4; fseek(f, 0, SEEK_SET);
  std::vector<int> hi(m); size_t got = fread(hi.data(), 4, m, f); fclose(f);
  int* di; cudaMalloc(&di, m * 4); cudaMemcpy(di, hi.data(), got * 4, cudaMemcpyHostToDevice);
  size_t tb = 200000ull * 512;
  float4* table; cudaMalloc(&table, tb); cudaMemset(table, 0, tb);
  float* out; cudaMalloc(&out, 4 << 20); cudaMemset(out, 0, 4 << 20);
  char* fl; cudaMalloc(&fl, 512ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int pw : {64, 128}) {
    long long warps = (m + pw - 1) / pw;
    int blocks = (int)((warps * 32 + 255) / 256);
    for (int mode = 0; mode < 5; ++mode) {
      int chunk = mode == 3 ? 4096 : 16384;
      float best = 1e30f, sum = 0;
      for (int r = 0; r < 12; ++r) {
        cudaMemsetAsync(fl, r, 512ull << 20);
        cudaEventRecord(a);
        if (mode == 0) gather_k<0, 8><<<blocks, 256>>>(table, tb, di, m, pw, out, chunk);
        else if (mode == 1 || mode == 3) gather_k<1, 8><<<blocks, 256>>>(table, tb, di, m, pw, out, chunk);
        else if (mode == 2) gather_k<2, 8><<<blocks, 256>>>(table, tb, di, m, pw, out, chunk);
        else gather_k<1, 8><<<blocks, 256>>>(table, tb / 2, di, m, pw, out, chunk);  // prefetch only the hot half
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (r >= 2) { best = std::min(best, ms); sum += ms; }
      }
      const char* names[] = {"no prefetch", "prefetch asc 16K", "prefetch desc 16K", "prefetch asc 4K", "prefetch first half"};
      printf("per_warp %d %-20s best %6.1f us  mean %6.1f us\n", pw, names[mode], best * 1e3, sum / 10 * 1e3);
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
