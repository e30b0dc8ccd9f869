// Microbenchmark: what bandwidth can 512-byte row gathers reach on this B200?
// (ceiling analysis for the SpMM merge kernel; not part of the library)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// each warp gathers `per_warp` rows (indices from idx), lane = float4 of a 512 B row
template <int U>
__global__ void gather_k(const float4* __restrict__ table, const int* __restrict__ idx, long long n_idx,
                         int per_warp, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  long long p0 = warp * per_warp;
  if (p0 >= n_idx) return;
  long long p1 = min(p0 + per_warp, n_idx);
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long b = p0; b < p1; b += 32) {
    int my = (b + lane < p1) ? idx[b + lane] : -1;
    int n = (int)min(32LL, p1 - b);
    for (int q0 = 0; q0 < n; q0 += U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int r = __shfl_sync(0xffffffffu, my, (q0 + u) & 31);
        v[u] = (q0 + u < n) ? __ldg(table + (size_t)r * 32 + lane) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
  out[warp * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

static float* g_flush = nullptr;
static bool g_do_flush = false;

template <int U>
float run_gather(const float4* t, const int* idx, long long n, int per_warp, int threads, float* out) {
  long long warps = (n + per_warp - 1) / per_warp;
  long long blocks = (warps * 32 + threads - 1) / threads;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) gather_k<U><<<blocks, threads>>>(t, idx, n, per_warp, out);
  const int reps = 10;
  float total = 0;
  for (int r = 0; r < reps; ++r) {
    if (g_do_flush) cudaMemsetAsync(g_flush, r, 512ull << 20);
    cudaEventRecord(a);
    gather_k<U><<<blocks, threads>>>(t, idx, n, per_warp, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    total += ms;
  }
  return total / reps;
}

int main(int argc, char** argv) {
  cudaMalloc(&g_flush, 512ull << 20);
  size_t nbytes = 1ull << 30;
  float4 *a, *b;
  cudaMalloc(&a, nbytes); cudaMalloc(&b, nbytes);
  cudaMemset(a, 0, nbytes);
  size_t n4 = nbytes / 16;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  copy_k<<<148 * 8, 512>>>(a, b, n4);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) copy_k<<<148 * 8, 512>>>(a, b, n4);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("copy: %.1f GB/s (read+write)\n", 2.0 * nbytes * 10 / (ms * 1e-3) / 1e9);

  const long long n = 2200000;
  std::vector<int> h(n);
  float* out; cudaMalloc(&out, 64 << 20);
  int* idx; cudaMalloc(&idx, n * sizeof(int));
  for (long long rows : {3000LL, 30000LL, 200000LL, 2000000LL}) {
    srand(1);
    for (long long i = 0; i < n; ++i) h[i] = (int)(((long long)rand() * 7919LL + rand()) % rows);
    cudaMemcpy(idx, h.data(), n * sizeof(int), cudaMemcpyHostToDevice);
    for (int pw : {32, 128}) {
      for (int thr : {256, 512}) {
        float m4 = run_gather<4>(a, idx, n, pw, thr, out);
        float m8 = run_gather<8>(a, idx, n, pw, thr, out);
        float m16 = run_gather<16>(a, idx, n, pw, thr, out);
        double gb = n * 512.0 / 1e9;
        printf("table %7lld rows (%6.1f MB) per_warp %3d thr %d: U4 %.1f  U8 %.1f  U16 %.1f GB/s  (best %.1f us)\n",
               rows, rows * 512.0 / 1e6, pw, thr, gb / (m4 * 1e-3), gb / (m8 * 1e-3), gb / (m16 * 1e-3),
               1e3 * std::min(m4, std::min(m8, m16)));
      }
    }
  }
  if (argc > 1) {  // real index stream (int32 binary), table rows = argv[2]
    FILE* f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END);
    long long m = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    std::vector<int> hi(m);
    size_t got = fread(hi.data(), 4, m, f);
    fclose(f);
    int* di; cudaMalloc(&di, m * 4);
    cudaMemcpy(di, hi.data(), got * 4, cudaMemcpyHostToDevice);
    for (int fl = 0; fl < 2; ++fl) {
      g_do_flush = fl;
      for (int pw : {64, 128}) {
        float m4 = run_gather<4>(a, di, m, pw, 256, out);
        float m8 = run_gather<8>(a, di, m, pw, 256, out);
        float m16 = run_gather<16>(a, di, m, pw, 256, out);
        double gb = m * 512.0 / 1e9;
        printf("real idx (%lld) flush=%d per_warp %d: U4 %.1f (%.1f us) U8 %.1f (%.1f us) U16 %.1f (%.1f us) GB/s\n",
               m, fl, pw, gb / (m4 * 1e-3), m4 * 1e3, gb / (m8 * 1e-3), m8 * 1e3, gb / (m16 * 1e-3), m16 * 1e3);
      }
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
