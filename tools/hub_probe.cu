// Microbenchmark: does serving the hottest dense rows from shared memory speed up
// 512-byte row gathers on the cfg2 index stream? (ceiling analysis for the hub
// variant; not part of the library)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hub_probe tools/hub_probe.cu
//   tools/hub_probe tools/cfg2_colidx.bin     (int32 column indices of cfg2's A)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

// grid-stride over chunks of `per_warp` indices; rows < H come from shared memory
template <int POL>
__device__ __forceinline__ float4 ldp(const float4* p) {
  float4 v;
  if constexpr (POL == 0) {
    v = __ldg(p);
  } else if constexpr (POL == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else if constexpr (POL == 2) {
    asm volatile("ld.global.nc.L1::evict_first.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  } else if constexpr (POL == 3) {
    v = __ldcg(p);
  } else {
    asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  }
  return v;
}

template <int U, int POL = 0>
__global__ void gather_hub(const float4* __restrict__ table, const int* __restrict__ idx, long long n_idx,
                           int per_warp, int H, float* __restrict__ out) {
  extern __shared__ float4 hub[];
  const int lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t < H * 32; t += blockDim.x) hub[t] = table[t];
  __syncthreads();
  const long long warps_total = (long long)gridDim.x * (blockDim.x >> 5);
  const long long warp0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long w = warp0; w * per_warp < n_idx; w += warps_total) {
    const long long p0 = w * per_warp;
    const long long p1 = min(p0 + per_warp, n_idx);
    for (long long b = p0; b < p1; b += 32) {
      int my = (b + lane < p1) ? idx[b + lane] : 0;
      int n = (int)min(32LL, p1 - b);
      for (int q0 = 0; q0 < n; q0 += U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int r = __shfl_sync(0xffffffffu, my, (q0 + u) & 31);
          if (q0 + u >= n) v[u] = make_float4(0, 0, 0, 0);
          else if (r < H) v[u] = hub[r * 32 + lane];
          else v[u] = ldp<POL>(table + (size_t)r * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
      }
    }
  }
  out[warp0 * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

static float* g_flush = nullptr;
static size_t g_reserve = 0;

template <int U, int POL = 0>
float run(const float4* t, const int* idx, long long n, int per_warp, int threads, int per_sm, int H, float* out) {
  const size_t smem = (size_t)H * 512 + g_reserve;
  cudaFuncSetAttribute(gather_hub<U, POL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int blocks = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) gather_hub<U, POL><<<blocks, threads, smem>>>(t, idx, n, per_warp, H, out);
  const int reps = 10;
  float total = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(g_flush, r, 512ull << 20);
    cudaEventRecord(a);
    gather_hub<U, POL><<<blocks, threads, smem>>>(t, idx, n, per_warp, H, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    total += ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return total / reps;
}

// same walk, but each lane copies its 16 bytes of a gathered row into a per-warp
// shared-memory ring with cp.async.cg (L2 -> SMEM, no L1 allocation); D rows in flight
template <int D>
__global__ void gather_cpasync(const float4* __restrict__ table, const int* __restrict__ idx, long long n_idx,
                               int per_warp, float* __restrict__ out) {
  extern __shared__ float4 ring_all[];
  const int lane = threadIdx.x & 31;
  float4* ring = ring_all + (threadIdx.x >> 5) * D * 32;
  const long long warps_total = (long long)gridDim.x * (blockDim.x >> 5);
  const long long warp0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long w = warp0; w * per_warp < n_idx; w += warps_total) {
    const long long p0 = w * per_warp;
    const long long p1 = min(p0 + per_warp, n_idx);
    const int n = (int)(p1 - p0);
    auto issue = [&](int q) {
      int r = q < n ? __ldg(idx + p0 + q) : 0;
      const unsigned s = (unsigned)__cvta_generic_to_shared(ring + (q % D) * 32 + lane);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(table + (size_t)r * 32 + lane),
                   "r"(q < n ? 16 : 0) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int q = 0; q < D - 1; ++q) issue(q);
    for (int q = 0; q < n; ++q) {
      issue(q + D - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
      const float4 v = ring[(q % D) * 32 + lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  out[warp0 * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
}

template <int D>
float run_cp(const float4* t, const int* idx, long long n, int per_warp, int threads, int per_sm, float* out) {
  const size_t smem = (size_t)(threads / 32) * D * 512;
  cudaFuncSetAttribute(gather_cpasync<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int blocks = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) gather_cpasync<D><<<blocks, threads, smem>>>(t, idx, n, per_warp, out);
  const int reps = 10;
  float total = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(g_flush, r, 512ull << 20);
    cudaEventRecord(a);
    gather_cpasync<D><<<blocks, threads, smem>>>(t, idx, n, per_warp, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    total += ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return total / reps;
}

// 256-bit loads: a half-warp covers a 512-byte row (8 floats per lane), so one warp
// instruction gathers two rows (indices q and q+1 of the warp's chunk); U pairs in flight
__device__ __forceinline__ void ld256(const float* p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
template <int U>
__global__ void gather256(const float* __restrict__ table, const int* __restrict__ idx, long long n_idx,
                          int per_warp, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;
  const long long warps_total = (long long)gridDim.x * (blockDim.x >> 5);
  const long long warp0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (long long w = warp0; w * per_warp < n_idx; w += warps_total) {
    const long long p0 = w * per_warp;
    const long long p1 = min(p0 + per_warp, n_idx);
    for (long long b = p0; b < p1; b += 32) {
      int my = (b + lane < p1) ? idx[b + lane] : -1;
      int n = (int)min(32LL, p1 - b);
      for (int q0 = 0; q0 < n; q0 += 2 * U) {
        float v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = q0 + 2 * u + half;
          int r = __shfl_sync(0xffffffffu, my, q & 31);
          if (q < n) ld256(table + (size_t)r * 128 + hl * 8, v[u]);
          else { for (int e = 0; e < 8; ++e) v[u][e] = 0.f; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += v[u][e];
      }
    }
  }
  float t = 0;
  for (int e = 0; e < 8; ++e) t += acc[e];
  out[warp0 * 32 + lane] = t;
}

template <int U>
float run256(const float* t, const int* idx, long long n, int per_warp, int threads, int per_sm, float* out) {
  const int blocks = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) gather256<U><<<blocks, threads>>>(t, idx, n, per_warp, out);
  const int reps = 10;
  float total = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(g_flush, r, 512ull << 20);
    cudaEventRecord(a);
    gather256<U><<<blocks, threads>>>(t, idx, n, per_warp, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    total += ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return total / reps;
}

int main(int argc, char** argv) {
  if (argc < 2) { printf("usage: hub_probe colidx.bin\n"); return 1; }
  cudaMalloc(&g_flush, 512ull << 20);
  FILE* f = fopen(argv[1], "rb");
  fseek(f, 0, SEEK_END);
  long long m = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  std::vector<int> hi(m);
  size_t got = fread(hi.data(), 4, m, f);
  fclose(f);
  int* di; cudaMalloc(&di, m * 4);
  cudaMemcpy(di, hi.data(), got * 4, cudaMemcpyHostToDevice);
  float4* table; cudaMalloc(&table, 200000ull * 512);
  cudaMemset(table, 0, 200000ull * 512);
  float* out; cudaMalloc(&out, 64 << 20);
  const double gb = m * 512.0 / 1e9;
  struct Cfg { int threads, per_sm, H; };
  for (Cfg c : {Cfg{256, 4, 0}, Cfg{256, 6, 0}, Cfg{256, 8, 0}}) {
    for (int pw : {32, 128}) {
      float m8 = run<8>(table, di, m, pw, c.threads, c.per_sm, c.H, out);
      float m16 = run<16>(table, di, m, pw, c.threads, c.per_sm, c.H, out);
      printf("thr %4d x%d/SM H %3d per_warp %3d: U8 %6.1f us (%6.0f GB/s)  U16 %6.1f us (%6.0f GB/s)\n", c.threads,
             c.per_sm, c.H, pw, m8 * 1e3, gb / (m8 * 1e-3), m16 * 1e3, gb / (m16 * 1e-3));
    }
  }
  for (int pw : {32, 64, 128}) {
    printf("256-bit per_warp %3d: U2 %.1f  U4 %.1f  U8 %.1f us  | x8/SM U4 %.1f\n", pw,
           1e3 * run256<2>((const float*)table, di, m, pw, 256, 4, out),
           1e3 * run256<4>((const float*)table, di, m, pw, 256, 4, out),
           1e3 * run256<8>((const float*)table, di, m, pw, 256, 4, out),
           1e3 * run256<4>((const float*)table, di, m, pw, 256, 8, out));
  }
  // shared memory reserved but unused (shrinks L1 like the merge kernel's staging does)
  for (int rsv_kb : {0, 16, 32, 46, 56}) {
    g_reserve = rsv_kb * 1024;
    printf("reserve %2d KB/CTA x4: U8 %.1f us\n", rsv_kb, 1e3 * run<8, 0>(table, di, m, 32, 256, 4, 0, out));
  }
  g_reserve = 0;
  for (int pw : {32, 128}) {
    printf("policy per_warp %3d: U8 ldg %.1f  no_alloc %.1f  evict_first %.1f  cg %.1f  evict_last %.1f | U4 ldg %.1f no_alloc %.1f cg %.1f | U6 ldg %.1f us\n", pw,
           1e3 * run<8, 0>(table, di, m, pw, 256, 4, 0, out), 1e3 * run<8, 1>(table, di, m, pw, 256, 4, 0, out),
           1e3 * run<8, 2>(table, di, m, pw, 256, 4, 0, out), 1e3 * run<8, 3>(table, di, m, pw, 256, 4, 0, out),
           1e3 * run<8, 4>(table, di, m, pw, 256, 4, 0, out), 1e3 * run<4, 0>(table, di, m, pw, 256, 4, 0, out),
           1e3 * run<4, 1>(table, di, m, pw, 256, 4, 0, out), 1e3 * run<4, 3>(table, di, m, pw, 256, 4, 0, out),
           1e3 * run<6, 0>(table, di, m, pw, 256, 4, 0, out));
  }
  struct CCfg { int threads, per_sm; };
  if (argc > 2)
  for (CCfg c : {CCfg{256, 4}, CCfg{256, 3}, CCfg{256, 2}, CCfg{512, 1}, CCfg{512, 2}}) {
    for (int pw : {32, 128}) {
      const int warps = c.threads / 32 * c.per_sm;
      float m8 = warps * 8 * 512 <= 220 * 1024 ? run_cp<8>(table, di, m, pw, c.threads, c.per_sm, out) : 0.f;
      float m12 = warps * 12 * 512 <= 220 * 1024 ? run_cp<12>(table, di, m, pw, c.threads, c.per_sm, out) : 0.f;
      float m16 = warps * 16 * 512 <= 220 * 1024 ? run_cp<16>(table, di, m, pw, c.threads, c.per_sm, out) : 0.f;
      float m24 = warps * 24 * 512 <= 220 * 1024 ? run_cp<24>(table, di, m, pw, c.threads, c.per_sm, out) : 0.f;
      printf("cp.async thr %4d x%d/SM per_warp %3d: D8 %6.1f  D12 %6.1f  D16 %6.1f  D24 %6.1f us\n", c.threads,
             c.per_sm, pw, m8 * 1e3, m12 * 1e3, m16 * 1e3, m24 * 1e3);
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
