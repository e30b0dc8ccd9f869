// Probe: are cfg2's 512-byte row gathers bound by how many L1 misses an SM keeps in flight?
// If so, gathers issued through the TMA engine (cp.async.bulk global -> shared, completion on an
// mbarrier; no L1 miss tracking involved) add in-flight capacity next to the LDG path.
// Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
//   tools/tma_probe tools/cfg2_colidx.bin
// Kernels (each warp walks `per_warp` consecutive indices of the stream, 512-byte rows):
//   ldg   : LDG.128 ring of U gathers (the merge kernel's scheme)
//   tma   : lane 0 issues one 512-byte bulk copy per row into a D-slot shared-memory ring
//           (one mbarrier per slot); all lanes read the slot with LDS.128
//   mixed : every other row through each path
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned phase) {
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int U>
__global__ void __launch_bounds__(256) ldg_k(const float4* __restrict__ table, const int* __restrict__ idx, long long n,
                                             int per_warp, float* out) {
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * 256LL + threadIdx.x) >> 5;
  long long p0 = gw * per_warp;
  if (p0 >= n) return;
  long long p1 = min(p0 + per_warp, n);
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long b = p0; b < p1; b += 32) {
    int my = (b + lane < p1) ? __ldg(idx + b + lane) : 0;
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

// MIX = 0: every row through the TMA ring; 1: even rows LDG (U-deep ring), odd rows TMA.
template <int D, int MIX>
__global__ void __launch_bounds__(256) tma_k(const float4* __restrict__ table, const int* __restrict__ idx, long long n,
                                             int per_warp, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float4* ring = reinterpret_cast<float4*>(sm) + (size_t)wid * D * 32;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + 8 * D * 512) + wid * D;
  if (lane == 0)
    for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long gw = (blockIdx.x * 256LL + threadIdx.x) >> 5;
  long long p0 = gw * per_warp;
  float4 acc = make_float4(0, 0, 0, 0);
  if (p0 < n) {
    long long p1 = min(p0 + per_warp, n);
    const int cnt = (int)(p1 - p0);
    constexpr int STEP = MIX ? 2 : 1;   // TMA rows: q = STEP*t + (STEP-1)
    const int nt = MIX ? cnt / 2 : cnt;
    auto issue = [&](int t) {
      if (lane == 0 && t < nt) {
        const int r = __ldg(idx + p0 + STEP * t + (STEP - 1));
        const int s = t % D;
        mbar_expect_tx(&bars[s], 512);
        bulk_g2s(ring + s * 32, table + (size_t)r * 32, 512, &bars[s]);
      }
    };
    for (int t = 0; t < D; ++t) issue(t);
    float4 pend = make_float4(0, 0, 0, 0);
    int next_ldg = 0;
    if (MIX && cnt > 0) pend = __ldg(table + (size_t)__ldg(idx + p0) * 32 + lane);
    for (int t = 0; t < nt; ++t) {
      const int s = t % D;
      if (MIX) {  // this turn's LDG row (issued one turn ahead)
        float4 v = pend;
        next_ldg = 2 * (t + 1);
        if (next_ldg < cnt) pend = __ldg(table + (size_t)__ldg(idx + p0 + next_ldg) * 32 + lane);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      mbar_wait(&bars[s], (t / D) & 1);
      float4 v = ring[s * 32 + lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      __syncwarp();
      issue(t + D);
    }
    if (MIX && (cnt & 1)) { acc.x += pend.x; }
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
  auto timeit = [&](auto launch, bool flush) {
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      if (flush) cudaMemsetAsync(fl, r, 512ull << 20);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (r >= 2) best = std::min(best, ms);
    }
    return best * 1e3f;
  };
  for (int fl_ : {1, 0}) {
    for (int pw : {64, 256}) {
      long long warps = (m + pw - 1) / pw;
      int blocks = (int)((warps * 32 + 255) / 256);
      float t_ldg = timeit([&] { ldg_k<8><<<blocks, 256>>>(table, di, m, pw, out); }, fl_);
      printf("flush=%d per_warp %3d  ldg U8          %6.1f us\n", fl_, pw, t_ldg);
      for (int d : {8, 16}) {
        size_t smem = 8ull * d * 512 + 8 * 8 * d;
        if (d == 8) {
          cudaFuncSetAttribute(tma_k<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          cudaFuncSetAttribute(tma_k<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          float t0 = timeit([&] { tma_k<8, 0><<<blocks, 256, smem>>>(table, di, m, pw, out); }, fl_);
          float t1 = timeit([&] { tma_k<8, 1><<<blocks, 256, smem>>>(table, di, m, pw, out); }, fl_);
          printf("flush=%d per_warp %3d  tma D8 %6.1f us | mixed D8 %6.1f us\n", fl_, pw, t0, t1);
        } else {
          cudaFuncSetAttribute(tma_k<16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          cudaFuncSetAttribute(tma_k<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          float t0 = timeit([&] { tma_k<16, 0><<<blocks, 256, smem>>>(table, di, m, pw, out); }, fl_);
          float t1 = timeit([&] { tma_k<16, 1><<<blocks, 256, smem>>>(table, di, m, pw, out); }, fl_);
          printf("flush=%d per_warp %3d  tma D16 %6.1f us | mixed D16 %6.1f us\n", fl_, pw, t0, t1);
        }
      }
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
