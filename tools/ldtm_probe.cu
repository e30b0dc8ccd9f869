// Throughput / latency of tcgen05.ld.32x32b.x4 (TMEM -> registers) as the COLTILE kernel issues it:
// batches of NB loads, one tcgen05.wait::ld, then 2 packed FMAs per load; W warps per SM.
// Answers: what does one SM's TMEM read path deliver (bytes / clk), and how long is one
// load -> wait round trip -- i.e. what bounds coltile_tmem_kernel once its instruction stream is lean.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ldtm_probe tools/ldtm_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NB, bool FMA>
__global__ void probe(float* out, long long* cycles, int reps) {
  __shared__ uint32_t tbase_s;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tbase_s;
  const uint32_t tq = tbase + ((uint32_t)(32 * (warp % 4)) << 16);
  // defined contents
  for (int c = 0; c < 512; c += 4)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(tq + c), "r"(0x3f800000u));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  __syncthreads();
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  uint32_t addr = tq + 4 * (tid & 7);
  const long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    uint32_t v[NB][4];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]) : "r"(addr));
      addr = tq + ((addr + 20) & 511 & ~3u);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (FMA) {
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        a0 = fmaf(1.0001f, __uint_as_float(v[u][0]), a0);
        a1 = fmaf(1.0001f, __uint_as_float(v[u][1]), a1);
        a2 = fmaf(1.0001f, __uint_as_float(v[u][2]), a2);
        a3 = fmaf(1.0001f, __uint_as_float(v[u][3]), a3);
      }
    } else {
#pragma unroll
      for (int u = 0; u < NB; ++u) a0 += __uint_as_float(v[u][0] ^ v[u][1] ^ v[u][2] ^ v[u][3]);
    }
  }
  const long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + tid] = a0 + a1 + a2 + a3;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int NB, bool FMA>
void run(int warps, float* d_out, long long* d_cyc) {
  const int reps = 8192;
  probe<NB, FMA><<<148, warps * 32>>>(d_out, d_cyc, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return; }
  long long cyc[148];
  cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += (double)cyc[i];
  mean /= 148;
  const double per_batch = mean / reps;               // cycles per batch per warp (latency of the round trip)
  const double loads = (double)reps * NB * warps;     // warp-loads per SM
  printf("warps %2d  batch %2d  %s: %7.1f cycles per batch per warp, %5.2f cycles per warp-load per SM, %6.1f B/clk/SM\n",
         warps, NB, FMA ? "+8 FMA/ld" : "xor only ", per_batch, mean / loads, loads * 512.0 / mean);
}

int main() {
  float* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 148 * 1024 * sizeof(float));
  cudaMalloc(&d_cyc, 148 * sizeof(long long));
  for (int warps : {1, 4, 8, 16, 32}) {
    run<1, true>(warps, d_out, d_cyc);
    run<4, true>(warps, d_out, d_cyc);
    run<8, true>(warps, d_out, d_cyc);
    run<16, false>(warps, d_out, d_cyc);
  }
  return 0;
}
