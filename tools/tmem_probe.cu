// Probe of the TMEM operand path used by the COLTILE-TMEM kernel (sm_100a):
// smem rows of 512 B -> tcgen05.cp.32x128b.warpx4 (broadcast to all four lane
// quarters) -> tcgen05.ld.32x32b.x4 per warp. Verifies the data layout and
// times tcgen05.ld throughput against LDS.128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t cp_desc(const void* smem_row) {
  // K-major, SWIZZLE_NONE: 32 rows of 16 B contiguous = 4 core matrices (8 x 16 B) at SBO = 128 B
  const uint64_t addr = (smem_u32(smem_row) >> 4) & 0x3fff;
  const uint64_t lbo = (128 >> 4) & 0x3fff;
  const uint64_t sbo = (128 >> 4) & 0x3fff;
  return addr | (lbo << 16) | (sbo << 32) | (1ull << 46);  // version 1, base offset 0, layout SWIZZLE_NONE
}

__global__ void probe(float* out, long long* cycles, int reps) {
  __shared__ __align__(1024) float rows[64][128];
  __shared__ uint32_t tbase_s;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 64 * 128; i += blockDim.x) rows[i / 128][i % 128] = (float)(i / 128) * 1000.f + (float)(i % 128);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tbase_s;
  if (tid == 0) {
    for (int j = 0; j < 64; ++j) {
      const uint64_t d = cp_desc(&rows[j][0]);
      const uint32_t taddr = tbase + 4 * j;
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(d));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait phase 0
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads j = warp*3 % 64 from its lane quarter
  const int j = (warp * 3) % 64;
  const uint32_t taddr = tbase + ((uint32_t)(32 * (warp % 4)) << 16) + 4 * j;
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[(tid * 4) + 0] = __uint_as_float(r0);
  out[(tid * 4) + 1] = __uint_as_float(r1);
  out[(tid * 4) + 2] = __uint_as_float(r2);
  out[(tid * 4) + 3] = __uint_as_float(r3);

  // throughput: tcgen05.ld x4 batches of 8 vs LDS.128
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    uint32_t v[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t a = tbase + ((uint32_t)(32 * (warp % 4)) << 16) + 4 * ((it * 8 + u) & 63);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]) : "r"(a));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += __uint_as_float(v[u][0]) + __uint_as_float(v[u][3]);
  }
  long long t1 = clock64();
  for (int it = 0; it < reps; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 x = *reinterpret_cast<const float4*>(&rows[(it * 8 + u) & 63][lane * 4]);
      acc += x.x + x.w;
    }
  }
  long long t2 = clock64();
  // latency of one 64-row chunk copy: 64 x tcgen05.cp + commit + mbarrier wait (thread 0 alone)
  long long t3 = 0, t4 = 0;
  if (tid == 0) {
    t3 = clock64();
    for (int it = 0; it < 32; ++it) {
      for (int j = 0; j < 64; ++j)
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase + 256 + 4 * j),
                     "l"(cp_desc(&rows[j][0])));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar)));
      const uint32_t par = (uint32_t)((it + 1) & 1);
      asm volatile(
          "{\n .reg .pred p;\n LAB_WAIT2:\n"
          " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra LAB_WAIT2;\n}\n" ::"r"(smem_u32(&mbar)), "r"(par));
    }
    t4 = clock64();
  }
  if (tid == 0) {
    cycles[0] = t1 - t0;
    cycles[1] = t2 - t1;
    cycles[2] = t4 - t3;
  }
  if (acc == 1234.5f) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  float* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 512 * 4 * sizeof(float));
  cudaMalloc(&d_cyc, 3 * sizeof(long long));
  const int reps = 4096;
  probe<<<1, 512>>>(d_out, d_cyc, reps);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  float h[512 * 4];
  long long cyc[3];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int tid = 0; tid < 512; ++tid) {
    const int warp = tid / 32, lane = tid % 32, j = (warp * 3) % 64;
    for (int e2 = 0; e2 < 4; ++e2) {
      const float want = (float)j * 1000.f + (float)(lane * 4 + e2);
      if (h[tid * 4 + e2] != want) {
        if (bad < 8) printf("mismatch tid %d e %d: got %f want %f\n", tid, e2, h[tid * 4 + e2], want);
        ++bad;
      }
    }
  }
  printf("layout check: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  const double n_ld = (double)reps * 8 * 16;  // warp-level loads per SM (16 warps)
  printf("tcgen05.ld.32x32b.x4: %.2f cycles per warp-load (16 warps, batches of 8)\n", (double)cyc[0] / (reps * 8));
  printf("LDS.128            : %.2f cycles per warp-load\n", (double)cyc[1] / (reps * 8));
  printf("64-row chunk copy (64 x tcgen05.cp.32x128b.warpx4 + commit + wait): %.0f cycles\n", (double)cyc[2] / 32);
  (void)n_ld;
  return 0;
}
