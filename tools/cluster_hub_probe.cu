// Microbenchmark: a CLUSTER-wide hub for the hottest dense rows.
// The H hottest rows of the 200000 x 128 fp32 operand (cfg2: low index = hot) are spread over the
// shared memories of a CL-CTA thread-block cluster (row r lives in CTA r % CL, slot r / CL); a
// gather of row r < H is served by `ld.shared::cluster` (DSMEM) from whichever CTA owns it, any
// other gather by LDG as in the shipped kernel. Same walk as hub_probe.cu (no FMA, no output).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_hub_probe tools/cluster_hub_probe.cu
//   tools/cluster_hub_probe tools/cfg2_colidx.bin
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ float4 ld_dsmem(unsigned addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ unsigned mapa(unsigned local, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

// MODE 0: hub rows from DSMEM; MODE 1: hub rows counted but still gathered by LDG (baseline with the
// same shared memory reserved); MODE 2: only the rows the CTA itself owns come from (local) SMEM.
template <int U, int MODE>
__global__ void gather_cluster_hub(const float4* __restrict__ table, const int* __restrict__ idx, long long n_idx,
                                   int per_warp, int H, int CL, float* __restrict__ out) {
  extern __shared__ float4 hub[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const int lane = threadIdx.x & 31;
  const int mine = (H + CL - 1 - (int)rank) / CL;  // rows r < H with r % CL == rank
  for (int t = threadIdx.x; t < mine * 32; t += blockDim.x) {
    const int slot = t >> 5;
    hub[t] = table[(size_t)(slot * CL + rank) * 32 + (t & 31)];
  }
  cluster.sync();
  const unsigned hub_base = (unsigned)__cvta_generic_to_shared(hub);
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
          else if (MODE == 0 && r < H)
            v[u] = ld_dsmem(mapa(hub_base + (unsigned)(((r / CL) * 32 + lane) * 16), (unsigned)(r % CL)));
          else if (MODE == 2 && r < H && (unsigned)(r % CL) == rank)
            v[u] = hub[(r / CL) * 32 + lane];
          else v[u] = __ldg(table + (size_t)r * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
      }
    }
  }
  out[warp0 * 32 + lane] = acc.x + acc.y + acc.z + acc.w;
  cluster.sync();  // no CTA may exit while a peer still reads its shared memory
}

static float* g_flush = nullptr;

template <int U, int MODE>
float run(const float4* t, const int* idx, long long n, int per_warp, int threads, int per_sm, int H, int CL,
          float* out) {
  auto kern = gather_cluster_hub<U, MODE>;
  const size_t smem = (size_t)((H + CL - 1) / CL) * 512;
  if (smem > 227 * 1024) return -1.f;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int blocks = 148 * per_sm;
  blocks -= blocks % CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, kern, t, idx, n, per_warp, H, CL, out);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(cudaGetLastError())); return -1.f; }
  const int reps = 10;
  float total = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(g_flush, r, 512ull << 20);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kern, t, idx, n, per_warp, H, CL, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    total += ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return -1.f; }
  return total / reps;
}

int main(int argc, char** argv) {
  if (argc < 2) { printf("usage: cluster_hub_probe colidx.bin\n"); return 1; }
  cudaMalloc(&g_flush, 512ull << 20);
  FILE* f = fopen(argv[1], "rb");
  if (!f) { printf("cannot open %s\n", argv[1]); return 1; }
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
  struct Cfg { int threads, per_sm, CL, H; };
  const Cfg cfgs[] = {
      {1024, 1, 8, 0},    {1024, 1, 8, 256},  {1024, 1, 8, 800},   {1024, 1, 8, 1600}, {1024, 1, 8, 3200},
      {1024, 1, 16, 0},   {1024, 1, 16, 1600}, {1024, 1, 16, 3200}, {1024, 1, 16, 6400},
      {512, 2, 8, 0},     {512, 2, 8, 800},   {512, 2, 8, 1600},
      {256, 4, 8, 0},     {256, 4, 8, 400},   {256, 4, 8, 800},
      {256, 4, 16, 400},  {256, 4, 16, 1600},
  };
  for (const Cfg& c : cfgs) {
    long long hits = 0;
    for (long long i = 0; i < m; ++i) hits += hi[i] < c.H;
    for (int pw : {32, 128}) {
      float d = run<8, 0>(table, di, m, pw, c.threads, c.per_sm, c.H, c.CL, out);
      float l = run<8, 1>(table, di, m, pw, c.threads, c.per_sm, c.H, c.CL, out);
      float s = run<8, 2>(table, di, m, pw, c.threads, c.per_sm, c.H, c.CL, out);
      printf("thr %4d x%d/SM cluster %2d H %4d (%4.1f%% of gathers, %3d KB/CTA) per_warp %3d: DSMEM hub %6.1f us | "
             "LDG only (same smem reserved) %6.1f us | own rows from local smem %6.1f us\n",
             c.threads, c.per_sm, c.CL, c.H, 100.0 * hits / m, (int)(((c.H + c.CL - 1) / c.CL) * 512 / 1024), pw,
             d * 1e3, l * 1e3, s * 1e3);
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
