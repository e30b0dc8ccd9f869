// Probe: does the B200's two-die L2 cap cfg2's gather, and does a die-aware split of the
// dense operand's columns lift it?  (ceiling analysis for the SpMM kernel; not part of the library)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/die_probe tools/die_probe.cu
//   tools/die_probe tools/cfg2_colidx.bin
// 1. SM -> die map: every SM times dependent L2 loads (ld.global.cg) to 64 addresses 4 KB
//    apart; an address is homed on one die, so SMs on the same die see the same near/far
//    pattern.  SMs are grouped by that pattern.
// 2. Uniform random 512-byte row gathers over tables of 16..112 MB (no flush): where does the
//    L2 stop holding the table?
// 3. cfg2's real index stream over a 200,000 x 128 fp32 table: every SM gathers whole rows
//    (baseline) vs. SMs of die d gather only columns [64d, 64d+64) of every row (each die's
//    L2 then needs half the table) vs. the same split with a group map unrelated to the dies.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }

__global__ void lat_k(const int* __restrict__ buf, int naddr, int stride_ints, unsigned* lat, int nsm_max, int iters) {
  extern __shared__ int pad[];
  if (threadIdx.x) return;
  unsigned s = smid();
  if (s >= (unsigned)nsm_max) return;
  pad[0] = 0;
  for (int a = 0; a < naddr; ++a) {
    const int* p = buf + (size_t)a * stride_ints;
    unsigned best = 0xffffffffu;
    int v = 0;
    for (int rep = 0; rep < 6; ++rep) {
      long long t0 = clock64();
      for (int c = 0; c < iters; ++c) {
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p + v));
      }
      long long t1 = clock64();
      pad[1 + (v & 7)] = v;
      unsigned d = (unsigned)((t1 - t0) / iters);
      if (rep > 0) best = min(best, d);
    }
    lat[s * naddr + a] = best;
  }
}

// MODE 0: every CTA gathers whole 512-byte rows.  MODE 1: a CTA on group g gathers the 256-byte
// half g of every row (two rows per warp instruction).  Work = chunks of the index stream taken
// from a per-group ticket counter (each group walks the whole stream once).
template <int MODE, int U>
__global__ void __launch_bounds__(256) gather_k(const float4* __restrict__ table, const int* __restrict__ idx,
                                                long long n, int chunk, const unsigned char* __restrict__ group,
                                                int* tickets, float* __restrict__ out) {
  __shared__ int s_c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = MODE ? group[smid()] : 0;
  const long long nchunks = (n + chunk - 1) / chunk;
  float4 acc = make_float4(0, 0, 0, 0);
  for (;;) {
    if (threadIdx.x == 0) s_c = atomicAdd(&tickets[g], 1);
    __syncthreads();
    const long long c = s_c;
    __syncthreads();
    if (c >= nchunks) break;
    const int per_warp = chunk / 8;
    long long p0 = c * chunk + (long long)warp * per_warp;
    long long p1 = min(p0 + per_warp, n);
    for (long long b = p0; b < p1; b += 32) {
      int my = (b + lane < p1) ? __ldg(idx + b + lane) : -1;
      int cnt = (int)min(32LL, p1 - b);
      if (MODE == 0) {
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
      } else {
        const int half = lane >> 4, sub = lane & 15;
        for (int q0 = 0; q0 < cnt; q0 += 2 * U) {
          float4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            int q = q0 + 2 * u + half;
            int r = __shfl_sync(0xffffffffu, my, q & 31);
            v[u] = (q < cnt) ? __ldg(table + (size_t)r * 32 + g * 16 + sub) : make_float4(0, 0, 0, 0);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
        }
      }
    }
  }
  out[(blockIdx.x * 256 + threadIdx.x) & ((1 << 20) - 1)] += acc.x + acc.y + acc.z + acc.w;
}

static float* g_flush = nullptr;

template <int MODE, int U>
float run(const float4* t, const int* idx, long long n, const unsigned char* grp, int* tickets, float* out,
          int ctas_per_sm, bool flush, int nsm) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int chunk = 2048;
  float best = 1e30f;
  for (int r = 0; r < 12; ++r) {
    if (flush) cudaMemsetAsync(g_flush, r, 512ull << 20);
    cudaMemsetAsync(tickets, 0, 8);
    cudaEventRecord(a);
    gather_k<MODE, U><<<nsm * ctas_per_sm, 256>>>(t, idx, n, chunk, grp, tickets, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) best = std::min(best, ms);
  }
  return best * 1e3f;  // us
}

int main(int argc, char** argv) {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&g_flush, 512ull << 20);
  // ---- 1. SM -> die map
  const int naddr = 64, stride = 1024;  // 4 KB apart
  int* buf; cudaMalloc(&buf, (size_t)naddr * stride * 4); cudaMemset(buf, 0, (size_t)naddr * stride * 4);
  unsigned* lat; cudaMalloc(&lat, nsm * naddr * 4); cudaMemset(lat, 0xff, nsm * naddr * 4);
  cudaFuncSetAttribute(lat_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  lat_k<<<nsm, 32, 150 * 1024>>>(buf, naddr, stride, lat, nsm, 32);
  printf("lat_k: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<unsigned> hl(nsm * naddr);
  cudaMemcpy(hl.data(), lat, hl.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<int> sig(nsm, 0);
  std::vector<unsigned char> die(nsm, 0);
  std::vector<std::vector<int>> far(nsm, std::vector<int>(naddr));
  for (int a = 0; a < naddr; ++a) {
    std::vector<unsigned> col;
    for (int s = 0; s < nsm; ++s) col.push_back(hl[s * naddr + a]);
    std::vector<unsigned> srt = col; std::sort(srt.begin(), srt.end());
    unsigned med = (srt[nsm / 2 - 1] + srt[nsm / 2]) / 2;
    for (int s = 0; s < nsm; ++s) far[s][a] = col[s] > med;
  }
  // group = agreement with SM 0's pattern
  int n0 = 0, ambiguous = 0;
  for (int s = 0; s < nsm; ++s) {
    int agree = 0;
    for (int a = 0; a < naddr; ++a) agree += far[s][a] == far[0][a];
    die[s] = agree * 2 < naddr;
    if (agree > naddr / 8 && agree < naddr - naddr / 8) ++ambiguous;
    n0 += die[s] == 0;
  }
  printf("die map: %d SMs with SM0, %d on the other die, %d ambiguous\n", n0, nsm - n0, ambiguous);
  printf("lat sample (SM0): ");
  for (int a = 0; a < 16; ++a) printf("%u ", hl[a]);
  printf("\nmap: ");
  for (int s = 0; s < nsm; ++s) printf("%d", die[s]);
  printf("\n");
  unsigned char *dgrp, *pgrp;
  cudaMalloc(&dgrp, 1024); cudaMalloc(&pgrp, 1024);
  cudaMemcpy(dgrp, die.data(), nsm, cudaMemcpyHostToDevice);
  std::vector<unsigned char> par(nsm);
  for (int s = 0; s < nsm; ++s) par[s] = s & 1;  // control: a split unrelated to the dies
  if (std::count(par.begin(), par.end(), 0) == n0) {}
  cudaMemcpy(pgrp, par.data(), nsm, cudaMemcpyHostToDevice);

  // ---- 2. table-size sweep
  size_t tbytes = 120ull << 20;
  float4* table; cudaMalloc(&table, tbytes); cudaMemset(table, 0, tbytes);
  float* out; cudaMalloc(&out, 4 << 20); cudaMemset(out, 0, 4 << 20);
  int* tickets; cudaMalloc(&tickets, 64);
  const long long n = 2200000;
  int* idx; cudaMalloc(&idx, n * 4);
  std::vector<int> h(n);
  for (int mb : {8, 16, 32, 48, 64, 80, 96, 112}) {
    long long rows = (long long)mb * (1 << 20) / 512;
    srand(1);
    for (long long i = 0; i < n; ++i) h[i] = (int)(((long long)rand() * 7919LL + rand()) % rows);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    float t0 = run<0, 8>(table, idx, n, dgrp, tickets, out, 4, false, nsm);
    float t1 = run<1, 8>(table, idx, n, dgrp, tickets, out, 4, false, nsm);
    float t2 = run<1, 8>(table, idx, n, pgrp, tickets, out, 4, false, nsm);
    double gb = n * 512.0 / 1e3;  // bytes / us -> GB/s * 1e-3
    printf("uniform table %4d MB: whole rows %6.1f us (%5.0f GB/s) | die split %6.1f us (%5.0f GB/s) | parity split %6.1f us (%5.0f GB/s)\n",
           mb, t0, gb / t0, t1, gb / t1, t2, gb / t2);
  }
  // ---- 3. real cfg2 stream
  if (argc > 1) {
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
    double gb = m * 512.0 / 1e3;
    for (int fl = 0; fl < 2; ++fl) {
      for (int cps : {2, 4, 8}) {
        float t0 = run<0, 8>(table, di, m, dgrp, tickets, out, cps, fl, nsm);
        float t1 = run<1, 8>(table, di, m, dgrp, tickets, out, cps, fl, nsm);
        float t2 = run<1, 8>(table, di, m, pgrp, tickets, out, cps, fl, nsm);
        float t3 = run<1, 4>(table, di, m, dgrp, tickets, out, cps, fl, nsm);
        printf("cfg2 stream flush=%d ctas/SM %d: whole rows %6.1f us (%5.0f GB/s) | die split U8 %6.1f us (%5.0f) U4 %6.1f us | parity split %6.1f us (%5.0f)\n",
               fl, cps, t0, gb / t0, t1, gb / t1, t3, t2, gb / t2);
      }
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
