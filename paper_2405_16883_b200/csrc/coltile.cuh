// K3: column-tiled CSR SpMM for wide dense operands (sm_100a).
//
// C[r, c0:c0+128] = sum_p val[p] * B[col[p], c0:c0+128] for a block of 64 rows.
// The dense operand is streamed through shared memory in 64-row chunks
// (cp.async double buffering, L2 -> SMEM, bypassing L1) and every staged row is
// reused by all rows of the block that hold that column (~6.4 at 10% density),
// so L2 traffic is (rows / 64) x |B| instead of nnz x 512 B of gathers. Each
// warp owns 8 rows x 128 columns of accumulators in registers; per stored
// entry a lane does one LDS.128 and four FFMAs. Row cursors advance
// monotonically through the sorted column indices of each row.
#pragma once

#include "stc_common.cuh"

namespace stc {

constexpr int CT_ROWS = 64;         // rows per CTA
constexpr int CT_COLS = 128;        // output columns per CTA (32 lanes x float4)
constexpr int CT_CHUNK = 64;        // staged B rows per stage
constexpr int CT_WARPS = 8;
constexpr int CT_RPW = CT_ROWS / CT_WARPS;  // rows per warp

STC_DEVICE void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
STC_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
STC_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int EPI, bool ADD>
__global__ void __launch_bounds__(256) coltile_kernel(int m, int n, int k, const int* __restrict__ rowptr,
                                                      const int* __restrict__ colidx,
                                                      const float* __restrict__ vals,
                                                      const float* __restrict__ B, long long ldb,
                                                      float* __restrict__ C, long long ldc,
                                                      const float* __restrict__ D, long long ldd) {
  extern __shared__ __align__(16) float smem[];  // [2][CT_CHUNK][CT_COLS]
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int row_base = blockIdx.x * CT_ROWS + warp * CT_RPW;
  const int c0 = blockIdx.y * CT_COLS;
  const int col = c0 + lane * 4;
  const bool col_ok = col < k;

  // per-row cursors and lane-parallel (col, val) batches
  int pcur[CT_RPW], pend[CT_RPW], bcol[CT_RPW];
  float bval[CT_RPW];
  float acc[CT_RPW][4];
#pragma unroll
  for (int r = 0; r < CT_RPW; ++r) {
    const int row = row_base + r;
    pcur[r] = row < m ? rowptr[row] : 0;
    pend[r] = row < m ? rowptr[row + 1] : 0;
    const int p = pcur[r] + lane;
    bcol[r] = p < pend[r] ? ld_stream(colidx + p) : INT_MAX;
    bval[r] = p < pend[r] ? ld_stream(vals + p) : 0.f;
    acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;
  }
  int bpos[CT_RPW];  // index of the next unconsumed entry inside the lane batch
#pragma unroll
  for (int r = 0; r < CT_RPW; ++r) bpos[r] = 0;

  auto stage = [&](int chunk, int buf) {
    const int j0 = chunk * CT_CHUNK;
    float* dst = smem + buf * CT_CHUNK * CT_COLS;
    // 64 rows x 32 float4 = 2048 16-byte copies, 8 per thread
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int idx = threadIdx.x + t * 256;
      const int jr = idx / 32, cq = idx % 32;
      const int j = j0 + jr;
      const int cc = c0 + cq * 4;
      const bool ok = (j < n) && (cc < k);
      cp_async16(dst + jr * CT_COLS + cq * 4, ok ? (const void*)(B + (long long)j * ldb + cc) : (const void*)B, ok);
    }
    cp_async_commit();
  };

  const int n_chunks = (n + CT_CHUNK - 1) / CT_CHUNK;
  if (n_chunks > 0) stage(0, 0);
  for (int ch = 0; ch < n_chunks; ++ch) {
    if (ch + 1 < n_chunks) {
      stage(ch + 1, (ch + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* tile = smem + (ch & 1) * CT_CHUNK * CT_COLS;
    const int jhi = (ch + 1) * CT_CHUNK;
    const int j0 = ch * CT_CHUNK;
#pragma unroll
    for (int r = 0; r < CT_RPW; ++r) {
      while (true) {
        const int c = __shfl_sync(0xffffffffu, bcol[r], bpos[r]);
        if (c >= jhi) break;  // INT_MAX once the row is exhausted
        const float v = __shfl_sync(0xffffffffu, bval[r], bpos[r]);
        if (col_ok) {
          const float4 x = *reinterpret_cast<const float4*>(tile + (c - j0) * CT_COLS + lane * 4);
          acc[r][0] = fmaf(v, x.x, acc[r][0]);
          acc[r][1] = fmaf(v, x.y, acc[r][1]);
          acc[r][2] = fmaf(v, x.z, acc[r][2]);
          acc[r][3] = fmaf(v, x.w, acc[r][3]);
        }
        if (++bpos[r] == 32) {
          pcur[r] += 32;
          const int p = pcur[r] + lane;
          bcol[r] = p < pend[r] ? ld_stream(colidx + p) : INT_MAX;
          bval[r] = p < pend[r] ? ld_stream(vals + p) : 0.f;
          bpos[r] = 0;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < CT_RPW; ++r) {
    const int row = row_base + r;
    if (row < m && col_ok) {
      float4 o = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      if constexpr (ADD) {
        const float4 d = *reinterpret_cast<const float4*>(D + (long long)row * ldd + col);
        o.x += d.x; o.y += d.y; o.z += d.z; o.w += d.w;
      }
      o.x = act<EPI>(o.x); o.y = act<EPI>(o.y); o.z = act<EPI>(o.z); o.w = act<EPI>(o.w);
      st_stream4(C + (long long)row * ldc + col, o);
    }
  }
}

}  // namespace stc
