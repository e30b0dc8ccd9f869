// EXPERIMENT RECORD (not built): the SMEM-staged COLTILE kernel that shipped before the
// Tensor-Memory kernel (csrc/coltile.cuh) replaced it. cfg3: 6.41 ms (SMEM-crossbar bound:
// one LDS.128 per 4 FFMA) vs 5.10 ms for the TMEM kernel. Needs the cp.async helpers now in
// stc_common.cuh and the per-row chunk_ptr plan (git history, spmm.cu stc_coltile_plan).
// K3: column-tiled CSR SpMM for wide dense operands (sm_100a).
//
// C[r, c0:c0+128] = sum_p val[p] * B[col[p], c0:c0+128] for a block of 128 rows.
//
// The dense operand is streamed through shared memory in CT_CHUNK-row chunks by
// a cp.async ring (L2 -> SMEM, bypassing L1); each staged row is reused by every
// row of the block that holds that column (~12.8 at 10% density), so L2 traffic
// is (rows/128) x |B[:, tile]| instead of nnz x 512 B of gathers. A plan-time
// table (`coltile_plan_kernel`) stores, per row, where each chunk's entries
// start, so a warp reads exactly the entries of (row, chunk) with one coalesced
// load — no searching, no dependent shuffles. 16 warps own 8 rows x 128 columns
// of accumulators each (lane = float4). Per entry the weight and column arrive
// by a broadcast LDS.64 from a per-warp scratch, the operand by one LDS.128, and
// four FFMAs consume them: the SMEM crossbar (about five wavefronts per entry)
// bounds the kernel near a quarter of the FP32 FMA peak.
#pragma once

#include "stc_common.cuh"

namespace stc {

constexpr int CT_ROWS = 128;        // rows per CTA
constexpr int CT_COLS = 128;        // output columns per CTA (32 lanes x float4)
constexpr int CT_CHUNK = 128;       // staged B rows per stage
constexpr int CT_STAGES = 3;
constexpr int CT_WARPS = 16;
constexpr int CT_THREADS = CT_WARPS * 32;
constexpr int CT_RPW = CT_ROWS / CT_WARPS;  // rows per warp
constexpr size_t CT_STAGE_FLOATS = (size_t)CT_CHUNK * CT_COLS;
constexpr int CT_SCRATCH = 256;     // staged (col, val) entries per warp and chunk
constexpr size_t CT_SMEM = CT_STAGES * CT_STAGE_FLOATS * sizeof(float) + (size_t)CT_WARPS * CT_SCRATCH * 8;

// Plan: chunk_ptr[row * (n_chunks + 1) + c] = first entry of `row` with col >= c * CT_CHUNK.
__global__ void coltile_plan_kernel(int m, int n_chunks, const int* __restrict__ rowptr,
                                    const int* __restrict__ colidx, int* __restrict__ chunk_ptr) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= m) return;
  const int a = rowptr[row], b = rowptr[row + 1];
  int* out = chunk_ptr + (long long)row * (n_chunks + 1);
  for (int c = lane; c <= n_chunks; c += 32) {
    // lower_bound of c*CT_CHUNK in colidx[a, b)
    int lo = a, hi = b;
    const int key = c * CT_CHUNK;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (colidx[mid] < key)
        lo = mid + 1;
      else
        hi = mid;
    }
    out[c] = lo;
  }
}


// Per-warp offsets of its CT_RPW rows' entries within one chunk: lane r (< CT_RPW)
// knows start(r), lane CT_RPW + r knows end(r); returns the exclusive prefix of the
// counts for row `lane % CT_RPW` and the total.
STC_DEVICE void chunk_layout(int bounds, int lane, int& my_off, int& total) {
  const int other = __shfl_xor_sync(0xffffffffu, bounds, CT_RPW);  // end for lanes < CT_RPW
  int cnt = (lane < CT_RPW) ? other - bounds : 0;
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < CT_RPW; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  my_off = incl - cnt;
  total = __shfl_sync(0xffffffffu, incl, CT_RPW - 1);
}

constexpr int CT_PREF = CT_SCRATCH / 32;  // prefetched items per lane

template <int EPI, bool ADD>
__global__ void __launch_bounds__(CT_THREADS, 1) coltile_kernel(int m, int n, int k, const int* __restrict__ chunk_ptr,
                                                               const int* __restrict__ colidx,
                                                               const float* __restrict__ vals,
                                                               const float* __restrict__ B, long long ldb,
                                                               float* __restrict__ C, long long ldc,
                                                               const float* __restrict__ D, long long ldd) {
  extern __shared__ __align__(16) float smem[];  // [CT_STAGES][CT_CHUNK][CT_COLS] + per-warp scratch
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int row_base = blockIdx.x * CT_ROWS + warp * CT_RPW;
  const int c0 = blockIdx.y * CT_COLS;
  const int col = c0 + lane * 4;
  const int n_chunks = (n + CT_CHUNK - 1) / CT_CHUNK;
  int2* scratch = reinterpret_cast<int2*>(smem + CT_STAGES * CT_STAGE_FLOATS) + warp * CT_SCRATCH;

  float acc[CT_RPW][4];
#pragma unroll
  for (int r = 0; r < CT_RPW; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;

  auto stage = [&](int chunk) {
    const int j0 = chunk * CT_CHUNK;
    float* dst = smem + (chunk % CT_STAGES) * CT_STAGE_FLOATS;
#pragma unroll
    for (int t = 0; t < (int)(CT_STAGE_FLOATS / 4) / CT_THREADS; ++t) {
      const int idx = threadIdx.x + t * CT_THREADS;
      const int jr = idx / 32, cq = idx % 32;
      const int j = j0 + jr;
      const int cc = c0 + cq * 4;
      const bool ok = (j < n) && (cc < k);
      cp_async16(dst + jr * CT_COLS + cq * 4, ok ? (const void*)(B + (long long)j * ldb + cc) : (const void*)B, ok);
    }
  };

  // lane r (< CT_RPW) reads the chunk start of row r, lane CT_RPW + r its end
  const int prow = row_base + (lane % CT_RPW);
  const bool prow_ok = lane < 2 * CT_RPW && prow < m;
  const int* cp_row = chunk_ptr + (long long)prow * (n_chunks + 1) + (lane >= CT_RPW ? 1 : 0);
  auto load_bounds = [&](int ch) { return (prow_ok && ch < n_chunks) ? ld_stream(cp_row + ch) : 0; };

  // prefetch of one chunk's entries into registers: item idx = t*32 + lane of the
  // concatenation of the warp's rows' entry ranges
  int pc[CT_PREF];
  float pv[CT_PREF];
  auto prefetch = [&](int bnd) {
    int my_off, total;
    chunk_layout(bnd, lane, my_off, total);
    int offs[CT_RPW], starts[CT_RPW];
#pragma unroll
    for (int r = 0; r < CT_RPW; ++r) {  // row r owns items [offs[r], offs[r+1])
      offs[r] = __shfl_sync(0xffffffffu, my_off, r);
      starts[r] = __shfl_sync(0xffffffffu, bnd, r);
    }
#pragma unroll
    for (int t = 0; t < CT_PREF; ++t) {
      const int idx = t * 32 + lane;
      pc[t] = INT_MAX;
      pv[t] = 0.f;
      if (idx < total) {
        int pos = 0;
#pragma unroll
        for (int r = 0; r < CT_RPW; ++r)
          if (idx >= offs[r]) pos = starts[r] + (idx - offs[r]);
        pc[t] = ld_stream(colidx + pos);
        pv[t] = ld_stream(vals + pos);
      }
    }
  };

#pragma unroll
  for (int s = 0; s < CT_STAGES - 1; ++s) {
    if (s < n_chunks) stage(s);
    cp_async_commit();
  }
  int b_cur = load_bounds(0);
  int b_next = load_bounds(1);
  prefetch(b_cur);
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int b_after = load_bounds(ch + 2);
    const int j0 = ch * CT_CHUNK;
    // publish this chunk's prefetched entries (column relative to the chunk)
#pragma unroll
    for (int t = 0; t < CT_PREF; ++t)
      if (pc[t] != INT_MAX) scratch[t * 32 + lane] = make_int2(pc[t] - j0, __float_as_int(pv[t]));
    cp_async_wait<CT_STAGES - 2>();
    __syncthreads();  // chunk ch staged for all; the slot refilled below is no longer read
    if (ch + CT_STAGES - 1 < n_chunks) stage(ch + CT_STAGES - 1);
    cp_async_commit();
    int my_off, total;
    chunk_layout(b_cur, lane, my_off, total);
    prefetch(b_next);  // next chunk's entries stream in while this one is consumed
    const float* tile = smem + (ch % CT_STAGES) * CT_STAGE_FLOATS + lane * 4;
#pragma unroll
    for (int r = 0; r < CT_RPW; ++r) {
      const int o0 = __shfl_sync(0xffffffffu, my_off, r);
      const int o1 = r + 1 < CT_RPW ? __shfl_sync(0xffffffffu, my_off, r + 1) : total;
      const int a = __shfl_sync(0xffffffffu, b_cur, r);
      int q = o0;
      const int qe = min(o1, CT_SCRATCH);
      for (; q + 4 <= qe; q += 4) {
        int2 it[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) it[u] = scratch[q + u];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 x = *reinterpret_cast<const float4*>(tile + it[u].x * CT_COLS);
          const float w = __int_as_float(it[u].y);
          acc[r][0] = fmaf(w, x.x, acc[r][0]);
          acc[r][1] = fmaf(w, x.y, acc[r][1]);
          acc[r][2] = fmaf(w, x.z, acc[r][2]);
          acc[r][3] = fmaf(w, x.w, acc[r][3]);
        }
      }
      for (; q < qe; ++q) {
        const int2 it = scratch[q];
        const float4 x = *reinterpret_cast<const float4*>(tile + it.x * CT_COLS);
        const float w = __int_as_float(it.y);
        acc[r][0] = fmaf(w, x.x, acc[r][0]);
        acc[r][1] = fmaf(w, x.y, acc[r][1]);
        acc[r][2] = fmaf(w, x.z, acc[r][2]);
        acc[r][3] = fmaf(w, x.w, acc[r][3]);
      }
      // overflow beyond the scratch capacity (dense rows): read entries directly
      for (int qq = max(o0, CT_SCRATCH); qq < o1; ++qq) {
        const int pos = a + (qq - o0);
        const float4 x = *reinterpret_cast<const float4*>(tile + (colidx[pos] - j0) * CT_COLS);
        const float w = vals[pos];
        acc[r][0] = fmaf(w, x.x, acc[r][0]);
        acc[r][1] = fmaf(w, x.y, acc[r][1]);
        acc[r][2] = fmaf(w, x.z, acc[r][2]);
        acc[r][3] = fmaf(w, x.w, acc[r][3]);
      }
    }
    __syncwarp();  // scratch is rewritten at the top of the next chunk
    b_cur = b_next;
    b_next = b_after;
  }
  cp_async_wait<0>();
#pragma unroll
  for (int r = 0; r < CT_RPW; ++r) {
    const int row = row_base + r;
    if (row < m && col < k) {
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
