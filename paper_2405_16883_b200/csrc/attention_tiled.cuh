// K7b: block-tiled fused sparse attention for masks with dense bands (sm_100a).
//
// A plan splits the mask into 64x64 (row-block, column-tile) tiles. Tiles that
// hold at least an eighth of their 4096 slots (e.g. the causal local window)
// are "dense tiles": their mask values are stored as a 64x64 float tile
// (NaN = absent). Everything else stays a CSR "remainder".
//
// attn_tile_kernel: one CTA per (row block, head). Q of the block is staged in
// SMEM once; for every dense tile, K and V of its 64 columns are staged and
//   S = scale * M .* (Q K^T)   (4x4 register tile per thread, LDS.128 operands)
//   online softmax per row    (row max / sum over the 16 threads of a row)
//   O += P V                  (4x4 register tile per thread)
// run on CUDA cores: each staged K/V row is reused by all 64 rows of the block
// instead of being gathered once per stored entry. The unnormalised (O, max,
// sum) of each row is written out; the per-row kernel then folds in the
// remainder entries with the same online softmax and normalises.
#pragma once

#include "stc_common.cuh"

namespace stc {

constexpr int AT_B = 64;          // rows per block, columns per tile
constexpr int AT_D = 64;          // head dim of the tiled path
constexpr int AT_THREADS = 256;
constexpr size_t AT_SMEM = 4ull * AT_B * AT_B * sizeof(float);  // Qt, Kt, V, Pt

struct TileArgs {
  int m, n, heads, n_blocks, dt_max;
  const int* tile_cols;     // [n_blocks][dt_max] column-tile index or -1
  const float* tile_vals;   // [n_blocks][dt_max][64][64] mask value, NaN = absent
  const float* Q;
  long long q_hs, q_rs;
  const float* K;
  long long k_hs, k_rs;
  const float* V;
  long long v_hs, v_rs;
  float scale;
  float* Opart;             // [H][M][64] unnormalised
  float2* ml;               // [H][M] (running max, running sum)
};

__global__ void __launch_bounds__(AT_THREADS, 3) attn_tile_kernel(TileArgs a) {
  extern __shared__ __align__(16) float sm[];
  float* Qt = sm;                    // [d][row]
  float* Kt = Qt + AT_B * AT_B;      // [d][col]
  float* Vs = Kt + AT_B * AT_B;      // [col][d]
  float* Pt = Vs + AT_B * AT_B;      // [col][row]
  const int b = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // rows 4ty..4ty+3, cols / d 4tx..4tx+3
  const int row0 = b * AT_B;
  const float* Qh = a.Q + h * a.q_hs;
  const float* Kh = a.K + h * a.k_hs;
  const float* Vh = a.V + h * a.v_hs;

  // lanes walk rows (consecutive r) for a fixed d-quad, so the transposed
  // scalar stores hit 32 distinct banks
  for (int idx = tid; idx < AT_B * (AT_D / 4); idx += AT_THREADS) {
    const int r = idx % AT_B, dq = (idx / AT_B) * 4;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row0 + r < a.m) q = *reinterpret_cast<const float4*>(Qh + (long long)(row0 + r) * a.q_rs + dq);
    Qt[(dq + 0) * AT_B + r] = q.x;
    Qt[(dq + 1) * AT_B + r] = q.y;
    Qt[(dq + 2) * AT_B + r] = q.z;
    Qt[(dq + 3) * AT_B + r] = q.w;
  }

  float o[4][4], mrow[4], lrow[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mrow[i] = -INFINITY;
    lrow[i] = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) o[i][e] = 0.f;
  }
  const unsigned hmask = 0xffffffffu;  // all lanes shuffle; width 16 keeps each row group apart

  for (int t = 0; t < a.dt_max; ++t) {
    const int tc = a.tile_cols[b * a.dt_max + t];
    if (tc < 0) break;
    __syncthreads();  // previous tile's operands fully consumed
    const int c0 = tc * AT_B;
    for (int idx = tid; idx < AT_B * (AT_D / 4); idx += AT_THREADS) {
      const int c = idx % AT_B, dq = (idx / AT_B) * 4;
      float4 kv = make_float4(0.f, 0.f, 0.f, 0.f), vv = kv;
      if (c0 + c < a.n) {
        kv = ld_gather4(Kh + (long long)(c0 + c) * a.k_rs + dq);
        vv = ld_gather4(Vh + (long long)(c0 + c) * a.v_rs + dq);
      }
      Kt[(dq + 0) * AT_B + c] = kv.x;
      Kt[(dq + 1) * AT_B + c] = kv.y;
      Kt[(dq + 2) * AT_B + c] = kv.z;
      Kt[(dq + 3) * AT_B + c] = kv.w;
      *reinterpret_cast<float4*>(Vs + c * AT_D + dq) = vv;
    }
    __syncthreads();

    float s[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 8
    for (int d = 0; d < AT_D; ++d) {
      const float4 q4 = *reinterpret_cast<const float4*>(Qt + d * AT_B + 4 * ty);
      const float4 k4 = *reinterpret_cast<const float4*>(Kt + d * AT_B + 4 * tx);
      const float qa[4] = {q4.x, q4.y, q4.z, q4.w};
      const float ka[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = fmaf(qa[i], ka[j], s[i][j]);
    }

    const float* mv_tile = a.tile_vals + ((long long)(b * a.dt_max + t) * AT_B) * AT_B;
    float p[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 mv4 = ld_stream4(mv_tile + (4 * ty + i) * AT_B + 4 * tx);
      const float mva[4] = {mv4.x, mv4.y, mv4.z, mv4.w};
      float tmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s[i][j] = isnan(mva[j]) ? -INFINITY : s[i][j] * mva[j] * a.scale;
        tmax = fmaxf(tmax, s[i][j]);
      }
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(hmask, tmax, w, 16));
      const float mnew = fmaxf(mrow[i], tmax);
      const float corr = (mnew == -INFINITY) ? 1.f : expf(mrow[i] - mnew);
      float rsum = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        p[i][j] = (s[i][j] == -INFINITY) ? 0.f : expf(s[i][j] - mnew);
        rsum += p[i][j];
      }
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1) rsum += __shfl_xor_sync(hmask, rsum, w, 16);
      lrow[i] = lrow[i] * corr + rsum;
      mrow[i] = mnew;
#pragma unroll
      for (int e = 0; e < 4; ++e) o[i][e] *= corr;
    }
    // P^T in SMEM, float4 slot of rows 4ty.. in column c swizzled to ty ^ ((c >> 2) & 7):
    // conflict-free stores here and broadcast loads in the PV loop
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 4 * tx + j;
      *reinterpret_cast<float4*>(Pt + c * AT_B + 4 * (ty ^ ((c >> 2) & 7))) =
          make_float4(p[0][j], p[1][j], p[2][j], p[3][j]);
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < AT_B; ++c) {
      const float4 p4 = *reinterpret_cast<const float4*>(Pt + c * AT_B + 4 * (ty ^ ((c >> 2) & 7)));
      const float4 v4 = *reinterpret_cast<const float4*>(Vs + c * AT_D + 4 * tx);
      const float pa[4] = {p4.x, p4.y, p4.z, p4.w};
      const float va[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[i][e] = fmaf(pa[i], va[e], o[i][e]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = row0 + 4 * ty + i;
    if (row >= a.m) continue;
    *reinterpret_cast<float4*>(a.Opart + ((long long)h * a.m + row) * AT_D + 4 * tx) =
        make_float4(o[i][0], o[i][1], o[i][2], o[i][3]);
    if (tx == 0) a.ml[(long long)h * a.m + row] = make_float2(mrow[i], lrow[i]);
  }
}

}  // namespace stc
