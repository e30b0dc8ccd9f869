// K7b: block-tiled fused sparse attention for masks with dense bands (sm_100a).
//
// A plan splits the mask into 64x64 (row-block, column-tile) tiles. Tiles that
// hold at least an eighth of their 4096 slots (e.g. the causal local window)
// are "dense tiles": their mask values are stored as a 64x64 float tile
// (NaN = absent). Everything else stays a CSR "remainder".
//
// attn_tile8_kernel: one CTA per (row block, head). Q of the block is staged in
// SMEM once; for every dense tile, K and V of its 64 columns are staged and
//   S = scale * M .* (Q K^T)   (8x8 register tile per thread, LDS.128 operands)
//   online softmax per row    (row max / sum over the 8 threads of a row)
//   O += P V                  (8x8 register tile per thread)
// run on CUDA cores: each staged K/V row is reused by all 64 rows of the block
// instead of being gathered once per stored entry. The unnormalised (O, max,
// sum) of each row is written out; the per-row kernel then folds in the
// remainder entries with the same online softmax and normalises.
#pragma once

#include "stc_common.cuh"

namespace stc {

constexpr int AT_B = 64;          // rows per block, columns per tile
constexpr int AT_D = 64;          // head dim of the tiled path

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

// ---------------------------------------------------------------------------
// attn_tile8_kernel (64 threads).
//
// Thread (ty, tx) = (tid / 8, tid % 8) owns rows {4ty..4ty+3, 32+4ty..32+4ty+3} and
// columns / head dims {4tx..4tx+3, 32+4tx..32+4tx+3}: per 4-wide slice of the
// reduction it issues 16 LDS.128 for 256 FMAs (a 4x4 tiling of 256 threads: 8 for
// 64, and SMEM-wavefront bound at 40 % FMA-pipe use — measured, cfg4 0.85 ms). Q, K and V are staged by
// cp.async (K and V of tile t+1 once tile t is done; P^T reuses K's buffer so that
// four CTAs fit an SM and cover each other's copies). K rows are stored with
// their 16-byte chunks XOR-swizzled by (row / 4) % 8 and P^T with its row chunks
// swizzled the same way, so the 8 lanes of a quarter-warp hit 8 bank groups.
// ---------------------------------------------------------------------------
constexpr int AT8_THREADS = 64;
constexpr size_t AT8_SMEM = 3ull * AT_B * AT_B * sizeof(float);  // Qs, Ks (aliased by Pt), Vs

STC_DEVICE int at8_row(int ty, int i) { return i < 4 ? 4 * ty + i : 32 + 4 * ty + (i - 4); }

__global__ void __launch_bounds__(AT8_THREADS, 4) attn_tile8_kernel(TileArgs a) {
  extern __shared__ __align__(16) float sm8[];
  float* Qs = sm8;                  // [row][d]
  float* Ks = Qs + AT_B * AT_B;     // [col][d], chunk-swizzled
  float* Vs = Ks + AT_B * AT_B;     // [col][d]
  float* Pt = Ks;                   // [col][row], row-chunk swizzled (K is dead once S is done)
  const int b = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x;
  const int tx = tid % 8, ty = tid / 8;
  const int row0 = b * AT_B;
  const float* Qh = a.Q + h * a.q_hs;
  const float* Kh = a.K + h * a.k_hs;
  const float* Vh = a.V + h * a.v_hs;
  const int* cols = a.tile_cols + (long long)b * a.dt_max;

  auto stage_rows = [&](float* dst, const float* src, long long rs, int r0, int limit, bool swz) {
    for (int idx = tid; idx < AT_B * 16; idx += AT8_THREADS) {
      const int r = idx / 16, dq = idx % 16;
      const bool ok = r0 + r < limit;
      const int slot = swz ? (dq ^ ((r >> 2) & 7)) : dq;
      cp_async16(dst + r * AT_D + slot * 4, ok ? (const void*)(src + (long long)(r0 + r) * rs + dq * 4) : (const void*)src,
                 ok);
    }
    cp_async_commit();
  };
  int n_t = 0;
  while (n_t < a.dt_max && cols[n_t] >= 0) ++n_t;
  stage_rows(Qs, Qh, a.q_rs, row0, a.m, false);
  if (n_t > 0) {
    stage_rows(Ks, Kh, a.k_rs, cols[0] * AT_B, a.n, true);
    stage_rows(Vs, Vh, a.v_rs, cols[0] * AT_B, a.n, false);
  }

  float o[8][8], mrow[8], lrow[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mrow[i] = -INFINITY;
    lrow[i] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) o[i][e] = 0.f;
  }

  for (int t = 0; t < n_t; ++t) {
    cp_async_wait<1>();  // Q and K(t) landed; V(t) may still be in flight
    __syncthreads();
    float s[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) s[i][j] = 0.f;
#pragma unroll 1
    for (int dq = 0; dq < 16; ++dq) {
      float4 q4[8], k4[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) q4[i] = *reinterpret_cast<const float4*>(Qs + at8_row(ty, i) * AT_D + dq * 4);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = at8_row(tx, j);
        k4[j] = *reinterpret_cast<const float4*>(Ks + c * AT_D + ((dq ^ ((c >> 2) & 7)) * 4));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[i][j] = fmaf(q4[i].x, k4[j].x, s[i][j]);
          s[i][j] = fmaf(q4[i].y, k4[j].y, s[i][j]);
          s[i][j] = fmaf(q4[i].z, k4[j].z, s[i][j]);
          s[i][j] = fmaf(q4[i].w, k4[j].w, s[i][j]);
        }
    }
    __syncthreads();  // every warp is done with Ks: P^T takes its place

    const float* mv_tile = a.tile_vals + ((long long)(b * a.dt_max + t) * AT_B) * AT_B;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = at8_row(ty, i);
      const float4 m0 = ld_stream4(mv_tile + r * AT_B + 4 * tx);
      const float4 m1 = ld_stream4(mv_tile + r * AT_B + 32 + 4 * tx);
      const float mva[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
      float tmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s[i][j] = isnan(mva[j]) ? -INFINITY : s[i][j] * mva[j] * a.scale;
        tmax = fmaxf(tmax, s[i][j]);
      }
#pragma unroll
      for (int w = 4; w >= 1; w >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, w));
      const float mnew = fmaxf(mrow[i], tmax);
      const float corr = (mnew == -INFINITY) ? 1.f : expf(mrow[i] - mnew);
      float rsum = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s[i][j] = (s[i][j] == -INFINITY) ? 0.f : expf(s[i][j] - mnew);
        rsum += s[i][j];
      }
#pragma unroll
      for (int w = 4; w >= 1; w >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, w);
      lrow[i] = lrow[i] * corr + rsum;
      mrow[i] = mnew;
#pragma unroll
      for (int e = 0; e < 8; ++e) o[i][e] *= corr;
    }
    // P^T: column c, row chunk rc (4 rows) stored at chunk rc ^ ((c >> 2) & 7)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = at8_row(tx, j);
      const int sw = (c >> 2) & 7;
      *reinterpret_cast<float4*>(Pt + c * AT_B + 4 * (ty ^ sw)) = make_float4(s[0][j], s[1][j], s[2][j], s[3][j]);
      *reinterpret_cast<float4*>(Pt + c * AT_B + 4 * ((8 + ty) ^ sw)) =
          make_float4(s[4][j], s[5][j], s[6][j], s[7][j]);
    }
    cp_async_wait<0>();  // V(t) landed
    __syncthreads();
#pragma unroll 2
    for (int c = 0; c < AT_B; ++c) {
      const int sw = (c >> 2) & 7;
      const float4 pa = *reinterpret_cast<const float4*>(Pt + c * AT_B + 4 * (ty ^ sw));
      const float4 pb = *reinterpret_cast<const float4*>(Pt + c * AT_B + 4 * ((8 + ty) ^ sw));
      const float4 va = *reinterpret_cast<const float4*>(Vs + c * AT_D + 4 * tx);
      const float4 vb = *reinterpret_cast<const float4*>(Vs + c * AT_D + 32 + 4 * tx);
      const float p8[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
      const float v8[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) o[i][e] = fmaf(p8[i], v8[e], o[i][e]);
    }
    __syncthreads();  // done with Vs and Pt: stream in the next tile's K and V
    if (t + 1 < n_t) {
      stage_rows(Ks, Kh, a.k_rs, cols[t + 1] * AT_B, a.n, true);
      stage_rows(Vs, Vh, a.v_rs, cols[t + 1] * AT_B, a.n, false);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + at8_row(ty, i);
    if (row >= a.m) continue;
    float* dst = a.Opart + ((long long)h * a.m + row) * AT_D;
    *reinterpret_cast<float4*>(dst + 4 * tx) = make_float4(o[i][0], o[i][1], o[i][2], o[i][3]);
    *reinterpret_cast<float4*>(dst + 32 + 4 * tx) = make_float4(o[i][4], o[i][5], o[i][6], o[i][7]);
    if (tx == 0) a.ml[(long long)h * a.m + row] = make_float2(mrow[i], lrow[i]);
  }
}

}  // namespace stc
