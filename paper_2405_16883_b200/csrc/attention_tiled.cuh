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

#include <type_traits>

#include "stc_common.cuh"

namespace stc {

constexpr int AT_B = 64;          // rows per block, columns per tile
constexpr int AT_D = 64;          // head dim of the tiled path
constexpr int AT_ABSENT = 0x7fc0ffee;  // score bits of an absent slot (a quiet NaN no FP op produces)

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
// attn_tile8_kernel<TXN> (8 * TXN threads; shipped with TXN = 16: 128 threads).
//
// Thread (ty, tx) = (tid / TXN, tid % TXN) owns rows {4ty..4ty+3, 32+4ty..32+4ty+3} and
// 64 / TXN columns / head dims (4tx..4tx+3, and 32+4tx.. when TXN = 8): per 4-wide slice
// of the reduction TXN = 16 issues 12 LDS.128 for 128 FMAs, TXN = 8 16 for 256 (a 4x4
// tiling of 256 threads: 8 for 64, SMEM-wavefront bound at 40 % FMA-pipe use — cfg4
// 0.85 ms; TXN = 8: 0.80 ms, 255 registers, 6 warps/SM; TXN = 16: 0.77 ms, 16 warps/SM). Q, K and V are staged by
// cp.async (K and V of tile t+1 once tile t is done; P^T reuses K's buffer so that
// four CTAs fit an SM and cover each other's copies). K rows are stored with
// their 16-byte chunks XOR-swizzled by (row / 4) % 8 and P^T with its row chunks
// swizzled the same way, so the 8 lanes of a quarter-warp hit 8 bank groups.
// Round 2: both products issue packed FMAs (FFMA2, stc_common.cuh). Q is staged
// transposed once per block (Qt[d][row]) so one LDS.128 yields four rows of a head
// dim: S accumulates as row pairs (S[i], S[i+1]) += (Qt[d][i], Qt[d][i+1]) * K[c][d],
// and O as head-dim pairs (O[e], O[e+1]) += P[i] * (V[c][e], V[c][e+1]) — 76 issue
// slots per 128 FMAs instead of 140, every sum in the same order as before.
// ---------------------------------------------------------------------------
constexpr size_t AT8_SMEM = 3ull * AT_B * AT_B * sizeof(float);  // Qt, Ks (aliased by Pt), Vs

// TXN threads share a row: TXN = 8 -> 8x8 register tiles (64 threads), TXN = 16 -> 8x4 (128 threads).
// Column / head-dim j of thread tx: (j / 4) * 4 * TXN + 4 * tx + j % 4.
template <int TXN>
STC_DEVICE int at8_col(int tx, int j) { return (j / 4) * 4 * TXN + 4 * tx + (j % 4); }
STC_DEVICE int at8_row(int ty, int i) { return i < 4 ? 4 * ty + i : 32 + 4 * ty + (i - 4); }

template <int TXN>
__global__ void __launch_bounds__(8 * TXN, 4) attn_tile8_kernel(TileArgs a) {
  constexpr int NT = 8 * TXN;   // threads
  constexpr int CW = 64 / TXN;  // columns (and head dims) per thread
  extern __shared__ __align__(16) float sm8[];
  float* Qt = sm8;                  // [d][row] (transposed once per block)
  float* Ks = Qt + AT_B * AT_B;     // [col][d], chunk-swizzled
  float* Vs = Ks + AT_B * AT_B;     // [col][d]
  float* Pt = Ks;                   // [col][row], row-chunk swizzled (K is dead once S is done)
  const int b = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x;
  const int tx = tid % TXN, ty = tid / TXN;
  const int row0 = b * AT_B;
  const float* Qh = a.Q + h * a.q_hs;
  const float* Kh = a.K + h * a.k_hs;
  const float* Vh = a.V + h * a.v_hs;
  const int* cols = a.tile_cols + (long long)b * a.dt_max;

  auto stage_rows = [&](float* dst, const float* src, long long rs, int r0, int limit, bool swz) {
    for (int idx = tid; idx < AT_B * 16; idx += NT) {
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
  for (int t = 0; t < n_t; ++t) STC_CHECK(cols[t] * AT_B < a.n, "dense tile outside the key range");
  if (n_t > 0) {
    stage_rows(Ks, Kh, a.k_rs, cols[0] * AT_B, a.n, true);
    stage_rows(Vs, Vh, a.v_rs, cols[0] * AT_B, a.n, false);
  }
  // Q^T: lane = row (conflict-free transposed stores), 16 bytes of a row per load
  for (int idx = tid; idx < AT_B * 16; idx += NT) {
    const int r = idx % AT_B, dq = idx / AT_B;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row0 + r < a.m) q = *reinterpret_cast<const float4*>(Qh + (long long)(row0 + r) * a.q_rs + dq * 4);
    Qt[(4 * dq + 0) * AT_B + r] = q.x;
    Qt[(4 * dq + 1) * AT_B + r] = q.y;
    Qt[(4 * dq + 2) * AT_B + r] = q.z;
    Qt[(4 * dq + 3) * AT_B + r] = q.w;
  }

  float o[8][CW], mrow[8], lrow[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mrow[i] = -INFINITY;
    lrow[i] = 0.f;
#pragma unroll
    for (int e = 0; e < CW; ++e) o[i][e] = 0.f;
  }

  for (int t = 0; t < n_t; ++t) {
    cp_async_wait<1>();  // K(t) landed; V(t) may still be in flight (Q^T: plain stores, same barrier)
    __syncthreads();
    float s[8][CW];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < CW; ++j) s[i][j] = 0.f;
#pragma unroll 1
    for (int dq = 0; dq < 16; ++dq) {
      float4 k4[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int c = at8_col<TXN>(tx, j);
        k4[j] = *reinterpret_cast<const float4*>(Ks + c * AT_D + ((dq ^ ((c >> 2) & 7)) * 4));
      }
#pragma unroll
      for (int dd = 0; dd < 4; ++dd) {  // head dim d = 4 dq + dd, ascending as before
        const float4 qa = *reinterpret_cast<const float4*>(Qt + (4 * dq + dd) * AT_B + 4 * ty);
        const float4 qb = *reinterpret_cast<const float4*>(Qt + (4 * dq + dd) * AT_B + 32 + 4 * ty);
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const float kd = dd == 0 ? k4[j].x : dd == 1 ? k4[j].y : dd == 2 ? k4[j].z : k4[j].w;
          fma2(s[0][j], s[1][j], kd, qa.x, qa.y);
          fma2(s[2][j], s[3][j], kd, qa.z, qa.w);
          fma2(s[4][j], s[5][j], kd, qb.x, qb.y);
          fma2(s[6][j], s[7][j], kd, qb.z, qb.w);
        }
      }
    }
    __syncthreads();  // every warp is done with Ks: P^T takes its place

    const float* mv_tile = a.tile_vals + ((long long)(b * a.dt_max + t) * AT_B) * AT_B;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = at8_row(ty, i);
      float mva[CW];
#pragma unroll
      for (int jq = 0; jq < CW / 4; ++jq) {
        const float4 m4 = ld_stream4(mv_tile + r * AT_B + at8_col<TXN>(tx, 4 * jq));
        mva[4 * jq] = m4.x; mva[4 * jq + 1] = m4.y; mva[4 * jq + 2] = m4.z; mva[4 * jq + 3] = m4.w;
      }
      float tmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        // absent slot -> a NaN with a private payload (fmaxf skips it; below it becomes
        // p = -0.0, "no entry"); a present entry's NaN score stays NaN, as in the reference
        s[i][j] = isnan(mva[j]) ? __int_as_float(AT_ABSENT) : s[i][j] * mva[j] * a.scale;
        tmax = fmaxf(tmax, s[i][j]);
      }
#pragma unroll
      for (int w = TXN / 2; w >= 1; w >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, w));
      const float mnew = fmaxf(mrow[i], tmax);
      const float corr = (mnew == -INFINITY) ? 1.f : expf(mrow[i] - mnew);
      float rsum = 0.f;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        s[i][j] = __float_as_int(s[i][j]) == AT_ABSENT ? -0.f : ((s[i][j] == -INFINITY) ? 0.f : expf(s[i][j] - mnew));
        rsum += s[i][j];
      }
#pragma unroll
      for (int w = TXN / 2; w >= 1; w >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, w);
      lrow[i] = lrow[i] * corr + rsum;
      mrow[i] = mnew;
#pragma unroll
      for (int e = 0; e < CW; ++e) o[i][e] *= corr;
    }
    // P^T: column c, row chunk rc (4 rows) stored at chunk rc ^ ((c >> 2) & 7)
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const int c = at8_col<TXN>(tx, j);
      const int sw = (c >> 2) & 7;
      *reinterpret_cast<float4*>(Pt + c * AT_B + 4 * (ty ^ sw)) = make_float4(s[0][j], s[1][j], s[2][j], s[3][j]);
      *reinterpret_cast<float4*>(Pt + c * AT_B + 4 * ((8 + ty) ^ sw)) =
          make_float4(s[4][j], s[5][j], s[6][j], s[7][j]);
    }
    cp_async_wait<0>();  // V(t) landed
    // Absent slots carry p = -0.0: with finite V rows their products add nothing, but 0 * Inf
    // would be NaN where the reference multiplies only stored entries. Each thread checks the
    // V chunks it staged; if any row of the tile is not finite, the PV loop skips absent slots.
    bool vfin = true;
    for (int idx = tid; idx < AT_B * 16; idx += NT) {
      const float4 v4 = *reinterpret_cast<const float4*>(Vs + (idx / 16) * AT_D + (idx % 16) * 4);
      vfin &= isfinite(v4.x) && isfinite(v4.y) && isfinite(v4.z) && isfinite(v4.w);
    }
    const bool v_finite = __syncthreads_and(vfin);
    auto pv = [&](auto masked) {
#pragma unroll 2
      for (int c = 0; c < AT_B; ++c) {
        const int sw = (c >> 2) & 7;
        const float4 pa = *reinterpret_cast<const float4*>(Pt + c * AT_B + 4 * (ty ^ sw));
        const float4 pb = *reinterpret_cast<const float4*>(Pt + c * AT_B + 4 * ((8 + ty) ^ sw));
        const float p8[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
        float v8[CW];
#pragma unroll
        for (int eq = 0; eq < CW / 4; ++eq) {
          const float4 v4 = *reinterpret_cast<const float4*>(Vs + c * AT_D + at8_col<TXN>(tx, 4 * eq));
          v8[4 * eq] = v4.x; v8[4 * eq + 1] = v4.y; v8[4 * eq + 2] = v4.z; v8[4 * eq + 3] = v4.w;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if constexpr (decltype(masked)::value) {
            if (signbit(p8[i])) continue;
          }
#pragma unroll
          for (int e = 0; e < CW; e += 2) fma2(o[i][e], o[i][e + 1], p8[i], v8[e], v8[e + 1]);
        }
      }
    };
    if (v_finite)
      pv(std::false_type{});
    else
      pv(std::true_type{});
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
#pragma unroll
    for (int eq = 0; eq < CW / 4; ++eq)
      *reinterpret_cast<float4*>(dst + at8_col<TXN>(tx, 4 * eq)) =
          make_float4(o[i][4 * eq], o[i][4 * eq + 1], o[i][4 * eq + 2], o[i][4 * eq + 3]);
    if (tx == 0) a.ml[(long long)h * a.m + row] = make_float2(mrow[i], lrow[i]);
  }
}

}  // namespace stc
