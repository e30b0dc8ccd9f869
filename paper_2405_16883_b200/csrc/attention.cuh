// K5 SDDMM, K6 row-segmented softmax and K7 fused sparse attention (sm_100a).
//
// Layout: one shared CSR mask (rowptr/colidx[/maskvals]) for all heads;
// Q [H][M][d], K/V [H][N][d] row-major (head strides given), scores/probs as
// [H][nnz] value arrays in the mask's order, O [H][M][d].
//
// A group of G = d/4 lanes owns one (head, row); each lane holds a float4 slice
// of q. For a batch of G stored entries every lane forms G partial dot
// products from G independent K-row gathers (G LDG.128 in flight per lane),
// then a transposed butterfly (G-1 shuffles) leaves the full dot product of
// entry l in lane l. The fused kernel keeps an online (running max / running
// sum) softmax and accumulates p * V_j without materialising S or P.
#pragma once

#include "stc_common.cuh"

namespace stc {

struct AttnArgs {
  int m, n, d, heads;
  const int* rowptr;
  const int* colidx;
  const float* maskv;      // nullable: implicit 1.0
  const float* Q;
  long long q_hs, q_rs;    // head / row strides (elements)
  const float* K;
  long long k_hs, k_rs;
  const float* V;
  long long v_hs, v_rs;
  float scale;
  long long nnz;
  float* S;                // [H][nnz] nullable (fused: written only if non-null)
  float* P;                // [H][nnz] nullable
  float* O;                // [H][M][d]
  long long o_hs, o_rs;
  const float* Opart;      // optional [H][M][d] unnormalised partial (dense tiles), d == 64
  const float2* ml;        // optional [H][M] running (max, sum) of the partial
};

// v[i] over lanes -> lane l holds sum over the group of the partials for entry l.
template <int G>
STC_DEVICE float transpose_reduce(float (&v)[G], int lane, unsigned mask) {
#pragma unroll
  for (int h = G / 2; h >= 1; h >>= 1) {
    const bool upper = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = upper ? v[i] : v[i + h];
      const float keep = upper ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(mask, send, h, G);
    }
  }
  return v[0];
}

// B partial sums over G lanes (B <= G, powers of two): lane l ends with the full
// sum of entry l % B (transposed stages inside aligned groups of B lanes, then a
// plain butterfly across the G / B groups).
template <int B, int G>
STC_DEVICE float transpose_reduce_b(float (&v)[B], int lane, unsigned mask) {
#pragma unroll
  for (int h = B / 2; h >= 1; h >>= 1) {
    const bool upper = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = upper ? v[i] : v[i + h];
      const float keep = upper ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(mask, send, h, G);
    }
  }
  float x = v[0];
#pragma unroll
  for (int h = B; h < G; h <<= 1) x += __shfl_xor_sync(mask, x, h, G);
  return x;
}

template <int G>
STC_DEVICE float group_max(float x, unsigned mask) {
#pragma unroll
  for (int h = G / 2; h >= 1; h >>= 1) x = fmaxf(x, __shfl_xor_sync(mask, x, h, G));
  return x;
}
template <int G>
STC_DEVICE float group_sum(float x, unsigned mask) {
#pragma unroll
  for (int h = G / 2; h >= 1; h >>= 1) x += __shfl_xor_sync(mask, x, h, G);
  return x;
}

// SDDMM: S[h, p] = scale * mask[p] * dot(Q[h,i,:], K[h,col[p],:])
template <int G, bool NARROW>
__global__ void __launch_bounds__(256) sddmm_kernel(AttnArgs a) {
  const int lane = threadIdx.x % G;
  const unsigned mask = subwarp_mask<G>();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int h = blockIdx.y;
  if (row >= a.m) return;
  const float4 q = *reinterpret_cast<const float4*>(a.Q + h * a.q_hs + (long long)row * a.q_rs + lane * 4);
  const float* Kh = a.K + h * a.k_hs + lane * 4;
  const unsigned krs = (unsigned)a.k_rs;
  if constexpr (NARROW) asm volatile("" : "+l"(Kh));  // see attention_body
  float* out = a.S + h * a.nnz;
  const int start = a.rowptr[row], end = a.rowptr[row + 1];
  for (int base = start; base < end; base += G) {
    const int n = min(G, end - base);
    const int my_col = (lane < n) ? ld_stream(a.colidx + base + lane) : 0;
    float part[G];
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int c = __shfl_sync(mask, my_col, t, G);
      float4 kv = make_float4(0.f, 0.f, 0.f, 0.f);
      STC_CHECK(t >= n || (c >= 0 && c < a.n), "SDDMM column outside K");
      if (t < n) kv = ld_gather4(NARROW ? Kh + (unsigned)c * krs : Kh + (long long)c * a.k_rs);
      part[t] = fmaf(q.x, kv.x, fmaf(q.y, kv.y, fmaf(q.z, kv.z, q.w * kv.w)));
    }
    const float s = transpose_reduce<G>(part, lane, mask);
    if (lane < n) {
      const float mv = a.maskv ? ld_stream(a.maskv + base + lane) : 1.f;
      st_stream1(out + base + lane, s * mv * a.scale);
    }
  }
}

// Row-segmented softmax over each row's stored entries, in place, all heads.
__global__ void __launch_bounds__(256) segsoftmax_kernel(int m, long long nnz, const int* __restrict__ rowptr,
                                                         float* __restrict__ vals) {
  const int lane = threadIdx.x % 32;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int h = blockIdx.y;
  if (row >= m) return;
  float* v = vals + h * nnz;
  const int start = rowptr[row], end = rowptr[row + 1];
  float mx = -INFINITY;
  for (int p = start + lane; p < end; p += 32) mx = fmaxf(mx, v[p]);
  mx = group_max<32>(mx, 0xffffffffu);
  float sum = 0.f;
  for (int p = start + lane; p < end; p += 32) sum += expf(v[p] - mx);
  sum = group_sum<32>(sum, 0xffffffffu);
  const float inv = 1.f / sum;
  for (int p = start + lane; p < end; p += 32) v[p] = expf(v[p] - mx) * inv;
}

// Fused: O[h,i,:] = sum_j softmax_j(scale * m_ij * q_i.k_j) * v_j with an online softmax.
// Entries are consumed in batches of B <= G (B = G/2 for wide heads keeps the
// V-row registers small enough for two CTAs' worth of extra warps per SM).
// VSMEM (the tiled path's remainder pass): the V rows of a batch do not wait in registers
// while the scores are reduced — each lane copies its 16-byte slice of every row into its own
// shared-memory slot with cp.async (no register, no cross-lane traffic: the lane reads back
// what it copied) and loads it when the probabilities are known. 32 registers fewer per
// thread: MINB CTAs per SM instead of 3, i.e. more batches of gathers in flight per SM.
#ifndef STC_ATTN_VSMEM_MINB
#define STC_ATTN_VSMEM_MINB 4
#endif
// NARROW: n * row stride of K and V below 2^31 elements (checked by the launcher), so a gathered row's
// offset is one 32-bit multiply instead of a 64 x 64-bit product per gather -- integer address
// arithmetic was 45 % of the remainder pass's instructions (IMAD 24 %, LEA 8 %, MOV 8 %, LDC 4 %).
template <int G, bool WRITE_S, bool VSMEM, bool NARROW = false>
STC_DEVICE void attention_body(const AttnArgs& a) {
  constexpr int B = G >= 16 ? G / 2 : G;
  extern __shared__ __align__(16) float4 vstage[];  // VSMEM: [B][256] float4, slot [t][thread]
  const int lane = threadIdx.x % G;
  const unsigned mask = subwarp_mask<G>();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int h = blockIdx.y;
  if (row >= a.m) return;
  const float4 q = *reinterpret_cast<const float4*>(a.Q + h * a.q_hs + (long long)row * a.q_rs + lane * 4);
  const float* Kh = a.K + h * a.k_hs + lane * 4;
  const float* Vh = a.V + h * a.v_hs + lane * 4;
  const unsigned krs = (unsigned)a.k_rs, vrs = (unsigned)a.v_rs;
  if constexpr (NARROW) {
    // keep the two row bases as opaque 64-bit registers: otherwise they are re-derived from the
    // kernel parameters for every gather (LDC + 64-bit add chain, 5-6 instructions per address)
    asm volatile("" : "+l"(Kh));
    asm volatile("" : "+l"(Vh));
  }
  auto krow = [&](int c) { return NARROW ? Kh + (unsigned)c * krs : Kh + (long long)c * a.k_rs; };
  auto vrow = [&](int c) { return NARROW ? Vh + (unsigned)c * vrs : Vh + (long long)c * a.v_rs; };
  const int start = a.rowptr[row], end = a.rowptr[row + 1];
  float run_max = -INFINITY, run_sum = 0.f;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  if (a.Opart) {  // continue the online softmax of the dense-tile pass
    const float2 mlv = a.ml[(long long)h * a.m + row];
    run_max = mlv.x;
    run_sum = mlv.y;
    o = *reinterpret_cast<const float4*>(a.Opart + ((long long)h * a.m + row) * 64 + lane * 4);
  }
  int next_col = (start + lane < end && lane < B) ? ld_stream(a.colidx + start + lane) : 0;
  for (int base = start; base < end; base += B) {
    const int n = min(B, end - base);
    const int my_col = next_col;
    float part[B];
    float4 vv[VSMEM ? 1 : B];
#pragma unroll
    for (int t = 0; t < B; ++t) {
      const int c = __shfl_sync(mask, my_col, t, G);
      float4 kv = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (!VSMEM) vv[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      STC_CHECK(t >= n || (c >= 0 && c < a.n), "attention column outside K/V");
      if constexpr (VSMEM)  // zero-filled past the row's end
        cp_async16(&vstage[t * 256 + threadIdx.x], vrow(t < n ? c : 0), t < n);
      if (t < n) {
        kv = ld_gather4(krow(c));
        if constexpr (!VSMEM) vv[t] = ld_gather4(vrow(c));
      }
      part[t] = fmaf(q.x, kv.x, fmaf(q.y, kv.y, fmaf(q.z, kv.z, q.w * kv.w)));
    }
    if constexpr (VSMEM) cp_async_commit();
    // indices of the next batch stream in while this one is reduced
    next_col = (base + B + lane < end && lane < B) ? ld_stream(a.colidx + base + B + lane) : 0;
    float s = transpose_reduce_b<B, G>(part, lane, mask);
    const bool mine = (lane % B) < n;  // lane l carries entry l % B
    const float mv = (mine && a.maskv) ? ld_stream(a.maskv + base + lane % B) : 1.f;
    s = mine ? s * mv * a.scale : -INFINITY;
    if constexpr (WRITE_S) {
      if (lane < n) a.S[h * a.nnz + base + lane] = s;
    }
    const float bmax = group_max<G>(s, mask);
    const float new_max = fmaxf(run_max, bmax);
    const float p = (mine && s != -INFINITY) ? expf(s - new_max) : 0.f;
    const float corr = (new_max == -INFINITY) ? 1.f : expf(run_max - new_max);
    // each entry appears in G / B lanes: count it once in the sum
    run_sum = run_sum * corr + group_sum<G>(lane < B ? p : 0.f, mask);
    o.x *= corr; o.y *= corr; o.z *= corr; o.w *= corr;
    if constexpr (VSMEM) cp_async_wait<0>();  // this thread's own copies: no barrier needed
#pragma unroll
    for (int t = 0; t < B; ++t) {
      const float pt = __shfl_sync(mask, p, t, G);
      const float4 v = VSMEM ? vstage[t * 256 + threadIdx.x] : vv[t];
      fma2(o.x, o.y, pt, v.x, v.y);  // packed FMAs (FFMA2), same roundings
      fma2(o.z, o.w, pt, v.z, v.w);
    }
    run_max = new_max;
  }
  const float inv = run_sum > 0.f ? 1.f / run_sum : 0.f;
  o.x *= inv; o.y *= inv; o.z *= inv; o.w *= inv;
  st_stream4(a.O + h * a.o_hs + (long long)row * a.o_rs + lane * 4, o);
  if constexpr (WRITE_S) {
    // P = exp(S - max) / sum, from the scores this group just wrote (parity mode)
    if (a.P) {
      __syncwarp(mask);
      for (int pp = start + lane; pp < end; pp += G)
        a.P[h * a.nnz + pp] = expf(a.S[h * a.nnz + pp] - run_max) * inv;
    }
  }
}

template <int G, bool WRITE_S, bool NARROW>
__global__ void __launch_bounds__(256) attention_kernel(AttnArgs a) {
  attention_body<G, WRITE_S, false, NARROW>(a);
}
template <int G, bool NARROW>
__global__ void __launch_bounds__(256, STC_ATTN_VSMEM_MINB) attention_vsmem_kernel(AttnArgs a) {
  attention_body<G, false, true, NARROW>(a);
}

}  // namespace stc
