// C-ABI entry points for SDDMM, segmented softmax and fused sparse attention.
#include "abi_util.cuh"
#include "attention.cuh"
#include "attention_tiled.cuh"

using namespace stc;

namespace {

constexpr int kThreads = 256;

int check_common(int m, int n, int d, int heads, const int* rowptr, long long nnz) {
  if (m < 0 || n < 0 || d < 0 || heads < 1 || nnz < 0) return fail(STC_EINVAL, "negative extent");
  if (nnz > INT32_MAX) return fail(STC_EUNSUPPORTED, "nnz exceeds int32 index range");
  if (heads > 65535) return fail(STC_EUNSUPPORTED, "more than 65535 heads");
  if (m && !rowptr) return fail(STC_EINVAL, "null rowptr");
  return STC_OK;
}

// every gathered row of K (and V) starts below 2^31 elements: the kernels take 32-bit row offsets
bool narrow_rows(const AttnArgs& a, bool with_v) {
  return (long long)a.n * a.k_rs < (1LL << 31) && (!with_v || (long long)a.n * a.v_rs < (1LL << 31));
}

bool dim_ok(int d) { return d == 4 || d == 8 || d == 16 || d == 32 || d == 64 || d == 128; }

template <int G>
int launch_sddmm(const AttnArgs& a, cudaStream_t st) {
  const dim3 grid((unsigned)ceil_div((long long)a.m * G, kThreads), a.heads);
  if (narrow_rows(a, false))
    sddmm_kernel<G, true><<<grid, kThreads, 0, st>>>(a);
  else
    sddmm_kernel<G, false><<<grid, kThreads, 0, st>>>(a);
  return check_launch("sddmm_kernel");
}

template <int G, bool WS>
int launch_attn(const AttnArgs& a, cudaStream_t st) {
  const dim3 grid((unsigned)ceil_div((long long)a.m * G, kThreads), a.heads);
  if (narrow_rows(a, true))
    attention_kernel<G, WS, true><<<grid, kThreads, 0, st>>>(a);
  else
    attention_kernel<G, WS, false><<<grid, kThreads, 0, st>>>(a);
  return check_launch("attention_kernel");
}

// the tiled path's remainder pass (d = 64): V rows staged through shared memory by cp.async
int launch_attn_vsmem(const AttnArgs& a, cudaStream_t st) {
  constexpr int G = 16;
  constexpr size_t smem = (size_t)(G / 2) * kThreads * sizeof(float4);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attention_vsmem_kernel<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(attention_vsmem_kernel<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  const dim3 grid((unsigned)ceil_div((long long)a.m * G, kThreads), a.heads);
  // 32-bit row offsets when every gathered row of K and V starts below 2^31 elements
  if (narrow_rows(a, true))
    attention_vsmem_kernel<G, true><<<grid, kThreads, smem, st>>>(a);
  else
    attention_vsmem_kernel<G, false><<<grid, kThreads, smem, st>>>(a);
  return check_launch("attention_vsmem_kernel");
}

template <bool WS>
int attn_by_d(const AttnArgs& a, cudaStream_t st) {
  switch (a.d / 4) {
    case 1: return launch_attn<1, WS>(a, st);
    case 2: return launch_attn<2, WS>(a, st);
    case 4: return launch_attn<4, WS>(a, st);
    case 8: return launch_attn<8, WS>(a, st);
    case 16: return launch_attn<16, WS>(a, st);
    default: return launch_attn<32, WS>(a, st);
  }
}

}  // namespace

extern "C" int stc_sddmm_csr_f32(int m, int n, int d, int heads, const int* rowptr, const int* colidx,
                                 const float* maskvals, long long nnz, const float* Q, long long q_hs,
                                 long long q_rs, const float* K, long long k_hs, long long k_rs, float scale,
                                 float* out_vals, void* stream) {
  STC_NVTX("stc_sddmm_csr_f32");
  int rc = check_common(m, n, d, heads, rowptr, nnz);
  if (rc) return rc;
  if (m == 0 || nnz == 0) return STC_OK;
  if (!dim_ok(d)) return fail(STC_EUNSUPPORTED, "head dim %d not in {4,8,16,32,64,128}", d);
  if (!colidx || !Q || !K || !out_vals) return fail(STC_EINVAL, "null pointer");
  if (!aligned16(Q) || !aligned16(K) || q_rs % 4 || k_rs % 4 || q_hs % 4 || k_hs % 4 || q_rs < d || k_rs < d)
    return fail(STC_EINVAL, "Q/K must be 16-byte aligned with strides that are multiples of 4 and >= d");
  AttnArgs a{};
  a.m = m; a.n = n; a.d = d; a.heads = heads;
  a.rowptr = rowptr; a.colidx = colidx; a.maskv = maskvals;
  a.Q = Q; a.q_hs = q_hs; a.q_rs = q_rs;
  a.K = K; a.k_hs = k_hs; a.k_rs = k_rs;
  a.scale = scale; a.nnz = nnz; a.S = out_vals;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (d / 4) {
    case 1: return launch_sddmm<1>(a, st);
    case 2: return launch_sddmm<2>(a, st);
    case 4: return launch_sddmm<4>(a, st);
    case 8: return launch_sddmm<8>(a, st);
    case 16: return launch_sddmm<16>(a, st);
    default: return launch_sddmm<32>(a, st);
  }
}

extern "C" int stc_segsoftmax_csr_f32(int m, int heads, const int* rowptr, long long nnz, float* vals,
                                      void* stream) {
  STC_NVTX("stc_segsoftmax_csr_f32");
  int rc = check_common(m, 0, 0, heads, rowptr, nnz);
  if (rc) return rc;
  if (m == 0 || nnz == 0) return STC_OK;
  if (!vals) return fail(STC_EINVAL, "null pointer");
  const dim3 grid((unsigned)ceil_div((long long)m * 32, kThreads), heads);
  segsoftmax_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(m, nnz, rowptr, vals);
  return check_launch("segsoftmax_kernel");
}

extern "C" int stc_sparse_attention_f32(int m, int n, int d, int heads, const int* rowptr, const int* colidx,
                                        const float* maskvals, long long nnz, const float* Q, long long q_hs,
                                        long long q_rs, const float* K, long long k_hs, long long k_rs,
                                        const float* V, long long v_hs, long long v_rs, float scale, float* O,
                                        long long o_hs, long long o_rs, float* S, float* P, void* stream) {
  STC_NVTX("stc_sparse_attention_f32");
  int rc = check_common(m, n, d, heads, rowptr, nnz);
  if (rc) return rc;
  if (m == 0) return STC_OK;
  if (!dim_ok(d)) return fail(STC_EUNSUPPORTED, "head dim %d not in {4,8,16,32,64,128}", d);
  if (!O || (nnz && (!colidx || !Q || !K || !V))) return fail(STC_EINVAL, "null pointer");
  if (P && !S) return fail(STC_EINVAL, "P output requires the S buffer");
  const bool ok = aligned16(Q) && aligned16(K) && aligned16(V) && aligned16(O) && q_rs % 4 == 0 &&
                  k_rs % 4 == 0 && v_rs % 4 == 0 && o_rs % 4 == 0 && q_hs % 4 == 0 && k_hs % 4 == 0 &&
                  v_hs % 4 == 0 && o_hs % 4 == 0 && q_rs >= d && k_rs >= d && v_rs >= d && o_rs >= d;
  if (!ok) return fail(STC_EINVAL, "Q/K/V/O must be 16-byte aligned with strides multiple of 4 and >= d");
  AttnArgs a{};
  a.m = m; a.n = n; a.d = d; a.heads = heads;
  a.rowptr = rowptr; a.colidx = colidx; a.maskv = maskvals;
  a.Q = Q; a.q_hs = q_hs; a.q_rs = q_rs;
  a.K = K; a.k_hs = k_hs; a.k_rs = k_rs;
  a.V = V; a.v_hs = v_hs; a.v_rs = v_rs;
  a.scale = scale; a.nnz = nnz; a.S = S; a.P = P;
  a.O = O; a.o_hs = o_hs; a.o_rs = o_rs;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return S ? attn_by_d<true>(a, st) : attn_by_d<false>(a, st);
}

extern "C" size_t stc_attention_tiled_workspace_bytes(int m, int heads) {
  if (m <= 0 || heads <= 0) return 0;
  return (size_t)heads * m * (AT_D * sizeof(float) + sizeof(float2));
}

extern "C" int stc_sparse_attention_tiled_f32(int m, int n, int d, int heads, int n_blocks, int dt_max,
                                              const int* tile_cols, const float* tile_vals, const int* rem_rowptr,
                                              const int* rem_colidx, const float* rem_vals, long long rem_nnz,
                                              const float* Q, long long q_hs, long long q_rs, const float* K,
                                              long long k_hs, long long k_rs, const float* V, long long v_hs,
                                              long long v_rs, float scale, float* O, long long o_hs, long long o_rs,
                                              void* ws, size_t ws_bytes, void* stream) {
  STC_NVTX("stc_sparse_attention_tiled_f32");
  int rc = check_common(m, n, d, heads, rem_rowptr, rem_nnz);
  if (rc) return rc;
  if (m == 0) return STC_OK;
  if (d != AT_D) return fail(STC_EUNSUPPORTED, "tiled attention needs head dim 64 (got %d)", d);
  if (n_blocks != (int)ceil_div(m, AT_B) || dt_max < 0) return fail(STC_EINVAL, "bad tile plan shape");
  if (!O || !Q || !K || !V || (dt_max && (!tile_cols || !tile_vals)) || (rem_nnz && (!rem_colidx || !rem_vals)))
    return fail(STC_EINVAL, "null pointer");
  const bool ok = aligned16(Q) && aligned16(K) && aligned16(V) && aligned16(O) && q_rs % 4 == 0 &&
                  k_rs % 4 == 0 && v_rs % 4 == 0 && o_rs % 4 == 0 && q_hs % 4 == 0 && k_hs % 4 == 0 &&
                  v_hs % 4 == 0 && o_hs % 4 == 0 && q_rs >= d && k_rs >= d && v_rs >= d && o_rs >= d;
  if (!ok) return fail(STC_EINVAL, "Q/K/V/O must be 16-byte aligned with strides multiple of 4 and >= d");
  const size_t need = stc_attention_tiled_workspace_bytes(m, heads);
  if (!ws || ws_bytes < need || !aligned16(ws)) return fail(STC_EWORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TileArgs t{};
  t.m = m; t.n = n; t.heads = heads; t.n_blocks = n_blocks; t.dt_max = dt_max;
  t.tile_cols = tile_cols; t.tile_vals = tile_vals;
  t.Q = Q; t.q_hs = q_hs; t.q_rs = q_rs;
  t.K = K; t.k_hs = k_hs; t.k_rs = k_rs;
  t.V = V; t.v_hs = v_hs; t.v_rs = v_rs;
  t.scale = scale;
  t.Opart = static_cast<float*>(ws);
  t.ml = reinterpret_cast<float2*>(t.Opart + (size_t)heads * m * AT_D);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attn_tile8_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AT8_SMEM);
    configured = true;
  }
  // 8x4 register tiles, 128 threads (8x8 with 64 threads measured 0.80 vs 0.77 ms on cfg4)
  attn_tile8_kernel<16><<<dim3(n_blocks, heads), 128, AT8_SMEM, st>>>(t);
  rc = check_launch("attn_tile8_kernel");
  if (rc) return rc;
  AttnArgs a{};
  a.m = m; a.n = n; a.d = d; a.heads = heads;
  a.rowptr = rem_rowptr; a.colidx = rem_colidx; a.maskv = rem_vals;
  a.Q = Q; a.q_hs = q_hs; a.q_rs = q_rs;
  a.K = K; a.k_hs = k_hs; a.k_rs = k_rs;
  a.V = V; a.v_hs = v_hs; a.v_rs = v_rs;
  a.scale = scale; a.nnz = rem_nnz;
  a.O = O; a.o_hs = o_hs; a.o_rs = o_rs;
  a.Opart = t.Opart;
  a.ml = t.ml;
#ifdef STC_ATTN_NO_VSMEM
  return launch_attn<16, false>(a, st);
#else
  return launch_attn_vsmem(a, st);
#endif
}
