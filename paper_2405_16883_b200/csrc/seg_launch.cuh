// Launch helpers of the segmented gather-reduce family, shared by the C-ABI
// translation units (spmm.cu: 32-bit gather offsets; spmm_wide.cu: 64-bit).
#pragma once

#include "abi_util.cuh"
#include "segreduce.cuh"

namespace stc {
namespace seg {

inline constexpr int kThreads = 256;
inline constexpr int kMaxIpg = 1024 * kEntryCost;  // items per group (in item units)

inline int choose_subw(int k, int vec) {
  for (int s : {4, 8, 16}) {
    if (s * vec >= k) return s;
  }
  return 32;
}

inline long long n_groups_for(int m, long long nnz, int ipg) { return ceil_div(merge_total_items(m, nnz), ipg); }

inline size_t merge_ws_bytes(int m, long long nnz, int k, int subw, int vec, int ipg, int batch) {
  const long long groups = n_groups_for(m, nnz, ipg);
  const int ng = kThreads / subw;
  const long long n_cta = ceil_div(groups, ng);
  const int sw = subw * vec;
  const long long slabs = ceil_div(k, sw);
  return (size_t)(2LL * batch * slabs * n_cta * sw * (long long)sizeof(float) +
                  batch * slabs * n_cta * (long long)sizeof(int));
}

struct Launch {
  int variant;
  int batch;
  cudaStream_t stream;
};

template <int SUBW, int VEC, int EPI, bool ADD, class Op>
int launch_seg(const SegOut& o, MergeShape ms, const Op& op, const Launch& L) {
  constexpr int SW = SUBW * VEC;
  constexpr int U = SUBW >= 8 ? Op::kRing : 4;
  const int slabs = (int)ceil_div(o.k, SW);
  if (o.m == 0 || slabs == 0) return STC_OK;
  if (L.variant == STC_VARIANT_ROW) {
    // a row's sub-warp loads SUBW entries at a time: keep up to 16 of their gathers in flight
    constexpr int UR = SUBW >= 16 ? 16 : (SUBW >= 8 ? 8 : 4);
    const dim3 grid((unsigned)ceil_div((long long)o.m * SUBW, kThreads), slabs, L.batch);
    row_kernel<SUBW, VEC, EPI, ADD, UR, Op><<<grid, dim3(kThreads), 0, L.stream>>>(o, ms, op);
    return check_launch("row_kernel");
  }
  constexpr int NG = kThreads / SUBW;
  ms.n_cta = (int)ceil_div(ms.n_groups, NG);
  if (ms.n_cta == 0) return STC_OK;
  const dim3 grid(ms.n_cta, slabs, L.batch);
  constexpr size_t smem = merge_smem_bytes<SUBW, VEC, Op>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(merge_kernel<SUBW, VEC, EPI, ADD, U, true, Op>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(merge_kernel<SUBW, VEC, EPI, ADD, U, false, Op>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  if (o.k % SW == 0)
    merge_kernel<SUBW, VEC, EPI, ADD, U, true, Op><<<grid, dim3(kThreads), smem, L.stream>>>(o, ms, op);
  else
    merge_kernel<SUBW, VEC, EPI, ADD, U, false, Op><<<grid, dim3(kThreads), smem, L.stream>>>(o, ms, op);
  return check_launch("merge_kernel");
}

template <int VEC, int EPI, bool ADD, template <int> class OpT>
int dispatch_subw(int subw, const SegOut& o, const MergeShape& ms, const OpT<VEC>& op, const Launch& L) {
  switch (subw) {
    case 4: return launch_seg<4, VEC, EPI, ADD>(o, ms, op, L);
    case 8: return launch_seg<8, VEC, EPI, ADD>(o, ms, op, L);
    case 16: return launch_seg<16, VEC, EPI, ADD>(o, ms, op, L);
    default: return launch_seg<32, VEC, EPI, ADD>(o, ms, op, L);
  }
}

template <int VEC, template <int> class OpT>
int dispatch_spmm(int epilogue, bool add, const SegOut& o, const MergeShape& ms, const OpT<VEC>& op,
                  const Launch& L) {
  const int subw = choose_subw(o.k, VEC);
  if (epilogue == STC_EPILOGUE_RELU)
    return add ? dispatch_subw<VEC, EPI_RELU, true>(subw, o, ms, op, L)
               : dispatch_subw<VEC, EPI_RELU, false>(subw, o, ms, op, L);
  return add ? dispatch_subw<VEC, EPI_NONE, true>(subw, o, ms, op, L)
             : dispatch_subw<VEC, EPI_NONE, false>(subw, o, ms, op, L);
}

// 64-bit gather entry points (spmm_wide.cu): dense operands of 2^32 elements or more
int spmm_wide(int vec, int epilogue, bool add, const SegOut& o, const MergeShape& ms, const int* colidx,
              const float* vals, const float* B, long long ldb, const Launch& L);
int mttkrp_wide(int vec, const SegOut& o, const MergeShape& ms, const int* jc, const int* kc, const float* vals,
                const float* B, long long ldb, const float* C, long long ldcf, int subw, const Launch& L);

}  // namespace seg
}  // namespace stc
