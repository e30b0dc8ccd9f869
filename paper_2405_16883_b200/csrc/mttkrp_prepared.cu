// C-ABI entry points of the prepared-item MTTKRP (segreduce_async.cuh): plan-time item build,
// plan of items per group for its kernel, and the launch.
#include "abi_util.cuh"
#include "seg_launch.cuh"
#include "segreduce_async.cuh"

using namespace stc;
using namespace stc::seg;

namespace {

template <int SUBW, int VEC>
int launch_async(const SegOut& o, MergeShape ms, const MttkrpItemsOp<VEC>& op, cudaStream_t st) {
  using Op = MttkrpItemsOp<VEC>;
  constexpr int SW = SUBW * VEC;
  constexpr int U = SUBW >= 8 ? Op::kRing : 4;
  constexpr int NG = kThreads / SUBW;
  const int slabs = (int)ceil_div(o.k, SW);
  if (o.m == 0 || slabs == 0) return STC_OK;
  ms.n_cta = (int)ceil_div(ms.n_groups, NG);
  if (ms.n_cta == 0) return STC_OK;
  const dim3 grid(ms.n_cta, slabs, 1);
  constexpr size_t smem = merge_async_smem_bytes<SUBW, VEC, Op>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(merge_async_kernel<SUBW, VEC, EPI_NONE, false, U, true, Op>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(merge_async_kernel<SUBW, VEC, EPI_NONE, false, U, false, Op>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  if (o.k % SW == 0)
    merge_async_kernel<SUBW, VEC, EPI_NONE, false, U, true, Op><<<grid, dim3(kThreads), smem, st>>>(o, ms, op);
  else
    merge_async_kernel<SUBW, VEC, EPI_NONE, false, U, false, Op><<<grid, dim3(kThreads), smem, st>>>(o, ms, op);
  return check_launch("merge_async_kernel");
}

template <int VEC>
int dispatch_async(int subw, const SegOut& o, const MergeShape& ms, const MttkrpItemsOp<VEC>& op, cudaStream_t st) {
  switch (subw) {
    case 4: return launch_async<4, VEC>(o, ms, op, st);
    case 8: return launch_async<8, VEC>(o, ms, op, st);
    case 16: return launch_async<16, VEC>(o, ms, op, st);
    default: return launch_async<32, VEC>(o, ms, op, st);
  }
}

template <int SUBW, int VEC>
int plan_ipg_async(int m, long long nnz, int k) {
  using Op = MttkrpItemsOp<VEC>;
  constexpr int U = SUBW >= 8 ? Op::kRing : 4;
  constexpr int NG = kThreads / SUBW;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto kern = merge_async_kernel<SUBW, VEC, EPI_NONE, false, U, true, Op>;
  const size_t smem = merge_async_smem_bytes<SUBW, VEC, Op>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  if (per_sm > Op::kMinBlocks) per_sm = Op::kMinBlocks;  // the register budget the kernel was compiled for
  const long long slabs = ceil_div(k, SUBW * VEC);
  const long long total = merge_total_items(m, nnz);
  long long ctas = (long long)sms * per_sm / slabs;  // CTAs per slab in one wave
  if (ctas < 1) ctas = 1;
  // one wave of groups when it fits the per-group item limit, else whole waves
  long long waves = ceil_div(total, ctas * NG * (long long)kMaxIpg);
  if (waves < 1) waves = 1;
  long long ipg = ceil_div(total, ctas * waves * NG);
  if (ipg < 32 * kEntryCost) ipg = 32 * kEntryCost;
  if (ipg > kMaxIpg) ipg = kMaxIpg;
  return (int)ipg;
}

}  // namespace

extern "C" size_t stc_mttkrp_items_bytes(long long nnz) {
  return nnz < 0 ? 0 : (size_t)nnz * sizeof(MttkrpOp<4>::Item);
}

extern "C" int stc_mttkrp_prepare_items(long long nnz, const int* jcrd, const int* kcrd, const float* vals,
                                        int n_j, long long ldb, int n_k, long long ldcf, void* items,
                                        void* stream) {
  STC_NVTX("stc_mttkrp_prepare_items");
  if (nnz < 0 || n_j < 0 || n_k < 0 || ldb < 0 || ldcf < 0) return fail(STC_EINVAL, "negative extent");
  if (nnz > INT32_MAX) return fail(STC_EUNSUPPORTED, "nnz exceeds int32 index range");
  if ((long long)(n_j + 1) * ldb >= (1LL << 32) || (long long)(n_k + 1) * ldcf >= (1LL << 32))
    return fail(STC_EUNSUPPORTED, "prepared items hold 32-bit gather offsets: factor of 2^32 elements or more");
  if (nnz == 0) return STC_OK;
  if (!jcrd || !kcrd || !vals || !items) return fail(STC_EINVAL, "null pointer");
  if (!aligned16(items)) return fail(STC_EINVAL, "items buffer must be 16-byte aligned");
  using Item = MttkrpOp<4>::Item;
  const int blocks = (int)std::min<long long>(ceil_div(nnz, 256), 148 * 32);
  mttkrp_items_kernel<Item><<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      nnz, jcrd, kcrd, vals, ldb, ldcf, static_cast<Item*>(items));
  return check_launch("mttkrp_items_kernel");
}

extern "C" int stc_mttkrp_prepared_items_per_group(int n_seg, long long nnz, int rank) {
  if (n_seg < 0 || nnz < 0 || rank < 1) return fail(STC_EINVAL, "bad plan arguments");
  const int vec = rank % 4 == 0 ? 4 : 1;
  const int subw = choose_subw(rank, vec);
  if (vec == 4) {
    switch (subw) {
      case 4: return plan_ipg_async<4, 4>(n_seg, nnz, rank);
      case 8: return plan_ipg_async<8, 4>(n_seg, nnz, rank);
      case 16: return plan_ipg_async<16, 4>(n_seg, nnz, rank);
      default: return plan_ipg_async<32, 4>(n_seg, nnz, rank);
    }
  }
  switch (subw) {
    case 4: return plan_ipg_async<4, 1>(n_seg, nnz, rank);
    case 8: return plan_ipg_async<8, 1>(n_seg, nnz, rank);
    case 16: return plan_ipg_async<16, 1>(n_seg, nnz, rank);
    default: return plan_ipg_async<32, 1>(n_seg, nnz, rank);
  }
}

extern "C" int stc_mttkrp_coo3_prepared_f32(int n_seg, int rank, const int* seg_ptr, const void* items,
                                            long long nnz, int n_j, const float* B, long long ldb, int n_k,
                                            const float* C, long long ldcf, float* M, long long ldm,
                                            const int* partition, int items_per_group, void* ws,
                                            size_t ws_bytes, void* stream) {
  STC_NVTX("stc_mttkrp_coo3_prepared_f32");
  if (n_seg < 0 || rank < 0 || nnz < 0 || n_j < 0 || n_k < 0) return fail(STC_EINVAL, "negative extent");
  if (nnz > INT32_MAX) return fail(STC_EUNSUPPORTED, "nnz exceeds int32 index range");
  if (n_seg == 0 || rank == 0) return STC_OK;
  if (!seg_ptr || !M || (nnz && (!items || !B || !C))) return fail(STC_EINVAL, "null pointer");
  if (ldb < rank || ldcf < rank || ldm < rank) return fail(STC_EINVAL, "leading dimension smaller than rank");
  if ((long long)(n_j + 1) * ldb >= (1LL << 32) || (long long)(n_k + 1) * ldcf >= (1LL << 32))
    return fail(STC_EUNSUPPORTED, "prepared items hold 32-bit gather offsets: factor of 2^32 elements or more");
  if (!aligned16(items)) return fail(STC_EINVAL, "items buffer must be 16-byte aligned");
  if (!partition || items_per_group < 1 || items_per_group > kMaxIpg)
    return fail(STC_EINVAL, "needs a merge-path partition with 1 <= items_per_group <= %d", kMaxIpg);
  const bool vec4 = rank % 4 == 0 && ldb % 4 == 0 && ldcf % 4 == 0 && ldm % 4 == 0 && aligned16(B) &&
                    aligned16(C) && aligned16(M);
  const int vec = vec4 ? 4 : 1;
  const int subw = choose_subw(rank, vec);
  const size_t need = merge_ws_bytes(n_seg, nnz, rank, subw, vec, items_per_group, 1);
  if (ws_bytes < need || (need && !ws)) return fail(STC_EWORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  SegOut o{n_seg, rank, seg_ptr, M, ldm, nullptr, 0};
  MergeShape ms{};
  const int sw = subw * vec;
  const long long n_cta = ceil_div(n_groups_for(n_seg, nnz, items_per_group), kThreads / subw);
  ms.starts = reinterpret_cast<const int2*>(partition);
  ms.n_groups = (int)n_groups_for(n_seg, nnz, items_per_group);
  ms.ipg = items_per_group;
  ms.head_buf = static_cast<float*>(ws);
  ms.tail_buf = ms.head_buf + ceil_div(rank, sw) * n_cta * sw;
  ms.counters = reinterpret_cast<int*>(ms.tail_buf + ceil_div(rank, sw) * n_cta * sw);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (vec4) {
    MttkrpItemsOp<4> op{static_cast<const MttkrpOp<4>::Item*>(items), B, C};
    op.limitb = (unsigned long long)n_j * ldb;
    op.limitc = (unsigned long long)n_k * ldcf;
    return dispatch_async<4>(subw, o, ms, op, st);
  }
  MttkrpItemsOp<1> op{static_cast<const MttkrpOp<1>::Item*>(items), B, C};
  op.limitb = (unsigned long long)n_j * ldb;
  op.limitc = (unsigned long long)n_k * ldcf;
  return dispatch_async<1>(subw, o, ms, op, st);
}
