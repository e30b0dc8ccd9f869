// 64-bit-gather instantiations of the segmented gather-reduce family (dense
// operands / factor matrices of 2^32 elements or more). A separate translation
// unit so the library's kernels compile in parallel.
#include "seg_launch.cuh"

namespace stc {
namespace seg {

int spmm_wide(int vec, int epilogue, bool add, const SegOut& o, const MergeShape& ms, const int* colidx,
              const float* vals, const float* B, long long ldb, const Launch& L) {
  if (vec == 4) {
    SpmmWideOp<4> op{};
    op.col = colidx;
    op.val = vals;
    op.B = B;
    op.ldb = ldb;
    return dispatch_spmm<4>(epilogue, add, o, ms, op, L);
  }
  SpmmWideOp<1> op{};
  op.col = colidx;
  op.val = vals;
  op.B = B;
  op.ldb = ldb;
  return dispatch_spmm<1>(epilogue, add, o, ms, op, L);
}

int mttkrp_wide(int vec, const SegOut& o, const MergeShape& ms, const int* jc, const int* kc, const float* vals,
                const float* B, long long ldb, const float* C, long long ldcf, int subw, const Launch& L) {
  if (vec == 4) {
    MttkrpWideOp<4> op{};
    op.jc = jc;
    op.kc = kc;
    op.val = vals;
    op.B = B;
    op.ldb = ldb;
    op.C = C;
    op.ldcf = ldcf;
    return dispatch_subw<4, EPI_NONE, false>(subw, o, ms, op, L);
  }
  MttkrpWideOp<1> op{};
  op.jc = jc;
  op.kc = kc;
  op.val = vals;
  op.B = B;
  op.ldb = ldb;
  op.C = C;
  op.ldcf = ldcf;
  return dispatch_subw<1, EPI_NONE, false>(subw, o, ms, op, L);
}

}  // namespace seg
}  // namespace stc
