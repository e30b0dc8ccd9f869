// C-ABI entry points for the segmented gather-reduce family:
// CSR SpMM (ROW / MERGE / COLTILE), batched CSR SpMM, COO SpMM, MTTKRP,
// plus the plan-time merge-path partition and COO row segmentation.
#include <cstdlib>

#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include "abi_util.cuh"
#include "coltile.cuh"
#include "seg_launch.cuh"

using namespace stc;

using namespace stc::seg;

namespace {

// ---- COLTILE plan: header {magic, n_chunks} | padded offsets | counts | chunk_ptr | CUB temp |
// packed entries (int2, 16-byte aligned). See coltile.cuh.
struct CttLayout {
  int n_chunks;
  long long n_slots, max_entries;
  size_t temp_bytes;
  long long offs, counts, chunk_ptr, temp, ent, total_ints;
};
inline CttLayout ctt_layout(int m, int n, long long nnz) {
  CttLayout l{};
  l.n_chunks = (int)ceil_div(n, CTT_BROWS);
  l.n_slots = ceil_div(m, CTT_ROWS) * l.n_chunks * CTT_ROWS;
  l.max_entries = nnz + (long long)(CTT_PAD - 1) * std::min<long long>(nnz, (long long)m * l.n_chunks);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int*)nullptr, (int*)nullptr, (int)(l.n_slots + 1));
  l.temp_bytes = tb;
  auto up4 = [](long long x) { return (x + 3) / 4 * 4; };
  l.offs = 4;
  l.counts = up4(l.offs + l.n_slots + 1);
  l.chunk_ptr = up4(l.counts + l.n_slots + 1);
  l.temp = up4(l.chunk_ptr + (long long)m * (l.n_chunks + 1));
  l.ent = up4(l.temp + (long long)((tb + 3) / 4));
  l.total_ints = l.ent + 2 * std::max<long long>(l.max_entries, 1);
  return l;
}

// Tiled tensor map of the dense operand for the COLTILE producer: fp32 [n rows, k columns], row
// pitch ldb, box = CTT_BROWS rows x CTT_COLS columns, out-of-range elements read as zero. The
// encoder is a driver entry point fetched through the runtime (the library does not link libcuda,
// so it still loads on a machine without a driver). False when the operand does not meet the
// tensor-map alignment rules (16-byte base and pitch) -- the kernel then copies row by row.
bool ctt_operand_map(const float* B, long long ldb, int n, int k, CUtensorMap* map) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<Encode>(fn);
  }();
  if (!encode || n <= 0 || k <= 0) return false;
  if (const char* e = std::getenv("STC_COLTILE_ROW_COPIES"); e && *e == '1') return false;  // tests: the other path
  if (reinterpret_cast<uintptr_t>(B) % 16 || (ldb * 4) % 16 || ldb * 4 >= (1LL << 40)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)n};
  const cuuint64_t pitch[1] = {(cuuint64_t)ldb * 4};
  const cuuint32_t box[2] = {(cuuint32_t)CTT_COLS, (cuuint32_t)CTT_BROWS};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(B), dims, pitch, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int EPI, bool ADD>
int launch_coltile_tmem(int m, int n, int k, long long nnz, const int* plan, const float* B, long long ldb, float* C,
                        long long ldc, const float* D, long long ldd, cudaStream_t st, const Launch& L) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(coltile_tmem_kernel<EPI, ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTT_SMEM);
    configured = true;
  }
  if (m == 0 || k == 0) return STC_OK;
  const CttLayout lay = ctt_layout(m, n, nnz);
  const dim3 grid((unsigned)ceil_div(m, CTT_ROWS), (unsigned)ceil_div(k, CTT_COLS));
  CUtensorMap bmap{};
  const int use_bmap = ctt_operand_map(B, ldb, n, k, &bmap) ? 1 : 0;
  coltile_tmem_kernel<EPI, ADD><<<grid, dim3(CTT_THREADS), CTT_SMEM, st>>>(
      m, n, k, plan + lay.offs, reinterpret_cast<const int2*>(plan + lay.ent), B, ldb, C, ldc, D, ldd, bmap, use_bmap);
  return check_launch("coltile_tmem_kernel");
}

// Shared validation + dispatch for every SpMM-shaped entry point.
int spmm_common(int batch, int m, int n, int k, const int* rowptr, const int* colidx, const float* vals,
                long long nnz, long long val_bs, const float* B, long long ldb, long long b_bs, float* C,
                long long ldc, long long c_bs, const float* D, long long ldd, int variant, int epilogue,
                const int* partition, int ipg, void* ws, size_t ws_bytes, void* stream) {
  STC_NVTX(variant == STC_VARIANT_COLTILE ? "stc_spmm/coltile"
           : variant == STC_VARIANT_MERGE ? "stc_spmm/merge" : "stc_spmm/row");
  if (m < 0 || n < 0 || k < 0 || nnz < 0 || batch < 1) return fail(STC_EINVAL, "negative extent");
  if (nnz > INT32_MAX) return fail(STC_EUNSUPPORTED, "nnz exceeds int32 index range");
  if (m == 0 || k == 0) return STC_OK;
  if (!rowptr || !C || (nnz && (!colidx || !vals || !B))) return fail(STC_EINVAL, "null pointer");
  if (ldb < k || ldc < k || (D && ldd < k)) return fail(STC_EINVAL, "leading dimension smaller than k");
  if (epilogue != STC_EPILOGUE_NONE && epilogue != STC_EPILOGUE_RELU)
    return fail(STC_EINVAL, "unknown epilogue %d", epilogue);
  // dense operands of 2^32 elements or more gather with 64-bit addresses (spmm_wide.cu)
  // (batched: B advances per batch in 64 bits, offsets are within one batch's operand)
  const bool wide = (long long)(n + 1) * ldb >= (1LL << 32);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec4 = (k % 4 == 0) && (ldb % 4 == 0) && (ldc % 4 == 0) && aligned16(B) && aligned16(C) &&
                    (!D || (ldd % 4 == 0 && aligned16(D))) && (val_bs % 4 == 0 || batch == 1) &&
                    (b_bs % 4 == 0) && (c_bs % 4 == 0);

  if (variant == STC_VARIANT_COLTILE) {  // operand staged in Tensor Memory; the plan carries A
    if (!vec4) return fail(STC_EUNSUPPORTED, "COLTILE needs k, ldb, ldc multiples of 4 and 16-byte alignment");
    if (batch != 1) return fail(STC_EUNSUPPORTED, "COLTILE is not batched");
    if (!partition) return fail(STC_EINVAL, "COLTILE needs its plan (stc_coltile_plan) as `partition`");
    const Launch L{variant, 1, st};
    if (epilogue == STC_EPILOGUE_RELU)
      return D ? launch_coltile_tmem<EPI_RELU, true>(m, n, k, nnz, partition, B, ldb, C, ldc, D, ldd, st, L)
               : launch_coltile_tmem<EPI_RELU, false>(m, n, k, nnz, partition, B, ldb, C, ldc, D, ldd, st, L);
    return D ? launch_coltile_tmem<EPI_NONE, true>(m, n, k, nnz, partition, B, ldb, C, ldc, D, ldd, st, L)
             : launch_coltile_tmem<EPI_NONE, false>(m, n, k, nnz, partition, B, ldb, C, ldc, D, ldd, st, L);
  }
  if (variant != STC_VARIANT_ROW && variant != STC_VARIANT_MERGE)
    return fail(STC_EINVAL, "unknown variant %d", variant);

  SegOut o{m, k, rowptr, C, ldc, D, ldd};
  MergeShape ms{};
  ms.batch_val_stride = val_bs;
  ms.batch_b_stride = b_bs;
  ms.batch_c_stride = c_bs;
  if (variant == STC_VARIANT_MERGE) {
    if (!partition) return fail(STC_EINVAL, "MERGE variant needs a partition");
    if (ipg < 1 || ipg > kMaxIpg) return fail(STC_EINVAL, "items_per_group must be in [1, %d]", kMaxIpg);
    const int vec = vec4 ? 4 : 1;
    const size_t need = merge_ws_bytes(m, nnz, k, choose_subw(k, vec), vec, ipg, batch);
    if (ws_bytes < need || (need && !ws))
      return fail(STC_EWORKSPACE, "workspace %zu bytes < %zu required", ws_bytes, need);
    const int sw = choose_subw(k, vec) * vec;
    const long long n_cta = ceil_div(n_groups_for(m, nnz, ipg), kThreads / choose_subw(k, vec));
    const long long slabs = ceil_div(k, sw);
    ms.starts = reinterpret_cast<const int2*>(partition);
    ms.n_groups = (int)n_groups_for(m, nnz, ipg);
    ms.ipg = ipg;
    ms.head_buf = static_cast<float*>(ws);
    ms.tail_buf = ms.head_buf + (long long)batch * slabs * n_cta * sw;
    ms.counters = reinterpret_cast<int*>(ms.tail_buf + (long long)batch * slabs * n_cta * sw);
  }
  const Launch L{variant, batch, st};
  if (wide) return spmm_wide(vec4 ? 4 : 1, epilogue, D != nullptr, o, ms, colidx, vals, B, ldb, L);
  if (vec4) {
    SpmmOp<4> op{colidx, vals, B, ldb};
    op.limit = (unsigned long long)n * ldb;
    return dispatch_spmm<4>(epilogue, D != nullptr, o, ms, op, L);
  }
  SpmmOp<1> op{colidx, vals, B, ldb};
  op.limit = (unsigned long long)n * ldb;
  return dispatch_spmm<1>(epilogue, D != nullptr, o, ms, op, L);
}

}  // namespace

namespace {
template <int SUBW, int VEC, class Op>
int plan_ipg(int m, long long nnz, int k, int batch) {
  constexpr int U = SUBW >= 8 ? Op::kRing : 4;
  constexpr int NG = kThreads / SUBW;
  constexpr int CAP = merge_stage_cap<SUBW, Op>();
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto kern = merge_kernel<SUBW, VEC, EPI_NONE, false, U, true, Op>;
  const size_t smem = merge_smem_bytes<SUBW, VEC, Op>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const long long slabs = ceil_div(k, SUBW * VEC);
  const long long total = merge_total_items(m, nnz);
  const long long cta_slots = (long long)sms * per_sm;
  // CTAs available per (slab, batch) in one wave
  long long ctas = cta_slots / (slabs * batch);
  if (ctas < 1) ctas = 1;
  const long long max_ipg = 8LL * CAP * kEntryCost < kMaxIpg ? 8LL * CAP * kEntryCost : kMaxIpg;  // a few windows
  long long waves = ceil_div(total, ctas * NG * max_ipg);
  if (waves < 1) waves = 1;
  long long ipg = ceil_div(total, ctas * waves * NG);
  if (ipg < 32 * kEntryCost) ipg = 32 * kEntryCost;
  if (ipg > kMaxIpg) ipg = kMaxIpg;
  return (int)ipg;
}
}  // namespace

extern "C" int stc_merge_plan_items_per_group(int m, long long nnz, int k, int batch, int kind) {
  if (m < 0 || nnz < 0 || k < 1 || batch < 1) return fail(STC_EINVAL, "bad plan arguments");
  const int vec = k % 4 == 0 ? 4 : 1;
  const int subw = choose_subw(k, vec);
  if (kind == 1) {
    if (vec == 4) {
      switch (subw) {
        case 4: return plan_ipg<4, 4, MttkrpOp<4>>(m, nnz, k, batch);
        case 8: return plan_ipg<8, 4, MttkrpOp<4>>(m, nnz, k, batch);
        case 16: return plan_ipg<16, 4, MttkrpOp<4>>(m, nnz, k, batch);
        default: return plan_ipg<32, 4, MttkrpOp<4>>(m, nnz, k, batch);
      }
    }
    switch (subw) {
      case 4: return plan_ipg<4, 1, MttkrpOp<1>>(m, nnz, k, batch);
      case 8: return plan_ipg<8, 1, MttkrpOp<1>>(m, nnz, k, batch);
      case 16: return plan_ipg<16, 1, MttkrpOp<1>>(m, nnz, k, batch);
      default: return plan_ipg<32, 1, MttkrpOp<1>>(m, nnz, k, batch);
    }
  }
  if (vec == 4) {
    switch (subw) {
      case 4: return plan_ipg<4, 4, SpmmOp<4>>(m, nnz, k, batch);
      case 8: return plan_ipg<8, 4, SpmmOp<4>>(m, nnz, k, batch);
      case 16: return plan_ipg<16, 4, SpmmOp<4>>(m, nnz, k, batch);
      default: return plan_ipg<32, 4, SpmmOp<4>>(m, nnz, k, batch);
    }
  }
  switch (subw) {
    case 4: return plan_ipg<4, 1, SpmmOp<1>>(m, nnz, k, batch);
    case 8: return plan_ipg<8, 1, SpmmOp<1>>(m, nnz, k, batch);
    case 16: return plan_ipg<16, 1, SpmmOp<1>>(m, nnz, k, batch);
    default: return plan_ipg<32, 1, SpmmOp<1>>(m, nnz, k, batch);
  }
}

extern "C" long long stc_coltile_plan_ints(int m, int n, long long nnz) {
  if (m < 0 || n < 0 || nnz < 0) return -1;
  if ((long long)ceil_div(m, CTT_ROWS) * ceil_div(n, CTT_BROWS) * CTT_ROWS + 1 >= INT32_MAX) return -1;
  const CttLayout lay = ctt_layout(m, n, nnz);
  if (lay.max_entries >= INT32_MAX) return -1;
  return lay.total_ints;
}

extern "C" int stc_coltile_plan(int m, int n, long long nnz, const int* rowptr, const int* colidx,
                                const float* vals, int* plan, long long plan_ints, void* stream) {
  STC_NVTX("stc_coltile_plan");
  if (m < 0 || n < 0 || nnz < 0) return fail(STC_EINVAL, "negative extent");
  if (!plan || !rowptr || (nnz && (!colidx || !vals))) return fail(STC_EINVAL, "null pointer");
  if ((long long)ceil_div(m, CTT_ROWS) * ceil_div(n, CTT_BROWS) * CTT_ROWS + 1 >= INT32_MAX)
    return fail(STC_EUNSUPPORTED, "COLTILE plan: m * ceil(n / 63) slots exceed int32");
  const CttLayout lay = ctt_layout(m, n, nnz);
  if (lay.max_entries >= INT32_MAX) return fail(STC_EUNSUPPORTED, "COLTILE plan exceeds int32 entries");
  if (plan_ints < lay.total_ints)
    return fail(STC_EINVAL, "plan buffer of %lld ints, need %lld", plan_ints, lay.total_ints);
  if (m == 0) return STC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* chunk_ptr = plan + lay.chunk_ptr;
  int* counts = plan + lay.counts;
  int* offs = plan + lay.offs;
  ctt_chunk_ptr_kernel<<<(unsigned)ceil_div(m, 8), 256, 0, st>>>(m, lay.n_chunks, rowptr, colidx, chunk_ptr);
  if (int rc = check_launch("ctt_chunk_ptr_kernel")) return rc;
  ctt_count_kernel<<<1184, 256, 0, st>>>(m, lay.n_chunks, lay.n_slots, chunk_ptr, counts);
  if (int rc = check_launch("ctt_count_kernel")) return rc;
  cudaMemsetAsync(counts + lay.n_slots, 0, sizeof(int), st);
  size_t tb = lay.temp_bytes;
  const cudaError_t e =
      cub::DeviceScan::ExclusiveSum(plan + lay.temp, tb, counts, offs, (int)(lay.n_slots + 1), st);
  if (e != cudaSuccess) return fail(STC_ELAUNCH, "coltile plan scan: %s", cudaGetErrorString(e));
  ctt_scatter_kernel<<<1184, 256, 0, st>>>(m, lay.n_chunks, chunk_ptr, colidx, vals, offs,
                                           reinterpret_cast<int2*>(plan + lay.ent));
  return check_launch("ctt_scatter_kernel");
}

// ---- long-row interleaving (plan time) -------------------------------------------------
namespace stc {
__global__ void merge_interleave_kernel(int m, long long nnz, const int* __restrict__ rowptr, const int* __restrict__ colidx,
                                  const float* __restrict__ vals, int span, int* __restrict__ colidx_out,
                                  float* __restrict__ vals_out) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nnz;
       p += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = m - 1;  // row r with rowptr[r] <= p < rowptr[r + 1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rowptr[mid] <= p)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int base = rowptr[lo];
    const int len = rowptr[lo + 1] - base;
    const int i = (int)(p - base);
    long long dst = p;
    if (len > span) {  // G interleaved sequences: entries j, j+G, j+2G, ... for j = 0..G-1
      const int G = (len + span - 1) / span, q = len / G, rem = len % G, j = i % G;
      dst = (long long)base + (long long)j * q + (j < rem ? j : rem) + i / G;
    }
    colidx_out[dst] = colidx[p];
    vals_out[dst] = vals[p];
  }
}
}  // namespace stc

extern "C" int stc_merge_interleave(int m, long long nnz, const int* rowptr, const int* colidx, const float* vals,
                                    int span, int* colidx_out, float* vals_out, void* stream) {
  STC_NVTX("stc_merge_interleave");
  if (m < 0 || nnz < 0 || span < 1) return fail(STC_EINVAL, "bad interleave arguments");
  if (m == 0 || nnz == 0) return STC_OK;
  if (!rowptr || !colidx || !vals || !colidx_out || !vals_out) return fail(STC_EINVAL, "null pointer");
  const long long blocks = std::min<long long>(ceil_div(nnz, 256), 148LL * 16);
  merge_interleave_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(m, nnz, rowptr, colidx, vals,
                                                                                    span, colidx_out, vals_out);
  return check_launch("merge_interleave_kernel");
}

extern "C" long long stc_merge_path_groups(int m, long long nnz, int items_per_group) {
  if (items_per_group < 1 || m < 0 || nnz < 0) return -1;
  return n_groups_for(m, nnz, items_per_group);
}

extern "C" int stc_merge_path_partition(int m, long long nnz, const int* rowptr, int items_per_group,
                                        int* starts, void* stream) {
  STC_NVTX("stc_merge_path_partition");
  if (m < 0 || nnz < 0 || items_per_group < 1) return fail(STC_EINVAL, "bad partition arguments");
  if (!rowptr || !starts) return fail(STC_EINVAL, "null pointer");
  if (((uintptr_t)starts & 7u) != 0) return fail(STC_EINVAL, "starts must be 8-byte aligned");
  const long long groups = n_groups_for(m, nnz, items_per_group);
  if (groups > INT32_MAX - 1) return fail(STC_EUNSUPPORTED, "too many groups");
  const long long n = groups + 1;
  merge_partition_kernel<<<(unsigned)ceil_div(n, kThreads), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      m, nnz, rowptr, items_per_group, (int)groups, reinterpret_cast<int2*>(starts));
  return check_launch("merge_partition_kernel");
}

extern "C" size_t stc_spmm_workspace_bytes(int m, long long nnz, int k, int variant, int items_per_group,
                                           int batch) {
  if (variant != STC_VARIANT_MERGE || items_per_group < 1 || m <= 0 || k <= 0) return 0;
  const size_t a = merge_ws_bytes(m, nnz, k, choose_subw(k, 4), 4, items_per_group, batch < 1 ? 1 : batch);
  const size_t b = merge_ws_bytes(m, nnz, k, choose_subw(k, 1), 1, items_per_group, batch < 1 ? 1 : batch);
  return a > b ? a : b;
}

extern "C" int stc_spmm_csr_f32(int m, int n, int k, const int* rowptr, const int* colidx, const float* vals,
                                long long nnz, const float* B, long long ldb, float* C, long long ldc,
                                const float* D, long long ldd, int variant, int epilogue,
                                const int* partition, int items_per_group, void* ws, size_t ws_bytes,
                                void* stream) {
  return spmm_common(1, m, n, k, rowptr, colidx, vals, nnz, 0, B, ldb, 0, C, ldc, 0, D, ldd, variant,
                     epilogue, partition, items_per_group, ws, ws_bytes, stream);
}

extern "C" int stc_spmm_csr_batched_f32(int batch, int m, int n, int k, const int* rowptr,
                                        const int* colidx, const float* vals, long long nnz,
                                        long long val_bstride, const float* B, long long ldb,
                                        long long b_bstride, float* C, long long ldc, long long c_bstride,
                                        int variant, int epilogue, const int* partition,
                                        int items_per_group, void* ws, size_t ws_bytes, void* stream) {
  if (batch > 65535) return fail(STC_EUNSUPPORTED, "batch > 65535");
  return spmm_common(batch, m, n, k, rowptr, colidx, vals, nnz, val_bstride, B, ldb, b_bstride, C, ldc,
                     c_bstride, nullptr, 0, variant, epilogue, partition, items_per_group, ws, ws_bytes,
                     stream);
}

extern "C" int stc_spmm_coo_f32(int n_seg, int n, int k, const int* seg_ptr, const int* cols,
                                const float* vals, long long nnz, const float* B, long long ldb, float* C,
                                long long ldc, int variant, const int* partition, int items_per_group,
                                void* ws, size_t ws_bytes, void* stream) {
  return spmm_common(1, n_seg, n, k, seg_ptr, cols, vals, nnz, 0, B, ldb, 0, C, ldc, 0, nullptr, 0, variant,
                     STC_EPILOGUE_NONE, partition, items_per_group, ws, ws_bytes, stream);
}

// ---- COO row segmentation (plan time) ----------------------------------------------

namespace {
__global__ void exclusive_from_counts_tail(const int* n_seg, int* seg_ptr, long long nnz) {
  seg_ptr[*n_seg] = (int)nnz;
}
}  // namespace

extern "C" size_t stc_coo_segments_temp_bytes(long long nnz) {
  size_t a = 0, b = 0;
  cub::DeviceRunLengthEncode::Encode(nullptr, a, (const int*)nullptr, (int*)nullptr, (int*)nullptr,
                                     (int*)nullptr, (int)nnz);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, (int)nnz);
  // counts buffer (nnz ints) + max of the two temporaries, 256-byte aligned pieces
  const size_t counts = ((size_t)nnz * sizeof(int) + 255) & ~size_t(255);
  return counts + ((a > b ? a : b) + 255) + 256;
}

extern "C" int stc_coo_segments(long long nnz, const int* rows, int* seg_rows, int* seg_ptr, int* n_seg_out,
                                void* temp, size_t temp_bytes, void* stream) {
  STC_NVTX("stc_coo_segments");
  if (nnz < 0 || nnz > INT32_MAX) return fail(STC_EUNSUPPORTED, "bad nnz");
  if (!seg_ptr || !n_seg_out || (nnz && (!rows || !seg_rows))) return fail(STC_EINVAL, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (nnz == 0) {
    cudaMemsetAsync(n_seg_out, 0, sizeof(int), st);
    cudaMemsetAsync(seg_ptr, 0, sizeof(int), st);
    return check_launch("coo_segments(empty)");
  }
  const size_t need = stc_coo_segments_temp_bytes(nnz);
  if (!temp || temp_bytes < need) return fail(STC_EWORKSPACE, "temp %zu < %zu", temp_bytes, need);
  char* base = static_cast<char*>(temp);
  base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base) + 255) & ~uintptr_t(255));
  int* counts = reinterpret_cast<int*>(base);
  char* tmp = base + (((size_t)nnz * sizeof(int) + 255) & ~size_t(255));
  size_t tmp_bytes = temp_bytes - (size_t)(tmp - static_cast<char*>(temp));
  cudaError_t e = cub::DeviceRunLengthEncode::Encode(tmp, tmp_bytes, rows, seg_rows, counts, n_seg_out,
                                                     (int)nnz, st);
  if (e != cudaSuccess) return fail(STC_ELAUNCH, "run-length encode: %s", cudaGetErrorString(e));
  tmp_bytes = temp_bytes - (size_t)(tmp - static_cast<char*>(temp));
  // exclusive sum over all nnz slots; slots past n_seg hold garbage counts but
  // seg_ptr[n_seg] is overwritten with nnz below and later slots are unused.
  e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, seg_ptr, (int)nnz, st);
  if (e != cudaSuccess) return fail(STC_ELAUNCH, "exclusive scan: %s", cudaGetErrorString(e));
  exclusive_from_counts_tail<<<1, 1, 0, st>>>(n_seg_out, seg_ptr, nnz);
  return check_launch("coo_segments");
}

// ---- MTTKRP ------------------------------------------------------------------------

namespace {
int mttkrp_common(int n_seg, int rank, const int* seg_ptr, const int* jcrd, const int* kcrd, const float* vals,
                  long long nnz, int n_j, const float* B, long long ldb, int n_k, const float* C, long long ldcf,
                  float* M, long long ldm, int variant, const int* partition, int items_per_group, void* ws,
                  size_t ws_bytes, void* stream) {
  if (n_seg < 0 || rank < 0 || nnz < 0) return fail(STC_EINVAL, "negative extent");
  if (nnz > INT32_MAX) return fail(STC_EUNSUPPORTED, "nnz exceeds int32 index range");
  if (n_seg == 0 || rank == 0) return STC_OK;
  if (!seg_ptr || !M || (nnz && (!jcrd || !kcrd || !vals || !B || !C))) return fail(STC_EINVAL, "null pointer");
  if (ldb < rank || ldcf < rank || ldm < rank) return fail(STC_EINVAL, "leading dimension smaller than rank");
  if (variant != STC_VARIANT_ROW && variant != STC_VARIANT_MERGE)
    return fail(STC_EUNSUPPORTED, "MTTKRP supports ROW and MERGE");
  if (n_j < 0 || n_k < 0) return fail(STC_EINVAL, "negative factor extent");
  const bool wide = (long long)(n_j + 1) * ldb >= (1LL << 32) || (long long)(n_k + 1) * ldcf >= (1LL << 32);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec4 = rank % 4 == 0 && ldb % 4 == 0 && ldcf % 4 == 0 && ldm % 4 == 0 && aligned16(B) &&
                    aligned16(C) && aligned16(M);
  const int vec = vec4 ? 4 : 1;
  const int subw = choose_subw(rank, vec);
  SegOut o{n_seg, rank, seg_ptr, M, ldm, nullptr, 0};
  MergeShape ms{};
  if (variant == STC_VARIANT_MERGE) {
    if (!partition || items_per_group < 1 || items_per_group > kMaxIpg)
      return fail(STC_EINVAL, "MERGE variant needs a partition with 1 <= items_per_group <= %d", kMaxIpg);
    const size_t need = merge_ws_bytes(n_seg, nnz, rank, subw, vec, items_per_group, 1);
    if (ws_bytes < need || (need && !ws)) return fail(STC_EWORKSPACE, "workspace %zu < %zu", ws_bytes, need);
    const int sw = subw * vec;
    const long long n_cta = ceil_div(n_groups_for(n_seg, nnz, items_per_group), kThreads / subw);
    ms.starts = reinterpret_cast<const int2*>(partition);
    ms.n_groups = (int)n_groups_for(n_seg, nnz, items_per_group);
    ms.ipg = items_per_group;
    ms.head_buf = static_cast<float*>(ws);
    ms.tail_buf = ms.head_buf + ceil_div(rank, sw) * n_cta * sw;
    ms.counters = reinterpret_cast<int*>(ms.tail_buf + ceil_div(rank, sw) * n_cta * sw);
  }
  const Launch L{variant, 1, st};
  if (wide) return mttkrp_wide(vec, o, ms, jcrd, kcrd, vals, B, ldb, C, ldcf, subw, L);
  if (vec4) {
    MttkrpOp<4> op{jcrd, kcrd, vals, B, ldb, C, ldcf};
    op.limitb = (unsigned long long)n_j * ldb;
    op.limitc = (unsigned long long)n_k * ldcf;
    return dispatch_subw<4, EPI_NONE, false>(subw, o, ms, op, L);
  }
  MttkrpOp<1> op{jcrd, kcrd, vals, B, ldb, C, ldcf};
  op.limitb = (unsigned long long)n_j * ldb;
  op.limitc = (unsigned long long)n_k * ldcf;
  return dispatch_subw<1, EPI_NONE, false>(subw, o, ms, op, L);
}
}  // namespace

extern "C" int stc_mttkrp_coo3_f32(int n_seg, int rank, const int* seg_ptr, const int* jcrd, const int* kcrd,
                                   const float* vals, long long nnz, int n_j, const float* B, long long ldb,
                                   int n_k, const float* C, long long ldcf, float* M, long long ldm, int variant,
                                   const int* partition, int items_per_group, void* ws, size_t ws_bytes,
                                   void* stream) {
  STC_NVTX("stc_mttkrp_coo3_f32");
  return mttkrp_common(n_seg, rank, seg_ptr, jcrd, kcrd, vals, nnz, n_j, B, ldb, n_k, C, ldcf, M, ldm, variant,
                       partition, items_per_group, ws, ws_bytes, stream);
}


#ifdef STC_DBG_TIMING
// Diagnostic build only: copy the per-group timing stamps of the last merge launch.
extern "C" int stc_debug_timing(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, stc::g_dbg, bytes);
}
#endif
