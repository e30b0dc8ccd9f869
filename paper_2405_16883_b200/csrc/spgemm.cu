// K9: sparse x sparse kernels on CSR operands.
//
//   SpGEMM  C(i,k) = A(i,j) * B(j,k)   (reference plan: [i, j, k], workspace over k,
//                                       engine.py:577-644 + Workspace engine.py:71-90)
//   union   C(i,j) = A(i,j) + B(i,j)   (two terms, _union_sorted engine.py:224-230)
//   product C(i,j) = A(i,j) * B(i,j)   (one term, _intersect_sorted engine.py:208-221)
//
// Structure follows the reference exactly: the SpGEMM output holds every (i,k)
// reached by a product (arithmetic zeros are kept), the union every coordinate
// of either operand, the product every common coordinate. Values keep the
// reference's order of accumulation: the workspace slot starts at 0.0 and adds
// the contributions in loop order — ascending j for SpGEMM (each contribution
// a_ij * b_jk), term order for the union ((0 + a) + b), and 0 + a * b for the
// product — evaluated in fp32.
//
// SpGEMM, B with at most kDenseMaxCols columns: a warp per row accumulates into
// a private SMEM window over all output columns (values + touched bitmask),
// walking j in ascending order — no sort, no product buffer. Wider B:
// expand-sort-compress, row by row: a warp per row writes the row's products
// (key k, value a*b) in (j, k) order; a stable segmented sort by k (CUB) keeps
// equal keys in ascending j; a warp per row then sums each run left to right. Union / product: a warp per row, each lane binary-searches its
// entries in the other operand's row; ballots give output ranks, so rows of any
// length spread over 32 lanes.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "abi_util.cuh"
#include "stc_common.cuh"

namespace stc {
namespace {

constexpr int kWarpsPerCta = 8;

STC_DEVICE int lower_bound(const int* __restrict__ a, int lo, int hi, int key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// cnt[i] = number of products of row i (sum of |B_j| over j in A_i); cnt[m] = 0
__global__ void spgemm_count_kernel(int m, const int* __restrict__ ap, const int* __restrict__ aj,
                                    const int* __restrict__ bp, long long* __restrict__ cnt) {
  const int row = blockIdx.x * kWarpsPerCta + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row > m) return;
  long long s = 0;
  if (row < m)
    for (int p = ap[row] + lane; p < ap[row + 1]; p += 32) {
      const int j = aj[p];
      s += bp[j + 1] - bp[j];
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) cnt[row] = s;
}

// products of row i at [ptr[i], ptr[i+1]) in (j asc, k asc) order
__global__ void spgemm_expand_kernel(int m, const int* __restrict__ ap, const int* __restrict__ aj,
                                     const float* __restrict__ av, const int* __restrict__ bp,
                                     const int* __restrict__ bj, const float* __restrict__ bv,
                                     const long long* __restrict__ ptr, int* __restrict__ keys,
                                     float* __restrict__ vals, int* __restrict__ seg) {
  const int row = blockIdx.x * kWarpsPerCta + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row > m) return;
  long long base = ptr[row];
  if (lane == 0) seg[row] = (int)base;
  if (row == m) return;
  for (int p = ap[row]; p < ap[row + 1]; ++p) {
    const int j = aj[p];
    const float a = av[p];
    const int b0 = bp[j], len = bp[j + 1] - b0;
    for (int t = lane; t < len; t += 32) {
      keys[base + t] = bj[b0 + t];
      vals[base + t] = a * bv[b0 + t];
    }
    base += len;
  }
}

// distinct keys per row of the sorted products
__global__ void spgemm_unique_kernel(int m, const int* __restrict__ seg, const int* __restrict__ keys,
                                     int* __restrict__ cnt) {
  const int row = blockIdx.x * kWarpsPerCta + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row > m) return;
  int s = 0;
  if (row < m)
    for (int p = seg[row] + lane; p < seg[row + 1]; p += 32) s += (p == seg[row] || keys[p] != keys[p - 1]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) cnt[row] = s;
}

// one output entry per run of equal keys, summed left to right from 0.0
__global__ void spgemm_compress_kernel(int m, const int* __restrict__ seg, const int* __restrict__ keys,
                                       const float* __restrict__ vals, const int* __restrict__ cp,
                                       int* __restrict__ ck, float* __restrict__ cv) {
  const int row = blockIdx.x * kWarpsPerCta + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= m) return;
  const int s = seg[row], e = seg[row + 1];
  int out = cp[row];
  for (int base = s; base < e; base += 32) {
    const int p = base + lane;
    const bool start = p < e && (p == s || keys[p] != keys[p - 1]);
    const unsigned ball = __ballot_sync(0xffffffffu, start);
    if (start) {
      const int key = keys[p];
      float acc = 0.0f + vals[p];
      for (int q = p + 1; q < e && keys[q] == key; ++q) acc += vals[q];
      const int o = out + __popc(ball & ((1u << lane) - 1u));
      ck[o] = key;
      cv[o] = acc;
    }
    out += __popc(ball);
  }
}

// ---- dense-window SpGEMM (B has at most kDenseMaxCols columns) ----------------------------
//
// A warp owns one row at a time and a private SMEM accumulator over all p output
// columns (fp32 values + a touched bitmask). It walks A's row in ascending j;
// for each j the lanes scatter B_j's entries (distinct k, so no conflicts):
// acc[k] = acc[k] + a*b, bit k set. __syncwarp between j steps keeps every
// acc[k] summed in ascending j from 0.0, deterministically. Phase 0 counts the
// set bits of the row; phase 1 emits (k, acc[k]) in ascending k by a ballot /
// popc scan over the bitmask words and clears what it read.
constexpr int kDenseMaxCols = 6144;

__host__ __device__ inline int dense_words(int p) { return (p + 31) / 32; }
__host__ __device__ inline size_t dense_warp_bytes(int p) {
  return (size_t)dense_words(p) * 4 + (size_t)((p + 31) / 32 * 32) * 4;
}

__global__ void spgemm_dense_kernel(int phase, int m, int p, const int* __restrict__ ap, const int* __restrict__ aj,
                                    const float* __restrict__ av, const int* __restrict__ bp,
                                    const int* __restrict__ bj, const float* __restrict__ bv,
                                    int* __restrict__ cnt, const int* __restrict__ cp, int* __restrict__ ck,
                                    float* __restrict__ cv) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int nw = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int words = dense_words(p);
  const int pad = words * 32;
  unsigned* bits = reinterpret_cast<unsigned*>(dsm) + warp * words;
  float* acc = reinterpret_cast<float*>(dsm + (size_t)nw * words * 4) + (size_t)warp * pad;
  for (int w = lane; w < words; w += 32) bits[w] = 0u;
  if (phase == 1)
    for (int k = lane; k < pad; k += 32) acc[k] = 0.0f;
  __syncwarp();
  for (int row = blockIdx.x * nw + warp; row < m; row += gridDim.x * nw) {
    for (int q = ap[row]; q < ap[row + 1]; ++q) {
      const int j = aj[q];
      const float a = av[q];
      for (int t = bp[j] + lane; t < bp[j + 1]; t += 32) {
        const int k = bj[t];
        STC_CHECK(k >= 0 && k < p, "SpGEMM column outside the dense window");
        atomicOr(&bits[k >> 5], 1u << (k & 31));
        if (phase == 1) acc[k] += a * bv[t];
      }
      __syncwarp();
    }
    if (phase == 0) {
      int c = 0;
      for (int w = lane; w < words; w += 32) {
        c += __popc(bits[w]);
        bits[w] = 0u;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) cnt[row] = c;
    } else {
      int out = cp[row];
      for (int base = 0; base < words; base += 32) {
        const int w = base + lane;
        unsigned b = w < words ? bits[w] : 0u;
        const int c = __popc(b);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        int o = out + incl - c;
        while (b) {
          const int bit = __ffs(b) - 1;
          b &= b - 1;
          const int k = w * 32 + bit;
          STC_CHECK(o < cp[row + 1], "SpGEMM row overflows its counted length");
          ck[o] = k;
          cv[o] = acc[k];
          acc[k] = 0.0f;
          ++o;
        }
        if (w < words) bits[w] = 0u;
        out += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncwarp();
  }
}

// ---- element-wise union (op 0) / intersection (op 1) ------------------------------------

// per row: |A_i ∩ B_i| (op 1) or |A_i| + |B_i| - |A_i ∩ B_i| (op 0); cnt[m] = 0
__global__ void ewise_count_kernel(int op, int m, const int* __restrict__ ap, const int* __restrict__ aj,
                                   const int* __restrict__ bp, const int* __restrict__ bj, int* __restrict__ cnt) {
  const int row = blockIdx.x * kWarpsPerCta + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row > m) return;
  int common = 0;
  int a0 = 0, a1 = 0, b0 = 0, b1 = 0;
  if (row < m) {
    a0 = ap[row], a1 = ap[row + 1], b0 = bp[row], b1 = bp[row + 1];
    for (int p = a0 + lane; p < a1; p += 32) {
      const int q = lower_bound(bj, b0, b1, aj[p]);
      common += (q < b1 && bj[q] == aj[p]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) common += __shfl_xor_sync(0xffffffffu, common, o);
  if (lane == 0) cnt[row] = op == 1 ? common : (a1 - a0) + (b1 - b0) - common;
}

__global__ void ewise_fill_kernel(int op, int m, const int* __restrict__ ap, const int* __restrict__ aj,
                                  const float* __restrict__ av, const int* __restrict__ bp,
                                  const int* __restrict__ bj, const float* __restrict__ bv,
                                  const int* __restrict__ cp, int* __restrict__ ck, float* __restrict__ cv) {
  const int row = blockIdx.x * kWarpsPerCta + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= m) return;
  const int a0 = ap[row], a1 = ap[row + 1], b0 = bp[row], b1 = bp[row + 1];
  const int c0 = cp[row];
  const unsigned below = (1u << lane) - 1u;
  // pass over A: position = |A < v| + |B < v| - |common < v| (union) or rank among commons
  int dups = 0;  // common entries before this chunk
  for (int base = a0; base < a1; base += 32) {
    const int p = base + lane;
    int key = 0, q = b1;
    bool found = false;
    if (p < a1) {
      key = aj[p];
      q = lower_bound(bj, b0, b1, key);
      found = q < b1 && bj[q] == key;
    }
    const unsigned fb = __ballot_sync(0xffffffffu, found);
    const int dup_before = dups + __popc(fb & below);
    if (p < a1) {
      if (op == 1) {
        if (found) {
          ck[c0 + dup_before] = key;
          cv[c0 + dup_before] = 0.0f + av[p] * bv[q];
        }
      } else {
        const int o = c0 + (p - a0) + (q - b0) - dup_before;
        ck[o] = key;
        cv[o] = found ? (0.0f + av[p]) + bv[q] : 0.0f + av[p];
      }
    }
    dups += __popc(fb);
  }
  if (op == 1) return;
  // pass over B: entries absent from A
  dups = 0;
  for (int base = b0; base < b1; base += 32) {
    const int p = base + lane;
    int key = 0, q = a1;
    bool found = false;
    if (p < b1) {
      key = bj[p];
      q = lower_bound(aj, a0, a1, key);
      found = q < a1 && aj[q] == key;
    }
    const unsigned fb = __ballot_sync(0xffffffffu, found);
    const int dup_before = dups + __popc(fb & below);
    if (p < b1 && !found) {
      const int o = c0 + (p - b0) + (q - a0) - dup_before;
      ck[o] = key;
      cv[o] = 0.0f + bv[p];
    }
    dups += __popc(fb);
  }
}

inline unsigned grid_rows(long long rows) { return (unsigned)ceil_div(rows, kWarpsPerCta); }
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t scan_ll_bytes(int n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const long long*)nullptr, (long long*)nullptr, n);
  return b;
}
size_t scan_int_bytes(int n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, n);
  return b;
}
size_t sort_bytes(int items, int segs) {
  size_t b = 0;
  cub::DeviceSegmentedSort::StableSortPairs(nullptr, b, (const int*)nullptr, (int*)nullptr, (const float*)nullptr,
                                            (float*)nullptr, items, segs, (const int*)nullptr, (const int*)nullptr);
  return b;
}

// SpGEMM workspace: keys/vals in + out, segment offsets (int32), counts, CUB temp
struct SpgemmWs {
  int *keys_in, *keys_out, *seg, *cnt;
  float *vals_in, *vals_out;
  void* tmp;
  size_t tmp_bytes;
};
size_t spgemm_ws_layout(int m, long long products, void* base, SpgemmWs* w) {
  const size_t P = (size_t)(products > 0 ? products : 1);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align256(off + bytes);
    return at;
  };
  const size_t o_ki = take(P * 4), o_ko = take(P * 4), o_vi = take(P * 4), o_vo = take(P * 4);
  const size_t o_seg = take(((size_t)m + 1) * 4), o_cnt = take(((size_t)m + 1) * 4);
  const size_t tb = std::max(sort_bytes((int)P, m > 0 ? m : 1), scan_int_bytes(m + 1));
  const size_t o_tmp = take(tb);
  if (w) {
    char* b = static_cast<char*>(base);
    w->keys_in = reinterpret_cast<int*>(b + o_ki);
    w->keys_out = reinterpret_cast<int*>(b + o_ko);
    w->vals_in = reinterpret_cast<float*>(b + o_vi);
    w->vals_out = reinterpret_cast<float*>(b + o_vo);
    w->seg = reinterpret_cast<int*>(b + o_seg);
    w->cnt = reinterpret_cast<int*>(b + o_cnt);
    w->tmp = b + o_tmp;
    w->tmp_bytes = tb;
  }
  return off + 256;  // slack: the caller's base need not be 256-byte aligned
}

void* align_base(void* p) {
  return reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
}

}  // namespace
}  // namespace stc

using namespace stc;

extern "C" size_t stc_spgemm_products_temp_bytes(int m) {
  if (m < 0) return 0;
  return align256(((size_t)m + 1) * sizeof(long long)) + scan_ll_bytes(m + 1) + 256;
}

extern "C" int stc_spgemm_products(int m, const int* a_rowptr, const int* a_colidx, const int* b_rowptr,
                                   long long* prod_ptr, void* temp, size_t temp_bytes, void* stream) {
  STC_NVTX("stc_spgemm_products");
  if (m < 0) return fail(STC_EINVAL, "negative extent");
  if (!a_rowptr || !b_rowptr || !prod_ptr) return fail(STC_EINVAL, "null pointer");
  const size_t need = stc_spgemm_products_temp_bytes(m);
  if (!temp || temp_bytes < need) return fail(STC_EWORKSPACE, "temp %zu < %zu", temp_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* b = static_cast<char*>(align_base(temp));
  long long* cnt = reinterpret_cast<long long*>(b);
  void* tmp = b + align256(((size_t)m + 1) * sizeof(long long));
  size_t tb = scan_ll_bytes(m + 1);
  spgemm_count_kernel<<<grid_rows(m + 1), kWarpsPerCta * 32, 0, st>>>(m, a_rowptr, a_colidx, b_rowptr, cnt);
  if (int rc = check_launch("spgemm_count_kernel")) return rc;
  const cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, prod_ptr, m + 1, st);
  if (e != cudaSuccess) return fail(STC_ELAUNCH, "spgemm product scan: %s", cudaGetErrorString(e));
  return check_launch("spgemm_products");
}

namespace {
bool use_dense(int p) { return p <= kDenseMaxCols; }

struct DenseLaunch {
  int warps;
  size_t smem;
  unsigned grid;
};
DenseLaunch dense_launch(int m, int p) {
  DenseLaunch d;
  const size_t per = dense_warp_bytes(p);
  int w = (int)((72u * 1024u) / per);
  d.warps = w < 1 ? 1 : (w > 8 ? 8 : w);
  d.smem = per * d.warps;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spgemm_dense_kernel, d.warps * 32, d.smem);
  const long long want = ceil_div(m, d.warps);
  const long long cap = (long long)sms * (per_sm > 0 ? per_sm : 1);
  d.grid = (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
  return d;
}
int launch_dense(int phase, int m, int p, const int* ap, const int* aj, const float* av, const int* bp,
                 const int* bj, const float* bv, int* cnt, const int* cp, int* ck, float* cv, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(spgemm_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  if (m == 0) return STC_OK;
  const DenseLaunch d = dense_launch(m, p);
  spgemm_dense_kernel<<<d.grid, d.warps * 32, d.smem, st>>>(phase, m, p, ap, aj, av, bp, bj, bv, cnt, cp, ck, cv);
  return check_launch("spgemm_dense_kernel");
}
size_t dense_ws_bytes(int m) { return align256(((size_t)m + 1) * 4) + scan_int_bytes(m + 1) + 256; }
}  // namespace

extern "C" size_t stc_spgemm_workspace_bytes(int m, int p, long long products) {
  if (m < 0 || p < 0 || products < 0) return 0;
  if (use_dense(p)) return dense_ws_bytes(m);
  if (products > INT32_MAX) return 0;
  return spgemm_ws_layout(m, products, nullptr, nullptr);
}

extern "C" int stc_spgemm_symbolic(int m, int p, const int* a_rowptr, const int* a_colidx, const float* a_vals,
                                   const int* b_rowptr, const int* b_colidx, const float* b_vals,
                                   const long long* prod_ptr, long long products, void* ws, size_t ws_bytes,
                                   int* c_rowptr, void* stream) {
  STC_NVTX("stc_spgemm_symbolic");
  if (m < 0 || p < 0 || products < 0) return fail(STC_EINVAL, "negative extent");
  if (!a_rowptr || !b_rowptr || !prod_ptr || !c_rowptr || !ws) return fail(STC_EINVAL, "null pointer");
  const size_t need = stc_spgemm_workspace_bytes(m, p, products);
  if (need == 0) return fail(STC_EUNSUPPORTED, "%lld products exceed the int32 range", products);
  if (ws_bytes < need) return fail(STC_EWORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_dense(p)) {
    char* b = static_cast<char*>(align_base(ws));
    int* cnt = reinterpret_cast<int*>(b);
    void* tmp = b + align256(((size_t)m + 1) * 4);
    cudaMemsetAsync(cnt + m, 0, sizeof(int), st);
    if (int rc = launch_dense(0, m, p, a_rowptr, a_colidx, a_vals, b_rowptr, b_colidx, b_vals, cnt, nullptr,
                              nullptr, nullptr, st))
      return rc;
    size_t tb = scan_int_bytes(m + 1);
    const cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, c_rowptr, m + 1, st);
    if (e != cudaSuccess) return fail(STC_ELAUNCH, "spgemm row scan: %s", cudaGetErrorString(e));
    return check_launch("spgemm_symbolic");
  }
  SpgemmWs w;
  spgemm_ws_layout(m, products, align_base(ws), &w);
  spgemm_expand_kernel<<<grid_rows(m + 1), kWarpsPerCta * 32, 0, st>>>(
      m, a_rowptr, a_colidx, a_vals, b_rowptr, b_colidx, b_vals, prod_ptr, w.keys_in, w.vals_in, w.seg);
  if (int rc = check_launch("spgemm_expand_kernel")) return rc;
  if (products > 0 && m > 0) {
    size_t tb = w.tmp_bytes;
    const cudaError_t e = cub::DeviceSegmentedSort::StableSortPairs(
        w.tmp, tb, w.keys_in, w.keys_out, w.vals_in, w.vals_out, (int)products, m, w.seg, w.seg + 1, st);
    if (e != cudaSuccess) return fail(STC_ELAUNCH, "spgemm segmented sort: %s", cudaGetErrorString(e));
  }
  spgemm_unique_kernel<<<grid_rows(m + 1), kWarpsPerCta * 32, 0, st>>>(m, w.seg, w.keys_out, w.cnt);
  if (int rc = check_launch("spgemm_unique_kernel")) return rc;
  size_t tb = w.tmp_bytes;
  const cudaError_t e = cub::DeviceScan::ExclusiveSum(w.tmp, tb, w.cnt, c_rowptr, m + 1, st);
  if (e != cudaSuccess) return fail(STC_ELAUNCH, "spgemm row scan: %s", cudaGetErrorString(e));
  return check_launch("spgemm_symbolic");
}

extern "C" int stc_spgemm_numeric(int m, int p, const int* a_rowptr, const int* a_colidx, const float* a_vals,
                                  const int* b_rowptr, const int* b_colidx, const float* b_vals, long long products,
                                  void* ws, size_t ws_bytes, const int* c_rowptr, int* c_colidx, float* c_vals,
                                  void* stream) {
  STC_NVTX("stc_spgemm_numeric");
  if (m < 0 || p < 0 || products < 0) return fail(STC_EINVAL, "negative extent");
  if (!ws || !c_rowptr) return fail(STC_EINVAL, "null pointer");
  const size_t need = stc_spgemm_workspace_bytes(m, p, products);
  if (need == 0) return fail(STC_EUNSUPPORTED, "%lld products exceed the int32 range", products);
  if (ws_bytes < need) return fail(STC_EWORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_dense(p))
    return launch_dense(1, m, p, a_rowptr, a_colidx, a_vals, b_rowptr, b_colidx, b_vals, nullptr, c_rowptr,
                        c_colidx, c_vals, st);
  SpgemmWs w;
  spgemm_ws_layout(m, products, align_base(ws), &w);
  spgemm_compress_kernel<<<grid_rows(m), kWarpsPerCta * 32, 0, st>>>(m, w.seg, w.keys_out, w.vals_out, c_rowptr,
                                                                     c_colidx, c_vals);
  return check_launch("spgemm_compress_kernel");
}

extern "C" size_t stc_csr_ewise_temp_bytes(int m) {
  if (m < 0) return 0;
  return align256(((size_t)m + 1) * sizeof(int)) + scan_int_bytes(m + 1) + 256;
}

extern "C" int stc_csr_ewise_symbolic(int op, int m, const int* a_rowptr, const int* a_colidx, const int* b_rowptr,
                                      const int* b_colidx, int* c_rowptr, void* temp, size_t temp_bytes,
                                      void* stream) {
  STC_NVTX("stc_csr_ewise_symbolic");
  if (op != STC_EWISE_UNION && op != STC_EWISE_INTERSECT) return fail(STC_EINVAL, "unknown element-wise op %d", op);
  if (m < 0) return fail(STC_EINVAL, "negative extent");
  if (!a_rowptr || !b_rowptr || !c_rowptr) return fail(STC_EINVAL, "null pointer");
  const size_t need = stc_csr_ewise_temp_bytes(m);
  if (!temp || temp_bytes < need) return fail(STC_EWORKSPACE, "temp %zu < %zu", temp_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* b = static_cast<char*>(align_base(temp));
  int* cnt = reinterpret_cast<int*>(b);
  void* tmp = b + align256(((size_t)m + 1) * sizeof(int));
  size_t tb = scan_int_bytes(m + 1);
  ewise_count_kernel<<<grid_rows(m + 1), kWarpsPerCta * 32, 0, st>>>(op, m, a_rowptr, a_colidx, b_rowptr,
                                                                     b_colidx, cnt);
  if (int rc = check_launch("ewise_count_kernel")) return rc;
  const cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, c_rowptr, m + 1, st);
  if (e != cudaSuccess) return fail(STC_ELAUNCH, "element-wise row scan: %s", cudaGetErrorString(e));
  return check_launch("ewise_symbolic");
}

extern "C" int stc_csr_ewise_f32(int op, int m, const int* a_rowptr, const int* a_colidx, const float* a_vals,
                                 const int* b_rowptr, const int* b_colidx, const float* b_vals, const int* c_rowptr,
                                 int* c_colidx, float* c_vals, void* stream) {
  STC_NVTX("stc_csr_ewise_f32");
  if (op != STC_EWISE_UNION && op != STC_EWISE_INTERSECT) return fail(STC_EINVAL, "unknown element-wise op %d", op);
  if (m < 0) return fail(STC_EINVAL, "negative extent");
  if (!a_rowptr || !b_rowptr || !c_rowptr) return fail(STC_EINVAL, "null pointer");
  if (m == 0) return STC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ewise_fill_kernel<<<grid_rows(m), kWarpsPerCta * 32, 0, st>>>(op, m, a_rowptr, a_colidx, a_vals, b_rowptr,
                                                                b_colidx, b_vals, c_rowptr, c_colidx, c_vals);
  return check_launch("ewise_fill_kernel");
}
