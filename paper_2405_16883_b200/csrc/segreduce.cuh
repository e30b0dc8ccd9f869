// Segmented gather-reduce over a row-compressed index stream (sm_100a).
//
// One kernel family serves every contraction on this path whose output row is
// a weighted sum of gathered dense vectors:
//   CSR SpMM        C[i,:]  = sum_p  val[p] * B[col[p], :]           (K1/K2/K3)
//   COO/DCSR SpMM   same, over the distinct rows of a sorted COO       (K4)
//   PV of attention O[h,i,:] = sum_p P[h,p] * V[h, col[p], :]         (K7 unfused)
//   MTTKRP          M[i,:]  = sum_p (T[p] * B[j[p],:]) * C[k[p],:]     (K8)
// The "gather op" (Op) supplies the per-entry item (indices + weight), how it
// is broadcast inside a sub-warp and how its dense operand is fetched; the
// walk, the carries and the epilogue are shared.
//
// Work decomposition ("merge path"): the row ends rowptr[1..m] and the entry
// positions 0..nnz-1 are merged into one sequence of m+nnz items; every
// sub-warp ("group") owns IPG consecutive items, found by a plan-time binary
// search (merge_partition_kernel). A group writes every row whose end item it
// owns; rows cut by group boundaries leave partial sums ("carries"):
//   * inside a CTA the carries are combined through shared memory;
//   * across CTAs each CTA leaves at most one tail carry and one head partial
//     in a global workspace and a fix-up kernel combines them in position
//     order and applies the epilogue.
// No atomics anywhere, so results are bit-reproducible run to run, and the
// epilogue (ReLU) is applied exactly once per row after its full reduction.
#pragma once

#include "stc_common.cuh"

namespace stc {

// ---------------------------------------------------------------------------
// Gather ops
// ---------------------------------------------------------------------------

template <int VEC>
struct SpmmOp {
  const int* col;     // [nnz]
  const float* val;   // [nnz] (batched: + batch * val_bstride)
  const float* B;     // dense operand, row-major with leading dim ldb
  long long ldb;

  struct Item {
    int c;
    float v;
  };
  struct Pre {
    Frag<VEC> b;
    float v;
  };
  STC_DEVICE Item load(long long p) const { return Item{ld_stream(col + p), ld_stream(val + p)}; }
  template <int SUBW>
  STC_DEVICE Item shfl(const Item& it, int src, unsigned mask) const {
    return Item{__shfl_sync(mask, it.c, src, SUBW), __shfl_sync(mask, it.v, src, SUBW)};
  }
  STC_DEVICE void fetch(const Item& it, int col0, Pre& pre, uint64_t pol) const {
    pre.b.load_gather(B + (long long)it.c * ldb + col0, pol);
    pre.v = it.v;
  }
  STC_DEVICE void accumulate(Frag<VEC>& acc, const Pre& pre) const {
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc.v[e] = fmaf(pre.v, pre.b.v[e], acc.v[e]);
  }
};

template <int VEC>
struct MttkrpOp {
  const int* jc;
  const int* kc;
  const float* val;
  const float* B;
  long long ldb;
  const float* C;
  long long ldcf;

  struct Item {
    int j, k;
    float v;
  };
  struct Pre {
    Frag<VEC> b, c;
    float v;
  };
  STC_DEVICE Item load(long long p) const {
    return Item{ld_stream(jc + p), ld_stream(kc + p), ld_stream(val + p)};
  }
  template <int SUBW>
  STC_DEVICE Item shfl(const Item& it, int src, unsigned mask) const {
    return Item{__shfl_sync(mask, it.j, src, SUBW), __shfl_sync(mask, it.k, src, SUBW),
                __shfl_sync(mask, it.v, src, SUBW)};
  }
  STC_DEVICE void fetch(const Item& it, int col0, Pre& pre, uint64_t pol) const {
    pre.b.load_gather(B + (long long)it.j * ldb + col0, pol);
    pre.c.load_gather(C + (long long)it.k * ldcf + col0, pol);
    pre.v = it.v;
  }
  STC_DEVICE void accumulate(Frag<VEC>& acc, const Pre& pre) const {
    // reference term order: (t * B[j,r]) * C[k,r]  (engine.py:394-402)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc.v[e] = fmaf(pre.v * pre.b.v[e], pre.c.v[e], acc.v[e]);
  }
};

// ---------------------------------------------------------------------------
// Output/epilogue context
// ---------------------------------------------------------------------------

struct SegOut {
  int m;                 // number of rows (segments)
  int k;                 // dense width
  const int* rowptr;     // [m+1]
  float* C;              // output rows, leading dim ldc
  long long ldc;
  const float* D;        // optional addend (same layout as C), may be null
  long long ldd;
};

template <int VEC, int EPI, bool ADD>
STC_DEVICE void write_row(const SegOut& o, int row, int col0, Frag<VEC> acc) {
  float* dst = o.C + (long long)row * o.ldc + col0;
  if constexpr (ADD) {
    Frag<VEC> d;
    d.load_plain(o.D + (long long)row * o.ldd + col0);
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc.v[e] += d.v[e];
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc.v[e] = act<EPI>(acc.v[e]);
  acc.store_stream(dst);
}

// ---------------------------------------------------------------------------
// Plan-time merge-path partition: starts[g] = (row, pos) at diagonal g*IPG.
// ---------------------------------------------------------------------------

__global__ void merge_partition_kernel(int m, long long nnz, const int* __restrict__ rowptr,
                                       int ipg, int n_groups, int2* __restrict__ starts) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > n_groups) return;
  const long long total = (long long)m + nnz;
  long long diag = (long long)g * ipg;
  if (diag > total) diag = total;
  // largest t in [0, m] with t == 0 || rowptr[t] + t <= diag  (monotone in t)
  int lo = 0, hi = m;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)rowptr[mid] + mid <= diag)
      lo = mid;
    else
      hi = mid - 1;
  }
  starts[g] = make_int2(lo, (int)(diag - lo));
}

// ---------------------------------------------------------------------------
// Merge-path segmented reduction
// ---------------------------------------------------------------------------

struct MergeShape {
  const int2* starts;    // [n_groups + 1]
  int n_groups;
  int ipg;               // items per group
  int n_cta;
  float* head_buf;       // [slabs][n_cta][slab_w]
  float* tail_buf;       // [slabs][n_cta][slab_w]
  long long batch_val_stride;   // batched (multi-head) variants: per-z offsets
  long long batch_b_stride;
  long long batch_c_stride;
};

template <int SUBW, int VEC, int EPI, bool ADD, int U, class Op>
__global__ void __launch_bounds__(256) merge_kernel(SegOut o, MergeShape ms, Op op) {
  constexpr int NG = 256 / SUBW;
  constexpr int SW = SUBW * VEC;
  __shared__ __align__(16) float Hs[NG][SW];
  __shared__ __align__(16) float Ts[NG][SW];
  __shared__ int Hrow[NG], Trow[NG];

  const int sub = threadIdx.x / SUBW;
  const int lane = threadIdx.x % SUBW;
  const unsigned mask = subwarp_mask<SUBW>();
  const int cta = blockIdx.x;
  const int slab = blockIdx.y;
  const int z = blockIdx.z;  // batch (head) index; shares the structure
  const int col0 = slab * SW + lane * VEC;
  const bool col_ok = col0 < o.k;
  const uint64_t pol = policy_evict_last();

  // batched views
  if (z) {
    op.val += z * ms.batch_val_stride;
    op.B += z * ms.batch_b_stride;
    o.C += z * ms.batch_c_stride;
    if constexpr (ADD) o.D += z * ms.batch_c_stride;
  }
  const long long zslab = ((long long)z * gridDim.y + slab) * ms.n_cta;

  const int g = min(cta * NG + sub, ms.n_groups);
  const int2 s = ms.starts[g];
  const int2 e = ms.starts[min(g + 1, ms.n_groups)];
  const int row0 = s.x;
  const int row_stop = e.x;   // rows [row0, row_stop) end inside this group
  const int p_end = e.y;

  int row = row0;
  int cur_start = (row < o.m) ? o.rowptr[row] : s.y;
  const bool head_mid = (row < o.m) && (s.y > cur_start);

  int rows_base = row;
  int re_lane = (rows_base + lane < row_stop) ? ld_stream(o.rowptr + rows_base + lane + 1) : INT_MAX;
  int cur_end = __shfl_sync(mask, re_lane, 0, SUBW);

  Frag<VEC> acc;
  acc.zero();
  if (lane == 0) {
    Hrow[sub] = -1;
    Trow[sub] = -1;
  }
  __syncwarp(mask);

  auto flush_and_advance = [&]() {
    if (row == row0 && head_mid) {
      if (col_ok) acc.store_plain(&Hs[sub][lane * VEC]);
      if (lane == 0) Hrow[sub] = row;
    } else if (col_ok) {
      write_row<VEC, EPI, ADD>(o, row, col0, acc);
    }
    acc.zero();
    ++row;
    cur_start = cur_end;
    if (row - rows_base == SUBW) {
      rows_base = row;
      re_lane = (rows_base + lane < row_stop) ? ld_stream(o.rowptr + rows_base + lane + 1) : INT_MAX;
    }
    cur_end = __shfl_sync(mask, re_lane, row - rows_base, SUBW);
  };

  for (int base = s.y; base < p_end; base += SUBW) {
    typename Op::Item it{};
    if (base + lane < p_end) it = op.load(base + lane);
    const int n = min(SUBW, p_end - base);
    for (int q0 = 0; q0 < n; q0 += U) {
      typename Op::Pre pre[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u;
        typename Op::Item iu = op.template shfl<SUBW>(it, q & (SUBW - 1), mask);
        if (q < n && col_ok) op.fetch(iu, col0, pre[u], pol);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u;
        if (q < n) {
          const int pp = base + q;
          while (pp >= cur_end) flush_and_advance();
          op.accumulate(acc, pre[u]);
        }
      }
    }
  }
  while (row < row_stop) flush_and_advance();
  // tail: the row still open at the end of this group's items
  if (row < o.m && p_end > cur_start && row == row_stop) {
    if (col_ok) acc.store_plain(&Ts[sub][lane * VEC]);
    if (lane == 0) Trow[sub] = row;
  }
  __syncthreads();

  // ---- CTA-level combine (position order: tails of earlier groups, then head) ----
  const int2 cs = ms.starts[min(cta * NG, ms.n_groups)];
  const bool cta_head_mid = (cs.x < o.m) && (cs.y > o.rowptr[cs.x]);
  const int hr = Hrow[sub];
  if (hr >= 0) {
    int lo = sub;
    while (lo > 0 && Trow[lo - 1] == hr) --lo;
    Frag<VEC> sum;
    sum.zero();
    if (col_ok) {
      for (int t = lo; t < sub; ++t) {
        Frag<VEC> part;
        part.load_plain(&Ts[t][lane * VEC]);
#pragma unroll
        for (int x = 0; x < VEC; ++x) sum.v[x] += part.v[x];
      }
      Frag<VEC> h;
      h.load_plain(&Hs[sub][lane * VEC]);
#pragma unroll
      for (int x = 0; x < VEC; ++x) sum.v[x] += h.v[x];
      if (lo == 0 && cta_head_mid && hr == cs.x) {
        sum.store_plain(ms.head_buf + (zslab + cta) * SW + lane * VEC);  // needs earlier CTAs
      } else {
        write_row<VEC, EPI, ADD>(o, hr, col0, sum);
      }
    }
  }
  if (sub == NG - 1 && Trow[sub] >= 0) {
    const int tr = Trow[sub];
    int lo = sub;
    while (lo > 0 && Trow[lo - 1] == tr && Hrow[lo] < 0) --lo;
    if (col_ok) {
      Frag<VEC> sum;
      sum.zero();
      for (int t = lo; t <= sub; ++t) {
        Frag<VEC> part;
        part.load_plain(&Ts[t][lane * VEC]);
#pragma unroll
        for (int x = 0; x < VEC; ++x) sum.v[x] += part.v[x];
      }
      sum.store_plain(ms.tail_buf + (zslab + cta) * SW + lane * VEC);
    }
  }
}

// Fix-up of rows cut by CTA boundaries: one sub-warp per boundary c >= 1 whose
// CTA finishes a row that began in an earlier CTA. Sums, in position order,
// the tail carries of CTAs c_first..c-1 and CTA c's head partial.
template <int SUBW, int VEC, int EPI, bool ADD>
__global__ void __launch_bounds__(256) merge_fixup_kernel(SegOut o, MergeShape ms) {
  constexpr int NG = 256 / SUBW;
  constexpr int SW = SUBW * VEC;
  const int lane = threadIdx.x % SUBW;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) / SUBW + 1;
  const int slab = blockIdx.y;
  const int z = blockIdx.z;
  if (c >= ms.n_cta) return;
  const int col0 = slab * SW + lane * VEC;
  if (col0 >= o.k) return;
  if (z) {
    o.C += z * ms.batch_c_stride;
    if constexpr (ADD) o.D += z * ms.batch_c_stride;
  }
  const long long zslab = ((long long)z * gridDim.y + slab) * ms.n_cta;

  const int2 cs = ms.starts[min(c * NG, ms.n_groups)];
  const int r = cs.x;
  if (r >= o.m) return;
  const int rstart = o.rowptr[r];
  if (cs.y <= rstart) return;  // boundary not inside row r
  if (c + 1 < ms.n_cta && ms.starts[min((c + 1) * NG, ms.n_groups)].x == r) return;  // not finished here
  const long long ci = (long long)NG * ms.ipg;
  const int c_first = (int)(((long long)rstart + r) / ci);

  Frag<VEC> sum;
  sum.zero();
  int t = c_first;
  for (; t + 4 <= c; t += 4) {
    Frag<VEC> p0, p1, p2, p3;
    p0.load_plain(ms.tail_buf + (zslab + t) * SW + lane * VEC);
    p1.load_plain(ms.tail_buf + (zslab + t + 1) * SW + lane * VEC);
    p2.load_plain(ms.tail_buf + (zslab + t + 2) * SW + lane * VEC);
    p3.load_plain(ms.tail_buf + (zslab + t + 3) * SW + lane * VEC);
#pragma unroll
    for (int x = 0; x < VEC; ++x) sum.v[x] = (((sum.v[x] + p0.v[x]) + p1.v[x]) + p2.v[x]) + p3.v[x];
  }
  for (; t < c; ++t) {
    Frag<VEC> p;
    p.load_plain(ms.tail_buf + (zslab + t) * SW + lane * VEC);
#pragma unroll
    for (int x = 0; x < VEC; ++x) sum.v[x] += p.v[x];
  }
  Frag<VEC> h;
  h.load_plain(ms.head_buf + (zslab + c) * SW + lane * VEC);
#pragma unroll
  for (int x = 0; x < VEC; ++x) sum.v[x] += h.v[x];
  write_row<VEC, EPI, ADD>(o, r, col0, sum);
}

// ---------------------------------------------------------------------------
// Row-split: one sub-warp per row (uniform, short rows; no carries)
// ---------------------------------------------------------------------------

template <int SUBW, int VEC, int EPI, bool ADD, int U, class Op>
__global__ void __launch_bounds__(256) row_kernel(SegOut o, MergeShape ms, Op op) {
  constexpr int SW = SUBW * VEC;
  const int lane = threadIdx.x % SUBW;
  const unsigned mask = subwarp_mask<SUBW>();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / SUBW;
  const int slab = blockIdx.y;
  const int z = blockIdx.z;
  if (row >= o.m) return;
  const int col0 = slab * SW + lane * VEC;
  const bool col_ok = col0 < o.k;
  const uint64_t pol = policy_evict_last();
  if (z) {
    op.val += z * ms.batch_val_stride;
    op.B += z * ms.batch_b_stride;
    o.C += z * ms.batch_c_stride;
    if constexpr (ADD) o.D += z * ms.batch_c_stride;
  }
  const int start = o.rowptr[row];
  const int end = o.rowptr[row + 1];
  Frag<VEC> acc;
  acc.zero();
  for (int base = start; base < end; base += SUBW) {
    typename Op::Item it{};
    if (base + lane < end) it = op.load(base + lane);
    const int n = min(SUBW, end - base);
    for (int q0 = 0; q0 < n; q0 += U) {
      typename Op::Pre pre[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        typename Op::Item iu = op.template shfl<SUBW>(it, (q0 + u) & (SUBW - 1), mask);
        if (q0 + u < n && col_ok) op.fetch(iu, col0, pre[u], pol);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u < n) op.accumulate(acc, pre[u]);
    }
  }
  if (col_ok) write_row<VEC, EPI, ADD>(o, row, col0, acc);
}

}  // namespace stc
