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
//     in a global workspace; the last CTA to publish a carry for a row (an
//     arrival counter per row) combines them in position order and applies the
//     epilogue — no second launch.
// No atomic accumulation: the only atomics are arrival counters, every sum runs
// in a fixed order, so results are bit-reproducible run to run, and the
// epilogue (ReLU) is applied exactly once per row after its full reduction.
#pragma once

#include "stc_common.cuh"

#ifndef STC_SPMM_LANE_OFF
#define STC_SPMM_LANE_OFF 2
#endif

namespace stc {

#ifdef STC_DBG_TIMING
// Diagnostic build only (tools/merge_balance_probe.py): per-group globaltimer stamps.
__device__ unsigned long long g_dbg[1 << 16][4];
STC_DEVICE unsigned long long dbg_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// ---------------------------------------------------------------------------
// Gather ops
// ---------------------------------------------------------------------------

// Items are staged in a "prepared" form: dense-operand row offsets are
// pre-multiplied by the leading dimension (32-bit element offsets; dense
// operands of 2^32 elements or more take the *WideOp forms below), so a gather
// is one IMAD.WIDE + one LDG.128. `shift(col0)` moves the dense pointers to the
// lane's first column once per kernel.
template <int VEC>
struct SpmmOp {
  const int* col;     // [nnz]
  const float* val;   // [nnz] (batched: + batch * val_bstride)
  const float* B;     // dense operand, row-major with leading dim ldb
  long long ldb;
  unsigned lane_off = 0;  // this lane's first column (added in 32-bit)
  unsigned long long limit = ~0ull;  // elements of B (checked build: every gather stays inside)

  static constexpr int kRing = 8;           // gathers in flight per group
  static constexpr bool kHoistItem = true;  // next fetch's item read one step ahead
  static constexpr int kMinBlocks = 4;      // resident CTAs per SM (register budget)
  static constexpr int kStageUnroll = 8;    // item loads per lane in flight while staging
  // staged items per CTA; the rest of SMEM stays L1, which the in-flight gathers need
  // (36 KB: 129 us on cfg2 against 100 us at 32 KB)
  static constexpr int kStageBytes = 32768;
  struct Item {
    unsigned off;
    float v;
  };
  // The weight is re-read from the staged item at accumulate time (LDS) so the
  // ring only holds the gathered vectors.
  struct Pre {
    Frag<VEC> b;
  };
  struct State {};
  STC_DEVICE Item load(long long p, bool /*first*/) const {
    return Item{(unsigned)((long long)ld_stream(col + p) * ldb), ld_stream(val + p)};
  }
  STC_DEVICE static Item dummy() { return Item{0u, 0.f}; }
  template <int SUBW>
  STC_DEVICE Item shfl(const Item& it, int src, unsigned mask) const {
    return Item{__shfl_sync(mask, it.off, src, SUBW), __shfl_sync(mask, it.v, src, SUBW)};
  }
#if STC_SPMM_LANE_OFF == 1
  // keep the lane's column offset in a register: without this it is recomputed for every gather
  // from %ctaid.y (an S2R and two integer ops on the address path of each entry)
  STC_DEVICE void shift(int col0) {
    lane_off = (unsigned)col0;
    asm volatile("" : "+r"(lane_off));
  }
#elif STC_SPMM_LANE_OFF == 2
  // ... or fold it into the operand base, held as an opaque 64-bit register
  STC_DEVICE void shift(int col0) {
    B += col0;
    limit -= (unsigned)col0 <= limit ? (unsigned)col0 : limit;
    asm volatile("" : "+l"(B));
    lane_off = 0;
  }
#else
  STC_DEVICE void shift(int col0) { lane_off = (unsigned)col0; }
#endif
  STC_DEVICE void fetch(const Item& it, Pre& pre) const {
    STC_CHECK((unsigned long long)(it.off + lane_off) + VEC <= limit, "SpMM gather outside B");
    pre.b.load_gather(B + (it.off + lane_off));
  }
  STC_DEVICE void accumulate(Frag<VEC>& acc, State&, const Pre& pre, const Item& it) const {
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc.v[e] = fmaf(it.v, pre.b.v[e], acc.v[e]);
  }
  STC_DEVICE static void init(State&) {}
  STC_DEVICE static void finish(Frag<VEC>&, State&) {}
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
  unsigned lane_off = 0;
  unsigned long long limitb = ~0ull, limitc = ~0ull;  // elements of B / C (checked build)

  // Entries are sorted by (i, j), so consecutive entries of one (i, j) fiber share
  // B[j,:]: it is gathered once per fiber (flag = first entry of a fiber) and held in
  // registers, and every entry adds its term (T * B[j,:]) * C[k,:] in entry order (the
  // reference's term order, engine.py:577-644) -- 3 ops per element. (The fiber-sum form
  // B[j,:] * sum_k T C[k,:] costs 5 ops per element with its open/close selects: cfg5
  // 135 -> 131 us; its loop alone 68 -> 53 us in a diagnostic build without gathers.)
#ifndef STC_MTTKRP_RING
#define STC_MTTKRP_RING 4
#endif
#ifndef STC_MTTKRP_SU
#define STC_MTTKRP_SU 2
#endif
  static constexpr int kRing = VEC == 4 ? STC_MTTKRP_RING : 8;
  static constexpr bool kHoistItem = false;
#ifndef STC_MTTKRP_MINB
#define STC_MTTKRP_MINB 3
#endif

#ifndef STC_MTTKRP_STAGE
#define STC_MTTKRP_STAGE 40960
#endif
  static constexpr int kMinBlocks = STC_MTTKRP_MINB;
  static constexpr int kStageUnroll = STC_MTTKRP_SU;  // item loads per lane in flight while staging (1: 130.6 us, 2: 129.1, 4: 129.0)
  static constexpr int kStageBytes = STC_MTTKRP_STAGE;  // 80-item windows (3 CTAs x 58 KB; 96-item windows: +15 % time)
  struct __align__(16) Item {
    unsigned offb, offc;
    float v;
    int flag;  // 1: first entry of a fiber (j differs from the previous entry's)
  };
  struct Pre {
    Frag<VEC> b, c;
  };
  struct State {
    Frag<VEC> b;  // the current fiber's B[j,:]
  };
  STC_DEVICE Item load(long long p, bool first) const {
    const int j = ld_stream(jc + p);
    const bool start = first || p == 0 || ld_stream(jc + p - 1) != j;
    return Item{(unsigned)((long long)j * ldb), (unsigned)((long long)ld_stream(kc + p) * ldcf), ld_stream(val + p),
                start ? 1 : 0};
  }
  STC_DEVICE static Item dummy() { return Item{0u, 0u, 0.f, 0}; }
  template <int SUBW>
  STC_DEVICE Item shfl(const Item& it, int src, unsigned mask) const {
    return Item{__shfl_sync(mask, it.offb, src, SUBW), __shfl_sync(mask, it.offc, src, SUBW),
                __shfl_sync(mask, it.v, src, SUBW), __shfl_sync(mask, it.flag, src, SUBW)};
  }
  STC_DEVICE void shift(int col0) { lane_off = (unsigned)col0; }
  STC_DEVICE void fetch(const Item& it, Pre& pre) const {
    STC_CHECK(!it.flag || (unsigned long long)(it.offb + lane_off) + VEC <= limitb, "MTTKRP gather outside B");
    STC_CHECK((unsigned long long)(it.offc + lane_off) + VEC <= limitc, "MTTKRP gather outside C");
#ifdef STC_DIAG_NOGATHER  // diagnostic builds only (tools/build_variant.sh): time without the gathers
    pre.b.v[0] = pre.c.v[0] = __int_as_float(it.offb ^ it.offc);
#else
    if (it.flag) pre.b.load_gather(B + (it.offb + lane_off));
    pre.c.load_gather(C + (it.offc + lane_off));
#endif
  }
  STC_DEVICE static void init(State& st) { st.b.zero(); }
  STC_DEVICE void accumulate(Frag<VEC>& acc, State& st, const Pre& pre, const Item& it) const {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      st.b.v[e] = it.flag ? pre.b.v[e] : st.b.v[e];
      acc.v[e] = fmaf(it.v * st.b.v[e], pre.c.v[e], acc.v[e]);
    }
  }
  STC_DEVICE static void finish(Frag<VEC>&, State&) {}

};

// 64-bit gathers for dense operands of 2^32 elements or more (e.g. 40 M-node
// graphs x 128 features, 20 GB): the item keeps the row index and the address is
// formed in 64 bits at fetch time (one more IMAD per gather than the prepared
// 32-bit offset). Same walk, carries and summation order as SpmmOp / MttkrpOp.
template <int VEC>
struct SpmmWideOp : SpmmOp<VEC> {
  using Item = typename SpmmOp<VEC>::Item;
  using Pre = typename SpmmOp<VEC>::Pre;
  STC_DEVICE Item load(long long p, bool /*first*/) const {
    return Item{(unsigned)ld_stream(this->col + p), ld_stream(this->val + p)};
  }
  STC_DEVICE void fetch(const Item& it, Pre& pre) const {
    pre.b.load_gather(this->B + (long long)it.off * this->ldb + this->lane_off);
  }
};

template <int VEC>
struct MttkrpWideOp : MttkrpOp<VEC> {
  using Item = typename MttkrpOp<VEC>::Item;
  using Pre = typename MttkrpOp<VEC>::Pre;
  STC_DEVICE Item load(long long p, bool first) const {
    const int j = ld_stream(this->jc + p);
    const bool start = first || p == 0 || ld_stream(this->jc + p - 1) != j;
    return Item{(unsigned)j, (unsigned)ld_stream(this->kc + p), ld_stream(this->val + p), start ? 1 : 0};
  }
  STC_DEVICE void fetch(const Item& it, Pre& pre) const {
    if (it.flag) pre.b.load_gather(this->B + (long long)it.offb * this->ldb + this->lane_off);
    pre.c.load_gather(this->C + (long long)it.offc * this->ldcf + this->lane_off);
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
  STC_CHECK(row >= 0 && row < o.m && col0 + VEC <= o.k, "output row outside C");
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
//
// Item costs: an entry weighs kEntryCost, a row end kRowCost. Entry q of row r
// starts at kEntryCost*q + kRowCost*r, the end of row r at
// kEntryCost*rowptr[r+1] + kRowCost*r; a group owns the items starting in its range.
// A row end costs about two gathers (per-group globaltimer stamps on cfg2: 0.147 us
// per entry + 0.282 us per row end, tools/merge_balance_probe.py), so kRowCost = 2:
// with unit weights groups of many short rows finish last. Together with the
// plan-time interleaving of long rows (ops.interleave_long_rows: every group inside
// a hub row then sees the same mix of hot and cold columns) the groups' finish
// times tighten from 66-100 us to 79-89 us and the cfg2 layer from 100.4 to 94.2 us
// (tools/interleave_probe.py; weights 1.5 / 1.75 / 2.5 / 3 measured 98.3 / 96.3 /
// 98.3 / 98.3 us).
// ---------------------------------------------------------------------------

#ifndef STC_ENTRY_COST
#define STC_ENTRY_COST 1
#endif
#ifndef STC_ROW_COST
#define STC_ROW_COST 2
#endif
constexpr int kEntryCost = STC_ENTRY_COST;
constexpr int kRowCost = STC_ROW_COST;

__host__ __device__ inline long long merge_total_items(int m, long long nnz) {
  return (long long)kRowCost * m + (long long)kEntryCost * nnz;
}

static __global__ void merge_partition_kernel(int m, long long nnz, const int* __restrict__ rowptr,
                                              int ipg, int n_groups, int2* __restrict__ starts) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > n_groups) return;
  const long long total = merge_total_items(m, nnz);
  long long diag = (long long)g * ipg;
  if (diag > total) diag = total;
  // t = row ends starting before diag: largest t in [0, m] with t == 0 ||
  // kEntryCost*rowptr[t] + kRowCost*(t-1) < diag (monotone in t)
  int lo = 0, hi = m;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)kEntryCost * rowptr[mid] + (long long)kRowCost * (mid - 1) < diag)
      lo = mid;
    else
      hi = mid - 1;
  }
  // entries q of row t starting before diag: kEntryCost*q + kRowCost*t < diag
  const long long x = diag - (long long)kRowCost * lo;
  long long p = x <= 0 ? 0 : (x + kEntryCost - 1) / kEntryCost;
  const long long p_lo = rowptr[lo];
  const long long p_hi = lo < m ? (long long)rowptr[lo + 1] : nnz;
  p = p < p_lo ? p_lo : (p > p_hi ? p_hi : p);
  starts[g] = make_int2(lo, (int)p);
}

// ---------------------------------------------------------------------------
// Merge-path segmented reduction
// ---------------------------------------------------------------------------

struct MergeShape {
  const int2* starts;    // [n_groups + 1]
  int n_groups;
  int ipg;               // items per group
  int n_cta;
  float* head_buf;       // [batch][slabs][n_cta][slab_w]
  float* tail_buf;       // [batch][slabs][n_cta][slab_w]
  int* counters;         // [batch][slabs][n_cta] arrival counters, zero between launches
  long long batch_val_stride;   // batched (multi-head) variants: per-z offsets
  long long batch_b_stride;
  long long batch_c_stride;
};

// Staging budget per CTA: 32 KB of items split over its NG groups (CAP items
// per group), plus CAP/4 row ends per group (restaged when a group owns more rows).
template <int SUBW, class Op>
__host__ __device__ constexpr int merge_stage_cap() {
  return Op::kStageBytes / ((256 / SUBW) * (int)sizeof(typename Op::Item));
}
template <int SUBW, class Op>
__host__ __device__ constexpr int merge_rows_cap() {
  return merge_stage_cap<SUBW, Op>() / 4 < 32 ? 32 : merge_stage_cap<SUBW, Op>() / 4;
}
constexpr int kStagePad = 8;  // dummy items after each window: branch-free prefetch

// Per-group strides of the staged windows, skewed so that the groups of one warp
// (which read different items in the same instruction) start in different banks.
__host__ __device__ constexpr int bank_skewed(int n, int elem_bytes) {
  const int per_line = 128 / elem_bytes;  // elements per 128-byte bank line
  return n + ((1 - n % per_line) + per_line) % per_line;
}
template <int SUBW, class Op>
__host__ __device__ constexpr int merge_item_stride() {
  return bank_skewed(merge_stage_cap<SUBW, Op>() + kStagePad, (int)sizeof(typename Op::Item));
}
template <int SUBW, class Op>
__host__ __device__ constexpr int merge_rend_stride() {
  return bank_skewed(merge_rows_cap<SUBW, Op>(), (int)sizeof(int));
}

// Dynamic shared memory of merge_kernel (independent of ipg: groups stream
// their items through a fixed-size window).
template <int SUBW, int VEC, class Op>
__host__ __device__ constexpr size_t merge_smem_bytes() {
  constexpr int NG = 256 / SUBW;
  constexpr int SW = SUBW * VEC;
  return (size_t)2 * NG * SW * sizeof(float)               // head / tail partials
         + (size_t)2 * NG * sizeof(int)                     // their row ids
         + (size_t)NG * merge_item_stride<SUBW, Op>() * sizeof(typename Op::Item)  // staged items window
         + (size_t)NG * merge_rend_stride<SUBW, Op>() * sizeof(int);                // staged row-end window
}

// CTA-level combine of the groups' head / tail partials (position order: tails of earlier
// groups, then the head) and the cross-CTA carry fix-up by the last arriving CTA. Shared by
// the staged and the register-pipelined merge kernels; called after a __syncthreads().
template <int SUBW, int VEC, int EPI, bool ADD>
STC_DEVICE void merge_combine(const SegOut& o, const MergeShape& ms, int sub, int lane, bool col_ok, int col0,
                              long long zslab, float* Hs, float* Ts, int* Hrow, int* Trow) {
  constexpr int NG = 256 / SUBW;
  constexpr int SW = SUBW * VEC;
  const int cta = blockIdx.x;
  // ---- CTA-level combine (position order: tails of earlier groups, then head) ----
  __shared__ int head_row_s, tail_row_s;
  if (threadIdx.x == 0) head_row_s = tail_row_s = -1;
  const int2 cs = ms.starts[min(cta * NG, ms.n_groups)];
  const bool cta_head_mid = (cs.x < o.m) && (cs.y > o.rowptr[cs.x]);
  __syncthreads();
  const int hr = Hrow[sub];
  if (hr >= 0) {
    int lo = sub;
    while (lo > 0 && Trow[lo - 1] == hr) --lo;
    const bool to_head = lo == 0 && cta_head_mid && hr == cs.x;  // began in an earlier CTA
    if (col_ok) {
      Frag<VEC> sum;
      sum.zero();
      for (int t = lo; t < sub; ++t) {
        Frag<VEC> part;
        part.load_plain(&Ts[t * SW + lane * VEC]);
#pragma unroll
        for (int x = 0; x < VEC; ++x) sum.v[x] += part.v[x];
      }
      Frag<VEC> h;
      h.load_plain(&Hs[sub * SW + lane * VEC]);
#pragma unroll
      for (int x = 0; x < VEC; ++x) sum.v[x] += h.v[x];
      if (to_head) {
        sum.store_plain(ms.head_buf + (zslab + cta) * SW + lane * VEC);
      } else {
        write_row<VEC, EPI, ADD>(o, hr, col0, sum);
      }
    }
    if (to_head && lane == 0) head_row_s = hr;
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
        part.load_plain(&Ts[t * SW + lane * VEC]);
#pragma unroll
        for (int x = 0; x < VEC; ++x) sum.v[x] += part.v[x];
      }
      sum.store_plain(ms.tail_buf + (zslab + cta) * SW + lane * VEC);
    }
    if (lane == 0) tail_row_s = tr;
  }

  // ---- rows cut by CTA boundaries: the last CTA to publish its carry for a row
  // sums every carry of that row in position order and writes it (no extra launch).
  // Carries are published with a gpu-scope fence before the arrival counter.
  __threadfence();
  __syncthreads();
  __shared__ int fix_row[2], fix_first[2], fix_last[2], n_fix;
  if (threadIdx.x == 0) {
    n_fix = 0;
    const long long ci = (long long)NG * ms.ipg;
    auto arrive = [&](int r, int c_last) {
      const int c_first = (int)(((long long)kEntryCost * o.rowptr[r] + (long long)kRowCost * r) / ci);
      const int need = c_last - c_first + 1;
      STC_CHECK(c_first >= 0 && c_first <= c_last && c_last < ms.n_cta, "carry chain outside the grid");
      int* ctr = ms.counters + zslab + c_last;
      if (atomicAdd(ctr, 1) + 1 == need) {
        *ctr = 0;  // every participant has arrived: reset for the next launch
        fix_row[n_fix] = r;
        fix_first[n_fix] = c_first;
        fix_last[n_fix] = c_last;
        ++n_fix;
      }
    };
    if (head_row_s >= 0) arrive(head_row_s, cta);
    if (tail_row_s >= 0) {
      const int r = tail_row_s;
      arrive(r, (int)(((long long)kEntryCost * o.rowptr[r + 1] + (long long)kRowCost * r) / ci));
    }
    __threadfence();
  }
  __syncthreads();
  for (int f = 0; f < n_fix; ++f) {
    const int r = fix_row[f], c_first = fix_first[f], c_last = fix_last[f];
    // sub-warp s sums tails c_first+s, c_first+s+NG, ... (ascending); sub-warp 0 then
    // adds the NG partials in order and the head: fixed order, spread over the CTA.
    Frag<VEC> sum;
    sum.zero();
    if (col_ok) {
      for (int t = c_first + sub; t < c_last; t += NG) {
        Frag<VEC> p;
        p.load_l2(ms.tail_buf + (zslab + t) * SW + lane * VEC);
#pragma unroll
        for (int x = 0; x < VEC; ++x) sum.v[x] += p.v[x];
      }
      sum.store_plain(&Ts[sub * SW + lane * VEC]);
    }
    __syncthreads();
    if (sub == 0 && col_ok) {
      Frag<VEC> tot;
      tot.zero();
      const int used = min(NG, c_last - c_first);
      for (int s2 = 0; s2 < used; ++s2) {
        Frag<VEC> p;
        p.load_plain(&Ts[s2 * SW + lane * VEC]);
#pragma unroll
        for (int x = 0; x < VEC; ++x) tot.v[x] += p.v[x];
      }
      Frag<VEC> h;
      h.load_l2(ms.head_buf + (zslab + c_last) * SW + lane * VEC);
#pragma unroll
      for (int x = 0; x < VEC; ++x) tot.v[x] += h.v[x];
      write_row<VEC, EPI, ADD>(o, r, col0, tot);
    }
    __syncthreads();
  }
}

// One sub-warp ("group") per `ipg` merge items. The group stages a window of
// its entries' items and of its rows' end offsets in shared memory (coalesced,
// one round trip per window), then streams the gathers through a U-deep
// register ring: the gather for entry q+U is issued while entry q is
// accumulated, independent of row boundaries, so U loads stay in flight
// across rows.
template <int SUBW, int VEC, int EPI, bool ADD, int U, bool FULL, class Op>
__global__ void __launch_bounds__(256, Op::kMinBlocks) merge_kernel(SegOut o, MergeShape ms, Op op) {
  static_assert(U <= kStagePad, "ring deeper than the staging pad");
  using Item = typename Op::Item;
  constexpr int NG = 256 / SUBW;
  constexpr int SW = SUBW * VEC;
  constexpr int CAP = merge_stage_cap<SUBW, Op>();
  constexpr int CAPR = merge_rows_cap<SUBW, Op>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* Hs = reinterpret_cast<float*>(smem_raw);                       // [NG][SW]
  float* Ts = Hs + NG * SW;                                             // [NG][SW]
  int* Hrow = reinterpret_cast<int*>(Ts + NG * SW);                     // [NG]
  int* Trow = Hrow + NG;                                                // [NG]
  Item* items_all = reinterpret_cast<Item*>(Trow + NG);                 // [NG][CAP]
  constexpr int IST = merge_item_stride<SUBW, Op>();
  constexpr int RST = merge_rend_stride<SUBW, Op>();
  int* rend_all = reinterpret_cast<int*>(items_all + NG * IST);         // [NG][RST]

  const int sub = threadIdx.x / SUBW;
  const int lane = threadIdx.x % SUBW;
  const unsigned mask = subwarp_mask<SUBW>();
  const int cta = blockIdx.x;
  const int slab = blockIdx.y;
  const int z = blockIdx.z;
  const int col0 = slab * SW + lane * VEC;
  const bool col_ok = FULL || col0 < o.k;
  Item* items = items_all + sub * IST;
  int* rend = rend_all + sub * RST;

  if (z) {
    op.val += z * ms.batch_val_stride;
    op.B += z * ms.batch_b_stride;
    o.C += z * ms.batch_c_stride;
    if constexpr (ADD) o.D += z * ms.batch_c_stride;
  }
  const long long zslab = ((long long)z * gridDim.y + slab) * ms.n_cta;
  op.shift(col0);

  const int g = min(cta * NG + sub, ms.n_groups);
  const int2 s = ms.starts[g];
  const int2 e = ms.starts[min(g + 1, ms.n_groups)];
  const int row0 = s.x;
  const int n_rows = e.x - s.x;   // rows whose end item this group owns
  const int n_nnz = e.y - s.y;    // entries this group accumulates
  STC_CHECK(n_rows >= 0 && n_nnz >= 0 && e.x <= o.m && n_nnz <= ms.ipg && n_rows <= ms.ipg,
            "merge partition: group range");
#ifdef STC_DBG_TIMING
  const unsigned long long t_start = dbg_timer();
#endif

  // row ends of rows [row0 + rb, row0 + rb + CAPR), relative to s.y
  int rb = 0;
  auto stage_rows = [&](int base) {
    __syncwarp(mask);
    for (int t = lane; t < CAPR && base + t < n_rows; t += SUBW) {
      rend[t] = ld_stream(o.rowptr + row0 + base + 1 + t) - s.y;
      STC_CHECK(rend[t] >= 0 && rend[t] <= n_nnz, "row end outside the group's entries");
    }
    __syncwarp(mask);
  };
  stage_rows(0);
  int first_start = 0;
  if (lane == 0) {
    first_start = (row0 < o.m) ? o.rowptr[row0] : s.y;
    Hrow[sub] = -1;
    Trow[sub] = -1;
  }
  first_start = __shfl_sync(mask, first_start, 0, SUBW);
  const bool head_mid = (row0 < o.m) && (s.y > first_start);

  int r = 0;                                        // current row = row0 + r
  int cur_end = n_rows > 0 ? rend[0] : INT_MAX;      // relative end of the current row
  int cur_start = first_start - s.y;                 // relative start (may be negative)
  Frag<VEC> acc;
  acc.zero();
  typename Op::State fst;
  Op::init(fst);

  auto flush = [&]() {
    Op::finish(acc, fst);
    const int row = row0 + r;
    if (r == 0 && head_mid) {
      if (col_ok) acc.store_plain(&Hs[sub * SW + lane * VEC]);
      if (lane == 0) Hrow[sub] = row;
    } else if (col_ok) {
      write_row<VEC, EPI, ADD>(o, row, col0, acc);
    }
    acc.zero();
    ++r;
    cur_start = cur_end;
    if (r - rb == CAPR) {
      rb = r;
      stage_rows(rb);
    }
    cur_end = r < n_rows ? rend[r - rb] : INT_MAX;
  };

  typename Op::Pre ring[U];
  for (int w0 = 0; w0 < n_nnz; w0 += CAP) {
    const int wn = min(CAP, n_nnz - w0);
    STC_CHECK(wn + kStagePad <= IST, "staging window overflows its stride");
    __syncwarp(mask);
    // SU loads per lane in flight before their SMEM stores (one latency per SU * SUBW items)
    constexpr int SU = Op::kStageUnroll;
#ifdef STC_DIAG_STAGE_ONCE  // diagnostic builds only: stage the first window and reuse it (wrong sums)
    if (w0 == 0)
#endif
    for (int t0 = 0; t0 < wn + kStagePad; t0 += SU * SUBW) {
      Item tmp[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int t = t0 + u * SUBW + lane;
        tmp[u] = t < wn ? op.load(s.y + w0 + t, w0 + t == 0) : Op::dummy();
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int t = t0 + u * SUBW + lane;
        if (t < wn + kStagePad) items[t] = tmp[u];
      }
    }
    __syncwarp(mask);
    int end_w = cur_end - w0;  // current row's end, relative to the window
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (col_ok) op.fetch(items[u], ring[u]);
    int q0 = 0;
    // the item of the next fetch is read from shared memory one step ahead, so the
    // gather's address does not wait on that LDS (the window's pad covers the overrun)
    // (SpMM only: MTTKRP's 16-byte items would spill at its register budget)
    Item nf = items[U];
    for (; q0 + U <= wn; q0 += U) {  // full ring turns: no bounds predicates
#pragma unroll
      for (int u = 0; u < U; ++u) {
        while (q0 + u >= end_w) {
          flush();
          end_w = cur_end - w0;
        }
        if constexpr (Op::kHoistItem) {
          const Item cur = nf;
          nf = items[q0 + u + 1 + U];
          op.accumulate(acc, fst, ring[u], items[q0 + u]);
          if (col_ok) op.fetch(cur, ring[u]);
        } else {
          op.accumulate(acc, fst, ring[u], items[q0 + u]);
          if (col_ok) op.fetch(items[q0 + u + U], ring[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {  // remainder of the window
      if (q0 + u < wn) {
        while (q0 + u >= end_w) {
          flush();
          end_w = cur_end - w0;
        }
        op.accumulate(acc, fst, ring[u], items[q0 + u]);
      }
    }
  }
  while (r < n_rows) flush();
  Op::finish(acc, fst);
  if (row0 + r < o.m && n_nnz > cur_start && r == n_rows) {
    if (col_ok) acc.store_plain(&Ts[sub * SW + lane * VEC]);
    if (lane == 0) Trow[sub] = row0 + r;
  }
#ifdef STC_DBG_TIMING
  if (lane == 0 && g < (1 << 16) && blockIdx.y == 0 && blockIdx.z == 0) {
    g_dbg[g][0] = t_start;
    g_dbg[g][1] = dbg_timer();
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_dbg[g][2] = (unsigned long long)n_rows | ((unsigned long long)smid << 32);
    g_dbg[g][3] = ((unsigned long long)n_nnz << 32) | (unsigned)(threadIdx.x / 32 + (blockIdx.x << 8));
  }
#endif
  __syncthreads();

  merge_combine<SUBW, VEC, EPI, ADD>(o, ms, sub, lane, col_ok, col0, zslab, Hs, Ts, Hrow, Trow);
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
  if (z) {
    op.val += z * ms.batch_val_stride;
    op.B += z * ms.batch_b_stride;
    o.C += z * ms.batch_c_stride;
    if constexpr (ADD) o.D += z * ms.batch_c_stride;
  }
  op.shift(col0);
  const int start = o.rowptr[row];
  const int end = o.rowptr[row + 1];
  Frag<VEC> acc;
  acc.zero();
  typename Op::State fst;
  Op::init(fst);
  typename Op::Item nxt{};
  if (start + lane < end) nxt = op.load(start + lane, lane == 0);
  for (int base = start; base < end; base += SUBW) {
    const typename Op::Item it = nxt;  // the next SUBW entries load while these are gathered
    if (base + SUBW + lane < end) nxt = op.load(base + SUBW + lane, false);
    const int n = min(SUBW, end - base);
    for (int q0 = 0; q0 < n; q0 += U) {
      typename Op::Pre pre[U];
      typename Op::Item iu[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        iu[u] = op.template shfl<SUBW>(it, (q0 + u) & (SUBW - 1), mask);
        if (q0 + u < n && col_ok) op.fetch(iu[u], pre[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u < n) op.accumulate(acc, fst, pre[u], iu[u]);
    }
  }
  Op::finish(acc, fst);
  if (col_ok) write_row<VEC, EPI, ADD>(o, row, col0, acc);
}

}  // namespace stc
