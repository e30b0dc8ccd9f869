// Merge-path segmented reduction over PREPARED items, staged asynchronously (sm_100a).
//
// Same decomposition, carries and summation order as merge_kernel (segreduce.cuh); what
// changes is how a group gets its items. merge_kernel builds them from the raw index /
// value streams into a large shared-memory window (one synchronous round trip per window,
// 40 KB of windows per CTA for MTTKRP, which leaves the SM 54 KB of L1 at 3 CTAs). Here the
// items were built once at plan time (`stc_mttkrp_prepare_items`: gather offsets already
// multiplied by the leading dimensions, fiber-start flags set) and each group streams them
// through a small circular buffer with cp.async: chunk c + NB - 1 is copied while chunk c is
// consumed, so staging costs no round trip and no registers, the gather ring runs across
// chunk boundaries without draining, and the CTA's shared memory shrinks to the carries
// plus NB * W items per group — the rest of the SM stays L1 for the factor-row gathers.
#pragma once

#include "segreduce.cuh"

namespace stc {

// MTTKRP over prepared 16-byte items {offset of B[j,:], offset of C[k,:], T, fiber-start flag}.
template <int VEC>
struct MttkrpItemsOp {
  using Base = MttkrpOp<VEC>;
  using Item = typename Base::Item;
  using Pre = typename Base::Pre;
  using State = typename Base::State;
  const Item* items;  // [nnz], entry order
  const float* B;
  const float* C;
  unsigned lane_off = 0;
  unsigned long long limitb = ~0ull, limitc = ~0ull;

#ifndef STC_MTTKRPA_RING
#define STC_MTTKRPA_RING 2
#endif
#ifndef STC_MTTKRPA_MINB
#define STC_MTTKRPA_MINB 4
#endif
#ifndef STC_MTTKRPA_CHUNKS
#define STC_MTTKRPA_CHUNKS 4
#endif
  static constexpr int kRing = VEC == 4 ? STC_MTTKRPA_RING : 8;
  static constexpr int kMinBlocks = STC_MTTKRPA_MINB;
  static constexpr int kChunks = STC_MTTKRPA_CHUNKS;  // chunks in the circular buffer (power of two)

  STC_DEVICE void shift(int col0) { lane_off = (unsigned)col0; }
  STC_DEVICE void fetch(const Item& it, Pre& pre) const {
    STC_CHECK(!it.flag || (unsigned long long)(it.offb + lane_off) + VEC <= limitb, "MTTKRP gather outside B");
    STC_CHECK((unsigned long long)(it.offc + lane_off) + VEC <= limitc, "MTTKRP gather outside C");
    if (it.flag) pre.b.load_gather(B + (it.offb + lane_off));
    pre.c.load_gather(C + (it.offc + lane_off));
  }
  STC_DEVICE static void init(State& st) { st.b.zero(); }
  STC_DEVICE void accumulate(Frag<VEC>& acc, State& st, const Pre& pre, const Item& it) const {
#pragma unroll
    for (int e = 0; e < VEC; ++e) st.b.v[e] = (it.flag & 1) ? pre.b.v[e] : st.b.v[e];
#ifndef STC_MTTKRP_NO_F2
    if constexpr (VEC % 2 == 0) {
      // packed halves (FMUL2 / FFMA2): each is exactly mul.rn / fma.rn, so the sums do not change;
      // half the issue slots of the product chain (cfg5 114.7 -> 112.7 us)
#pragma unroll
      for (int e = 0; e < VEC; e += 2) {
        float t0, t1;
        mul2(t0, t1, it.v, st.b.v[e], st.b.v[e + 1]);
        fma2v(acc.v[e], acc.v[e + 1], t0, t1, pre.c.v[e], pre.c.v[e + 1]);
      }
      return;
    }
#endif
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc.v[e] = fmaf(it.v * st.b.v[e], pre.c.v[e], acc.v[e]);
  }
  STC_DEVICE static void finish(Frag<VEC>&, State&) {}
  // a group starts mid-fiber: its first entry must load B[j,:] whatever the stored flag says
  STC_DEVICE static void mark_first(Item& it) { it.flag |= 1; }
};

// Plan-time item build: one thread per entry.
template <class Item>
__global__ void mttkrp_items_kernel(long long nnz, const int* __restrict__ jc, const int* __restrict__ kc,
                                    const float* __restrict__ val, long long ldb, long long ldcf,
                                    Item* __restrict__ items) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nnz;
       p += (long long)gridDim.x * blockDim.x) {
    const int j = jc[p];
    const bool start = p == 0 || jc[p - 1] != j;
    items[p] = Item{(unsigned)((long long)j * ldb), (unsigned)((long long)kc[p] * ldcf), val[p], start ? 1 : 0};
  }
}

// 8-entry chunks (16 KB of item rings per CTA) against 16 (32 KB): cfg5 116.8 -> 110.6 us -- the L1 the
// rings leave is what keeps the hot factor rows resident under ~1000 in-flight gather lines per SM
#ifndef STC_ASYNC_CHUNK
#define STC_ASYNC_CHUNK 8
#endif
template <int SUBW>
__host__ __device__ constexpr int async_chunk() {
  // entries per cp.async group: every lane copies at least one item
  return SUBW > STC_ASYNC_CHUNK ? SUBW : STC_ASYNC_CHUNK;
}
template <int SUBW, class Op>
__host__ __device__ constexpr int async_ring_items() {
  return async_chunk<SUBW>() * Op::kChunks;
}
template <int SUBW, class Op>
__host__ __device__ constexpr int async_item_stride() {
  return bank_skewed(async_ring_items<SUBW, Op>(), (int)sizeof(typename Op::Item));
}
#ifndef STC_ASYNC_UNROLL
#define STC_ASYNC_UNROLL 0
#endif
template <int W, int U>
__host__ __device__ constexpr int async_unroll() {
  // entries per unrolled body of the chunk loop (0: the whole chunk)
  return STC_ASYNC_UNROLL > 0 && STC_ASYNC_UNROLL < W && STC_ASYNC_UNROLL % U == 0 && W % STC_ASYNC_UNROLL == 0
             ? STC_ASYNC_UNROLL
             : W;
}
#ifndef STC_ASYNC_ROWS
#define STC_ASYNC_ROWS 32
#endif
constexpr int kAsyncRows = STC_ASYNC_ROWS;  // staged row ends per group (restaged when a group owns more)
template <int SUBW, int VEC, class Op>
__host__ __device__ constexpr size_t merge_async_smem_bytes() {
  constexpr int NG = 256 / SUBW;
  constexpr int SW = SUBW * VEC;
  return (size_t)2 * NG * SW * sizeof(float) + (size_t)2 * NG * sizeof(int) +
         (size_t)NG * async_item_stride<SUBW, Op>() * sizeof(typename Op::Item) +
         (size_t)NG * bank_skewed(kAsyncRows, (int)sizeof(int)) * sizeof(int);
}

template <int SUBW, int VEC, int EPI, bool ADD, int U, bool FULL, class Op>
__global__ void __launch_bounds__(256, Op::kMinBlocks) merge_async_kernel(SegOut o, MergeShape ms, Op op) {
  using Item = typename Op::Item;
  static_assert(sizeof(Item) == 16, "cp.async staging copies 16-byte items");
  constexpr int NG = 256 / SUBW;
  constexpr int SW = SUBW * VEC;
  constexpr int W = async_chunk<SUBW>();
  constexpr int NB = Op::kChunks;
  constexpr int RING = W * NB;
  static_assert((RING & (RING - 1)) == 0 && NB >= 3, "circular buffer: power of two, at least 3 chunks");
  static_assert(U <= W && W % U == 0, "gather ring deeper than a chunk");
  constexpr int IST = async_item_stride<SUBW, Op>();
  constexpr int CAPR = kAsyncRows;
  constexpr int RST = bank_skewed(CAPR, (int)sizeof(int));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* Hs = reinterpret_cast<float*>(smem_raw);                       // [NG][SW]
  float* Ts = Hs + NG * SW;                                             // [NG][SW]
  int* Hrow = reinterpret_cast<int*>(Ts + NG * SW);                     // [NG]
  int* Trow = Hrow + NG;                                                // [NG]
  Item* items_all = reinterpret_cast<Item*>(Trow + NG);                 // [NG][IST]
  int* rend_all = reinterpret_cast<int*>(items_all + NG * IST);         // [NG][RST]

  const int sub = threadIdx.x / SUBW;
  const int lane = threadIdx.x % SUBW;
  const unsigned mask = subwarp_mask<SUBW>();
  const int cta = blockIdx.x;
  const int slab = blockIdx.y;
  const int col0 = slab * SW + lane * VEC;
  const bool col_ok = FULL || col0 < o.k;
  Item* items = items_all + sub * IST;
  int* rend = rend_all + sub * RST;
  const long long zslab = (long long)slab * ms.n_cta;
  op.shift(col0);

  const int g = min(cta * NG + sub, ms.n_groups);
  const int2 s = ms.starts[g];
  const int2 e = ms.starts[min(g + 1, ms.n_groups)];
  const int row0 = s.x;
  const int n_rows = e.x - s.x;   // rows whose end item this group owns
  const int n_nnz = e.y - s.y;    // entries this group accumulates
  STC_CHECK(n_rows >= 0 && n_nnz >= 0 && e.x <= o.m && n_nnz <= ms.ipg && n_rows <= ms.ipg,
            "merge partition: group range");

  // chunk c = entries [c * W, c * W + W) of the group -> circular buffer (zero-filled past the
  // group's range: a zero item gathers row 0 of C and is never accumulated)
  const Item* gitems = op.items + s.y;
  auto issue = [&](int c) {
#pragma unroll
    for (int t = lane; t < W; t += SUBW) {
      const int p = c * W + t;
      const bool in = p < n_nnz;
      cp_async16(&items[p & (RING - 1)], gitems + (in ? p : 0), in);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int c = 0; c < NB - 1; ++c) issue(c);

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
  int cur_end = n_rows > 0 ? rend[0] : INT_MAX;      // end of the current row, relative to s.y
  int cur_start = first_start - s.y;                 // its start (may be negative)
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
  // the warp's groups run the same number of chunk steps (a warp-uniform loop keeps the
  // uniform datapath usable: descriptors and bases stay in uniform registers); a group past
  // its own range sees zero-filled items and the `left` guard below
  const int n_chunks = __reduce_max_sync(0xffffffffu, (n_nnz + W - 1) / W);
  int end_w = cur_end;  // current row's end relative to the chunk being consumed
  for (int c = 0; c < n_chunks; ++c) {
    __syncwarp(mask);               // every lane has left chunk c - 1: its slots may be overwritten
    issue(c + NB - 1);
    cp_async_wait<NB - 2>();        // this lane's copies of chunks <= c + 1 have landed ...
    __syncwarp(mask);               // ... and every other lane's
    // slots of chunk c and of chunk c + 1: every item access below is base + constant
    const Item* cur = items + (c & (NB - 1)) * W;
    const Item* nxt = items + ((c + 1) & (NB - 1)) * W;
    if (c == 0) {
      if (lane == 0) Op::mark_first(items[0]);
      __syncwarp(mask);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (col_ok) op.fetch(cur[u], ring[u]);
    }
    const int cw = c * W;
    end_w = cur_end - cw;
    // Fast path, taken warp-wide: every group of the warp has a full chunk with no row end in it
    // (most chunks: a group owns ~350 entries and one or two row ends). Straight-line code with no
    // flush scaffolding, so the operand bases and load descriptors stay in uniform registers.
    if (__all_sync(0xffffffffu, cw + W <= n_nnz && end_w >= W)) {
#pragma unroll
      for (int t = 0; t < W; ++t) {
        op.accumulate(acc, fst, ring[t % U], cur[t]);
        if (col_ok) op.fetch(t + U < W ? cur[t + U] : nxt[t + U - W], ring[t % U]);
      }
    } else if (cw + W <= n_nnz) {  // full chunk: W / U ring turns, entry t + U lies in this chunk or the next
      // unrolled F entries at a time (F a multiple of the ring depth, so ring slots stay
      // static): the fully unrolled chunk with its inlined flush paths is ~25 k SASS lines
      // and stalls on instruction fetch (no_instruction 9 % of samples at F = W = 16)
      constexpr int F = async_unroll<W, U>();
#pragma unroll 1
      for (int tb = 0; tb < W; tb += F) {
#pragma unroll
        for (int q = 0; q < F; ++q) {
          const int t = tb + q;
          while (t >= end_w) {
            flush();
            end_w = cur_end - cw;
          }
          op.accumulate(acc, fst, ring[q % U], cur[t]);
          if (col_ok) {
            if constexpr (F == W)
              op.fetch(t + U < W ? cur[t + U] : nxt[t + U - W], ring[q % U]);
            else
              op.fetch(items[(cw + t + U) & (RING - 1)], ring[q % U]);
          }
        }
      }
    } else if (cw < n_nnz) {  // the group's last, partial chunk (items past the range are zero: harmless gathers)
      const int left = n_nnz - cw;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        if (t < left) {
          while (t >= end_w) {
            flush();
            end_w = cur_end - cw;
          }
          op.accumulate(acc, fst, ring[t % U], cur[t]);
          if (t + U < W && col_ok) op.fetch(cur[t + U], ring[t % U]);
        }
      }
    }
  }
  cp_async_wait<0>();
  while (r < n_rows) flush();
  Op::finish(acc, fst);
  if (row0 + r < o.m && n_nnz > cur_start && r == n_rows) {
    if (col_ok) acc.store_plain(&Ts[sub * SW + lane * VEC]);
    if (lane == 0) Trow[sub] = row0 + r;
  }
  __syncthreads();

  merge_combine<SUBW, VEC, EPI, ADD>(o, ms, sub, lane, col_ok, col0, zslab, Hs, Ts, Hrow, Trow);
}

}  // namespace stc
