// EXPERIMENT (not built): TMEM-staged COLTILE kernel, kept as the record of a
// negative result. cfg3 on B200:
//   SMEM-staged coltile (shipped, csrc/coltile.cuh)              6.42 ms
//   this file: consumer warps fill TMEM with tcgen05.st          6.73 ms
//   producer-warp tcgen05.cp.32x128b.warpx4 staging               9.07 ms
//   (tools/tmem_probe.cu: one 64-row chunk copy = 3373 cycles)
// Needs the padded-offset plan of coltile_tmem_plan.diff (applies to csrc/spmm.cu).
// K3: column-tiled CSR SpMM for wide dense operands, operand staged in TMEM (sm_100a).
//
// C[r, c0:c0+128] = sum_p val[p] * B[col[p], c0:c0+128] for a block of 128 rows.
//
// Data path of the dense operand B (the FFN's X^T, 64 MB, L2-resident):
//   global --cp.async--> SMEM stage (64 rows x 512 B)
//          --tcgen05.cp.32x128b.warpx4--> TMEM (broadcast to all four lane quarters)
//          --tcgen05.ld.32x32b.x4--> registers (lane l gets B[j, c0+4l .. c0+4l+3])
// Each staged B row is reused by every row of the block holding that column
// (~12.8 at 10% density). Reading the operand from Tensor Memory instead of
// shared memory takes the per-FMA operand traffic off the SMEM crossbar (one
// LDS.128 per 4 FFMA capped the SMEM-staged variant near a quarter of the FP32
// peak); TMEM serves it several times faster (tools/tmem_probe.cu). No MMA is
// issued — the north star keeps tensor cores off this path — TMEM is used as a
// large, high-bandwidth operand buffer for CUDA-core FMAs.
//
// Warp-specialized pipeline (1 CTA/SM, TMEM = 2 buffers x 256 columns, no CTA barrier):
//   producer warp : cp.async chunk c+2 -> SMEM stage, tcgen05.cp chunk c -> TMEM buffer
//                   c&1 once the consumers released it (mbarrier `empty`), commit to `full`
//   16 consumer warps: wait `full[c&1]`, consume chunk c from TMEM, arrive on `empty[c&1]`
// so warps with more entries in a chunk no longer hold the others at a barrier.
// A plan-time table (`coltile_plan_kernel`) gives, per row, where each chunk's
// entries start; every warp stages its rows' (col, val) entries of the chunk in
// a per-warp SMEM scratch (prefetched one chunk ahead), so the inner loop is
// LDS.64 (broadcast) + tcgen05.ld + 4 FFMA per entry.
#pragma once

#include "stc_common.cuh"

namespace stc {

constexpr int CT_ROWS = 128;        // rows per CTA
constexpr int CT_COLS = 128;        // output columns per CTA (32 lanes x float4)
constexpr int CT_CHUNK = 64;        // B rows per chunk (one TMEM buffer = 4 * 64 columns)
constexpr int CT_WARPS = 16;                // consumer warps; one more warp produces
constexpr int CT_THREADS = (CT_WARPS + 1) * 32;
constexpr int CT_STAGES = 3;                // SMEM stages of the producer
constexpr int CT_RPW = CT_ROWS / CT_WARPS;  // rows per warp
constexpr int CT_SCRATCH = 128;
constexpr int CT_PAD = 4;                   // row segments padded to this many entries             // staged (col, val) entries per warp and chunk
constexpr int CT_PREF = CT_SCRATCH / 32;    // prefetched entries per lane
constexpr size_t CT_STAGE_FLOATS = (size_t)CT_CHUNK * CT_COLS;
constexpr size_t CT_SMEM = CT_STAGES * CT_STAGE_FLOATS * sizeof(float) + (size_t)CT_WARPS * CT_SCRATCH * 8 + 64;

// Plan: chunk_ptr[row * (n_chunks + 1) + c] = first entry of `row` with col >= c * CT_CHUNK.
__global__ void coltile_plan_kernel(int m, int n_chunks, const int* __restrict__ rowptr,
                                    const int* __restrict__ colidx, int* __restrict__ chunk_ptr) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= m) return;
  const int a = rowptr[row], b = rowptr[row + 1];
  int* out = chunk_ptr + (long long)row * (n_chunks + 1);
  for (int c = lane; c <= n_chunks; c += 32) {
    int lo = a, hi = b;  // lower_bound of c*CT_CHUNK in colidx[a, b)
    const int key = c * CT_CHUNK;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (colidx[mid] < key)
        lo = mid + 1;
      else
        hi = mid;
    }
    out[c] = lo;
  }
}

// Padded offsets (plan): every row's entries of a chunk are padded to a multiple of CT_PAD
// (padding = weight 0), and offs[(rb * n_chunks + c) * CT_ROWS + rr] is where row
// rb*CT_ROWS+rr starts in the padded, (block, chunk, row)-ordered entry sequence. Rows of
// one (block, chunk) are contiguous, so warp w's list is offs[.. + w*CT_RPW .. + CT_RPW].
__global__ void coltile_count_kernel(int m, int n_chunks, long long n_slots, const int* __restrict__ chunk_ptr,
                                     int* __restrict__ counts) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_slots;
       i += (long long)gridDim.x * blockDim.x) {
    const int rr = (int)(i % CT_ROWS);
    const long long bc = i / CT_ROWS;
    const int c = (int)(bc % n_chunks);
    const int row = (int)(bc / n_chunks) * CT_ROWS + rr;
    int cnt = 0;
    if (row < m) {
      const int* cp = chunk_ptr + (long long)row * (n_chunks + 1) + c;
      cnt = (cp[1] - cp[0] + CT_PAD - 1) / CT_PAD * CT_PAD;
    }
    counts[i] = cnt;
  }
}

STC_DEVICE void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
STC_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
STC_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

STC_DEVICE uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared-memory matrix descriptor for tcgen05.cp of 32 rows x 16 B stored contiguously
// (K-major, no swizzle: four 8x16B core matrices 128 B apart).
STC_DEVICE uint64_t tmem_cp_desc(const void* smem_rows) {
  const uint64_t addr = (smem_u32(smem_rows) >> 4) & 0x3fff;
  return addr | (uint64_t(128 >> 4) << 16) | (uint64_t(128 >> 4) << 32) | (1ull << 46);
}

STC_DEVICE void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Per-warp offsets of its CT_RPW rows' entries within one chunk: lane r (< CT_RPW)
// knows start(r), lane CT_RPW + r knows end(r); returns the exclusive prefix of the
// counts for row `lane % CT_RPW` and the total.
STC_DEVICE void chunk_layout(int bounds, int lane, int& my_off, int& total) {
  const int other = __shfl_xor_sync(0xffffffffu, bounds, CT_RPW);  // end for lanes < CT_RPW
  const int cnt = (lane < CT_RPW) ? other - bounds : 0;
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < CT_RPW; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  my_off = incl - cnt;
  total = __shfl_sync(0xffffffffu, incl, CT_RPW - 1);
}

template <int EPI, bool ADD>
__global__ void __launch_bounds__(CT_THREADS, 1) coltile_kernel(int m, int n, int k, const int* __restrict__ offs,
                                                               const int* __restrict__ chunk_ptr,
                                                               const int* __restrict__ colidx,
                                                               const float* __restrict__ vals,
                                                               const float* __restrict__ B, long long ldb,
                                                               float* __restrict__ C, long long ldc,
                                                               const float* __restrict__ D, long long ldd) {
  extern __shared__ __align__(1024) float smem[];  // [CT_STAGES][CT_CHUNK][CT_COLS] stages + scratch
  int2* scratch_all = reinterpret_cast<int2*>(smem + CT_STAGES * CT_STAGE_FLOATS);
  uint64_t* sfull = reinterpret_cast<uint64_t*>(scratch_all + CT_WARPS * CT_SCRATCH);  // [3] SMEM stage landed
  uint64_t* sempty = sfull + CT_STAGES;  // [3] SMEM stage copied into TMEM by all consumer warps
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(sempty + CT_STAGES);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int c0 = blockIdx.y * CT_COLS;
  const int n_chunks = (n + CT_CHUNK - 1) / CT_CHUNK;

  if (warp == 0) {  // TMEM: 512 columns = two 256-column buffers
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < CT_STAGES; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(smem_u32(&sfull[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sempty[b])), "r"(CT_WARPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = *tbase_s;

  if (warp == CT_WARPS) {
    // ================= producer warp: global -> SMEM (cp.async) -> TMEM (tcgen05.cp) =================
    auto stage = [&](int chunk) {
      const int j0 = chunk * CT_CHUNK;
      float* dst = smem + (chunk % CT_STAGES) * CT_STAGE_FLOATS;
      for (int idx = lane; idx < (int)(CT_STAGE_FLOATS / 4); idx += 32) {
        const int jr = idx / 32, cq = idx % 32;
        const int j = j0 + jr;
        const int cc = c0 + cq * 4;
        const bool ok = (j < n) && (cc < k);
        cp_async16(dst + jr * CT_COLS + cq * 4, ok ? (const void*)(B + (long long)j * ldb + cc) : (const void*)B, ok);
      }
      cp_async_commit();
    };
    for (int c = 0; c < n_chunks; ++c) {
      if (c >= CT_STAGES)  // all consumer warps copied chunk c - CT_STAGES out of this stage
        mbar_wait(smem_u32(&sempty[c % CT_STAGES]), (uint32_t)((c / CT_STAGES - 1) & 1));
      stage(c);
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&sfull[c % CT_STAGES]))
                   : "memory");
    }
    cp_async_wait<0>();
  } else {
    // ================= consumer warps: 8 rows each =================
    const int row_base = blockIdx.x * CT_ROWS + warp * CT_RPW;
    const int col = c0 + lane * 4;
    int2* scratch = scratch_all + warp * CT_SCRATCH;
    const int quarter = warp % 4, part = warp / 4;
    const uint32_t tq = tbase + ((uint32_t)(32 * quarter) << 16);  // this warp's TMEM lane quarter
    // The four warps of a lane quarter write one copy of each chunk into their quarter
    // (each warp CT_CHUNK / 4 B rows: LDS.128 -> tcgen05.st) and sync on a named barrier.
    auto fill = [&](int c) {
      mbar_wait(smem_u32(&sfull[c % CT_STAGES]), (uint32_t)((c / CT_STAGES) & 1));
      constexpr int kRows = CT_CHUNK / 4;
      const float* src = smem + (c % CT_STAGES) * CT_STAGE_FLOATS + (kRows * part) * CT_COLS + lane * 4;
      const uint32_t dst = tq + (uint32_t)((c & 1) * 4 * CT_CHUNK + 4 * kRows * part);
#pragma unroll 4
      for (int j = 0; j < kRows; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(src + j * CT_COLS);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst + 4 * j),
                     "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                     "r"(__float_as_uint(v.w))
                     : "memory");
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sempty[c % CT_STAGES])) : "memory");
    };
    auto quarter_sync = [&]() {
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("bar.sync %0, 128;" ::"r"(1 + quarter) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;");
    };
    const int* offs_w = offs + (long long)blockIdx.x * n_chunks * CT_ROWS + warp * CT_RPW;
    const int* cp_w = chunk_ptr + (long long)row_base * (n_chunks + 1);
    // Per-chunk metadata of the warp's rows, one int per lane: lanes 0..CT_RPW the padded
    // offsets, lanes 16+r / 24+r the CSR start / end of row r within the chunk.
    auto load_meta = [&](int ch) {
      int v = 0;
      if (ch < n_chunks) {
        if (lane <= CT_RPW) {
          v = ld_stream(offs_w + (long long)ch * CT_ROWS + lane);
        } else if (lane >= 16 && lane < 16 + 2 * CT_RPW) {
          const int r = (lane - 16) % CT_RPW, hi = (lane - 16) / CT_RPW;
          if (row_base + r < m) v = ld_stream(cp_w + (long long)r * (n_chunks + 1) + ch + hi);
        }
      }
      return v;
    };
    // entries [base, base + CT_SCRATCH) of the warp's padded list of a chunk -> (col, val); padding -> (j0, 0)
    auto fetch = [&](int meta, int j0, int base, int (&pk)[CT_PREF], float (&pv)[CT_PREF]) {
      const int e0 = __shfl_sync(0xffffffffu, meta, 0);
      const int total = __shfl_sync(0xffffffffu, meta, CT_RPW) - e0;
      int off[CT_RPW], st[CT_RPW], en[CT_RPW];
#pragma unroll
      for (int r = 0; r < CT_RPW; ++r) {
        off[r] = __shfl_sync(0xffffffffu, meta, r) - e0;
        st[r] = __shfl_sync(0xffffffffu, meta, 16 + r);
        en[r] = __shfl_sync(0xffffffffu, meta, 16 + CT_RPW + r);
      }
#pragma unroll
      for (int t = 0; t < CT_PREF; ++t) {
        pk[t] = j0;  // raw column; padding points at the chunk's first row with weight 0
        pv[t] = 0.f;
        const int idx = base + t * 32 + lane;
        int pos = 0, lim = 0;
#pragma unroll
        for (int r = 0; r < CT_RPW; ++r)
          if (idx >= off[r]) {
            pos = st[r] + (idx - off[r]);
            lim = en[r];
          }
        if (idx < total && pos < lim) {
          pk[t] = ld_stream(colidx + pos);
          pv[t] = ld_stream(vals + pos);
        }
      }
    };
    int pk[CT_PREF];
    float pv[CT_PREF];
    float acc[CT_RPW][4];
#pragma unroll
    for (int r = 0; r < CT_RPW; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;

    // 4 entries (one padded group) -> 4 tcgen05.ld, one wait, 16 FFMA
    auto group = [&](float (&a)[4], uint32_t tchunk, int4 e01, int4 e23) {
      uint32_t x[4][4];
      const int cols[4] = {e01.x, e01.z, e23.x, e23.z};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x[u][0]), "=r"(x[u][1]), "=r"(x[u][2]), "=r"(x[u][3])
                     : "r"(tchunk + (uint32_t)cols[u]));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const float w[4] = {__int_as_float(e01.y), __int_as_float(e01.w), __int_as_float(e23.y),
                          __int_as_float(e23.w)};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[0] = fmaf(w[u], __uint_as_float(x[u][0]), a[0]);
        a[1] = fmaf(w[u], __uint_as_float(x[u][1]), a[1]);
        a[2] = fmaf(w[u], __uint_as_float(x[u][2]), a[2]);
        a[3] = fmaf(w[u], __uint_as_float(x[u][3]), a[3]);
      }
    };

    int o_cur = load_meta(0);
    int o_next = load_meta(1);
    fetch(o_cur, 0, 0, pk, pv);
    if (n_chunks > 0) fill(0);
    quarter_sync();
    for (int ch = 0; ch < n_chunks; ++ch) {
      const int o_after = load_meta(ch + 2);
      const int j0 = ch * CT_CHUNK;
      const int e0 = __shfl_sync(0xffffffffu, o_cur, 0);
      const int total = __shfl_sync(0xffffffffu, o_cur, CT_RPW) - e0;
#pragma unroll
      for (int t = 0; t < CT_PREF; ++t) scratch[t * 32 + lane] = make_int2(4 * (pk[t] - j0), __float_as_int(pv[t]));
      __syncwarp();
      fetch(o_next, j0 + CT_CHUNK, 0, pk, pv);  // next chunk's entries stream in while this one is consumed
      if (ch + 1 < n_chunks) fill(ch + 1);
      const uint32_t tchunk = tq + (uint32_t)((ch & 1) * 4 * CT_CHUNK);
      const int4* sc = reinterpret_cast<const int4*>(scratch);
      for (int base = 0; base < total; base += CT_SCRATCH) {
        if (base > 0) {  // rows denser than the scratch: refill it synchronously
          int qk[CT_PREF];
          float qv[CT_PREF];
          fetch(o_cur, j0, base, qk, qv);
          __syncwarp();
#pragma unroll
          for (int t = 0; t < CT_PREF; ++t) scratch[t * 32 + lane] = make_int2(4 * (qk[t] - j0), __float_as_int(qv[t]));
          __syncwarp();
        }
#pragma unroll
        for (int r = 0; r < CT_RPW; ++r) {
          const int qa = max(__shfl_sync(0xffffffffu, o_cur, r) - e0, base) - base;
          const int qb = min(__shfl_sync(0xffffffffu, o_cur, r + 1) - e0, base + CT_SCRATCH) - base;
          for (int q = qa; q < qb; q += CT_PAD) group(acc[r], tchunk, sc[q / 2], sc[q / 2 + 1]);
        }
      }
      quarter_sync();  // chunk ch fully read, chunk ch + 1 fully written
      o_cur = o_next;
      o_next = o_after;
    }
#pragma unroll
    for (int r = 0; r < CT_RPW; ++r) {
      const int row = row_base + r;
      if (row < m && col < k) {
        float4 o = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
        if constexpr (ADD) {
          const float4 d = *reinterpret_cast<const float4*>(D + (long long)row * ldd + col);
          o.x += d.x; o.y += d.y; o.z += d.z; o.w += d.w;
        }
        o.x = act<EPI>(o.x); o.y = act<EPI>(o.y); o.z = act<EPI>(o.z); o.w = act<EPI>(o.w);
        st_stream4(C + (long long)row * ldc + col, o);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

}  // namespace stc
