// K3: column-tiled CSR SpMM with the dense operand staged in Tensor Memory (sm_100a).
//
// C[r, c0:c0+128] = sum_p val[p] * B[col[p], c0:c0+128] for a block of 224 rows (28 consumer warps x 8 rows).
//
// Operand path:  global --one tiled TMA copy per chunk (tensor map)--> SMEM stage (63 B rows x
//                512 B + one all-zero row that padding entries point at)
//                --LDS.128 + tcgen05.st (one fill warp per TMEM lane quarter)--> TMEM
//                --tcgen05.ld.32x32b.x4 (28 consumer warps)--> registers (lane l: B[j, c0+4l .. c0+4l+3])
// Each staged row is reused by every row of the block holding that column (~12.8
// at 10 % density). Reading the operand from TMEM takes it off the SMEM crossbar,
// which caps an SMEM-staged kernel near a quarter of the FP32 peak (the previous
// design, round 1: cfg3 6.41 ms; this kernel: 5.10 ms in round 1, 2.83 ms now).
// No MMA is issued — tensor cores stay off this path (north star); TMEM serves as
// a wide operand buffer for CUDA-core FMAs.
//
// Entry path: the plan (`stc_coltile_plan`) re-encodes A per (224-row block,
// 63-column chunk, row) as packed entries {TMEM address of B[col] for the row's warp and
// the chunk's buffer, value bits}, each row padded to an even count with a zero-weight entry
// that points at the chunk's all-zero slot — the inner loop adds nothing to the addresses it
// loads and has no masked case. A warp's list for a chunk is contiguous: it is copied into
// SMEM with cp.async one chunk ahead, and the inner loop is two LDS.128 (4 entries) + 4
// tcgen05.ld + one wait::ld + 8 FFMA2 (a row's odd pair: half of that).
// The plan carries the VALUES of A (it is the prepared form of the matrix, like a
// cuSPARSE SpMM preprocess): rebuild it when the values change.
//
// Pipeline (1 CTA/SM, 1024 threads, TMEM = 2 buffers x 256 columns, all hand-offs by mbarrier):
//   fill warp q    : (q = 0 also issues the TMA copies, two chunks ahead: one
//   (4 warps)        cp.async.bulk.tensor.2d, 63 x 128 box, zero fill past n / k, into stage c % 3
//                    once all four fill warps have left chunk c - 1's stage -- `sempty`; an operand
//                    that cannot be mapped falls back to one bulk copy per 512-byte row, 63 of
//                    which cost the TMA engine ~2900 cycles per chunk: cfg3 4.71 -> 3.84 ms with
//                    the tiled copy.) Waits for the stage (`sfull`, transaction bytes) and for its
//                    quarter's buffer c & 1 to be read (`tfree[q]`), copies the 64 slots into the
//                    quarter (LDS.128 -> tcgen05.st), then arrives on `tfull[q]` and `sempty`.
//   28 consumer    : wait `tfull[quarter]`, consume chunk c from TMEM, arrive on `tfree[quarter]`.
//   warps            (Round 2: the consumers used to copy the chunks themselves, interleaved with
//                    their group loop, and met at a named barrier per quarter: 3.84 -> 3.61 ms.
//                    tcgen05.cp.32x128b.warpx4 as the copy engine was measured too: ~40 cycles per
//                    512-byte row during which tcgen05.ld does not proceed -- 5.75 ms.)
#pragma once

#include <cuda.h>  // CUtensorMap (the type only: the encoder is fetched through the runtime, spmm.cu)

#include <type_traits>

#include "stc_common.cuh"

namespace stc {

#ifndef CTT_GROUP_UNROLL
#define CTT_GROUP_UNROLL 1
#endif
constexpr int kGroupUnroll = CTT_GROUP_UNROLL;    // groups per unrolled body of a row's loop
#ifndef CTT_CONSUMER_WARPS
#define CTT_CONSUMER_WARPS 28
#endif
// Consumer warps (a multiple of 4: warp % 4 = TMEM lane quarter). The group loop is a chain of
// dependent latencies (list LDS -> R2UR -> tcgen05.ld -> wait::ld -> FFMA2), so it is the number of
// resident warps that sets the rate: cfg3 3.61 ms at 16 warps (96 registers), 3.34 at 20, 3.10 at 24,
// 2.93 at 28 (64 registers, 224-row blocks: 2368 CTAs = 16 full waves of 148).
constexpr int CTT_WARPS = CTT_CONSUMER_WARPS;
constexpr int CTT_RPW = 8;                        // rows per consumer warp
constexpr int CTT_ROWS = CTT_WARPS * CTT_RPW;
constexpr int CTT_COLS = 128;
constexpr int CTT_CHUNK = 64;                     // operand slots per chunk in SMEM / TMEM
constexpr int CTT_BROWS = CTT_CHUNK - 1;          // B rows per chunk; the last slot is an all-zero row
constexpr int CTT_FILL_WARPS = 4;                  // one per TMEM lane quarter: SMEM stage -> TMEM
constexpr int CTT_THREADS = (CTT_WARPS + CTT_FILL_WARPS) * 32;  // 1024 threads, 64 registers each
constexpr int CTT_STAGES = 3;
constexpr int CTT_PAD = 2;                        // row segments padded to this many entries (one 16-byte list element)
constexpr int CTT_ECAP = 128;                     // staged entries per warp and chunk
constexpr int CTT_ZERO_SLOT = 4 * CTT_BROWS;      // TMEM column of the zero row inside a chunk's buffer
constexpr size_t CTT_STAGE_FLOATS = (size_t)CTT_CHUNK * CTT_COLS;
constexpr size_t CTT_SMEM = CTT_STAGES * CTT_STAGE_FLOATS * sizeof(float)  // B stages
                            + (size_t)CTT_WARPS * 2 * CTT_ECAP * 8          // entry lists (double)
                            + 256;                                          // barriers, TMEM address

STC_DEVICE uint32_t ctt_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

STC_DEVICE void ctt_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// ---- plan -----------------------------------------------------------------------------------
// chunk_ptr[row * (n_chunks + 1) + c] = first entry of `row` with col >= c * CTT_BROWS
__global__ void ctt_chunk_ptr_kernel(int m, int n_chunks, const int* __restrict__ rowptr,
                                     const int* __restrict__ colidx, int* __restrict__ chunk_ptr) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= m) return;
  const int a = rowptr[row], b = rowptr[row + 1];
  int* out = chunk_ptr + (long long)row * (n_chunks + 1);
  for (int c = lane; c <= n_chunks; c += 32) {
    int lo = a, hi = b;
    const int key = c * CTT_BROWS;
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

// padded entry count of every (block, chunk, row-in-block) slot; slot order = list order
__global__ void ctt_count_kernel(int m, int n_chunks, long long n_slots, const int* __restrict__ chunk_ptr,
                                 int* __restrict__ counts) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_slots;
       i += (long long)gridDim.x * blockDim.x) {
    const int rr = (int)(i % CTT_ROWS);
    const long long bc = i / CTT_ROWS;
    const int c = (int)(bc % n_chunks);
    const int row = (int)(bc / n_chunks) * CTT_ROWS + rr;
    int cnt = 0;
    if (row < m) {
      const int* cp = chunk_ptr + (long long)row * (n_chunks + 1) + c;
      cnt = (cp[1] - cp[0] + CTT_PAD - 1) / CTT_PAD * CTT_PAD;
    }
    counts[i] = cnt;
  }
}

__global__ void ctt_scatter_kernel(int m, int n_chunks, const int* __restrict__ chunk_ptr,
                                   const int* __restrict__ colidx, const float* __restrict__ vals,
                                   const int* __restrict__ offs, int2* __restrict__ ent) {
  const long long n_pairs = (long long)m * n_chunks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pairs;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / n_chunks), c = (int)(i % n_chunks);
    const int* cp = chunk_ptr + (long long)row * (n_chunks + 1) + c;
    const int a = cp[0], b = cp[1];
    const long long slot = ((long long)(row / CTT_ROWS) * n_chunks + c) * CTT_ROWS + row % CTT_ROWS;
    int e = offs[slot];
    // the entry carries its full TMEM address (the kernel's allocation starts at column 0):
    // lane quarter of the row's consumer warp, TMEM buffer of the chunk, 4 columns per B row
    const int base = ((32 * (((row % CTT_ROWS) / CTT_RPW) % 4)) << 16) + (c & 1) * 4 * CTT_CHUNK;
    for (int p = a; p < b; ++p) ent[e++] = make_int2(base + 4 * (colidx[p] - c * CTT_BROWS), __float_as_int(vals[p]));
    // padding: weight 0 on the chunk's all-zero slot -- 0 * 0, never 0 * Inf / NaN from a B
    // row the matrix row does not reference, and the kernel needs no tail case
    for (int q = b - a; q % CTT_PAD; ++q) ent[e++] = make_int2(base + CTT_ZERO_SLOT, 0);
  }
}

// ---- kernel ---------------------------------------------------------------------------------
template <int EPI, bool ADD>
__global__ void __launch_bounds__(CTT_THREADS, 1)
    coltile_tmem_kernel(int m, int n, int k, const int* __restrict__ offs, const int2* __restrict__ ent,
                        const float* __restrict__ B, long long ldb, float* __restrict__ C, long long ldc,
                        const float* __restrict__ D, long long ldd, const __grid_constant__ CUtensorMap bmap,
                        int use_bmap) {
  extern __shared__ __align__(1024) float smem[];
  int2* lists = reinterpret_cast<int2*>(smem + CTT_STAGES * CTT_STAGE_FLOATS);  // [warp][2][ECAP]
  uint64_t* sfull = reinterpret_cast<uint64_t*>(lists + CTT_WARPS * 2 * CTT_ECAP);  // stage landed (TMA bytes)
  uint64_t* sempty = sfull + CTT_STAGES;   // stage copied out by the four fill warps
  uint64_t* tfull = sempty + CTT_STAGES;   // [quarter][buffer]: TMEM buffer of the quarter written
  uint64_t* tfree = tfull + 8;             // [quarter][buffer]: ... read by the quarter's four consumer warps
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tfree + 8);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int c0 = blockIdx.y * CTT_COLS;
  const int n_chunks = (n + CTT_BROWS - 1) / CTT_BROWS;

  // slot 63 of every stage is the zero row: the operand copies fill slots 0..62 only
  for (int t = threadIdx.x; t < CTT_STAGES * CTT_COLS; t += CTT_THREADS)
    smem[(t / CTT_COLS) * CTT_STAGE_FLOATS + (size_t)CTT_BROWS * CTT_COLS + t % CTT_COLS] = 0.f;
  if (warp == 0) {  // TMEM: 512 columns = two 256-column buffers
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(ctt_smem_u32(tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < CTT_STAGES; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ctt_smem_u32(&sfull[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ctt_smem_u32(&sempty[b])), "r"(CTT_FILL_WARPS));
    }
    for (int b = 0; b < 8; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ctt_smem_u32(&tfull[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ctt_smem_u32(&tfree[b])), "r"(CTT_WARPS / 4));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = *tbase_s;
  // all 512 columns are allocated (the allocation waits until the SM's TMEM is free), so it
  // starts at lane 0, column 0: the plan's entries carry absolute TMEM addresses (no
  // per-load address add in the inner loop)
  STC_CHECK(tbase == 0u, "TMEM allocation does not start at column 0");

  if (warp >= CTT_WARPS) {
    // ---------------- fill warp of lane quarter q ----------------
    // B chunk c -> SMEM stage c % 3 (TMA, issued by the fill warp of quarter 0, two chunks ahead)
    const int row_bytes = 4 * min(CTT_COLS, k - c0);  // multiple of 16 (k % 4 == 0)
    auto stage_in = [&](int c) {
      const int s = c % CTT_STAGES;
      const int j0 = c * CTT_BROWS;
      const int rows = min(CTT_BROWS, n - j0);
      float* dst = smem + s * CTT_STAGE_FLOATS;
      const uint32_t bar = ctt_smem_u32(&sfull[s]);
      if (use_bmap) {
        // one tiled copy per chunk: the 63 x 128 box of B at (row j0, column c0); rows past n and
        // columns past k arrive as zeros and count towards the transaction bytes. (63 row copies
        // of 512 bytes keep the TMA engine busy ~2900 cycles per chunk, longer than the
        // consumers need for it: they waited on the stage for 18 % of their samples.)
        if (lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                       "r"((uint32_t)(CTT_BROWS * CTT_COLS * sizeof(float)))
                       : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  ctt_smem_u32(dst)),
              "l"(&bmap), "r"(c0), "r"(j0), "r"(bar)
              : "memory");
        }
        __syncwarp();
        return;
      }
      if (rows < CTT_BROWS || row_bytes < 4 * CTT_COLS) {  // zero what the copies do not cover
        for (int idx = lane; idx < (int)(CTT_STAGE_FLOATS / 4); idx += 32) {
          const int jr = idx / 32, cq = idx % 32;
          if (jr < CTT_BROWS && (jr >= rows || 16 * cq >= row_bytes))
            *reinterpret_cast<float4*>(dst + jr * CTT_COLS + cq * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rows * row_bytes)
                     : "memory");
      __syncwarp();
      STC_CHECK(j0 + rows <= n && c0 + row_bytes / 4 <= k, "B chunk outside the operand");
      for (int jr = lane; jr < rows; jr += 32)  // the warp's lanes issue the row copies in parallel
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                ctt_smem_u32(dst + jr * CTT_COLS)),
            "l"(B + (long long)(j0 + jr) * ldb + c0), "r"(row_bytes), "r"(bar)
            : "memory");
      __syncwarp();
    };
    // SMEM stage -> TMEM buffer c & 1 of the quarter:
    // lane l holds B[j, c0 + 4l .. + 3] of every staged row j (LDS.128) and stores it to columns
    // 4j .. 4j + 3 of its quarter (tcgen05.st); the zero row (slot 63) is copied like the others
    const int q = warp - CTT_WARPS;  // == warp % 4: the quarter this warp may access
    const uint32_t tq = tbase + ((uint32_t)(32 * q) << 16);
    if (q == 0)
      for (int c = 0; c < min(CTT_STAGES - 1, n_chunks); ++c) stage_in(c);
    for (int c = 0; c < n_chunks; ++c) {
      const int s = c % CTT_STAGES, b = c & 1;
      if (q == 0 && c + CTT_STAGES - 1 < n_chunks) {  // chunk c + 2 into the stage chunk c - 1 has left
        if (c >= 1) ctt_mbar_wait(ctt_smem_u32(&sempty[(c - 1) % CTT_STAGES]), (uint32_t)(((c - 1) / CTT_STAGES) & 1));
        stage_in(c + CTT_STAGES - 1);
      }
      if (c >= 2) ctt_mbar_wait(ctt_smem_u32(&tfree[2 * q + b]), (uint32_t)((c / 2 - 1) & 1));  // chunk c - 2 read
      ctt_mbar_wait(ctt_smem_u32(&sfull[s]), (uint32_t)((c / CTT_STAGES) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float* src = smem + s * CTT_STAGE_FLOATS + lane * 4;
      const uint32_t dst = tq + (uint32_t)(b * 4 * CTT_CHUNK);
#pragma unroll 8
      for (int j = 0; j < CTT_CHUNK; ++j) {  // (unrolled: the loads run ahead of the TMEM stores)
        const float4 v = *reinterpret_cast<const float4*>(src + j * CTT_COLS);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst + 4 * j),
                     "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                     "r"(__float_as_uint(v.w))
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ctt_smem_u32(&tfull[2 * q + b])) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ctt_smem_u32(&sempty[s])) : "memory");
      }
    }
  } else {
    // ---------------- consumers: 8 rows x 128 columns each ----------------
    const int row_base = blockIdx.x * CTT_ROWS + warp * CTT_RPW;
    const int quarter = warp % 4;
    int2* mylists = lists + warp * 2 * CTT_ECAP;
    const int* offs_w = offs + (long long)blockIdx.x * n_chunks * CTT_ROWS + warp * CTT_RPW;
    // lanes 0..CTT_RPW: the warp's row boundaries in the padded list of chunk ch
    auto load_meta = [&](int ch) {
      return (lane <= CTT_RPW && ch < n_chunks) ? ld_stream(offs_w + (long long)ch * CTT_ROWS + lane) : 0;
    };
    auto stage_list = [&](int ch, int meta) {  // cp.async of chunk ch's list (skipped if it overflows)
      if (ch < n_chunks) {
        const int e0 = __shfl_sync(0xffffffffu, meta, 0);
        const int total = __shfl_sync(0xffffffffu, meta, CTT_RPW) - e0;
        if (total <= CTT_ECAP) {
          int2* dst = mylists + (ch & 1) * CTT_ECAP;
          for (int i = lane; i < total / 2; i += 32) cp_async16(dst + 2 * i, ent + e0 + 2 * i, true);
        }
      }
      cp_async_commit();
    };

    float acc[CTT_RPW][4];
#pragma unroll
    for (int r = 0; r < CTT_RPW; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;
    // 4 entries -> 4 tcgen05.ld, one wait, 8 packed FMAs (a padding entry: weight 0 on the zero slot)
    auto group = [&](float (&a)[4], int4 e01, int4 e23) {
      uint32_t x[4][4];
      const int taddr[4] = {e01.x, e01.z, e23.x, e23.z};  // absolute TMEM addresses (plan)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        STC_CHECK((uint32_t)taddr[u] >> 16 == 32u * quarter && (taddr[u] & 0xffff) < 512,
                  "COLTILE entry outside the warp's TMEM lane quarter");
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x[u][0]), "=r"(x[u][1]), "=r"(x[u][2]), "=r"(x[u][3])
                     : "r"(taddr[u]));
      // the loaded registers pass through the wait, so no use of them can be scheduled above it
      asm volatile("tcgen05.wait::ld.sync.aligned;"
                   : "+r"(x[0][0]), "+r"(x[0][1]), "+r"(x[0][2]), "+r"(x[0][3]), "+r"(x[1][0]), "+r"(x[1][1]),
                     "+r"(x[1][2]), "+r"(x[1][3]), "+r"(x[2][0]), "+r"(x[2][1]), "+r"(x[2][2]), "+r"(x[2][3]),
                     "+r"(x[3][0]), "+r"(x[3][1]), "+r"(x[3][2]), "+r"(x[3][3])
                   :
                   : "memory");
      const float w[4] = {__int_as_float(e01.y), __int_as_float(e01.w), __int_as_float(e23.y),
                          __int_as_float(e23.w)};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        // packed FMAs (FFMA2, value broadcast): 8 issue slots per group instead of 16
        fma2(a[0], a[1], w[u], __uint_as_float(x[u][0]), __uint_as_float(x[u][1]));
        fma2(a[2], a[3], w[u], __uint_as_float(x[u][2]), __uint_as_float(x[u][3]));
      }
    };
    // a row's last pair when its padded count is not a multiple of 4 (rows are padded to pairs:
    // 0.5 padding entries per row and chunk on average instead of 1.5 with groups of 4 only)
    auto pair = [&](float (&a)[4], int4 e01) {
      uint32_t x[2][4];
      const int taddr[2] = {e01.x, e01.z};
#pragma unroll
      for (int u = 0; u < 2; ++u)
        STC_CHECK((uint32_t)taddr[u] >> 16 == 32u * quarter && (taddr[u] & 0xffff) < 512,
                  "COLTILE entry outside the warp's TMEM lane quarter");
#pragma unroll
      for (int u = 0; u < 2; ++u)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x[u][0]), "=r"(x[u][1]), "=r"(x[u][2]), "=r"(x[u][3])
                     : "r"(taddr[u]));
      asm volatile("tcgen05.wait::ld.sync.aligned;"
                   : "+r"(x[0][0]), "+r"(x[0][1]), "+r"(x[0][2]), "+r"(x[0][3]), "+r"(x[1][0]), "+r"(x[1][1]),
                     "+r"(x[1][2]), "+r"(x[1][3])
                   :
                   : "memory");
      const float w[2] = {__int_as_float(e01.y), __int_as_float(e01.w)};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        fma2(a[0], a[1], w[u], __uint_as_float(x[u][0]), __uint_as_float(x[u][1]));
        fma2(a[2], a[3], w[u], __uint_as_float(x[u][2]), __uint_as_float(x[u][3]));
      }
    };

    int meta = load_meta(0);
    int meta_next = load_meta(1);
    stage_list(0, meta);
    for (int ch = 0; ch < n_chunks; ++ch) {
      const int meta_after = load_meta(ch + 2);
      stage_list(ch + 1, meta_next);
      cp_async_wait<1>();  // chunk ch's list has landed (ch + 1's may be in flight)
      __syncwarp();
      const int e0 = __shfl_sync(0xffffffffu, meta, 0);
      const int total = __shfl_sync(0xffffffffu, meta, CTT_RPW) - e0;
      STC_CHECK(total >= 0 && total % CTT_PAD == 0, "COLTILE chunk list length");
      // lane r: pairs of row r in this chunk; the rows' pairs are contiguous in the list, so one
      // pointer walks it (chunks denser than the staged list read it straight from global memory)
      const int npair = (__shfl_down_sync(0xffffffffu, meta, 1) - meta) / CTT_PAD;
      auto rows = [&](const int4* gp) {  // one int4 = one pair of entries
#pragma unroll
        for (int r = 0; r < CTT_RPW; ++r) {
          const int nr = __shfl_sync(0xffffffffu, npair, r);
          STC_CHECK(nr >= 0 && nr * CTT_PAD <= total, "COLTILE row list outside the chunk list");
#pragma unroll kGroupUnroll
          for (int g = 0; g < (nr >> 1); ++g, gp += 2) group(acc[r], gp[0], gp[1]);
          if (nr & 1) pair(acc[r], *gp++);
        }
      };
      // chunk ch is in buffer ch & 1 of this quarter once the quarter's fill warp has stored it
      ctt_mbar_wait(ctt_smem_u32(&tfull[2 * quarter + (ch & 1)]), (uint32_t)((ch / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (total <= CTT_ECAP)
        rows(reinterpret_cast<const int4*>(mylists + (ch & 1) * CTT_ECAP));  // LDS
      else
        rows(reinterpret_cast<const int4*>(ent + e0));                       // LDG
      // every load of this chunk has completed (each group waits): hand the buffer back
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ctt_smem_u32(&tfree[2 * quarter + (ch & 1)]))
                     : "memory");
      meta = meta_next;
      meta_next = meta_after;
    }
    cp_async_wait<0>();
    const int col = c0 + lane * 4;
#pragma unroll
    for (int r = 0; r < CTT_RPW; ++r) {
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
