/* stc.h — C ABI of the B200-native sparse-contraction library (libstc.so).
 *
 * The reference (arxiv 2405.16883 "Scorch", package `sparsetc`) has no native
 * layer: its hot path is the Python interpreter in
 * /root/reference/pkg/src/sparsetc/engine.py. Each entry point below replaces
 * one interpreted loop nest of that engine; the citation names it.
 *
 * Conventions
 *   - All pointers are DEVICE pointers (CUDA global memory) except `stream`,
 *     which is a cudaStream_t passed as void*. The library never allocates or
 *     frees: scratch comes from a caller-provided workspace whose size is
 *     given by the matching *_workspace_bytes query.
 *   - Indices are int32, values float32, leading dimensions in elements.
 *   - Launches are asynchronous and stream-ordered; nothing synchronises.
 *   - Return 0 on success, negative on error (STC_E*); the message is
 *     available from stc_last_error() (thread-local). No exceptions cross
 *     the ABI. There is no CPU fallback.
 *   - Results are deterministic: no atomics; every output row is reduced in
 *     a fixed order.
 */
#ifndef STC_H_
#define STC_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STC_ABI_VERSION 3  /* 2: L2-persisting entry points removed, stc_fsum_segments_f64 added; 3: prepared-item MTTKRP */

#define STC_OK 0
#define STC_EINVAL (-1)       /* null / misaligned pointer, bad shape        */
#define STC_EUNSUPPORTED (-2) /* shape or variant not supported             */
#define STC_ELAUNCH (-3)      /* CUDA launch error (cudaGetLastError)       */
#define STC_EWORKSPACE (-4)   /* workspace too small                        */

/* SpMM kernel variants — the device form of the reference planner's choice
 * of loop order and tiling (scheduler.py:347, tiling.py:53):
 *   ROW     one sub-warp per row (loop order [i,j,k], rows uniform)
 *   MERGE   nnz-balanced merge-path split with atomics-free carries
 *           (same loop order, power-law rows)
 *   COLTILE column-tiled, dense operand staged in shared memory and
 *           Tensor Memory (tile set {k} with a wide k)                                    */
#define STC_VARIANT_ROW 0
#define STC_VARIANT_MERGE 1
#define STC_VARIANT_COLTILE 2

#define STC_EPILOGUE_NONE 0
#define STC_EPILOGUE_RELU 1

#define STC_EWISE_UNION 0     /* C = A + B over the union of patterns        */
#define STC_EWISE_INTERSECT 1 /* C = A .* B over the intersection            */

int stc_abi_version(void);
const char* stc_last_error(void);

/* Number of kernels this library has launched in the process (all threads).
 * Used by bench.py to report how many native launches a timed region made. */
long long stc_launch_count(void);


/* Merge-path partition of a compressed row structure (plan time).
 * Groups own `items_per_group` consecutive items of the merged sequence
 * (m row ends weighing 2 items each — a row flush costs about two gathers —
 * and nnz entries of 1 item; a group owns the items starting in its range).
 * Writes (row, pos) int pairs for groups 0..n_groups into `starts`
 * (2*(n_groups+1) ints).                                                     */
long long stc_merge_path_groups(int m, long long nnz, int items_per_group);
int stc_merge_path_partition(int m, long long nnz, const int* rowptr, int items_per_group,
                             int* starts, void* stream);

/* Plan-time interleaving of long rows for the MERGE variant: writes a copy of
 * (colidx, vals) in which every row longer than `span` entries (the span of one
 * merge group, i.e. items_per_group) is stored as G = ceil(len / span) interleaved
 * sequences (entries 0, G, 2G, ..., then 1, G + 1, ...); shorter rows are copied.
 * A group covering part of a hub row then gathers from the whole row's column
 * range (hot and cold columns alike) instead of one sorted slice of it. Feed the
 * copy to stc_spmm_csr_f32 (same rowptr); the row sums change only in order.   */
int stc_merge_interleave(int m, long long nnz, const int* rowptr, const int* colidx, const float* vals,
                         int span, int* colidx_out, float* vals_out, void* stream);

/* Plan-time choice of items_per_group for the MERGE variant: the merged
 * sequence is cut into exactly enough groups to fill whole waves of resident
 * CTAs on this device (one wave when a group's staging window allows), so no
 * partial last wave idles SMs. `kind` 0 = SpMM, 1 = MTTKRP.                  */
int stc_merge_plan_items_per_group(int m, long long nnz, int k, int batch, int kind);

/* Plan of the COLTILE variant (B operand staged in Tensor Memory): A re-encoded
 * per (224-row block, 63-column chunk, row) as packed {Tensor Memory address
 * of the operand row, value} entries, each row padded to an even count with a
 * zero-weight entry on an all-zero operand slot (the layout is private to the
 * kernel). The kernel stages B through a tiled TMA copy: it builds a tensor
 * map of B per launch (B and its pitch must be 16-byte aligned, as for every
 * vectorised variant); the encoder is a driver entry point fetched through the
 * runtime, and when it is unavailable -- or STC_COLTILE_ROW_COPIES=1 is set in
 * the environment, a test hook -- B is staged by one bulk copy per row instead
 * (same results, slower).
 * The plan CARRIES A's VALUES (the prepared form of A, like a cuSPARSE SpMM
 * preprocess): rebuild it whenever the values change. stc_coltile_plan_ints
 * gives its size in int32 (-1 if unsupported); pass it as the `partition` of a
 * COLTILE SpMM with the same m, n, nnz (colidx / vals are then not read).    */
long long stc_coltile_plan_ints(int m, int n, long long nnz);
int stc_coltile_plan(int m, int n, long long nnz, const int* rowptr, const int* colidx, const float* vals,
                     int* plan, long long plan_ints, void* stream);

/* Workspace for the MERGE variant (carry buffers + per-CTA arrival counters);
 * 0 for ROW/COLTILE. It must be ZERO-FILLED once when allocated; every launch
 * leaves the counters at zero again.                                        */
size_t stc_spmm_workspace_bytes(int m, long long nnz, int k, int variant, int items_per_group,
                                int batch);

/* CSR SpMM  C[i,:] = act(sum_{p in row i} vals[p] * B[colidx[p], :] + D[i,:])
 * Replaces the dense-output driver + vectorised tail of the reference,
 * engine.py:487-573 (`_run_dense_output`, `vector_sink`), for
 * C(i,k) = A(i,j) * B(j,k) [+ D(i,k)] with A CSR, B/D dense.
 * B of any size: below 2^32 elements the gathers use prepared 32-bit offsets,
 * at or above it 64-bit addresses (same walk and summation order).
 * n = columns of A (rows of B); D nullable; `partition` = the merge-path
 * starts for MERGE, the chunk plan for COLTILE, ignored for ROW.            */
int stc_spmm_csr_f32(int m, int n, int k, const int* rowptr, const int* colidx, const float* vals,
                     long long nnz, const float* B, long long ldb, float* C, long long ldc,
                     const float* D, long long ldd, int variant, int epilogue, const int* partition,
                     int items_per_group, void* ws, size_t ws_bytes, void* stream);

/* Batched CSR SpMM over a shared structure (multi-head O(h,i,d)=P(h,i,j)*V(h,j,d),
 * reference plan [dense,dense,compressed] x dense, engine.py:487-573):
 * per batch z the values start at vals + z*val_bstride, B at B + z*b_bstride,
 * C (and D) at C + z*c_bstride.                                              */
int stc_spmm_csr_batched_f32(int batch, int m, int n, int k, const int* rowptr, const int* colidx,
                             const float* vals, long long nnz, long long val_bstride,
                             const float* B, long long ldb, long long b_bstride, float* C,
                             long long ldc, long long c_bstride, int variant, int epilogue,
                             const int* partition, int items_per_group, void* ws, size_t ws_bytes,
                             void* stream);

/* Distinct-row segmentation of a sorted COO row column (plan time):
 * seg_rows[s] = s-th distinct row, seg_ptr[s] = its first entry,
 * seg_ptr[n_seg] = nnz; *n_seg_out (device int) = number of segments.
 * This is the compressed i-level the reference builds for a COO/DCSR SpMM
 * or MTTKRP output (`_SparseOutputBuilder`, engine.py:233-253).             */
size_t stc_coo_segments_temp_bytes(long long nnz);
int stc_coo_segments(long long nnz, const int* rows, int* seg_rows, int* seg_ptr, int* n_seg_out,
                     void* temp, size_t temp_bytes, void* stream);

/* COO SpMM over precomputed segments: C[s,:] = sum_{p in seg s} vals[p]*B[cols[p],:].
 * Output is the dense level of the reference's [compressed, dense] result
 * (engine.py:577-644 with a 1-D Workspace, engine.py:71-90).                */
int stc_spmm_coo_f32(int n_seg, int n, int k, const int* seg_ptr, const int* cols,
                     const float* vals, long long nnz, const float* B, long long ldb, float* C,
                     long long ldc, int variant, const int* partition, int items_per_group, void* ws,
                     size_t ws_bytes, void* stream);

/* SDDMM  S[h,p] = scale * maskvals[p] * dot(Q[h,i,:], K[h,colidx[p],:])
 * (maskvals nullable = 1.0). Replaces `_run_sparse_output` + the vectorised
 * reduction tail, engine.py:577-644 and :413-432, for
 * S(i,j) = M(i,j) * Q(i,d) * K(j,d). d in {4,8,16,32,64,128}.               */
int stc_sddmm_csr_f32(int m, int n, int d, int heads, const int* rowptr, const int* colidx,
                      const float* maskvals, long long nnz, const float* Q, long long q_hs,
                      long long q_rs, const float* K, long long k_hs, long long k_rs, float scale,
                      float* out_vals, void* stream);

/* Row-segmented softmax of each row's stored values, in place, for `heads`
 * consecutive [nnz] value arrays. No reference symbol (the grammar has only
 * + and *); restated in oracle/.                          */
int stc_segsoftmax_csr_f32(int m, int heads, const int* rowptr, long long nnz, float* vals,
                           void* stream);

/* Fused sparse attention O = softmax_rows(scale * M .* (Q K^T)) V with an
 * online softmax; S and P (nullable) are written only when non-null
 * (parity mode). Composition of the three reference expressions SDDMM,
 * softmax and SpMM (engine.py:577-644, 487-573).                            */
int stc_sparse_attention_f32(int m, int n, int d, int heads, const int* rowptr, const int* colidx,
                             const float* maskvals, long long nnz, const float* Q, long long q_hs,
                             long long q_rs, const float* K, long long k_hs, long long k_rs,
                             const float* V, long long v_hs, long long v_rs, float scale, float* O,
                             long long o_hs, long long o_rs, float* S, float* P, void* stream);

/* Block-tiled fused attention (head dim 64) for masks with dense bands: the
 * plan (built by paper_2405_16883_b200.ops.attention_tile_plan) lists for every
 * 64-row block up to dt_max dense 64-column tiles (tile_cols, -1 padded) with
 * their mask values (tile_vals, NaN = absent) and a CSR remainder of all other
 * entries. Dense tiles run as register-tiled QK^T / PV on CUDA cores with an
 * online softmax; the remainder continues the same softmax per row.
 * Workspace: stc_attention_tiled_workspace_bytes(m, heads).                 */
size_t stc_attention_tiled_workspace_bytes(int m, int heads);
int stc_sparse_attention_tiled_f32(int m, int n, int d, int heads, int n_blocks, int dt_max, const int* tile_cols,
                                   const float* tile_vals, const int* rem_rowptr, const int* rem_colidx,
                                   const float* rem_vals, long long rem_nnz, const float* Q, long long q_hs,
                                   long long q_rs, const float* K, long long k_hs, long long k_rs, const float* V,
                                   long long v_hs, long long v_rs, float scale, float* O, long long o_hs,
                                   long long o_rs, void* ws, size_t ws_bytes, void* stream);

/* MTTKRP over a sorted COO 3-tensor, segmented by distinct i:
 * M[s,:] = sum_{p in seg s} (vals[p] * B[j[p],:]) * C[k[p],:], terms added in entry
 * order; B[j,:] is gathered once per run of equal j (an (i, j) fiber).
 * B has n_j rows, C has n_k rows (below 2^32 elements the gathers use prepared 32-bit
 * offsets, at or above it 64-bit addresses; any size that fits in memory).
 * Replaces `_run_sparse_output` with the (i,r) Workspace, engine.py:577-644,
 * 71-90, for M(i,r) = T(i,j,k) * B(j,r) * C(k,r).                           */
int stc_mttkrp_coo3_f32(int n_seg, int rank, const int* seg_ptr, const int* jcrd, const int* kcrd,
                        const float* vals, long long nnz, int n_j, const float* B, long long ldb,
                        int n_k, const float* C, long long ldcf, float* M, long long ldm, int variant,
                        const int* partition, int items_per_group, void* ws, size_t ws_bytes,
                        void* stream);

/* Prepared form of the same contraction (ABI 3). `stc_mttkrp_prepare_items` rewrites the
 * entry streams once, at plan time, as 16-byte items {element offset of B[j,:], element
 * offset of C[k,:], T, first-entry-of-an-(i,j)-fiber flag} for the given leading dimensions
 * (`items`: stc_mttkrp_items_bytes(nnz) bytes, 16-byte aligned; 32-bit offsets, so factors
 * below 2^32 elements). `stc_mttkrp_coo3_prepared_f32` then runs the merge-path reduction
 * with the items streamed through small per-group circular buffers by cp.async (no staging
 * round trips, and the SM keeps its L1 for the factor rows): same partition format, workspace
 * (stc_spmm_workspace_bytes with the MERGE variant), summation order and results as
 * stc_mttkrp_coo3_f32 with STC_VARIANT_MERGE. Call it with the ldb / ldcf the items were
 * prepared for; `stc_mttkrp_prepared_items_per_group` plans the partition granularity for
 * its kernel. Replaces the same loop nest, engine.py:577-644.                               */
size_t stc_mttkrp_items_bytes(long long nnz);
int stc_mttkrp_prepare_items(long long nnz, const int* jcrd, const int* kcrd, const float* vals, int n_j,
                             long long ldb, int n_k, long long ldcf, void* items, void* stream);
int stc_mttkrp_prepared_items_per_group(int n_seg, long long nnz, int rank);
int stc_mttkrp_coo3_prepared_f32(int n_seg, int rank, const int* seg_ptr, const void* items, long long nnz,
                                 int n_j, const float* B, long long ldb, int n_k, const float* C,
                                 long long ldcf, float* M, long long ldm, const int* partition,
                                 int items_per_group, void* ws, size_t ws_bytes, void* stream);

/* ---- device-side construction --------------------------
 * Exact duplicate folding: out[s] = fsum(vals[starts[s] .. starts[s+1])), the correctly
 * rounded float64 sum that Python's math.fsum returns (Shewchuk expansion + half-even
 * correction), bit for bit; replaces the reference's per-coordinate fsum in
 * build_from_entries (tensor.py:238-241). Where fsum raises, out[s] is a NaN with the
 * payload below (-inf + inf: ValueError; intermediate overflow: OverflowError).         */
#define STC_FSUM_INF_MINUS_INF 0x7ff8dead00000001LL
#define STC_FSUM_OVERFLOW 0x7ff8dead00000002LL
int stc_fsum_segments_f64(long long n_seg, const long long* starts, const double* vals, double* out,
                          void* stream);

/* ---- sparse x sparse on CSR operands ------------------
 * SpGEMM C(i,k) = A(i,j) * B(j,k), CSR x CSR -> CSR, replacing the reference's
 * workspace plan ([i,j,k], Workspace over k: engine.py:577-644, 71-90). Output
 * structure = every (i,k) reached by a product (arithmetic zeros are kept);
 * values = 0.0 + a_ij1*b_j1k + a_ij2*b_j2k + ... in ascending j (fp32).
 * Three phases, sizes read back by the caller between them:
 *   1. stc_spgemm_products: prod_ptr[m+1] = exclusive scan of per-row product
 *      counts; products = prod_ptr[m] (temp: stc_spgemm_products_temp_bytes).
 *   2. stc_spgemm_symbolic: writes c_rowptr[m+1] (workspace `ws` of
 *      stc_spgemm_workspace_bytes(m, p, products) bytes; p = columns of B).
 *   3. stc_spgemm_numeric: c_colidx / c_vals (c_rowptr[m] entries).
 * B with p <= 6144 columns: a per-warp SMEM accumulator over the whole output
 * row; wider B: expand, stable segmented sort, compress (products < 2^31).   */
size_t stc_spgemm_products_temp_bytes(int m);
int stc_spgemm_products(int m, const int* a_rowptr, const int* a_colidx, const int* b_rowptr,
                        long long* prod_ptr, void* temp, size_t temp_bytes, void* stream);
size_t stc_spgemm_workspace_bytes(int m, int p, long long products);
int stc_spgemm_symbolic(int m, int p, const int* a_rowptr, const int* a_colidx, const float* a_vals,
                        const int* b_rowptr, const int* b_colidx, const float* b_vals,
                        const long long* prod_ptr, long long products, void* ws, size_t ws_bytes,
                        int* c_rowptr, void* stream);
int stc_spgemm_numeric(int m, int p, const int* a_rowptr, const int* a_colidx, const float* a_vals,
                       const int* b_rowptr, const int* b_colidx, const float* b_vals, long long products,
                       void* ws, size_t ws_bytes, const int* c_rowptr, int* c_colidx, float* c_vals,
                       void* stream);

/* Element-wise CSR (same shape): STC_EWISE_UNION C = A + B (two terms, the
 * reference's _union_sorted, engine.py:224-230; value (0 + a) + b, or 0 + a /
 * 0 + b where only one side stores the coordinate), STC_EWISE_INTERSECT
 * C = A .* B (_intersect_sorted, engine.py:208-221; value 0 + a * b).
 * stc_csr_ewise_symbolic writes c_rowptr[m+1] (temp: stc_csr_ewise_temp_bytes);
 * stc_csr_ewise_f32 fills c_colidx / c_vals.                                  */
size_t stc_csr_ewise_temp_bytes(int m);
int stc_csr_ewise_symbolic(int op, int m, const int* a_rowptr, const int* a_colidx, const int* b_rowptr,
                           const int* b_colidx, int* c_rowptr, void* temp, size_t temp_bytes, void* stream);
int stc_csr_ewise_f32(int op, int m, const int* a_rowptr, const int* a_colidx, const float* a_vals,
                      const int* b_rowptr, const int* b_colidx, const float* b_vals, const int* c_rowptr,
                      int* c_colidx, float* c_vals, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STC_H_ */
