/* stc_oracle.c — float64 C restatement of the reference engine's arithmetic.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * CPU-baseline leg of bench.py; never by the product package.
 *
 * Each function keeps the exact summation order of
 * /root/reference/pkg/src/sparsetc/engine.py so results are bit-identical to
 * sparsetc.execute (and to oracle/restate.py); build with -ffp-contract=off so
 * no multiply-add is fused. Rows are independent, so OpenMP splits rows.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* C[i,:] = sum over the row's entries, ascending position, from 0.0, of
 * a_ij * B[j,:] (engine.py:487-565, vector_sink :551-560); then + D, then ReLU.
 * rows [r0, r1) only (bounded samples). */
void orc_spmm_csr_f64(int64_t r0, int64_t r1, const int64_t* rowptr, const int64_t* colidx,
                      const double* vals, const double* B, int64_t k, const double* D, int relu,
                      double* C) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = r0; i < r1; ++i) {
    double* c = C + (i - r0) * k;
    for (int64_t x = 0; x < k; ++x) c[x] = 0.0;
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const double a = vals[p];
      const double* b = B + colidx[p] * k;
      for (int64_t x = 0; x < k; ++x) {
        const double t = a * b[x];
        c[x] = c[x] + t;
      }
    }
    if (D) {
      const double* d = D + i * k;
      for (int64_t x = 0; x < k; ++x) c[x] = c[x] + d[x];
    }
    if (relu)
      for (int64_t x = 0; x < k; ++x) c[x] = c[x] > 0.0 ? c[x] : 0.0;
  }
}

/* S[p] = m_p * sum_blocks( sum_{x in block} q[i,x]*k[j,x] ) with blocks of
 * `tile` (tile <= 0: one block), partial sums from 0.0 left to right
 * (engine.py:404-461). */
void orc_sddmm_csr_f64(int64_t m, const int64_t* rowptr, const int64_t* colidx, const double* maskvals,
                       const double* Q, const double* K, int64_t d, int64_t tile, double* S) {
  if (tile <= 0) tile = d;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < m; ++i) {
    const double* q = Q + i * d;
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const double* kk = K + colidx[p] * d;
      double total = 0.0;
      for (int64_t lo = 0; lo < d; lo += tile) {
        const int64_t hi = lo + tile < d ? lo + tile : d;
        double part = 0.0;
        for (int64_t x = lo; x < hi; ++x) {
          const double t = q[x] * kk[x];
          part = part + t;
        }
        total = total + part;
      }
      S[p] = (maskvals ? maskvals[p] : 1.0) * total;
    }
  }
}

/* Row softmax over each row's stored values: exp(s - max) / sum (no reference symbol). */
void orc_segsoftmax_f64(int64_t m, const int64_t* rowptr, const double* S, double* P) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < m; ++i) {
    const int64_t a = rowptr[i], b = rowptr[i + 1];
    if (a == b) continue;
    double mx = -INFINITY;
    for (int64_t p = a; p < b; ++p) mx = S[p] > mx ? S[p] : mx;
    double sum = 0.0;
    for (int64_t p = a; p < b; ++p) sum += exp(S[p] - mx);
    for (int64_t p = a; p < b; ++p) P[p] = exp(S[p] - mx) / sum;
  }
}

/* M[s,:] = sum over the segment's entries, in order, from 0.0, of
 * (t * B[j,:]) * C[k,:] (b_first) or (t * C[k,:]) * B[j,:] (engine.py:394-402, 81-83). */
void orc_mttkrp_f64(int64_t n_seg, const int64_t* seg_ptr, const int64_t* jc, const int64_t* kc,
                    const double* vals, const double* B, const double* C, int64_t R, int b_first,
                    double* M) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t s = 0; s < n_seg; ++s) {
    double* out = M + s * R;
    for (int64_t r = 0; r < R; ++r) out[r] = 0.0;
    for (int64_t p = seg_ptr[s]; p < seg_ptr[s + 1]; ++p) {
      const double t = vals[p];
      const double* b = B + jc[p] * R;
      const double* c = C + kc[p] * R;
      for (int64_t r = 0; r < R; ++r) {
        const double v = b_first ? (t * b[r]) * c[r] : (t * c[r]) * b[r];
        out[r] = out[r] + v;
      }
    }
  }
}
