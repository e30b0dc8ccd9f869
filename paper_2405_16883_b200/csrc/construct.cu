// Device-side format construction helpers.
//
// Duplicate folding of build_from_entries / from_arrays: the reference sums the values of
// a repeated coordinate exactly, with Python's math.fsum (`/root/reference/pkg/src/
// sparsetc/tensor.py:238-241`), and stores the correctly rounded float64 result; this
// package then rounds that to float32 once. `stc_fsum_segments_f64` reproduces fsum on the
// device, one thread per group of equal coordinates, bit for bit: Shewchuk's exact
// floating-point expansion (every partial sum kept as non-overlapping doubles, TwoSum per
// component), then the round-half-even correction of the final summation step that
// CPython's fsum applies (the published msum algorithm). Non-finite inputs follow fsum's
// special sum: a NaN input gives NaN, an infinity the infinity. Where fsum raises, the
// group's result is a NaN with a reserved payload the host turns into the same exception:
// +Inf together with -Inf (ValueError "-inf + inf in fsum", STC_FSUM_INF_MINUS_INF) and an
// intermediate overflow of finite inputs (OverflowError, STC_FSUM_OVERFLOW).
#include <cmath>

#include "abi_util.cuh"
#include "stc_common.cuh"

namespace stc {

constexpr int kFsumPartials = 64;  // an exact double expansion needs at most ~40 components

__device__ double fsum_group(const double* __restrict__ v, long long a, long long b) {
  double p[kFsumPartials];
  int n = 0;
  double special = 0.0, inf_sum = 0.0;
  for (long long q = a; q < b; ++q) {
    double x = v[q];
    const double xsave = x;
    int i = 0;
    for (int j = 0; j < n; ++j) {
      double y = p[j];
      if (fabs(x) < fabs(y)) {
        const double t = x;
        x = y;
        y = t;
      }
      const double hi = __dadd_rn(x, y);
      const double lo = __dsub_rn(y, __dsub_rn(hi, x));
      if (lo != 0.0) p[i++] = lo;
      x = hi;
    }
    n = i;
    if (x != 0.0) {
      if (!isfinite(x)) {
        // a non-finite partial: intermediate overflow of finite inputs, or an Inf / NaN input
        if (isfinite(xsave)) return __longlong_as_double(STC_FSUM_OVERFLOW);
        if (isinf(xsave)) inf_sum += xsave;
        special += xsave;
        n = 0;
      } else if (n < kFsumPartials) {
        p[n++] = x;
      }
    }
  }
  if (special != 0.0) return isnan(inf_sum) ? __longlong_as_double(STC_FSUM_INF_MINUS_INF) : special;
  double hi = 0.0;
  if (n > 0) {
    double lo = 0.0;
    --n;
    hi = p[n];
    // sum the partials from the top, stopping at the first inexact step
    while (n > 0) {
      const double x = hi;
      const double y = p[--n];
      hi = __dadd_rn(x, y);
      const double yr = __dsub_rn(hi, x);
      lo = __dsub_rn(y, yr);
      if (lo != 0.0) break;
    }
    // round-half-even correction: if the remaining partials push the exact value past the
    // halfway point of the last rounding, step hi one ulp in their direction
    if (n > 0 && ((lo < 0.0 && p[n - 1] < 0.0) || (lo > 0.0 && p[n - 1] > 0.0))) {
      const double y = lo * 2.0;
      const double x = __dadd_rn(hi, y);
      const double yr = __dsub_rn(x, hi);
      if (y == yr) hi = x;
    }
  }
  return hi;
}

__global__ void fsum_segments_kernel(long long n_seg, const long long* __restrict__ starts,
                                     const double* __restrict__ v, double* __restrict__ out) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n_seg;
       s += (long long)gridDim.x * blockDim.x) {
    const long long a = starts[s], b = starts[s + 1];
    out[s] = (b - a == 1) ? v[a] : fsum_group(v, a, b);
  }
}

}  // namespace stc

extern "C" int stc_fsum_segments_f64(long long n_seg, const long long* starts, const double* vals, double* out,
                                     void* stream) {
  STC_NVTX("stc_fsum_segments_f64");
  if (n_seg < 0) return stc::fail(STC_EINVAL, "negative segment count");
  if (n_seg == 0) return STC_OK;
  if (!starts || !vals || !out) return stc::fail(STC_EINVAL, "null pointer");
  const long long blocks = std::min<long long>((n_seg + 255) / 256, 148LL * 32);
  stc::fsum_segments_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(n_seg, starts, vals,
                                                                                            out);
  return stc::check_launch("fsum_segments_kernel");
}
