// Shared device/host helpers for the fp64 tensor-Chebyshev engine (sm_100a).
//
// Layout vocabulary used across the kernels:
//   * "dense tensor"  : C-order (n_1, ..., n_J) fp64, node / coefficient index l_J fastest
//                       (the reference's CoefTensor.coefficients layout, S/chebnd.py:33-54).
//   * "eval layout"   : the same coefficients viewed as a matrix (R, K) where the trailing q
//                       modes are merged into K = n_{J-q+1}...n_J and the leading J-q modes into
//                       R rows; rows are padded to Kp = roundup(K, 4) columns and the row count to
//                       R8 = roundup(R, 8), all padding zero.  This is the operand layout of the
//                       DMMA evaluator (K2) and is what the build (K1) writes.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cb {

constexpr int kMaxDims = 12;

// Status block written by kernels (device) and decoded by the host shim.
//   w[0] : non-finite input seen (count, saturating)
//   w[1] : domain violation seen (|x| > 1 + CLAMP_TOL)
//   w[2..3] : bit pattern of the worst |x| among violators (atomicMax on the u64 image)
struct Status {
  unsigned int nonfinite;
  unsigned int domain;
  unsigned long long worst_bits;
};

// S/cheb1d.py:22  CLAMP_TOL
constexpr double kClampTol = 1e-12;

// Division by a runtime-invariant unsigned divisor (Granlund-Montgomery, 32-bit numerators).
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  FastDiv() = default;
  __host__ explicit FastDiv(uint32_t div) : d(div) {
    uint32_t l = 0;
    while ((1ull << l) < div) ++l;
    s = l;
    m = static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - div)) / div + 1ull);
    if (div == 1) { m = 0; s = 0; }
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    uint64_t t = __umulhi(x, m);
    return static_cast<uint32_t>((t + x) >> s);
  }
  __device__ __forceinline__ void divmod(uint32_t x, uint32_t& q, uint32_t& r) const {
    q = div(x);
    r = x - q * d;
  }
};

// Clamp a reference-variable coordinate the way clamp_reference does (S/cheb1d.py:127-135):
// non-finite or |x| > 1 + tol flags the status block; the value is clipped to [-1, 1].
__device__ __forceinline__ double clamp_ref(double x, Status* st) {
  double ax = fabs(x);
  if (!isfinite(x)) {
    if (st) atomicAdd(&st->nonfinite, 1u);
    return 0.0;
  }
  if (ax > 1.0 + kClampTol && st) {
    atomicAdd(&st->domain, 1u);
    atomicMax(&st->worst_bits, static_cast<unsigned long long>(__double_as_longlong(ax)));
  }
  return fmin(1.0, fmax(-1.0, x));
}

// Entry M0[l][k] of the node-samples -> coefficients matrix (S/solver.py:162-171, the matrix form
// of cheb_transform S/cheb1d.py:138-170):  s_l * w_k * cos(pi * l * k / N), s = (1/N, 2/N, ...,
// 2/N, 1/N), w = (1/2, 1, ..., 1, 1/2).  The cosine argument is reduced exactly in integers to
// [0, pi/2] so that the mirrored entries used by the even/odd fold are exact negatives and the
// entries at l*k = N/2 (mod N) are exact zeros.
__host__ __device__ inline double transform_entry(int l, int k, int N) {
  if (N == 0) return 1.0;
  long long m = (static_cast<long long>(l) * k) % (2LL * N);   // angle pi*m/N, m in [0, 2N)
  if (m > N) m = 2LL * N - m;                                   // cos symmetric about pi
  double sign = 1.0;
  if (2 * m > N) { m = N - m; sign = -1.0; }                    // cos(pi - a) = -cos(a)
  double c;
  if (2 * m == N) c = 0.0;
  else {
#ifdef __CUDA_ARCH__
    c = cospi(static_cast<double>(m) / static_cast<double>(N));
#else
    c = cos(3.141592653589793238462643383279502884 * static_cast<double>(m) / static_cast<double>(N));
#endif
  }
  double s = (l == 0 || l == N) ? 1.0 / N : 2.0 / N;
  double w = (k == 0 || k == N) ? 0.5 : 1.0;
  return sign * c * s * w;
}

// T_l(x) for l = 0..n-1 by the three-term recurrence (S/chebnd.py:135-144, _row_basis).
__device__ __forceinline__ void cheb_row(double x, int n, double* out, int stride) {
  double t0 = 1.0, t1 = x;
  if (n > 0) out[0] = 1.0;
  if (n > 1) out[stride] = x;
  double x2 = 2.0 * x;
  for (int l = 2; l < n; ++l) {
    double t2 = fma(x2, t1, -t0);
    out[l * stride] = t2;
    t0 = t1;
    t1 = t2;
  }
}

}  // namespace cb
