// Collocation solver on the device: the Bellman sweep, the safeguarded
// Newton maximiser and the fixed-point driver of the reference solver (S/solver.py).
//
// One warp per (player i, state node p) runs the whole best response of _best_response_block
// (S/solver.py:359-409) for that node:
//   1. bind the other players' current controls in the control-space drift stacks
//      (Step 1, :374-379) -> the drift polynomial in the player's own control, (K, J);
//   2. drift at the K own-control nodes, Euler successor, clip to the state box, clamp count
//      (:382-386), one lane per own-control node;
//   3. the player's value interpolant at the successor (:389-397) — nested accumulation over the
//      state modes, dim 1 innermost, exactly the reference's binding order;
//   4. objective delta*(stage + v) (:399-401), the 1-D fit M0 @ objective (:404);
//   5. _maximise_block (:262-323): projected Newton on f', endpoints, and the 257-point scan +
//      60-step bisection fallback (the scan spread over the 32 lanes).
// The per-row maximiser follows numpy's arithmetic operation for operation (this file is
// compiled with -fmad=false; numpy's pairwise summation is reproduced), so on identical
// coefficient rows it is bitwise identical to the reference (tested).
//
// The driver (`solve`, :495-570) captures [sweep (+ convergence test by its last warp) -> refit
// (K1 transform)] pairs in a CUDA graph; the sup-norm change per player is reduced with atomicMax on the IEEE bits
// (non-negative doubles order like their bit patterns) and the stopping test runs on the device,
// so the host only polls a flag once per graph launch.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include "../../include/chebnash_b200.h"
#include "cb_common.cuh"
#include "cb_kernels.h"

namespace cb {

namespace {

constexpr int kSweepWarps = 4;
constexpr int kSolverMaxJ = CB_MAX_PLAYERS;
constexpr int kKMax = CB_MAX_CONTROL_NODES;
constexpr int kSolverMaxN = 64;  // state nodes per dimension
constexpr int kScanPoints = 257;   // S/solver.py:52
constexpr int kBisect = 60;        // :53
constexpr int kNewtonIter = 30;    // :50
constexpr double kNewtonTol = 1e-12;  // :51

struct SolveCtl {
  long long it;          // next sweep index (0-based)
  long long max_iters;
  long long iterations;  // set when done
  int done;
  int converged;
  unsigned err;          // non-finite objective seen
  unsigned arrived;      // warps of the running sweep that finished (last one runs the stopping test)
};

struct SweepArgs {
  cb_game_t g;
  long long NP;
  const double* nodes;
  const double* drift;             // node-major drift tensors (cb_solver_drift_layout)
  long long dofs[kSolverMaxJ];     // per-player offsets into `drift`
  const double* coef;
  const double* v_old;
  const double* u_old;
  double* v_new;
  double* u_new;
  unsigned long long* clamp;      // single-sweep counter (solve: clamp_base[it])
  unsigned long long* hist_base;  // solve only: (max_iters, J) sup changes as IEEE bits
  unsigned long long* clamp_base;
  SolveCtl* ctl;                  // solve only
  Status* st;                     // single sweep: non-finite flag
  int coef_smem;                  // stage all J value tensors in shared memory (one L2 round trip)
  int drift_blk;                  // doubles per warp of the staged drift block (0: read from L2)
};

// numpy's pairwise summation for n <= 128 (umath loops: 8 partial sums, then a fixed tree).
__device__ double np_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = r + a[i];
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res = res + a[i];
  return res;
}

// _clenshaw_last (S/solver.py:226-236) for one row.
__device__ double clenshaw_row(const double* c, int L, double x) {
  if (L == 1) return c[0];
  const double x2 = 2.0 * x;
  double b1 = 0.0, b2 = 0.0;
  for (int k = L - 1; k >= 1; --k) {
    const double t = c[k] + x2 * b1 - b2;
    b2 = b1;
    b1 = t;
  }
  return c[0] + x * b1 - b2;
}

// derivative_array (S/cheb1d.py:230-249): p (L) -> q (L-1)
__device__ void deriv_row(const double* p, int L, double* q) {
  const int n = L - 1;
  q[n - 1] = 2.0 * n * p[n];
  if (n >= 2) q[n - 2] = 2.0 * (n - 1) * p[n - 1];
  for (int l = n - 3; l >= 0; --l) q[l] = q[l + 2] + 2.0 * (l + 1) * p[l + 1];
  q[0] *= 0.5;
}

__device__ __forceinline__ double np_sign(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : (v == 0.0 ? 0.0 : v)); }
__device__ __forceinline__ double clip1(double v) { return fmin(fmax(v, -1.0), 1.0); }

// 60 bisection steps on sign(f') (S/solver.py:252-257) as 12 rounds of a depth-5 speculative
// search: lane j (1..31) evaluates the midpoint of the bracket that sequential bisection would
// reach at heap node j, a ballot resolves five levels at once.  Every midpoint is formed by the
// same 0.5*(lo+hi) from the same brackets as the sequential loop, so lo/hi are bitwise identical.
template <typename F>
__device__ __forceinline__ void bisect_warp(F&& q1_at, double& lo, double& hi, double s_lo) {
  const int lane = threadIdx.x & 31;
  for (int round = 0; round < kBisect / 5; ++round) {
    bool same = false;
    if (lane >= 1) {
      double l = lo, h = hi;
      const int depth = 31 - __clz(lane);  // path bits below the leading one
      for (int b = depth - 1; b >= 0; --b) {
        const double mid = 0.5 * (l + h);
        if ((lane >> b) & 1) l = mid;
        else h = mid;
      }
      same = np_sign(q1_at(0.5 * (l + h))) == s_lo;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, same);
    int node = 1;
    for (int lev = 0; lev < 5; ++lev) {
      const double mid = 0.5 * (lo + hi);
      if ((mask >> node) & 1u) {
        lo = mid;
        node = 2 * node + 1;
      } else {
        hi = mid;
        node = 2 * node;
      }
    }
  }
}

// _maximise_block for one row held in shared memory (c, L); all 32 lanes call it and get the
// same (x, f).  q1 / q2: per-warp scratch (L-1, L-2).
__device__ void warp_maximise(const double* c, int L, double x0, bool always_scan, double* q1, double* q2,
                              double& x_out, double& f_out) {
  const int lane = threadIdx.x & 31;
  double alt[kKMax];
  for (int l = 0; l < L; ++l) alt[l] = (l & 1) ? -c[l] : c[l];
  const double f_hi = np_sum(c, L);
  const double f_lo = np_sum(alt, L);
  if (L <= 2) {
    x_out = (f_hi >= f_lo) ? 1.0 : -1.0;
    f_out = fmax(f_hi, f_lo);
    return;
  }
  if (lane == 0) {
    deriv_row(c, L, q1);
    deriv_row(q1, L - 1, q2);
  }
  __syncwarp();
  double x = clip1(x0);
  bool moving = true, failed = false;
  for (int it = 0; it < kNewtonIter; ++it) {
    const double f1 = clenshaw_row(q1, L - 1, x);
    const double f2 = clenshaw_row(q2, L - 2, x);
    const bool tiny = fabs(f2) <= 1e-300;
    const double raw = x - f1 / (tiny ? 1.0 : f2);
    const double xn = clip1(raw);
    if (moving && ((!tiny && raw != xn) || tiny)) failed = true;
    moving = moving && !tiny;
    const double dx = fabs(xn - x);
    if (moving) x = xn;
    moving = moving && (dx > kNewtonTol);
    if (!moving) break;
  }
  failed = failed || moving;
  failed = failed || (clenshaw_row(q2, L - 2, x) >= 0.0);
  if (always_scan) failed = true;
  double best_x = x, best_f = clenshaw_row(c, L, x);
  if (f_lo > best_f) {
    best_x = -1.0;
    best_f = f_lo;
  }
  if (f_hi > best_f) {
    best_x = 1.0;
    best_f = f_hi;
  }
  if (failed) {
    // dense scan over linspace(-1, 1, 257) (exact binary fractions), first maximum wins
    double bv = -INFINITY;
    int bj = kScanPoints;
    for (int j = lane; j < kScanPoints; j += 32) {
      const double xs = (j == kScanPoints - 1) ? 1.0 : -1.0 + j * (2.0 / (kScanPoints - 1));
      const double v = clenshaw_row(c, L, xs);
      if (v > bv || bj == kScanPoints) {
        bv = v;
        bj = j;
      }
    }
    for (int o = 16; o >= 1; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov > bv || (ov == bv && oj < bj)) {
        bv = ov;
        bj = oj;
      }
    }
    auto xs_at = [](int j) { return (j == kScanPoints - 1) ? 1.0 : -1.0 + j * (2.0 / (kScanPoints - 1)); };
    const double x_scan = xs_at(bj);
    double lo = xs_at(bj > 0 ? bj - 1 : 0);
    double hi = xs_at(bj < kScanPoints - 1 ? bj + 1 : kScanPoints - 1);
    const double s_lo = np_sign(clenshaw_row(q1, L - 1, lo));
    bisect_warp([&](double xm) { return clenshaw_row(q1, L - 1, xm); }, lo, hi, s_lo);
    const double x_ref = 0.5 * (lo + hi);
    const double x_fb = (clenshaw_row(c, L, x_ref) >= bv) ? x_ref : x_scan;
    double cf = clenshaw_row(c, L, x_fb);
    if (cf > best_f) {
      best_x = x_fb;
      best_f = cf;
    }
    cf = clenshaw_row(c, L, x_scan);
    if (cf > best_f) {
      best_x = x_scan;
      best_f = cf;
    }
  }
  x_out = best_x;
  f_out = best_f;
}

// Register-resident form of warp_maximise for a compile-time row length LT (3..16): the same
// operations in the same order (bitwise identical results), with the coefficient, derivative and
// second-derivative rows unrolled into registers instead of re-read from shared memory.
template <int LT>
__device__ __forceinline__ double clen_t(const double* c, double x) {
  if constexpr (LT == 1) {
    return c[0];
  } else {
    const double x2 = 2.0 * x;
    double b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int k = LT - 1; k >= 1; --k) {
      const double t = c[k] + x2 * b1 - b2;
      b2 = b1;
      b1 = t;
    }
    return c[0] + x * b1 - b2;
  }
}

template <int LT>
__device__ __forceinline__ double np_sum_t(const double* a) {
  if constexpr (LT < 8) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < LT; ++i) r = r + a[i];
    return r;
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    constexpr int full = LT - (LT % 8);
#pragma unroll
    for (int i = 8; i < full; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int i = full; i < LT; ++i) res = res + a[i];
    return res;
  }
}

template <int LT>
__device__ __forceinline__ void deriv_t(const double* p, double* q) {
  constexpr int n = LT - 1;
  q[n - 1] = 2.0 * n * p[n];
  if constexpr (n >= 2) q[n - 2] = 2.0 * (n - 1) * p[n - 1];
#pragma unroll
  for (int l = n - 3; l >= 0; --l) q[l] = q[l + 2] + 2.0 * (l + 1) * p[l + 1];
  q[0] *= 0.5;
}

template <int LT>
__device__ void warp_maximise_t(const double* cs, double x0, bool always_scan, double& x_out, double& f_out) {
  const int lane = threadIdx.x & 31;
  double c[LT], alt[LT], q1[LT - 1], q2[LT - 2];
#pragma unroll
  for (int l = 0; l < LT; ++l) {
    c[l] = cs[l];
    alt[l] = (l & 1) ? -c[l] : c[l];
  }
  const double f_hi = np_sum_t<LT>(c);
  const double f_lo = np_sum_t<LT>(alt);
  deriv_t<LT>(c, q1);
  deriv_t<LT - 1>(q1, q2);
  double x = clip1(x0);
  bool moving = true, failed = false;
  for (int it = 0; it < kNewtonIter; ++it) {
    const double f1 = clen_t<LT - 1>(q1, x);
    const double f2 = clen_t<LT - 2>(q2, x);
    const bool tiny = fabs(f2) <= 1e-300;
    const double raw = x - f1 / (tiny ? 1.0 : f2);
    const double xn = clip1(raw);
    if (moving && ((!tiny && raw != xn) || tiny)) failed = true;
    moving = moving && !tiny;
    const double dx = fabs(xn - x);
    if (moving) x = xn;
    moving = moving && (dx > kNewtonTol);
    if (!moving) break;
  }
  failed = failed || moving;
  failed = failed || (clen_t<LT - 2>(q2, x) >= 0.0);
  if (always_scan) failed = true;
  double best_x = x, best_f = clen_t<LT>(c, x);
  if (f_lo > best_f) {
    best_x = -1.0;
    best_f = f_lo;
  }
  if (f_hi > best_f) {
    best_x = 1.0;
    best_f = f_hi;
  }
  if (failed) {
    double bv = -INFINITY;
    int bj = kScanPoints;
    for (int j = lane; j < kScanPoints; j += 32) {
      const double xs = (j == kScanPoints - 1) ? 1.0 : -1.0 + j * (2.0 / (kScanPoints - 1));
      const double v = clen_t<LT>(c, xs);
      if (v > bv || bj == kScanPoints) {
        bv = v;
        bj = j;
      }
    }
    for (int o = 16; o >= 1; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov > bv || (ov == bv && oj < bj)) {
        bv = ov;
        bj = oj;
      }
    }
    auto xs_at = [](int j) { return (j == kScanPoints - 1) ? 1.0 : -1.0 + j * (2.0 / (kScanPoints - 1)); };
    const double x_scan = xs_at(bj);
    double lo = xs_at(bj > 0 ? bj - 1 : 0);
    double hi = xs_at(bj < kScanPoints - 1 ? bj + 1 : kScanPoints - 1);
    const double s_lo = np_sign(clen_t<LT - 1>(q1, lo));
    bisect_warp([&](double xm) { return clen_t<LT - 1>(q1, xm); }, lo, hi, s_lo);
    const double x_ref = 0.5 * (lo + hi);
    const double x_fb = (clen_t<LT>(c, x_ref) >= bv) ? x_ref : x_scan;
    double cf = clen_t<LT>(c, x_fb);
    if (cf > best_f) {
      best_x = x_fb;
      best_f = cf;
    }
    cf = clen_t<LT>(c, x_scan);
    if (cf > best_f) {
      best_x = x_scan;
      best_f = cf;
    }
  }
  x_out = best_x;
  f_out = best_f;
}

// row-length dispatch: registers for 3 <= L <= 16, the shared-memory form otherwise
__device__ void warp_maximise_any(const double* c, int L, double x0, bool always_scan, double* q1, double* q2,
                                  double& x_out, double& f_out) {
  switch (L) {
#define CB_MX(v) case v: warp_maximise_t<v>(c, x0, always_scan, x_out, f_out); return;
    CB_MX(3) CB_MX(4) CB_MX(5) CB_MX(6) CB_MX(7) CB_MX(8) CB_MX(9) CB_MX(10) CB_MX(11) CB_MX(12) CB_MX(13)
    CB_MX(14) CB_MX(15) CB_MX(16)
#undef CB_MX
    default: warp_maximise(c, L, x0, always_scan, q1, q2, x_out, f_out); return;
  }
}

// Value interpolant of one player at a point: coefficients with reversed axes (l_J, ..., l_1),
// i.e. dim 0 is the memory-fastest axis; nested accumulation, dim 0 innermost (the reference's
// binding order).  The innermost row runs in scalar registers; the outer levels (fixed-size arrays
// indexed by unrolled constants, so they stay in registers) are touched once per row.
__device__ double eval_reversed(const double* C, int J, const int* np, const double* pt) {
  double x2[kSolverMaxJ], t[kSolverMaxJ], tp[kSolverMaxJ], acc[kSolverMaxJ];
  int dig[kSolverMaxJ], nn[kSolverMaxJ];
  long long rows = 1;
#pragma unroll
  for (int d = 0; d < kSolverMaxJ; ++d) {
    const bool on = d < J;
    x2[d] = on ? 2.0 * pt[d] : 0.0;
    t[d] = 1.0;
    tp[d] = on ? pt[d] : 0.0;  // T_{-1} := x so that T_1 = 2x*T_0 - T_{-1} = x
    acc[d] = 0.0;
    dig[d] = 0;
    nn[d] = on ? np[d] : 1;
    if (on && d > 0) rows *= np[d];
  }
  const int n0 = nn[0];
  const double xx2 = x2[0], x0 = 0.5 * x2[0];
  double result = 0.0;
  for (long long row = 0; row < rows; ++row, C += n0) {
    double a0 = 0.0, t0 = 1.0, tp0 = x0;
    for (int l = 0; l < n0; ++l) {
      a0 = a0 + C[l] * t0;
      const double tn = xx2 * t0 - tp0;
      tp0 = t0;
      t0 = tn;
    }
    double v = a0;
    bool carry = true;
#pragma unroll
    for (int L = 1; L < kSolverMaxJ; ++L) {
      if (carry && L < J) {
        acc[L] = acc[L] + v * t[L];
        const double tn = x2[L] * t[L] - tp[L];
        tp[L] = t[L];
        t[L] = tn;
        if (++dig[L] < nn[L]) {
          carry = false;
        } else {
          v = acc[L];
          acc[L] = 0.0;
          dig[L] = 0;
          t[L] = 1.0;
          tp[L] = 0.5 * x2[L];
          if (L == J - 1) result = v;
        }
      }
    }
    if (J == 1) result = v;
  }
  return result;
}

// stopping test of solve (:551-556): sup-norm change below tol -> converged.  Run by the last
// warp of each sweep (after every warp's history update is visible).
__device__ void solve_finish(SolveCtl* ctl, const unsigned long long* hist_base, int J, double tol) {
  const long long it = ctl->it;
  ctl->it = it + 1;
  if (ctl->err) {
    ctl->done = 1;
    ctl->iterations = it + 1;
    return;
  }
  double dmax = 0.0;
  for (int i = 0; i < J; ++i) dmax = fmax(dmax, __longlong_as_double(static_cast<long long>(hist_base[it * J + i])));
  if (dmax < tol) {
    ctl->done = 1;
    ctl->converged = 1;
    ctl->iterations = it + 1;
  } else if (it + 1 >= ctl->max_iters) {
    ctl->done = 1;
    ctl->iterations = it + 1;
  }
}

__global__ void __launch_bounds__(kSweepWarps * 32) sweep_kernel(const __grid_constant__ SweepArgs a) {
  __shared__ double sT[kSweepWarps][kSolverMaxJ - 1][kKMax];   // bound players' basis rows
  __shared__ double sAcc[kSweepWarps][kKMax * kSolverMaxJ];      // drift polynomial (K, J)
  __shared__ double sObj[kSweepWarps][kKMax];
  __shared__ double sCoef[kSweepWarps][kKMax];
  __shared__ double sQ1[kSweepWarps][kKMax];
  __shared__ double sQ2[kSweepWarps][kKMax];
  __shared__ double sPt[kSweepWarps][kKMax][kSolverMaxJ];        // successor points (reference coords)
  __shared__ double sTv[kSweepWarps][kSolverMaxJ][kSolverMaxN];  // value basis rows of one successor
  extern __shared__ __align__(16) double sdyn[];
  const cb_game_t& g = a.g;
  const int J = g.J;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long task = static_cast<long long>(blockIdx.x) * kSweepWarps + warp;
  const bool done = a.ctl ? (a.ctl->done != 0) : false;  // grid-uniform
  if (done) {  // converged earlier in this graph launch: carry the fields forward
    if (task < J * a.NP && lane == 0) {
      const long long ip = task;
      a.v_new[ip] = a.v_old[ip];
      a.u_new[ip] = a.u_old[ip];
    }
    return;
  }
  // the value tensors of all players, staged once per block (coalesced)
  double* sC = sdyn;
  double* sD = sdyn + (a.coef_smem ? J * a.NP : 0);
  if (a.coef_smem) {
    for (long long e = threadIdx.x; e < J * a.NP; e += blockDim.x) sC[e] = __ldg(a.coef + e);
  }
  __syncthreads();
  if (task >= J * a.NP) return;
  const int i = static_cast<int>(task / a.NP);
  const long long p = task - static_cast<long long>(i) * a.NP;
  const long long ip = static_cast<long long>(i) * a.NP + p;
  const long long it = a.ctl ? a.ctl->it : 0;
  const int K = g.nu[i];
  const double u_scale = 2.0 / g.U_max;
  const double p_scale = 2.0 / g.P_max;

  // 1. basis rows of the bound players' current controls at this node (Step 1, :374-379)
  //    (small per-player arrays are indexed only by unrolled constants -> registers)
  int bsz[kSolverMaxJ - 1], bdim[kSolverMaxJ - 1];
  long long NB = 1;
#pragma unroll
  for (int t = 0; t < kSolverMaxJ - 1; ++t) {
    bdim[t] = t < i ? t : t + 1;
    bsz[t] = (t < J - 1) ? g.nu[bdim[t]] : 1;
    NB *= bsz[t];
  }
  // this node's drift block D_i[p] (NB, K, J), prefetched into shared memory while the basis rows
  // are formed
  const double* D = a.drift + a.dofs[i] + static_cast<long long>(p) * NB * K * J;
  if (a.drift_blk) {
    double* dst = sD + warp * a.drift_blk;
    for (long long e = lane; e < NB * K * J; e += 32) dst[e] = __ldg(D + e);
    D = dst;
  }
  if (lane < J - 1) {
    const int bd = lane < i ? lane : lane + 1;
    const int bs = g.nu[bd];
    const double x = a.u_old[static_cast<long long>(bd) * a.NP + p] * u_scale - 1.0;
    double* row = sT[warp][lane];
    row[0] = 1.0;
    if (bs > 1) row[1] = x;
    const double x2 = 2.0 * x;
    for (int l = 2; l < bs; ++l) row[l] = x2 * row[l - 1] - row[l - 2];
  }
  __syncwarp();
  // 2. bind: acc[l_own * J + comp] = sum over bound tuples b of prod T * D_i[p][b][l_own][comp];
  //    the node-major layout makes each b a contiguous (K, J) block: coalesced lane reads
  {
    const int KJ = K * J;
    for (int r = lane; r < KJ; r += 32) {
      int tt[kSolverMaxJ - 1];
#pragma unroll
      for (int t = 0; t < kSolverMaxJ - 1; ++t) tt[t] = 0;
      double acc = 0.0;
#pragma unroll 4
      for (int b = 0; b < static_cast<int>(NB); ++b) {
        double w = sT[warp][0][tt[0]];
#pragma unroll
        for (int t = 1; t < kSolverMaxJ - 1; ++t)
          if (t < J - 1) w = w * sT[warp][t][tt[t]];
        acc = acc + w * D[static_cast<long long>(b) * KJ + r];
        bool carry = true;  // next bound tuple (last bound player fastest)
#pragma unroll
        for (int t = kSolverMaxJ - 2; t >= 0; --t) {
          if (carry && t < J - 1) {
            if (++tt[t] < bsz[t]) carry = false;
            else tt[t] = 0;
          }
        }
      }
      sAcc[warp][r] = acc;
    }
  }
  __syncwarp();
  // 3. own-control node k = lane: drift, successor, value, objective
  unsigned clamped = 0;
  if (lane < K) {
    const int k = lane;
    const double rn = g.rnodes[i][k];
    double gk[kSolverMaxJ];
#pragma unroll
    for (int c = 0; c < kSolverMaxJ; ++c) gk[c] = 0.0;
    double T0 = 1.0, T1 = rn;
    for (int l = 0; l < K; ++l) {
      const double Tl = (l == 0) ? 1.0 : (l == 1 ? rn : (2.0 * rn) * T1 - T0);
      if (l >= 2) {
        T0 = T1;
        T1 = Tl;
      }
#pragma unroll
      for (int c = 0; c < kSolverMaxJ; ++c)
        if (c < J) gk[c] = gk[c] + Tl * sAcc[warp][l * J + c];
    }
#pragma unroll
    for (int c = 0; c < kSolverMaxJ; ++c) {
      if (c < J) {
        const double nxt = a.nodes[p * J + c] + g.h * gk[c];
        const double cl = fmin(fmax(nxt, 0.0), g.P_max);
        clamped += (cl != nxt) ? 1u : 0u;
        sPt[warp][k][c] = cl * p_scale - 1.0;
      }
    }
  }
  __syncwarp();
  // value interpolant at the K successors: one lane per point for small tensors; the whole warp
  // per point (flat coefficient index split over lanes, T tables in smem, shuffle reduction) when
  // the tensor has more than 128 coefficients
  double vnext = 0.0;
  const double* Ci = (a.coef_smem ? sC : a.coef) + static_cast<long long>(i) * a.NP;
  if (a.NP <= 128) {
    if (lane < K) vnext = eval_reversed(Ci, J, g.np, sPt[warp][lane]);
  } else {
    int d0[kSolverMaxJ], d32[kSolverMaxJ];
    {
      int r0 = lane, r32 = 32;
      for (int d = 0; d < J; ++d) {
        d0[d] = r0 % g.np[d];
        r0 /= g.np[d];
        d32[d] = r32 % g.np[d];
        r32 /= g.np[d];
      }
    }
    for (int k = 0; k < K; ++k) {
      if (lane < J) {
        const double x = sPt[warp][k][lane];
        double* row = sTv[warp][lane];
        row[0] = 1.0;
        if (g.np[lane] > 1) row[1] = x;
        const double x2 = 2.0 * x;
        for (int l = 2; l < g.np[lane]; ++l) row[l] = x2 * row[l - 1] - row[l - 2];
      }
      __syncwarp();
      int dg[kSolverMaxJ];
      for (int d = 0; d < J; ++d) dg[d] = d0[d];
      double part = 0.0;
      for (long long e = lane; e < a.NP; e += 32) {
        double w = sTv[warp][0][dg[0]];
        for (int d = 1; d < J; ++d) w = w * sTv[warp][d][dg[d]];
        part = part + w * Ci[e];
        int carry = 0;  // flat index += 32 in the mixed radix of the tensor
        for (int d = 0; d < J; ++d) {
          dg[d] += d32[d] + carry;
          carry = 0;
          while (dg[d] >= g.np[d]) {
            dg[d] -= g.np[d];
            ++carry;
          }
        }
      }
      for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == k) vnext = part;
      __syncwarp();
    }
  }
  if (lane < K) {
    const int k = lane;
    const double un = g.unodes[i][k];
    const double gain = un * (g.A[i] - 0.5 * un);
    const double xi = a.nodes[p * J + i];
    const double damage = 0.5 * g.phi[i] * (xi * xi);
    const double stage = g.h * (gain - damage);
    const double obj = g.delta * (stage + vnext);
    if (!isfinite(obj)) {
      if (a.ctl) atomicOr(&a.ctl->err, 1u);
      if (a.st) atomicOr(&a.st->nonfinite, 1u);
    }
    sObj[warp][k] = obj;
  }
  __syncwarp();
  // 4. 1-D fit in the own control: coef_l = sum_k M0[l][k] obj_k, M0 = diag(s) B^T diag(w)
  if (lane < K) {
    const int l = lane, n = K - 1;
    const double s = (l == 0 || l == n) ? 1.0 / n : 2.0 / n;
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
      const double rn = g.rnodes[i][k];
      double Tl = 1.0;
      if (l >= 1) {
        double t0 = 1.0, t1 = rn;
        const double r2 = 2.0 * rn;
        for (int m = 2; m <= l; ++m) {
          const double tn = r2 * t1 - t0;
          t0 = t1;
          t1 = tn;
        }
        Tl = t1;
      }
      const double w = (k == 0 || k == n) ? 0.5 : 1.0;
      acc = acc + (s * (Tl * w)) * sObj[warp][k];
    }
    sCoef[warp][l] = acc;
  }
  __syncwarp();
  // 5. maximise from the warm start
  double xb, fb;
  warp_maximise_any(sCoef[warp], K, a.u_old[ip] * u_scale - 1.0, false, sQ1[warp], sQ2[warp], xb, fb);
  for (int o = 16; o >= 1; o >>= 1) clamped += __shfl_xor_sync(0xffffffffu, clamped, o);
  if (lane == 0) {
    a.u_new[ip] = (xb + 1.0) * (0.5 * g.U_max);
    a.v_new[ip] = fb;
    unsigned long long* cl = a.ctl ? a.clamp_base + it : a.clamp;
    if (cl && clamped) atomicAdd(cl, static_cast<unsigned long long>(clamped));
    if (a.ctl) {
      const double d = fabs(fb - a.v_old[ip]);
      atomicMax(a.hist_base + it * J + i, static_cast<unsigned long long>(__double_as_longlong(d)));
      __threadfence();
      if (atomicAdd(&a.ctl->arrived, 1u) == static_cast<unsigned>(J * a.NP) - 1u) {
        __threadfence();
        a.ctl->arrived = 0;
        solve_finish(a.ctl, a.hist_base, J, g.tol);
      }
    }
  }
}

__global__ void solve_init_kernel(SolveCtl* ctl, long long max_iters) {
  ctl->it = 0;
  ctl->max_iters = max_iters;
  ctl->iterations = 0;
  ctl->done = 0;
  ctl->converged = 0;
  ctl->err = 0;
}

__global__ void maximise_rows_kernel(long long m, int L, const double* coef, const double* x0, double* x, double* f,
                                     int always_scan) {
  __shared__ double sC[kSweepWarps][kKMax];
  __shared__ double sQ1[kSweepWarps][kKMax];
  __shared__ double sQ2[kSweepWarps][kKMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long row = static_cast<long long>(blockIdx.x) * kSweepWarps + warp;
  if (row >= m) return;
  if (lane < L) sC[warp][lane] = coef[row * L + lane];
  __syncwarp();
  double xb, fb;
  warp_maximise_any(sC[warp], L, x0[row], always_scan != 0, sQ1[warp], sQ2[warp], xb, fb);
  if (lane == 0) {
    x[row] = xb;
    f[row] = fb;
  }
}


// Closed-loop rollouts (simulate, S/solver.py:597-629): one warp per trajectory.  Per step the
// lanes share the policy evaluation (flat coefficient index split across lanes, weights from
// per-dim T tables in shared memory, warp-shuffle reduction), then lane 0 clips the controls,
// records the row and takes the clipped Euler step of the drift (S/game.py:140-168).
constexpr int kSimWarps = 4;
constexpr int kSimMaxN = 64;

__global__ void __launch_bounds__(kSimWarps * 32) simulate_kernel(const __grid_constant__ cb_game_t g, long long B,
                                                                  const double* __restrict__ pol,
                                                                  const double* __restrict__ p0, long long n_steps,
                                                                  double* __restrict__ states,
                                                                  double* __restrict__ controls) {
  __shared__ double sT[kSimWarps][kSolverMaxJ][kSimMaxN];
  __shared__ double sP[kSimWarps][kSolverMaxJ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long b = static_cast<long long>(blockIdx.x) * kSimWarps + warp;
  if (b >= B) return;
  const int J = g.J;
  long long N = 1;
  for (int d = 0; d < J; ++d) N *= g.np[d];
  const double scale = 2.0 / g.P_max;
  double rowsum[kSolverMaxJ];
  for (int i = 0; i < J; ++i) {
    double s = 0.0;
    for (int j = 0; j < J; ++j) s = s + g.K[i][j];
    rowsum[i] = s;
  }
  if (lane < J) sP[warp][lane] = p0[b * J + lane];
  __syncwarp();
  for (long long t = 0; t <= n_steps; ++t) {
    // basis tables T_l(scale * p_d - 1)
    if (lane < J) {
      const double x = scale * sP[warp][lane] - 1.0;
      double* row = sT[warp][lane];
      row[0] = 1.0;
      if (g.np[lane] > 1) row[1] = x;
      const double x2 = 2.0 * x;
      for (int l = 2; l < g.np[lane]; ++l) row[l] = x2 * row[l - 1] - row[l - 2];
    }
    __syncwarp();
    double u[kSolverMaxJ];
    for (int i = 0; i < J; ++i) {
      const double* C = pol + static_cast<long long>(i) * N;
      double acc = 0.0;
      for (long long e = lane; e < N; e += 32) {
        long long rem = e;
        double w = 1.0;
        for (int d = J - 1; d >= 0; --d) {
          const long long q = rem / g.np[d];
          w = w * sT[warp][d][rem - q * g.np[d]];
          rem = q;
        }
        acc = acc + w * C[e];
      }
      for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      u[i] = fmin(fmax(acc, 0.0), g.U_max);
    }
    if (lane == 0) {
      double* srow = states + (b * (n_steps + 1) + t) * J;
      double* crow = controls + (b * (n_steps + 1) + t) * J;
      double p[kSolverMaxJ];
      for (int d = 0; d < J; ++d) {
        p[d] = sP[warp][d];
        srow[d] = p[d];
        crow[d] = u[d];
      }
      if (t < n_steps) {
        for (int i = 0; i < J; ++i) {
          double ex = 0.0;
          for (int j = 0; j < J; ++j) ex = ex + p[j] * g.K[i][j];
          const double gi = (ex - p[i] * rowsum[i]) / g.m[i] - g.c[i] * p[i] + g.beta[i] * u[i];
          sP[warp][i] = fmin(fmax(p[i] + g.h * gi, 0.0), g.P_max);
        }
      }
    }
    __syncwarp();
  }
}


// Node-major drift tensors D_i[p][b][l_own][comp] (the reference's _PlayerWork.coeffs layout,
// S/solver.py:183-189) from the J control-space stacks (nu_1..nu_J, N_P): one thread per element.
__global__ void drift_layout_kernel(const __grid_constant__ cb_game_t g, long long NP, const double* __restrict__ stacks,
                                    double* __restrict__ drift, int i, long long total) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int J = g.J, K = g.nu[i];
  long long rem = e;
  const int comp = static_cast<int>(rem % J);
  rem /= J;
  const int lown = static_cast<int>(rem % K);
  rem /= K;
  long long NB = 1;
  for (int j = 0; j < J; ++j)
    if (j != i) NB *= g.nu[j];
  long long b = rem % NB;
  const long long p = rem / NB;
  int l[kSolverMaxJ];
  l[i] = lown;
  for (int j = J - 1; j >= 0; --j) {
    if (j == i) continue;
    l[j] = static_cast<int>(b % g.nu[j]);
    b /= g.nu[j];
  }
  long long off = 0, selems = NP;
  for (int j = 0; j < J; ++j) {
    off = off * g.nu[j] + l[j];
    selems *= g.nu[j];
  }
  drift[e] = stacks[comp * selems + off * NP + p];
}


// Refit of small value fields in ONE launch (instead of one fiber pass per mode): block b
// transforms player b's node values (np_J, ..., np_1 as C order, dim 1 fastest) along every mode
// in shared memory with the unfolded DCT-I matrix (transform_entry, exact angle reduction) and
// writes the reversed-axis coefficient tensor.  Used when N_P <= 4096 and every np_d <= 64.
constexpr int kRefitThreads = 256;

__global__ void __launch_bounds__(kRefitThreads) refit_small_kernel(const __grid_constant__ cb_game_t g, long long NP,
                                                                    const double* __restrict__ v,
                                                                    double* __restrict__ coef) {
  extern __shared__ __align__(16) double rs[];
  double* A = rs;             // [NP]
  double* B = rs + NP;        // [NP]
  double* M = rs + 2 * NP;    // [64 * 64] matrix of the current mode
  const int i = blockIdx.x;
  for (long long e = threadIdx.x; e < NP; e += blockDim.x) A[e] = v[i * NP + e];
  long long stride = 1;  // element stride of dim d (dim 0 fastest)
  for (int d = 0; d < g.J; ++d) {
    const int n = g.np[d], N = n - 1;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) M[e] = transform_entry(e / n, e % n, N);
    __syncthreads();
    const long long fibers = NP / n;
    for (long long f = threadIdx.x; f < fibers * n; f += blockDim.x) {
      const long long fib = f / n;
      const int l = static_cast<int>(f - fib * n);
      const long long base = (fib / stride) * stride * n + (fib % stride);
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc = fma(M[l * n + k], A[base + k * stride], acc);
      B[base + l * stride] = acc;
    }
    __syncthreads();
    double* t = A;
    A = B;
    B = t;
    stride *= n;
  }
  for (long long e = threadIdx.x; e < NP; e += blockDim.x) coef[i * NP + e] = A[e];
}


// Closed-form linear-quadratic equilibrium (the reference's validation oracle, S/oracle.py:65-163):
// the exact Bellman update of quadratic values V_i = p'Q_i p + b_i'p + d_i and affine feedback
// u_i = e_i + f_i'p, iterated in coefficient space on one thread (J <= 8: a few hundred flops per
// update).  State vector: [Q (J,J,J)][b (J,J)][d (J)][e (J)][f (J,J)].
struct LQOut {
  long long iterations;
  int status;  // 0 ok, 1 interior maximisation not concave, 2 no fixed point within max_iters
  int pad;
};

__device__ int lq_update(const cb_game_t& g, const double* Q, const double* b, const double* d, const double* e,
                         const double* f, double* Qn, double* bn, double* dn, double* en, double* fn) {
  const int J = g.J;
  const double h = g.h, delta = g.delta;
  double D[kSolverMaxJ][kSolverMaxJ];
  for (int r = 0; r < J; ++r) {
    double rs = 0.0;
    for (int c = 0; c < J; ++c) rs = rs + g.K[r][c];
    for (int c = 0; c < J; ++c) D[r][c] = (g.K[r][c] - (r == c ? rs : 0.0)) / g.m[r] - (r == c ? g.c[r] : 0.0);
  }
  for (int i = 0; i < J; ++i) {
    const double* Qi = Q + i * J * J;
    const double* bi = b + i * J;
    double M[kSolverMaxJ][kSolverMaxJ], w[kSolverMaxJ], z[kSolverMaxJ];
    for (int r = 0; r < J; ++r) {
      const double Er = (r != i) ? e[r] : 0.0;
      w[r] = h * g.beta[r] * Er;
      z[r] = (r == i) ? h * g.beta[i] : 0.0;
      for (int c = 0; c < J; ++c) {
        const double Frc = (r != i) ? f[r * J + c] : 0.0;
        M[r][c] = (r == c ? 1.0 : 0.0) + h * (D[r][c] + g.beta[r] * Frc);
      }
    }
    // z'Qi z, z'Qi (row vector), Qi w
    double zQ[kSolverMaxJ], Qw[kSolverMaxJ];
    for (int c = 0; c < J; ++c) {
      double s1 = 0.0, s2 = 0.0;
      for (int r = 0; r < J; ++r) {
        s1 = s1 + z[r] * Qi[r * J + c];
        s2 = s2 + Qi[c * J + r] * w[r];
      }
      zQ[c] = s1;
      Qw[c] = s2;
    }
    double zQz = 0.0;
    for (int c = 0; c < J; ++c) zQz = zQz + zQ[c] * z[c];
    const double denom = h - 2.0 * zQz;
    if (!(denom > 0.0)) return 1;
    double t = 0.0;
    for (int r = 0; r < J; ++r) t = t + z[r] * (2.0 * Qw[r] + bi[r]);
    const double e_new = (h * g.A[i] + t) / denom;
    double f_new[kSolverMaxJ];
    for (int c = 0; c < J; ++c) {
      double s = 0.0;
      for (int r = 0; r < J; ++r) s = s + (2.0 * zQ[r]) * M[r][c];
      f_new[c] = s / denom;
    }
    double Mt[kSolverMaxJ][kSolverMaxJ], wt[kSolverMaxJ];
    for (int r = 0; r < J; ++r) {
      wt[r] = w[r] + e_new * z[r];
      for (int c = 0; c < J; ++c) Mt[r][c] = M[r][c] + z[r] * f_new[c];
    }
    // Qn_i = delta * (h * stage_quad + Mt' Qi Mt), symmetrised
    double QM[kSolverMaxJ][kSolverMaxJ];
    for (int r = 0; r < J; ++r)
      for (int c = 0; c < J; ++c) {
        double s = 0.0;
        for (int k = 0; k < J; ++k) s = s + Qi[r * J + k] * Mt[k][c];
        QM[r][c] = s;
      }
    double* Qo = Qn + i * J * J;
    for (int r = 0; r < J; ++r)
      for (int c = 0; c < J; ++c) {
        double s = 0.0;
        for (int k = 0; k < J; ++k) s = s + Mt[k][r] * QM[k][c];
        double sq = -0.5 * f_new[r] * f_new[c];
        if (r == i && c == i) sq -= 0.5 * g.phi[i];
        Qo[r * J + c] = delta * (h * sq + s);
      }
    for (int r = 0; r < J; ++r)
      for (int c = r + 1; c < J; ++c) {
        const double a = 0.5 * (Qo[r * J + c] + Qo[c * J + r]);
        Qo[r * J + c] = a;
        Qo[c * J + r] = a;
      }
    // bn_i = delta * (h (A_i - e_new) f_new + Mt' (2 Qi wt + bi))
    double v2[kSolverMaxJ];
    for (int r = 0; r < J; ++r) {
      double s = 0.0;
      for (int k = 0; k < J; ++k) s = s + Qi[r * J + k] * wt[k];
      v2[r] = 2.0 * s + bi[r];
    }
    for (int c = 0; c < J; ++c) {
      double s = 0.0;
      for (int k = 0; k < J; ++k) s = s + Mt[k][c] * v2[k];
      bn[i * J + c] = delta * (h * (g.A[i] - e_new) * f_new[c] + s);
    }
    double wQw = 0.0, bw = 0.0;
    for (int r = 0; r < J; ++r) {
      double s = 0.0;
      for (int k = 0; k < J; ++k) s = s + Qi[r * J + k] * wt[k];
      wQw = wQw + wt[r] * s;
      bw = bw + bi[r] * wt[r];
    }
    dn[i] = delta * (h * (g.A[i] * e_new - 0.5 * e_new * e_new) + wQw + bw + d[i]);
    en[i] = e_new;
    for (int c = 0; c < J; ++c) fn[i * J + c] = f_new[c];
  }
  return 0;
}

// mode 0: one update of `state`; mode 1: lq_solve from the zero value function (S/oracle.py:112-163)
__global__ void lq_kernel(const __grid_constant__ cb_game_t g, double* state, double* work, long long max_iters,
                          double tol, int mode, LQOut* res) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int J = g.J;
  const int nQ = J * J * J, nb = J * J;
  const int n = nQ + 2 * nb + 2 * J;
  double* cur = state;
  double* nxt = work;
  auto parts = [&](double* base, double*& Q, double*& b, double*& d, double*& e, double*& f) {
    Q = base;
    b = base + nQ;
    d = b + nb;
    e = d + J;
    f = e + J;
  };
  double *Q, *b, *d, *e, *f, *Qn, *bn, *dn, *en, *fn;
  parts(cur, Q, b, d, e, f);
  parts(nxt, Qn, bn, dn, en, fn);
  res->status = 0;
  res->iterations = 0;
  if (mode == 0) {
    res->status = lq_update(g, Q, b, d, e, f, Qn, bn, dn, en, fn);
    for (int k = 0; k < n; ++k) cur[k] = nxt[k];
    res->iterations = 1;
    return;
  }
  for (int k = 0; k < n; ++k) cur[k] = 0.0;
  for (int i = 0; i < J; ++i) e[i] = g.A[i];
  long long it = 1;
  bool settled = false;
  for (; it <= max_iters; ++it) {
    const int st = lq_update(g, Q, b, d, e, f, Qn, bn, dn, en, fn);
    if (st) {
      res->status = st;
      res->iterations = it;
      return;
    }
    double change = 0.0;
    for (int k = 0; k < nQ + nb; ++k) change = fmax(change, fabs(nxt[k] - cur[k]));
    for (int k = nQ + nb + J; k < n; ++k) change = fmax(change, fabs(nxt[k] - cur[k]));
    for (int k = 0; k < n; ++k) cur[k] = nxt[k];
    if (change < tol) {
      settled = true;
      break;
    }
  }
  if (!settled) {
    res->status = 2;
    res->iterations = max_iters;
    return;
  }
  // constant term: one update from d = 0, then d_i = d_once_i / (1 - delta)
  for (int i = 0; i < J; ++i) d[i] = 0.0;
  res->status = lq_update(g, Q, b, d, e, f, Qn, bn, dn, en, fn);
  for (int i = 0; i < J; ++i) d[i] = dn[i] / (1.0 - g.delta);
  res->iterations = it;
}

long long nodes_of(const cb_game_t& g) {
  long long n = 1;
  for (int d = 0; d < g.J; ++d) n *= g.np[d];
  return n;
}

// per-player element counts / offsets of the node-major drift tensors
long long drift_offsets(const cb_game_t& g, long long* dofs) {
  const long long NP = nodes_of(g);
  long long total = 0;
  for (int i = 0; i < g.J; ++i) {
    long long NB = 1;
    for (int j = 0; j < g.J; ++j)
      if (j != i) NB *= g.nu[j];
    if (dofs) dofs[i] = total;
    total += NP * NB * g.nu[i] * g.J;
  }
  return total;
}

constexpr int kSweepDynSmem = 160 * 1024;

cudaError_t launch_sweep(SweepArgs a, cudaStream_t s) {
  const long long tasks = a.g.J * a.NP;
  const long long blocks = (tasks + kSweepWarps - 1) / kSweepWarps;
  // shared-memory staging: all value tensors (<= 64 KB) and one drift block per warp (<= 24 KB),
  // used only while the grid still fits in one wave (static smem + staging per block, <= 4 blocks
  // per SM by registers); otherwise both are read from L2
  long long blk = 0;
  for (int i = 0; i < a.g.J; ++i) {
    long long NB = 1;
    for (int j = 0; j < a.g.J; ++j)
      if (j != i) NB *= a.g.nu[j];
    const long long b = NB * a.g.nu[i] * a.g.J;
    if (b > blk) blk = b;
  }
  const bool coef_ok = tasks * 8 <= 64 * 1024, drift_ok = blk * 8 <= 24 * 1024;
  const size_t dyn = (coef_ok ? tasks * 8 : 0) + (drift_ok ? blk * 8 * kSweepWarps : 0);
  const long long per_sm = std::min<long long>(4, (227 * 1024) / (44 * 1024 + static_cast<long long>(dyn)));
  const bool stage = blocks <= per_sm * num_sms();
  a.coef_smem = (stage && coef_ok) ? 1 : 0;
  a.drift_blk = (stage && drift_ok) ? static_cast<int>(blk) : 0;
  const size_t bytes = stage ? dyn : 0;
  ensure_smem_attr(reinterpret_cast<const void*>(sweep_kernel), kSweepDynSmem);
  sweep_kernel<<<static_cast<unsigned>(blocks), kSweepWarps * 32, bytes, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

// refit (S/solver.py:441-449): node values (J, N_P) viewed as (J, np_J, ..., np_1) -> reversed-axis
// coefficient tensors, one K1 transform over axes 1..J
cudaError_t refit(const cb_game_t& g, const double* v, double* coef, cudaStream_t s) {
  const long long NP = nodes_of(g);
  bool small = NP <= 4096;
  for (int d = 0; d < g.J; ++d) small = small && g.np[d] <= 64;
  if (small) {
    const size_t bytes = sizeof(double) * (2 * NP + 64 * 64);
    ensure_smem_attr(reinterpret_cast<const void*>(refit_small_kernel), static_cast<int>(bytes));
    refit_small_kernel<<<g.J, kRefitThreads, bytes, s>>>(g, NP, v, coef);
    count_launch();
    return cudaGetLastError();
  }
  long long shape[kSolverMaxJ + 1];
  shape[0] = g.J;
  for (int d = 0; d < g.J; ++d) shape[1 + d] = g.np[g.J - 1 - d];
  return transform_axes(g.J + 1, shape, 1, g.J + 1, v, coef, nullptr, 0, nullptr, s);
}

}  // namespace

cudaError_t bellman_sweep(const cb_game_t& g, const double* nodes, const double* drift, const double* coef,
                          const double* v, const double* u, double* v_out, double* u_out,
                          unsigned long long* clamped, Status* st, cudaStream_t stream) {
  SweepArgs a{};
  a.g = g;
  a.NP = nodes_of(g);
  a.nodes = nodes;
  a.drift = drift;
  drift_offsets(g, a.dofs);
  a.coef = coef;
  a.v_old = v;
  a.u_old = u;
  a.v_new = v_out;
  a.u_new = u_out;
  a.clamp = clamped;
  a.st = st;
  return launch_sweep(a, stream);
}

long long drift_elems(const cb_game_t& g) { return drift_offsets(g, nullptr); }

cudaError_t drift_layout(const cb_game_t& g, const double* stacks, double* drift, cudaStream_t stream) {
  const long long NP = nodes_of(g);
  long long dofs[kSolverMaxJ];
  drift_offsets(g, dofs);
  for (int i = 0; i < g.J; ++i) {
    long long NB = 1;
    for (int j = 0; j < g.J; ++j)
      if (j != i) NB *= g.nu[j];
    const long long total = NP * NB * g.nu[i] * g.J;
    drift_layout_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(g, NP, stacks, drift + dofs[i],
                                                                                      i, total);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

long long solve_work_bytes(const cb_game_t& g, long long max_iters) {
  return max_iters * g.J * 8 + max_iters * 8 + 64;
}

cudaError_t solve(const cb_game_t& g, const double* nodes, const double* drift, double* v, double* u, double* coef,
                  void* work, long long max_iters, long long* iterations, int* converged, int* nonfinite,
                  cudaStream_t stream) {
  const long long NP = nodes_of(g);
  const long long JN = g.J * NP;
  unsigned long long* hist = static_cast<unsigned long long*>(work);
  unsigned long long* clampc = hist + max_iters * g.J;
  SolveCtl* ctl = reinterpret_cast<SolveCtl*>(clampc + max_iters);
  cudaError_t e = cudaMemsetAsync(work, 0, static_cast<size_t>(solve_work_bytes(g, max_iters)), stream);
  if (e != cudaSuccess) return e;
  solve_init_kernel<<<1, 1, 0, stream>>>(ctl, max_iters);
  count_launch();
  e = refit(g, v, coef, stream);  // initial interpolants of buffer 0
  if (e != cudaSuccess) return e;

  SweepArgs a{};
  a.g = g;
  a.NP = NP;
  a.nodes = nodes;
  a.drift = drift;
  drift_offsets(g, a.dofs);
  a.hist_base = hist;
  a.clamp_base = clampc;
  a.ctl = ctl;
  // graph body: two sweeps (buffer 0 -> 1 -> 0), each followed by its refit and stopping test
  const int pairs = max_iters >= 256 ? 32 : static_cast<int>((max_iters + 1) / 2);
  cudaStream_t cs;
  e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const long long launches0 = launch_count();
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  for (int r = 0; r < pairs && e == cudaSuccess; ++r) {
    for (int half = 0; half < 2 && e == cudaSuccess; ++half) {
      const long long src = half * JN, dst = (1 - half) * JN;
      a.coef = coef + src;
      a.v_old = v + src;
      a.u_old = u + src;
      a.v_new = v + dst;
      a.u_new = u + dst;
      e = launch_sweep(a, cs);
      if (e == cudaSuccess) e = refit(g, v + dst, coef + dst, cs);
    }
  }
  cudaError_t e2 = cudaStreamEndCapture(cs, &graph);
  if (e == cudaSuccess) e = e2;
  const long long captured = launch_count() - launches0;  // counted once while capturing
  const long long per_launch = captured;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  SolveCtl h{};
  // the capture stream waits for the setup work on `stream`; results flow back the same way
  cudaEvent_t ev = nullptr;
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev, 0);
  long long launched = 0;
  while (e == cudaSuccess) {
    e = cudaGraphLaunch(exec, cs);
    if (e != cudaSuccess) break;
    launched += per_launch;
    e = cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess || h.done) break;
  }
  for (long long k = captured; k < launched; ++k) count_launch();  // graph replays run the same kernels
  if (e == cudaSuccess) e = cudaEventRecord(ev, cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, ev, 0);
  if (ev) cudaEventDestroy(ev);
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess) return e;
  *iterations = h.iterations;
  *converged = h.converged;
  *nonfinite = h.err ? 1 : 0;
  return cudaSuccess;
}

cudaError_t simulate(const cb_game_t& g, long long B, const double* policies, const double* p0, long long n_steps,
                     double* states, double* controls, cudaStream_t stream) {
  if (B <= 0) return cudaSuccess;
  const long long blocks = (B + kSimWarps - 1) / kSimWarps;
  simulate_kernel<<<static_cast<unsigned>(blocks), kSimWarps * 32, 0, stream>>>(g, B, policies, p0, n_steps, states,
                                                                               controls);
  count_launch();
  return cudaGetLastError();
}

cudaError_t lq(const cb_game_t& g, double* state, double* work, long long max_iters, double tol, int mode,
               long long* iterations, int* status, cudaStream_t stream) {
  LQOut* dres = reinterpret_cast<LQOut*>(work + (g.J * g.J * g.J + 2 * g.J * g.J + 2 * g.J));
  lq_kernel<<<1, 32, 0, stream>>>(g, state, work, max_iters, tol, mode, dres);
  count_launch();
  LQOut h{};
  cudaError_t e = cudaMemcpyAsync(&h, dres, sizeof(h), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  *iterations = h.iterations;
  *status = h.status;
  return cudaSuccess;
}

cudaError_t maximise_rows(long long m, int L, const double* coef, const double* x0, double* x, double* f,
                          int always_scan, cudaStream_t stream) {
  if (m <= 0) return cudaSuccess;
  const long long blocks = (m + kSweepWarps - 1) / kSweepWarps;
  maximise_rows_kernel<<<static_cast<unsigned>(blocks), kSweepWarps * 32, 0, stream>>>(m, L, coef, x0, x, f,
                                                                                       always_scan);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cb
