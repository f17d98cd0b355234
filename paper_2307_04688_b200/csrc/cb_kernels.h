// Internal (C++) entry points shared between the kernel translation units and the C-ABI layer.
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "cb_common.cuh"
#include "../../include/chebnash_b200.h"

namespace cb {

// Largest mode size the C ABI accepts (degree 4095); modes above 34 / 128 take the generic paths.
constexpr int kMaxModeSize = 4096;

// make_basis nodes on [lo, hi] (S/cheb1d.py:97-103): descending, endpoints pinned exactly.
inline void make_nodes(double lo, double hi, long long n, double* out) {
  const long long N = n - 1;
  for (long long k = 0; k <= N; ++k) {
    double v;
    if (N == 0) v = 0.5 * (lo + hi);
    else if (k == 0) v = hi;
    else if (k == N) v = lo;
    else v = 0.5 * (hi - lo) * cos(3.141592653589793 * static_cast<double>(k) / static_cast<double>(N)) + 0.5 * (lo + hi);
    out[k] = v;
  }
}

// Eval layout of a J-mode coefficient tensor: the trailing q modes merged into K columns
// (padded to Kp, a multiple of 4), the leading J-q modes into R rows (padded to R8, a multiple
// of 8).  See cb_common.cuh and DESIGN.md §3.
struct EvalLayout {
  int J;
  long long n[kMaxDims];
  int q;
  long long R, R8, K, Kp;
  long long elems() const { return R8 * Kp; }
};

// Choose q (1..J) maximising the DMMA tile efficiency R*K / (R8*Kp) subject to the build's
// contiguous-tile budget; ties -> smaller q.
EvalLayout make_eval_layout(int J, const long long* n);

// Per-device one-time cudaFuncSetAttribute(MaxDynamicSharedMemorySize).
void ensure_smem_attr(const void* func, int bytes, bool max_carveout = false);
int num_sms();
// cuTensorMapEncodeTiled via the runtime's driver entry point (nullptr when unavailable).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
// Process-wide count of kernels launched by this library (reported as gpu_launches by bench.py).
void count_launch();
long long launch_count();

// K1 build / generic axis transform (cb_build.cu).
cudaError_t transform_axes(int ndim, const long long* shape, int a0, int a1, const double* in, double* out,
                           Status* st, int check_finite, const EvalLayout* evl, cudaStream_t stream);

// K2 scattered evaluator (cb_eval.cu).
struct AdvectSpec {
  long long node_begin;     // first flat node index (C order) evaluated by this call
  double A[kMaxDims * kMaxDims];  // drift g(x) = A x (row-major J x J), in interval units
  double dt;
  double lo[kMaxDims], hi[kMaxDims];  // state box per dim (the grid basis interval)
  int source;               // subtract dt*|x|^2 of the (unclipped) node
  int npeers;               // > 0: store results into peers[r][node] (full node-value buffers) instead of out
  double* peers[8];
  const double* node_tab;   // device node table [J][node_pitch] (required when a mode has > 64 nodes)
  int node_pitch;
};
const char* last_eval_plan();  // kernel / plan chosen by the last eval_points on this thread
// tensor_coeffs + eval_points in one call (one fused launch for small J = 2 tensors)
cudaError_t build_eval_points(const EvalLayout& L, const long long* shape, const double* values, long long M,
                              const double* points, double* out, double* coef, Status* st, cudaStream_t stream);
cudaError_t eval_points(const EvalLayout& L, const double* coef, long long M, const double* points,
                        const AdvectSpec* adv, double* out, Status* st, int force_generic, cudaStream_t stream);

// K3 / stack contractions (cb_axis.cu).
//   in  : dense (A, n, R, Q) ;  E : (k, n) row-major ;  out[a*oA + j*oJ + r*oR + q] .
cudaError_t contract_axis(long long A, int n, long long R, long long Q, int k, const double* E, const double* in,
                          double* out, long long oA, long long oJ, long long oR, cudaStream_t stream);
//   out[m*oM + r*oR] = sum_l T_l(x_m) in[m*sM + l*sL + r*sR]   (x_m clamped, status checked)
//   (W non-null: weights W[m*n + l] replace T_l(x_m); clamp: apply clamp_reference to x)
cudaError_t contract_diagonal(long long Mcount, int n, long long R, const double* x, const double* W, int clamp,
                              const double* in, long long sM, long long sL, long long sR, double* out, long long oM,
                              long long oR, Status* st, cudaStream_t stream);
cudaError_t derivative(long long rows, int L, const double* in, double* out, cudaStream_t stream);
// all J evaluation matrices of a structured evaluation in one launch: matrix d (k[d] x size[d])
// at out + sum_{j<d} k[j]*size[j]; points clamped (clamp_reference) into st
cudaError_t basis_matrices(int J, const long long* k, const double* const* x, const long long* size, double* out,
                           Status* st, cudaStream_t stream);
cudaError_t basis_matrix(long long k, const double* x, int size, double* out, Status* st, int clamp,
                         cudaStream_t stream);
cudaError_t gather_index(long long rest, long long count, long long* flat, cudaStream_t stream);
cudaError_t gather_take_f(int ndim_in, const long long* shape_in, const double* in, long long nsel, const long long* flat,
                          int ndim_out, const long long* shape_out, double* out, cudaStream_t stream);
// eval_grid: J successive rotating mode products with k_j x n_j evaluation matrices.
cudaError_t eval_grid(const EvalLayout& L, const double* coef, const long long* k, const double* const* E,
                      double* out, double* work, long long work_elems, cudaStream_t stream);
long long eval_grid_work_elems(const EvalLayout& L, const long long* k);

// Collocation solver (cb_solver.cu).
long long drift_elems(const cb_game_t& g);
cudaError_t drift_layout(const cb_game_t& g, const double* stacks, double* drift, cudaStream_t stream);
cudaError_t bellman_sweep(const cb_game_t& g, const double* nodes, const double* drift, const double* coef,
                          const double* v, const double* u, double* v_out, double* u_out,
                          unsigned long long* clamped, Status* st, cudaStream_t stream);
long long solve_work_bytes(const cb_game_t& g, long long max_iters);
cudaError_t solve(const cb_game_t& g, const double* nodes, const double* drift, double* v, double* u, double* coef,
                  void* work, long long max_iters, long long* iterations, int* converged, int* nonfinite,
                  cudaStream_t stream);
cudaError_t simulate(const cb_game_t& g, long long B, const double* policies, const double* p0, long long n_steps,
                     double* states, double* controls, cudaStream_t stream);
cudaError_t lq(const cb_game_t& g, double* state, double* work, long long max_iters, double tol, int mode,
               long long* iterations, int* status, cudaStream_t stream);
cudaError_t maximise_rows(long long m, int L, const double* coef, const double* x0, double* x, double* f,
                          int always_scan, cudaStream_t stream);

}  // namespace cb
