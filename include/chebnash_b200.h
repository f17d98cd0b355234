/*
 * chebnash_b200 — C ABI of the B200-native fp64 tensor-Chebyshev engine.
 *
 * Drop-in boundary for the hot path of the reference package `chebnash` (arXiv 2307.04688):
 * J-dimensional tensor-product Chebyshev interpolation inside the time-stepping solver.  The
 * reference has no FFI layer — its boundary is the Python API re-exported by
 * pkg/src/chebnash/__init__.py:11-57 — so every entry point below names the reference function
 * it replaces (file:line, paths relative to pkg/src/chebnash/).  The Python shim
 * paper_2307_04688_b200/ binds these with ctypes and keeps the reference signatures
 * (see INTEGRATION.md).
 *
 * Conventions
 *   - Plain pointers and sizes only.  `d_*` pointers are device (CUDA global) memory owned by the
 *     caller; the library never allocates or frees caller memory.  `stream` is a cudaStream_t
 *     passed as void* (NULL = legacy default stream).  All calls are asynchronous on `stream`.
 *   - Return value: CB_OK (0) or a CB_E* code; cb_last_error() gives a thread-local message.
 *   - `d_status` (optional, may be NULL) points to a 16-byte device block
 *       { uint32 nonfinite; uint32 domain; uint64 worst_abs_bits; }
 *     that kernels update: nonfinite != 0 -> "must be finite" ValueError; domain != 0 ->
 *     "evaluation point outside [-1, 1] beyond tolerance: |x| = <worst>" ValueError
 *     (cheb1d.py:127-135, chebnd.py:179-185).  The caller zeroes it before the call.
 *   - Dense tensors are C-order (n_1, ..., n_J) fp64 (chebnd.py:33-54).  Coefficients consumed by
 *     the evaluators are in the "eval layout" described by cb_eval_layout().
 *   - Re-entrant, with two documented exceptions to "no global mutable state": mutex-guarded
 *     per-device caches (kernel attributes, cb_advect_loop's instantiated graphs, advected-node
 *     tables for modes above 64 nodes), and the __constant__ slot that holds cb_eval_grid's
 *     evaluation matrices (every DFMA of the structured passes reads them as constant operands).
 *     Eager cb_eval_grid / cb_eval_grid_targets calls on different streams and threads are
 *     ordered through that slot by an internal event guard; a cb_eval_grid captured into a CUDA
 *     graph bypasses the guard, so such a graph must not be replayed concurrently with another
 *     cb_eval_grid (captured or eager) on another stream.
 *   - Input range: 1 <= J <= 12 modes (the tensor-core evaluators up to J = 8, above that the
 *     Clenshaw / generic evaluators), mode sizes 1..4096 (degree <= 4095), at most 2^31
 *     elements per tensor.
 */
#ifndef CHEBNASH_B200_H
#define CHEBNASH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CB_ABI_VERSION 1

enum {
  CB_OK = 0,
  CB_EINVAL = 1,     /* bad shape / argument (reference raises ValueError) */
  CB_ENONFINITE = 2, /* non-finite objective in a sweep / non-concave LQ update (FloatingPointError) */
  CB_ENOFIX = 3,     /* LQ coefficient iteration did not settle (RuntimeError) */
  CB_ECUDA = 4       /* CUDA runtime error */
};

int cb_abi_version(void);
const char* cb_last_error(void);

/* Number of kernels this library has launched in the process, including the kernels of each
 * cb_advect_loop step-pair graph replay (captured launches count when they are replayed). */
int64_t cb_kernel_launches(void);

/* Description of the evaluator kernel / plan chosen by the last cb_eval_points or
 * cb_eval_advected call on this thread (diagnostics, bench reporting). */
const char* cb_last_eval_plan(void);

/* Device inventory: number of visible CUDA devices (0 without a GPU), SM count and compute
 * capability of the current device.  Never fails on a CPU-only host. */
int cb_runtime_info(int* device_count, int* sm_count, int* cc_major, int* cc_minor);

/* Eval layout of a J-mode tensor with sizes n[0..J-1]:
 *   out[0]=q (trailing modes merged into columns), out[1]=R (rows), out[2]=R8 (rows padded to 8),
 *   out[3]=K (columns), out[4]=Kp (columns padded to 4), out[5]=R8*Kp (elements to allocate).
 * Host-only. */
int cb_eval_layout(int J, const int64_t* n, int64_t* out6);

/* Dense C-order (n_1..n_J) <-> eval layout (zero padding written by pack).  Used when a
 * CoefTensor is constructed from user coefficients (chebnd.py:33-54) and when its
 * `.coefficients` are read back. */
int cb_pack_eval(int J, const int64_t* n, const double* d_dense, double* d_eval, void* stream);
int cb_unpack_eval(int J, const int64_t* n, const double* d_eval, double* d_dense, void* stream);

/* K1 — tensor_coeffs (chebnd.py:162-190; cheb_transform cheb1d.py:138-170 per mode).
 * d_samples: dense (n_1..n_J) node values, entry (k_1..k_J) at the descending nodes
 * (make_basis cheb1d.py:73-104).  d_coef: eval layout, cb_eval_layout()[5] doubles.
 * Non-finite samples set d_status->nonfinite. */
int cb_tensor_coeffs(int J, const int64_t* n, const double* d_samples, double* d_coef, void* d_status, void* stream);

/* K1 generic — apply the node->coefficient transform along the consecutive axes [a0, a1) of a
 * dense C-order array of `ndim` dims.  Covers stack_coeffs (chebnd.py:193-206: axes 0..J-1 of
 * (n_1..n_J, N_P)), cheb_transform(values, axis) (cheb1d.py:138-170: one axis) and
 * coeffs_from_samples (cheb1d.py:173-195).  d_out may equal d_in. */
int cb_transform_axes(int ndim, const int64_t* shape, int a0, int a1, const double* d_in, double* d_out,
                      void* d_status, int check_finite, void* stream);

/* K2 — batched scattered evaluation: the solver's value evaluator solver.py:388-397 with the
 * semantics of eval_full chebnd.py:315-327 (clamp_reference cheb1d.py:127-135).
 * d_points: (M, J) row-major reference coordinates in [-1, 1]; d_out: (M,).
 * flags bit 0: force the DFMA fallback kernel (testing). */
int cb_eval_points(int J, const int64_t* n, const double* d_coef, int64_t M, const double* d_points, double* d_out,
                   void* d_status, int flags, void* stream);

/* K1 + K2 in one call — tensor_coeffs chebnd.py:162-190 followed by the evaluation at `M` points
 * (the per-sweep refit + evaluate of the solver, solver.py:441-449 then :388-397), for loops whose
 * steps are too small to amortise two launches.  d_values: (n_1..n_J) node values; d_coef receives
 * the eval-layout coefficients exactly as cb_tensor_coeffs writes them; d_out: (M,) values,
 * bitwise those of cb_tensor_coeffs + cb_eval_points.  Small J = 2 tensors (modes <= 34, e.g.
 * BASELINE config 1's 17 x 17) run as ONE fused launch; every other shape as the two calls. */
int cb_build_eval_points(int J, const int64_t* n, const double* d_values, int64_t M, const double* d_points,
                         double* d_out, double* d_coef, void* d_status, void* stream);

/* K2 from host buffers — the same evaluation with (M, J) points and (M,) results in HOST memory
 * (pinned for overlap): the points are copied up, evaluated and copied back in chunks on two
 * internal copy streams so the PCIe transfers overlap the evaluator (solver.py:388-397 as called
 * from host code).  d_points_ws (M*J doubles) and d_out_ws (M doubles) are device work buffers.
 * Asynchronous with respect to the host: results are in h_out once `stream` has completed.
 * Bitwise identical to cb_eval_points on the same inputs. */
int cb_eval_points_host(int J, const int64_t* n, const double* d_coef, int64_t M, const double* h_points,
                        double* h_out, double* d_points_ws, double* d_out_ws, void* d_status, int flags,
                        void* stream);

/* K4 building block — evaluate at advected grid nodes (solver.py:383-397 with a fixed linear
 * drift): for flat C-order node indices i in [node_begin, node_begin+count):
 *   x = grid node i on the box [lo, hi]^J (make_basis nodes), y = clip(x + dt*A x, lo, hi),
 *   d_out[i - node_begin] = V(y) - (source ? dt*|x|^2 : 0),  V given by d_coef (eval layout).
 * A: host J x J row-major.  lo, hi: host arrays of J. */
int cb_eval_advected(int J, const int64_t* n, const double* d_coef, int64_t node_begin, int64_t count,
                     const double* A, double dt, const double* lo, const double* hi, int source, double* d_out,
                     void* stream);

/* K4 with the exchange fused in (node-sharded loop across GPUs): as
 * cb_eval_advected, but every result V(y_i) is stored into ALL G buffers d_full[r][i] (each the
 * base of one rank's full node-value array, peers mapped over NVLink with cb_ipc_import), so the
 * evaluation kernel itself performs the per-step all-gather.  Replaces the slab evaluation +
 * NCCL all-gather of dist.ShardedAdvectLoop (the reference's block sweep S/solver.py:412-438
 * with its barrier before _refit :441-449).  d_full: host array of G <= 8 device pointers. */
int cb_eval_advected_peers(int J, const int64_t* n, const double* d_coef, int64_t node_begin, int64_t count,
                           const double* A, double dt, const double* lo, const double* hi, int source,
                           double* const* d_full, int G, void* stream);

/* CUDA IPC for the peer buffers of cb_eval_advected_peers.  cb_ipc_export writes a 72-byte
 * record (cudaIpcMemHandle_t of the allocation holding d_ptr + the byte offset of d_ptr in it);
 * cb_ipc_import maps a record exported by another process (same node) and returns the peer's
 * pointer and the mapping base to pass to cb_ipc_close. */
int cb_ipc_export(const void* d_ptr, void* record72);
int cb_ipc_import(const void* record72, void** d_ptr_out, void** d_base_out);
int cb_ipc_close(void* d_base);

/* K4 — device-resident time loop on one GPU (solver.py:541-550 skeleton, BASELINE configs 3/5b):
 *   repeat `steps` times:  C = tensor_coeffs(V);  V <- eval_advected(C) (source on).
 * d_values: dense (n_1..n_J) V_0 in, V_steps out.  d_tmp: same size scratch.  d_coef: eval-layout
 * scratch.  use_graph != 0 captures the step pair in a CUDA graph (no per-step host work). */
int cb_advect_loop(int J, const int64_t* n, double* d_values, double* d_tmp, double* d_coef, int steps,
                   const double* A, double dt, const double* lo, const double* hi, void* d_status, int use_graph,
                   void* stream);

/* Single-axis contraction with an evaluation matrix E (k x n, row-major):
 *   out[a*oA + j*oJ + r*oR + q] = sum_l E[j*n + l] * in[((a*n + l)*R + r)*Q + q]
 * eval_axis (chebnd.py:209-240) = (A=1, Q=1 | Q=N_P, oR=k*Q, oJ=Q ...), _bind_rows (:152-154),
 * _bind_shared (:147-149). */
int cb_contract_axis(int64_t A, int n, int64_t R, int64_t Q, int k, const double* d_E, const double* d_in,
                     double* d_out, int64_t oA, int64_t oJ, int64_t oR, void* stream);

/* Diagonal contraction: out[m*oM + r*oR] = sum_l w_{m,l} * in[m*sM + l*sL + r*sR] with
 * w_{m,l} = T_l(x_m) (x clamped like clamp_reference when clamp != 0) or, when d_W is non-NULL,
 * w_{m,l} = d_W[m*n + l].  eval_diagonal_batch (chebnd.py:275-312), _bind_diagonal (:157-159),
 * clenshaw with batch axes (cheb1d.py:198-214). */
int cb_contract_diagonal(int64_t M, int n, int64_t R, const double* d_x, const double* d_W, int clamp,
                         const double* d_in, int64_t sM, int64_t sL, int64_t sR, double* d_out, int64_t oM, int64_t oR,
                         void* d_status, void* stream);

/* derivative_array (cheb1d.py:230-249): rows of L coefficients -> rows of L-1 derivative
 * coefficients (reference variable). */
int cb_derivative(int64_t rows, int L, const double* d_in, double* d_out, void* stream);

/* basis_matrix (chebnd.py:114-132; clamp != 0) and _row_basis (:135-144; clamp == 0):
 * d_out (k, size) row-major, B[j, l] = T_l(x_j). */
int cb_basis_matrix(int64_t k, const double* d_x, int size, double* d_out, void* d_status, int clamp, void* stream);

/* make_gather_index (chebnd.py:243-272): d_flat[i] = (i % rest) + rest*(count+1)*(i / rest). */
int cb_gather_index(int64_t rest, int64_t count, int64_t* d_flat, void* stream);

/* GatherIndex.take (chebnd.py:97-111): Fortran-order gather between C-contiguous arrays:
 * out_F[i] = in_F[flat[i]] for i < nsel. */
int cb_gather_take(int ndim_in, const int64_t* shape_in, const double* d_in, int64_t nsel, const int64_t* d_flat,
                   int ndim_out, const int64_t* shape_out, double* d_out, void* stream);

/* K3 — structured evaluation on a tensor-product target grid: J successive eval_axis mode
 * products (chebnd.py:209-233; paper pagemtimes P:385-417).  d_E[j]: device (k_j x n_j)
 * row-major evaluation matrices T_l(t_{j,i}).  d_out: dense (k_1..k_J).  d_work: scratch of
 * cb_eval_grid_workspace() doubles. */
int64_t cb_eval_grid_workspace(int J, const int64_t* n, const int64_t* k);
int cb_eval_grid(int J, const int64_t* n, const double* d_coef, const int64_t* k, const double* const* d_E,
                 double* d_out, double* d_work, int64_t work_elems, void* stream);

/* cb_eval_grid from the target coordinates (eval_axis's basis_matrix step included, chebnd.py:
 * 224-233): d_targets[j] holds k_j reference coordinates of dim j (clamp_reference, errors into
 * d_status); all J evaluation matrices are formed in ONE launch into d_E_ws (sum_j k_j*n_j
 * doubles, matrix j at offset sum_{i<j} k_i*n_i), then the mode-product passes run. */
int cb_eval_grid_targets(int J, const int64_t* n, const double* d_coef, const int64_t* k,
                         const double* const* d_targets, double* d_E_ws, void* d_status, double* d_out,
                         double* d_work, int64_t work_elems, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Collocation solver: the Bellman sweep of solver.py on the device.
 * ------------------------------------------------------------------------------------------- */
#define CB_MAX_PLAYERS 8
#define CB_MAX_CONTROL_NODES 32

/* GameSpec (game.py:29-107) + the derived constants a sweep needs.  Node enumeration of the
 * state grid is dimension 1 fastest (game.py:117-126): node p has coordinates nodes[p*J + d]. */
typedef struct {
  int J;                                   /* players = state dimensions, 2..8 */
  int np[CB_MAX_PLAYERS];                  /* state nodes per dimension, Np_d + 1 (2..64) */
  int nu[CB_MAX_PLAYERS];                  /* control nodes per player, Nu_i + 1 (2..32) */
  double h, delta, P_max, U_max, tol;      /* Euler step, 1 - rho*h, boxes, stopping tolerance */
  double A[CB_MAX_PLAYERS], phi[CB_MAX_PLAYERS];
  double K[CB_MAX_PLAYERS][CB_MAX_PLAYERS];            /* exchange matrix (game.py:140-151) */
  double beta[CB_MAX_PLAYERS], c[CB_MAX_PLAYERS], m[CB_MAX_PLAYERS];
  double unodes[CB_MAX_PLAYERS][CB_MAX_CONTROL_NODES]; /* make_basis(Nu_i, 0, U_max).nodes */
  double rnodes[CB_MAX_PLAYERS][CB_MAX_CONTROL_NODES]; /* reference_nodes(Nu_i) */
} cb_game_t;

/* Node-major drift tensors D_i[p][b][l_own][comp] (the reference's _PlayerWork.coeffs,
 * solver.py:183-189) from the J control-space drift stacks (precompute_dynamics_stack,
 * solver.py:141-159: each (nu_1, ..., nu_J, N_P) C-order, concatenated).  Done once per game;
 * d_drift holds cb_solver_drift_elems() doubles. */
int64_t cb_solver_drift_elems(const cb_game_t* game);
int cb_solver_drift_layout(const cb_game_t* game, const double* d_stacks, double* d_drift, void* stream);

/* One synchronous best-response sweep over all players and nodes: _run_sweep + _best_response_block
 * (solver.py:359-438), one warp per (player, node).
 *   d_nodes  (N_P, J) state nodes;  d_drift: cb_solver_drift_layout() of the drift stacks;
 *   d_coef   (J, N_P) value coefficients of the current fields, player i's tensor stored with
 *            REVERSED axes (l_J, ..., l_1) — exactly cb_transform_axes over axes 1..J of the node
 *            values viewed as (J, np_J, ..., np_1), i.e. _refit (solver.py:441-449) without a copy;
 *   d_v, d_u (J, N_P) current values / policy -> d_v_out, d_u_out (J, N_P);
 *   d_clamped: uint64 counter, incremented by the number of clamped successor components.
 * A non-finite objective sets d_status->nonfinite (FloatingPointError, solver.py:400-401). */
int cb_bellman_sweep(const cb_game_t* game, const double* d_nodes, const double* d_drift, const double* d_coef,
                     const double* d_v, const double* d_u, double* d_v_out, double* d_u_out, uint64_t* d_clamped,
                     void* d_status, void* stream);

/* Device work bytes for cb_solve (history + clamp counts + control block). */
int64_t cb_solve_work_bytes(const cb_game_t* game, int64_t max_iters);

/* Fixed-point driver `solve` (solver.py:495-570) run on the device: sweeps + refits captured in
 * CUDA graphs, convergence tested on the device (sup-norm change < tol), no host work per sweep.
 * d_v, d_u, d_coef each hold TWO (J, N_P) buffers; the initial fields are in buffer 0.  On return
 * the final fields are in buffer (*iterations % 2).  d_work layout (cb_solve_work_bytes):
 *   [max_iters * J doubles: per-sweep per-player sup change][max_iters uint64: clamp counts][ctl].
 * Returns CB_ENONFINITE if a sweep produced a non-finite objective (*iterations = that sweep). */
int cb_solve(const cb_game_t* game, const double* d_nodes, const double* d_drift, double* d_v, double* d_u,
             double* d_coef, void* d_work, int64_t max_iters, int64_t* iterations, int* converged, void* stream);

/* Closed-loop rollouts `simulate` (solver.py:597-629), batched over `batch` initial states:
 * u_t = clip(policy(p_t), 0, U_max), p_{t+1} = clip(p_t + h g(p_t, u_t), 0, P_max) (game.py:165-168).
 * d_policies: the J policy interpolants (fit_policy, solver.py:577-583), dense C-order
 * (np_1..np_J) each, concatenated; d_p0 (batch, J); d_states, d_controls (batch, n_steps+1, J). */
int cb_simulate(const cb_game_t* game, int64_t batch, const double* d_policies, const double* d_p0, int64_t n_steps,
                double* d_states, double* d_controls, void* stream);

/* Closed-form linear-quadratic equilibrium (the reference's validation oracle, oracle.py:65-163):
 * d_state = [Q (J,J,J)][b (J,J)][d (J)][e (J)][f (J,J)] (device doubles).  mode 0: one exact
 * Bellman update of d_state (lq_bellman_update); mode 1: lq_solve from the zero value function
 * (iterate until the (Q, b, e, f) change < tol, then close the constant term).  d_work holds
 * J^3 + 2J^2 + 2J doubles + 16 bytes.  Synchronous (returns the iteration count).  Errors:
 * CB_ENONFINITE (not concave), CB_ENOFIX (no fixed point within max_iters). */
int cb_lq(const cb_game_t* game, double* d_state, double* d_work, int64_t max_iters, double tol, int mode,
          int64_t* iterations, void* stream);

/* Safeguarded maximiser _maximise_block (solver.py:262-323) on m rows of L coefficients
 * (reference variable on [-1, 1]) from warm starts d_x0: d_x, d_f (m,).  always_scan != 0 adds the
 * dense-scan candidate for every row (newton_maximize, solver.py:326-356). */
int cb_maximise_rows(int64_t m, int L, const double* d_coef, const double* d_x0, double* d_x, double* d_f,
                     int always_scan, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CHEBNASH_B200_H */
