// K3 (structured evaluation) and the single-axis contractions behind the stack / axis API.
//
//   contract_axis     : out[a, j, r, q] (any strides) = sum_l E[j, l] in[a, l, r, q]
//                       - eval_axis on a CoefTensor (S/chebnd.py:209-233, _bind_rows :152-154)
//                         = A=1, Q=1, out (rest, k) "rotated";
//                       - eval_axis on a TensorStack (:234-240, _bind_shared :147-149) = Q = N_P;
//                       - _bind_shared / _bind_rows layouts directly.
//   contract_diagonal : out[m, r] = sum_l T_l(x_m) in[m, l, r]   (eval_diagonal_batch :275-312,
//                       _bind_diagonal :157-159) with arbitrary strides.
//   eval_grid         : J successive rotating mode products with k_j x n_j evaluation matrices
//                       (the paper's pagemtimes evaluation P:385-417; BASELINE config 5a).
//   basis_matrix, gather_index, gather_take_f : S/chebnd.py:114-132, 243-272, 97-111.
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "cb_common.cuh"
#include "cb_kernels.h"

namespace cb {

namespace {

constexpr int kAxThreads = 256;

struct AxisParams {
  const double* E;
  const double* in;
  double* out;
  long long A, R, Q;
  int n, k;
  long long oA, oJ, oR;
  long long total;  // A*k*R*Q
};

// generic: one thread per output element, q fastest then r, j, a
__global__ void __launch_bounds__(kAxThreads) contract_axis_generic(AxisParams p) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < p.total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long q = e % p.Q;
    long long t = e / p.Q;
    long long r = t % p.R;
    t /= p.R;
    int j = static_cast<int>(t % p.k);
    long long a = t / p.k;
    const double* src = p.in + (a * p.n * p.R + r) * p.Q + q;
    const double* er = p.E + static_cast<long long>(j) * p.n;
    double acc = 0.0;
    for (int l = 0; l < p.n; ++l) acc = fma(__ldg(er + l), src[static_cast<long long>(l) * p.R * p.Q], acc);
    p.out[a * p.oA + j * p.oJ + r * p.oR + q] = acc;
  }
}

// Fast rotating product (A = 1, Q = 1): in (n, R) -> out (R, k), out[r, j] = sum_l E[j, l] in[l, r].
// A CTA owns kRT consecutive r; each thread keeps 2 input columns in registers (compile-time n)
// and produces their k outputs; the (kRT x k) output tile is staged in smem and stored
// contiguously (the tile is a contiguous block of the output).
constexpr int kRT = 256;   // rows per CTA (2 per thread, 128 threads)
constexpr int kRotThreads = 128;

template <int NT>
__global__ void __launch_bounds__(kRotThreads) rotate_fixed(const double* __restrict__ E, const double* __restrict__ in,
                                                            double* __restrict__ out, long long R, int k) {
  extern __shared__ __align__(16) double sm[];
  double* Es = sm;                         // [k][NT]
  double* Os = sm + ((k * NT + 1) & ~1);   // [kRT][k]
  for (int e = threadIdx.x; e < k * NT; e += blockDim.x) Es[e] = E[e];
  for (long long r0 = static_cast<long long>(blockIdx.x) * kRT; r0 < R; r0 += static_cast<long long>(gridDim.x) * kRT) {
    const int rows = static_cast<int>(min(static_cast<long long>(kRT), R - r0));
    double v0[NT], v1[NT];
    const int ra = threadIdx.x, rb = threadIdx.x + kRotThreads;
#pragma unroll
    for (int l = 0; l < NT; ++l) {
      v0[l] = (ra < rows) ? __ldg(in + static_cast<long long>(l) * R + r0 + ra) : 0.0;
      v1[l] = (rb < rows) ? __ldg(in + static_cast<long long>(l) * R + r0 + rb) : 0.0;
    }
    __syncthreads();  // Es ready / previous tile stored
    for (int j = 0; j < k; ++j) {
      const double* er = Es + j * NT;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int l = 0; l < NT; ++l) {
        const double w = er[l];
        a0 = fma(w, v0[l], a0);
        a1 = fma(w, v1[l], a1);
      }
      Os[ra * k + j] = a0;
      Os[rb * k + j] = a1;
    }
    __syncthreads();
    double* dst = out + r0 * k;
    const int cnt = rows * k;
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) dst[e] = Os[e];
  }
}

template <int TN>
struct Tag { static constexpr int value = TN; };

template <typename F>
bool dispatch_rot(int n, F&& f) {
  switch (n) {
#define CB_CASE(v) case v: f(Tag<v>{}); return true;
    CB_CASE(1) CB_CASE(2) CB_CASE(3) CB_CASE(4) CB_CASE(5) CB_CASE(6) CB_CASE(7) CB_CASE(8)
    CB_CASE(9) CB_CASE(10) CB_CASE(11) CB_CASE(12) CB_CASE(13) CB_CASE(14) CB_CASE(15) CB_CASE(16)
    CB_CASE(17) CB_CASE(18) CB_CASE(19) CB_CASE(20) CB_CASE(21) CB_CASE(22) CB_CASE(23) CB_CASE(24)
    CB_CASE(25) CB_CASE(26) CB_CASE(27) CB_CASE(28) CB_CASE(29) CB_CASE(30) CB_CASE(31) CB_CASE(32)
    CB_CASE(33) CB_CASE(34)
#undef CB_CASE
    default: return false;
  }
}

struct DiagParams {
  const double* x;
  const double* W;   // optional (M, n) row-major weights; replaces T_l(x_m) when non-null
  const double* in;
  double* out;
  Status* st;
  long long M, R;
  int n;
  long long sM, sL, sR, oM, oR;
  int m_fast;  // thread index varies m fastest (input stride along m is 1)
  int clamp;   // apply clamp_reference semantics to x
};

__global__ void __launch_bounds__(kAxThreads) contract_diagonal_kernel(DiagParams p) {
  const long long total = p.M * p.R;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long m, r;
    if (p.m_fast) {
      m = e % p.M;
      r = e / p.M;
    } else {
      r = e % p.R;
      m = e / p.R;
    }
    const double* src = p.in + m * p.sM + r * p.sR;
    if (p.W) {
      const double* w = p.W + m * p.n;
      double acc = 0.0;
      for (int l = 0; l < p.n; ++l) acc = fma(__ldg(w + l), src[l * p.sL], acc);
      p.out[m * p.oM + r * p.oR] = acc;
      continue;
    }
    // only the r == 0 thread of each member reports domain errors (one report per point)
    const double x = p.clamp ? clamp_ref(__ldg(p.x + m), r == 0 ? p.st : nullptr) : __ldg(p.x + m);
    const double x2 = 2.0 * x;
    double t0 = 1.0, t1 = x;
    double acc = src[0];
    if (p.n > 1) acc = fma(x, src[p.sL], acc);
    for (int l = 2; l < p.n; ++l) {
      const double t2 = fma(x2, t1, -t0);
      t0 = t1;
      t1 = t2;
      acc = fma(t2, src[l * p.sL], acc);
    }
    p.out[m * p.oM + r * p.oR] = acc;
  }
}

__global__ void basis_matrix_kernel(long long k, const double* x, int size, double* out, Status* st, int clamp) {
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < k;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    double v = __ldg(x + j);
    if (clamp) v = clamp_ref(v, st);
    cheb_row(v, size, out + j * size, 1);
  }
}

// All J evaluation matrices of a structured evaluation in one launch: thread per target point
// (dim d found from the prefix sums), row j of E_d = T_0..T_{n_d - 1}(clamp_reference(t_{d,j})).
struct BasisBatch {
  const double* x[kMaxDims];
  double* out[kMaxDims];
  long long kcum[kMaxDims + 1];
  int size[kMaxDims];
  int J;
  Status* st;
};

__global__ void basis_batch_kernel(const __grid_constant__ BasisBatch p) {
  const long long total = p.kcum[p.J];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int d = 0;
    while (d + 1 < p.J && i >= p.kcum[d + 1]) ++d;
    const long long j = i - p.kcum[d];
    const double v = clamp_ref(__ldg(p.x[d] + j), p.st);
    cheb_row(v, p.size[d], p.out[d] + j * p.size[d], 1);
  }
}

__global__ void gather_index_kernel(long long rest, long long count, long long* flat) {
  const long long total = rest * count;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long m = i / rest, r = i - m * rest;
    flat[i] = r + rest * (count + 1) * m;
  }
}

constexpr int kMaxTakeDims = 12;
struct TakeParams {
  int nd_in, nd_out;
  long long shp_in[kMaxTakeDims], str_in[kMaxTakeDims];
  long long shp_out[kMaxTakeDims], str_out[kMaxTakeDims];
  const double* in;
  const long long* flat;
  double* out;
  long long nsel;
};

__device__ __forceinline__ long long f_to_c(long long f, int nd, const long long* shp, const long long* str) {
  long long off = 0;
  for (int d = 0; d < nd; ++d) {
    const long long q = f / shp[d];
    off += (f - q * shp[d]) * str[d];
    f = q;
  }
  return off;
}

__global__ void gather_take_kernel(TakeParams p) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.nsel;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long src = f_to_c(p.flat[i], p.nd_in, p.shp_in, p.str_in);
    const long long dst = f_to_c(i, p.nd_out, p.shp_out, p.str_out);
    p.out[dst] = p.in[src];
  }
}

// derivative_array (S/cheb1d.py:230-249): one row of (rows, L) coefficients per thread.
__global__ void derivative_kernel(long long rows, int L, const double* in, double* out) {
  const int n = L - 1;
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double* p = in + r * L;
    double* q = out + r * n;
    q[n - 1] = 2.0 * n * p[n];
    if (n >= 2) q[n - 2] = 2.0 * (n - 1) * p[n - 1];
    for (int l = n - 3; l >= 0; --l) q[l] = q[l + 2] + 2.0 * (l + 1) * p[l + 1];
    q[0] *= 0.5;
  }
}


// K3 fused final pair of structured modes:  in (n, n, R') -> out (R', k, k)
//   out[r'][ia][ib] = sum_{la, lb} Ea[ia][la] Eb[ib][lb] in[la][lb][r'].
// A CTA owns RT consecutive r'.  Step 1 contracts lb (Z[la][r'][ib]), step 2 contracts la and
// writes the (RT x k x k) output tile with lanes along ib (contiguous in memory).  The evaluation
// matrices ride in the kernel parameters (constant bank): every FMA takes them as a direct
// operand, each thread keeps its n inputs in registers and produces k outputs (k independent
// FMA chains).  Saves the write + re-read of the largest intermediate (13 x 25^5 for config 5a).
// Evaluation matrices of the structured passes live in two constant-memory slots, filled by a
// stream-ordered device-to-device copy right before the kernel that reads them (no host sync);
// every DFMA then takes its matrix entry as a constant-bank operand.  Calls on different streams
// are ordered through ConstSlotGuard (eval_grid).
// Mode d's (K x N) matrix sits at offset d*K*N: a uniform grid (every mode the same (N, K)) is
// uploaded once per call (one copy when the matrices are contiguous), other plans per pass.
constexpr int kCETotal = 4096;
__constant__ double cGridE[kCETotal];

template <int N, int K, int DA>
struct Fused2Params {
  const double* in;
  double* out;
  long long R;
};

#ifndef CB_F2_RT
#define CB_F2_RT 8
#endif
#ifndef CB_F2_WARPS
#define CB_F2_WARPS 7
#endif
#ifndef CB_F2_MINB
#define CB_F2_MINB 6
#endif
constexpr int kF2RT = CB_F2_RT;         // r' per tile
constexpr int kF2Warps = CB_F2_WARPS;   // 7 warps x 6 CTAs / SM for 8 r' per tile
constexpr int kF2Threads = kF2Warps * 32;
constexpr int kWSRT = 8;                // r' per tile of the DMMA form (its n-tiles are 8 columns)
constexpr int kF2IB = 5;       // K <= 25 (5 blocks)       // outputs per thread item (compile-time constant-bank indices)
#ifndef CB_F2_IB2
#define CB_F2_IB2 25
#endif
constexpr int kF2IB2 = CB_F2_IB2;   // step 2: outputs per thread item (its N inputs are loaded once per item)

// step 1, output block B: z[ib] for ib in [B*5, B*5+5) from the N inputs v (row la, column rt)
template <int N, int K, int DA, int B>
__device__ __forceinline__ void f2_step1(const Fused2Params<N, K, DA>& p, const double* v, double* z) {
#pragma unroll
  for (int j = 0; j < kF2IB; ++j) {
    const int ib = B * kF2IB + j;
    if (ib < K) {
      double acc = 0.0;
#pragma unroll
      for (int lb = 0; lb < N; ++lb) acc = fma(cGridE[(DA + 1) * K * N + ib * N + lb], v[lb], acc);
      z[ib] = acc;
    }
  }
}

template <int N, int K, int DA, int B>
__device__ __forceinline__ void f2_step2(const Fused2Params<N, K, DA>& p, const double* v, double* dst) {
#pragma unroll
  for (int j = 0; j < kF2IB2; ++j) {
    const int ia = B * kF2IB2 + j;
    if (ia < K) {
      double acc = 0.0;
#pragma unroll
      for (int la = 0; la < N; ++la) acc = fma(cGridE[DA * K * N + ia * N + la], v[la], acc);
      dst[ia * K] = acc;
    }
  }
}

template <int N, int K, int DA>
__global__ void __launch_bounds__(kF2Threads, CB_F2_MINB) fused2_kernel(const __grid_constant__ Fused2Params<N, K, DA> p) {
  extern __shared__ __align__(16) double f2sm[];
  double* sX = f2sm;                   // [N*N][RT]
  double* sZ = f2sm + N * N * kF2RT;   // [N][RT][K]
  constexpr int NB = (K + kF2IB - 1) / kF2IB;
  constexpr int C1 = (N * kF2RT + 31) / 32;   // 32-row chunks of step 1 (per output block)
  constexpr int C2 = (K * kF2RT + 31) / 32;   // 32-item chunks of step 2 (per output block)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // one tile per CTA (no persistent loop: keeps the constant-bank operands from being hoisted
  // into registers across iterations)
  {
    const long long r0 = static_cast<long long>(blockIdx.x) * kF2RT;
    const int rt_n = static_cast<int>(min(static_cast<long long>(kF2RT), p.R - r0));
    // cp.async: every element of the tile in flight at once (a load loop serialises on the
    // global-memory latency: long-scoreboard stalls were 36 % of the last pass's samples)
    // pairs of columns: one 16-byte copy where the global address is 16-byte aligned
    for (int e2 = threadIdx.x; e2 < N * N * kF2RT / 2; e2 += blockDim.x) {
      const int row = e2 / (kF2RT / 2), rt = 2 * (e2 % (kF2RT / 2));
      const double* g = p.in + static_cast<long long>(row) * p.R + r0 + rt;
      double* d = sX + row * kF2RT + rt;
      if (rt + 1 < rt_n && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(d))),
                     "l"(g)
                     : "memory");
      } else {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (rt + i < rt_n) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(d + i))),
                         "l"(g + i)
                         : "memory");
          } else {
            d[i] = 0.0;
          }
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // step 1: Z[la][rt][ib] = sum_lb Eb[ib][lb] X[la][lb][rt]; task = (block, chunk), warp-uniform block
#pragma unroll
    for (int it = 0; it < (NB * C1 + kF2Warps - 1) / kF2Warps; ++it) {
      const int task = warp + it * kF2Warps;
      if (task >= NB * C1) break;
      const int blk = task / C1, w = (task % C1) * 32 + lane;
      if (w < N * kF2RT) {
        const int la = w / kF2RT, rt = w % kF2RT;
        double v[N];
#pragma unroll
        for (int lb = 0; lb < N; ++lb) v[lb] = sX[(la * N + lb) * kF2RT + rt];
        double* z = sZ + (la * kF2RT + rt) * K;
        switch (blk) {
          case 0: f2_step1<N, K, DA, 0>(p, v, z); break;
          case 1: if constexpr (NB > 1) f2_step1<N, K, DA, 1>(p, v, z); break;
          case 2: if constexpr (NB > 2) f2_step1<N, K, DA, 2>(p, v, z); break;
          case 3: if constexpr (NB > 3) f2_step1<N, K, DA, 3>(p, v, z); break;
          default: if constexpr (NB > 4) f2_step1<N, K, DA, 4>(p, v, z); break;
        }
      }
    }
    __syncthreads();
    // step 2: out[r0+rt][ia][ib] = sum_la Ea[ia][la] Z[la][rt][ib]; lanes along ib (contiguous)
    constexpr int NB2 = (K + kF2IB2 - 1) / kF2IB2;
#pragma unroll
    for (int it = 0; it < (NB2 * C2 + kF2Warps - 1) / kF2Warps; ++it) {
      const int task = warp + it * kF2Warps;
      if (task >= NB2 * C2) break;
      const int blk = task / C2, w = (task % C2) * 32 + lane;
      const int rt = w / K, ib = w % K;
      if (w < K * kF2RT && rt < rt_n) {
        double v[N];
#pragma unroll
        for (int la = 0; la < N; ++la) v[la] = sZ[(la * kF2RT + rt) * K + ib];
        double* dst = p.out + (r0 + rt) * (K * K) + ib;
        switch (blk) {
          case 0: f2_step2<N, K, DA, 0>(p, v, dst); break;
          case 1: if constexpr (NB2 > 1) f2_step2<N, K, DA, 1>(p, v, dst); break;
          case 2: if constexpr (NB2 > 2) f2_step2<N, K, DA, 2>(p, v, dst); break;
          case 3: if constexpr (NB2 > 3) f2_step2<N, K, DA, 3>(p, v, dst); break;
          default: if constexpr (NB2 > 4) f2_step2<N, K, DA, 4>(p, v, dst); break;
        }
      }
    }
  }
}

// Mode-d matrix into its constant offset (stream-ordered device-to-device copy).
template <int N, int K>
cudaError_t upload_const(int d, const double* E, cudaStream_t stream) {
  if ((d + 1) * K * N > kCETotal) return cudaErrorInvalidValue;
  return cudaMemcpyToSymbolAsync(cGridE, E, sizeof(double) * K * N, sizeof(double) * d * K * N,
                                 cudaMemcpyDeviceToDevice, stream);
}

// Fused pair of modes (DA, DA+1); `uploaded`: their matrices are already in the constant bank.
template <int N, int K, int DA>
cudaError_t launch_fused2_at(const double* Ea, const double* Eb, bool uploaded, const double* in, double* out,
                             long long R, cudaStream_t stream) {
  static_assert((DA + 2) * K * N <= kCETotal, "constant bank too small");
  cudaError_t e = cudaSuccess;
  if (!uploaded) {
    e = upload_const<N, K>(DA, Ea, stream);
    if (e == cudaSuccess) e = upload_const<N, K>(DA + 1, Eb, stream);
  }
  if (e != cudaSuccess) return e;
  Fused2Params<N, K, DA> p;
  p.in = in;
  p.out = out;
  p.R = R;
  const long long g = (R + kF2RT - 1) / kF2RT;
  if (g > 0x7fffffffLL) return cudaErrorInvalidValue;
  const size_t smem = sizeof(double) * (N * N + N * K) * kF2RT;
  ensure_smem_attr(reinterpret_cast<const void*>(fused2_kernel<N, K, DA>), 200 * 1024);
  fused2_kernel<N, K, DA><<<static_cast<unsigned>(g), kF2Threads, smem, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Fused pair 13 -> 25 on the FP64 tensor cores (DMMA.8x8x4).  The DFMA form above is issue-bound
// (2.27 instructions per DFMA, a quarter of them the LDCU.128 uniform loads sm_100 needs for
// 64-bit constant operands); here a mode product is a 25 x 13 by 13 x (8 columns) GEMM per
// n-tile: rows 0..23 as 3 DMMA m-tiles over 4 k-steps (l = 13..15 zero-padded), row 24 on DFMA
// from the SAME B fragments (lane partial over its l = 4 ks + tq, reduced over tq by two
// shuffles).  The evaluation-matrix fragments live in registers (loaded once per step), so an
// n-tile of 8 columns issues 12 DMMA + 4 DFMA + 4 LDS + 4 SHFL + stores instead of 81 DFMA +
// 41 LDCU + loads.  Same tile as the DFMA kernel: in (13, 13, R) -> out (R, 25, 25), 8 r' per tile;
// step 1 contracts the FIRST mode into shared memory, step 2 the second into global memory, so
// the DMMA rows of step 2 are ib, contiguous in the output (64-byte runs per store; the other
// order scattered 8-byte stores over 8 rows: 1.00 vs 0.75 ms).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma884_axis(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// A-operand fragments of a 25 x 13 evaluation matrix E (row-major): 3 m-tiles x 4 k-steps for rows
// 0..23 (zero for l >= 13) and the row-24 entries of this lane's l.
struct FDFrags {
  double a[3][4];
  double e24[4];
};
__device__ __forceinline__ void fd_load_frags(const double* __restrict__ E, int gq, int tq, FDFrags& f) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int l = ks * 4 + tq;
    const bool ok = l < 13;
#pragma unroll
    for (int m = 0; m < 3; ++m) f.a[m][ks] = ok ? __ldg(E + (m * 8 + gq) * 13 + l) : 0.0;
    f.e24[ks] = ok ? __ldg(E + 24 * 13 + l) : 0.0;
  }
}

// ------------------------------------------------------------------------------------------
// Warp-specialised form of the DMMA fused pair: two producer warps run step 1 (first mode) of
// tile i+1 while four consumer warps run step 2 (second mode) of tile i, each group keeping ITS
// evaluation-matrix fragments in registers for the whole persistent loop (the one-role form
// reloaded 16 fragments per thread per step and spent a quarter of its time in tile loads and
// CTA-wide barriers).  X tiles and the intermediate Z are double-buffered in shared memory; the
// groups hand Z over with named barriers (bar.arrive / bar.sync, 192 threads).
// ------------------------------------------------------------------------------------------
#ifndef CB_WS_P
#define CB_WS_P 2
#endif
#ifndef CB_WS_C
#define CB_WS_C 4
#endif
constexpr int kWSP = CB_WS_P, kWSC = CB_WS_C;           // producer / consumer warps
constexpr int kWSThreads = (kWSP + kWSC) * 32;
constexpr int kWSXP = 8, kWSZP = 204;                   // smem pitches (doubles)
constexpr int kWSCtas = 3;

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Two n-tiles of one GEMM step interleaved (6 independent DMMA chains per warp instead of 3: an
// n-tile alone is a chain of four dependent k-steps, ~300 cycles of latency for 192 of issue).
// bptr(i, l) -> shared-memory address of B[l][column gq] of n-tile i; store(i, c, p24) writes it.
template <typename BPtr, typename Store>
__device__ __forceinline__ void fd_ntile_pair(const FDFrags& f, int tq, bool two, BPtr bptr, Store store) {
  double bf[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int l = ks * 4 + tq;
      bf[i][ks] = (l < 13 && (i == 0 || two)) ? *bptr(i, l) : 0.0;
    }
  double c[2][3][2] = {};
  double p24[2] = {0.0, 0.0};
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
      for (int m = 0; m < 3; ++m) dmma884_axis(c[i][m][0], c[i][m][1], f.a[m][ks], bf[i][ks]);
      p24[i] = fma(f.e24[ks], bf[i][ks], p24[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    p24[i] += __shfl_xor_sync(0xffffffffu, p24[i], 1);
    p24[i] += __shfl_xor_sync(0xffffffffu, p24[i], 2);
  }
  store(0, c[0], p24[0]);
  if (two) store(1, c[1], p24[1]);
}

__global__ void __launch_bounds__(kWSThreads, kWSCtas)
    fused2_dmma_ws_kernel(const double* __restrict__ in, double* __restrict__ out, long long R,
                          const double* __restrict__ Ea, const double* __restrict__ Eb) {
  constexpr int N = 13, K = 25, RT = kWSRT;
  constexpr int XS = N * N * kWSXP, ZS = N * kWSZP;
  extern __shared__ __align__(16) double wssm[];
  double* sXb = wssm;             // [2][N*N][kWSXP]
  double* sZb = wssm + 2 * XS;    // [2][N][kWSZP]   (col = rt * 25 + ia)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const long long ntiles = (R + RT - 1) / RT;
  if (static_cast<long long>(blockIdx.x) >= ntiles) return;
  const int n_my = static_cast<int>((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);  // tiles of this CTA
  enum { FULL0 = 1, EMPTY0 = 3, PBAR = 5 };
  FDFrags f;
  if (warp < kWSP) {
    // ---------------- producers: X tile loads + step 1 ----------------
    fd_load_frags(Ea, gq, tq, f);
    const int ptid = threadIdx.x;   // 0..63
    auto prefetch = [&](long long tile, double* sX) {
      const long long r0 = tile * RT;
      const int rt_n = static_cast<int>(min(static_cast<long long>(RT), R - r0));
      for (int e2 = ptid; e2 < N * N * RT / 2; e2 += kWSP * 32) {
        const int row = e2 / (RT / 2), rt = 2 * (e2 % (RT / 2));
        const double* g = in + static_cast<long long>(row) * R + r0 + rt;
        double* d = sX + row * kWSXP + rt;
        if (rt + 1 < rt_n && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(d))),
                       "l"(g)
                       : "memory");
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (rt + i < rt_n) {
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(d + i))),
                           "l"(g + i)
                           : "memory");
            } else {
              d[i] = 0.0;
            }
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    prefetch(blockIdx.x, sXb);
    for (int it = 0; it < n_my; ++it) {
      const int b = it & 1;
      // both producer warps are done with X buffer b^1 (tile it-1) before it is refilled
      named_sync(PBAR, kWSP * 32);
      if (it + 1 < n_my) {
        prefetch(blockIdx.x + static_cast<long long>(it + 1) * gridDim.x, sXb + (b ^ 1) * XS);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      named_sync(PBAR, kWSP * 32);   // tile `it` visible to both producer warps
      if (it >= 2) named_sync(EMPTY0 + b, kWSThreads);   // consumers finished Z buffer b (tile it-2)
      const double* sX = sXb + b * XS;
      double* sZ = sZb + b * ZS;
      for (int lb = warp; lb < N; lb += 2 * kWSP) {
        const int lb2 = lb + kWSP;
        fd_ntile_pair(
            f, tq, lb2 < N,
            [&](int i, int la) { return sX + (la * N + (i ? lb2 : lb)) * kWSXP + gq; },
            [&](int i, const double (*c)[2], double p24) {
              double* z = sZ + (i ? lb2 : lb) * kWSZP;
#pragma unroll
              for (int m = 0; m < 3; ++m) {
                z[(2 * tq) * K + m * 8 + gq] = c[m][0];
                z[(2 * tq + 1) * K + m * 8 + gq] = c[m][1];
              }
              if (tq == 0) z[gq * K + 24] = p24;
            });
      }
      named_arrive(FULL0 + b, kWSThreads);
    }
  } else {
    // ---------------- consumers: step 2 + output stores ----------------
    fd_load_frags(Eb, gq, tq, f);
    const int cw = warp - kWSP;
    for (int it = 0; it < n_my; ++it) {
      const int b = it & 1;
      const long long r0 = (blockIdx.x + static_cast<long long>(it) * gridDim.x) * RT;
      const int rt_n = static_cast<int>(min(static_cast<long long>(RT), R - r0));
      named_sync(FULL0 + b, kWSThreads);
      const double* sZ = sZb + b * ZS;
      for (int t = cw; t < (RT * K) / 8; t += 2 * kWSC) {
        const int t2 = t + kWSC;
        fd_ntile_pair(
            f, tq, t2 < (RT * K) / 8,
            [&](int i, int lb) { return sZ + lb * kWSZP + (i ? t2 : t) * 8 + gq; },
            [&](int i, const double (*c)[2], double p24) {
              const int c0 = (i ? t2 : t) * 8;
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int col = c0 + 2 * tq + j;
                const int rt = col / K, ia = col - rt * K;
                if (rt < rt_n) {
                  double* dst = out + (r0 + rt) * (K * K) + ia * K + gq;
#pragma unroll
                  for (int m = 0; m < 3; ++m) dst[m * 8] = c[m][j];
                }
              }
              if (tq == 0) {
                const int col = c0 + gq;
                const int rt = col / K, ia = col - rt * K;
                if (rt < rt_n) out[(r0 + rt) * (K * K) + ia * K + 24] = p24;
              }
            });
      }
      // hand Z buffer b back (only if a later tile of this CTA will refill it)
      if (it + 2 < n_my) named_arrive(EMPTY0 + b, kWSThreads);
    }
  }
}

cudaError_t launch_fused2_dmma_ws(const double* Ea, const double* Eb, const double* in, double* out, long long R,
                                  cudaStream_t stream) {
  long long g = (R + kWSRT - 1) / kWSRT;
  const size_t smem = sizeof(double) * (2 * 13 * 13 * kWSXP + 2 * 13 * kWSZP);
  ensure_smem_attr(reinterpret_cast<const void*>(fused2_dmma_ws_kernel), 200 * 1024, true);
  static int per_sm = 0;   // resident CTAs per SM (persistent grid = exactly one wave)
  if (per_sm == 0) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fused2_dmma_ws_kernel, kWSThreads, smem) != cudaSuccess || nb < 1)
      nb = 1;
    per_sm = nb;
    if (std::getenv("CB_GRID_VERBOSE")) std::fprintf(stderr, "fused2_dmma_ws_kernel: %d CTAs/SM, %zu B smem\n", nb, smem);
  }
  const long long resident = static_cast<long long>(num_sms()) * per_sm;
  if (g > resident) g = resident;
  fused2_dmma_ws_kernel<<<static_cast<unsigned>(g), kWSThreads, smem, stream>>>(in, out, R, Ea, Eb);
  count_launch();
  return cudaGetLastError();
}

template <int N, int K>
cudaError_t launch_fused2(int d, const double* Ea, const double* Eb, bool uploaded, const double* in, double* out,
                          long long R, cudaStream_t stream) {
  switch (d) {
#define CB_F2(v) case v: return launch_fused2_at<N, K, v>(Ea, Eb, uploaded, in, out, R, stream);
    CB_F2(0) CB_F2(1) CB_F2(2) CB_F2(3) CB_F2(4) CB_F2(5) CB_F2(6)
#undef CB_F2
    default: return cudaErrorInvalidValue;
  }
}


// Rotating single-mode pass with the (K x N) evaluation matrix in the kernel parameters:
//   out[r][j] = sum_l E[j][l] in[l][r].  One row per thread, one 256-row tile per CTA (no
//   persistent loop, so the constant operands stay in the bank), output staged in shared memory
//   and written as one contiguous block.
template <int N, int K, int D>
struct RotParams {
  const double* in;
  double* out;
  long long R;
};

constexpr int kRCThreads = 256;

template <int N, int K, int D>
__global__ void __launch_bounds__(kRCThreads) rotate_const(const __grid_constant__ RotParams<N, K, D> p) {
  extern __shared__ __align__(16) double rcs[];   // [256][K]
  const long long r0 = static_cast<long long>(blockIdx.x) * kRCThreads;
  const int rows = static_cast<int>(min(static_cast<long long>(kRCThreads), p.R - r0));
  const int r = threadIdx.x;
  if (r < rows) {
    double v[N];
#pragma unroll
    for (int l = 0; l < N; ++l) v[l] = __ldg(p.in + static_cast<long long>(l) * p.R + r0 + r);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) acc = fma(cGridE[D * K * N + j * N + l], v[l], acc);
      rcs[r * K + j] = acc;
    }
  }
  __syncthreads();
  double* dst = p.out + r0 * K;
  const int cnt = rows * K;
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) dst[e] = rcs[e];
}

template <int N, int K, int D>
cudaError_t launch_rotate_const_at(const double* E, bool uploaded, const double* in, double* out, long long R,
                                   cudaStream_t stream) {
  static_assert((D + 1) * K * N <= kCETotal, "constant bank too small");
  if (!uploaded) {
    cudaError_t e = upload_const<N, K>(D, E, stream);
    if (e != cudaSuccess) return e;
  }
  RotParams<N, K, D> p;
  p.in = in;
  p.out = out;
  p.R = R;
  const long long g = (R + kRCThreads - 1) / kRCThreads;
  if (g > 0x7fffffffLL) return cudaErrorInvalidValue;
  const size_t smem = sizeof(double) * kRCThreads * K;
  ensure_smem_attr(reinterpret_cast<const void*>(rotate_const<N, K, D>), 200 * 1024);
  rotate_const<N, K, D><<<static_cast<unsigned>(g), kRCThreads, smem, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int N, int K>
cudaError_t launch_rotate_const(int d, const double* E, bool uploaded, const double* in, double* out, long long R,
                                cudaStream_t stream) {
  switch (d) {
#define CB_RO(v) case v: return launch_rotate_const_at<N, K, v>(E, uploaded, in, out, R, stream);
    CB_RO(0) CB_RO(1) CB_RO(2) CB_RO(3) CB_RO(4) CB_RO(5) CB_RO(6) CB_RO(7)
#undef CB_RO
    default: return cudaErrorInvalidValue;
  }
}

unsigned grid_for(long long total, int threads) {
  long long g = (total + threads - 1) / threads;
  const long long cap = static_cast<long long>(num_sms()) * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

}  // namespace

cudaError_t contract_axis(long long A, int n, long long R, long long Q, int k, const double* E, const double* in,
                          double* out, long long oA, long long oJ, long long oR, cudaStream_t stream) {
  if (A <= 0 || R <= 0 || Q <= 0 || k <= 0) return cudaSuccess;
  // fast rotating path
  if (A == 1 && Q == 1 && oJ == 1 && oR == k && n <= 34) {
    const size_t smem = sizeof(double) * (((k * n + 1) & ~1) + static_cast<size_t>(kRT) * k);
    if (smem <= 200 * 1024) {
      bool done = dispatch_rot(n, [&](auto tag) {
        constexpr int NT = decltype(tag)::value;
        ensure_smem_attr(reinterpret_cast<const void*>(rotate_fixed<NT>), 200 * 1024);
        long long g = (R + kRT - 1) / kRT;
        const long long cap = static_cast<long long>(num_sms()) * 8;
        if (g > cap) g = cap;
        rotate_fixed<NT><<<static_cast<unsigned>(g), kRotThreads, smem, stream>>>(E, in, out, R, k);
  count_launch();
      });
      if (done) return cudaGetLastError();
    }
  }
  AxisParams p{E, in, out, A, R, Q, n, k, oA, oJ, oR, A * k * R * Q};
  contract_axis_generic<<<grid_for(p.total, kAxThreads), kAxThreads, 0, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t contract_diagonal(long long Mcount, int n, long long R, const double* x, const double* W, int clamp,
                              const double* in, long long sM, long long sL, long long sR, double* out, long long oM,
                              long long oR, Status* st, cudaStream_t stream) {
  if (Mcount <= 0 || R <= 0) return cudaSuccess;
  DiagParams p{x, W, in, out, st, Mcount, R, n, sM, sL, sR, oM, oR, sM == 1 ? 1 : 0, clamp};
  contract_diagonal_kernel<<<grid_for(Mcount * R, kAxThreads), kAxThreads, 0, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t derivative(long long rows, int L, const double* in, double* out, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  derivative_kernel<<<grid_for(rows, 128), 128, 0, stream>>>(rows, L, in, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t basis_matrix(long long k, const double* x, int size, double* out, Status* st, int clamp,
                         cudaStream_t stream) {
  if (k <= 0) return cudaSuccess;
  basis_matrix_kernel<<<grid_for(k, 128), 128, 0, stream>>>(k, x, size, out, st, clamp);
  count_launch();
  return cudaGetLastError();
}

cudaError_t basis_matrices(int J, const long long* k, const double* const* x, const long long* size, double* out,
                           Status* st, cudaStream_t stream) {
  if (J < 1 || J > kMaxDims) return cudaErrorInvalidValue;
  BasisBatch p{};
  p.J = J;
  p.st = st;
  p.kcum[0] = 0;
  long long off = 0;
  for (int d = 0; d < J; ++d) {
    p.x[d] = x[d];
    p.out[d] = out + off;
    p.size[d] = static_cast<int>(size[d]);
    p.kcum[d + 1] = p.kcum[d] + k[d];
    off += k[d] * size[d];
  }
  if (p.kcum[J] <= 0) return cudaSuccess;
  basis_batch_kernel<<<grid_for(p.kcum[J], 128), 128, 0, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t gather_index(long long rest, long long count, long long* flat, cudaStream_t stream) {
  if (rest * count <= 0) return cudaSuccess;
  gather_index_kernel<<<grid_for(rest * count, 256), 256, 0, stream>>>(rest, count, flat);
  count_launch();
  return cudaGetLastError();
}

cudaError_t gather_take_f(int ndim_in, const long long* shape_in, const double* in, long long nsel, const long long* flat,
                          int ndim_out, const long long* shape_out, double* out, cudaStream_t stream) {
  if (nsel <= 0) return cudaSuccess;
  if (ndim_in > kMaxTakeDims || ndim_out > kMaxTakeDims) return cudaErrorInvalidValue;
  TakeParams p{};
  p.nd_in = ndim_in;
  p.nd_out = ndim_out;
  long long s = 1;
  for (int d = ndim_in - 1; d >= 0; --d) {
    p.shp_in[d] = shape_in[d];
    p.str_in[d] = s;
    s *= shape_in[d];
  }
  s = 1;
  for (int d = ndim_out - 1; d >= 0; --d) {
    p.shp_out[d] = shape_out[d];
    p.str_out[d] = s;
    s *= shape_out[d];
  }
  p.in = in;
  p.flat = flat;
  p.out = out;
  p.nsel = nsel;
  gather_take_kernel<<<grid_for(nsel, 256), 256, 0, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}


// Orders uses of the constant slots (cGridE) across streams: a call waits for the previous call's
// last reader (per device) before its first slot copy and records itself on exit.  Skipped while
// the stream is being captured into a graph (the graph's own order applies).
struct ConstSlotGuard {
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static cudaEvent_t& last(int dev) {
    static cudaEvent_t ev[64] = {};
    return ev[dev & 63];
  }
  std::lock_guard<std::mutex> lock;
  cudaStream_t stream;
  int dev = 0;
  bool active = false;
  cudaError_t err = cudaSuccess;
  explicit ConstSlotGuard(cudaStream_t s) : lock(mu()), stream(s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    err = cudaStreamIsCapturing(stream, &cs);
    if (err != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return;
    cudaEvent_t& ev = last(dev);
    if (!ev) err = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(stream, ev, 0);
    active = err == cudaSuccess;
  }
  ~ConstSlotGuard() {
    if (active) cudaEventRecord(last(dev), stream);
  }
};

// the last two modes fused when their sizes have an instantiated kernel (launch_fused2)
static bool grid_fuse_last_two(const EvalLayout& L, const long long* k) {
  const int J = L.J;
  if (J < 3 || L.n[J - 2] != L.n[J - 1] || k[J - 2] != k[J - 1]) return false;
  const long long n = L.n[J - 1], kk = k[J - 1];
  return (n == 13 && kk == 25) || (n == 5 && kk == 4);
}

long long eval_grid_work_elems(const EvalLayout& L, const long long* k) {
  long long dense = 1;
  for (int d = 0; d < L.J; ++d) dense *= L.n[d];
  dense = dense / L.K * L.Kp;  // the passes may carry the K padding (q = 2 fused path)
  long long mx = dense;
  long long cur = dense;
  for (int d = 0; d + 1 < L.J; ++d) {
    cur = cur / L.n[d] * k[d];
    if (cur > mx) mx = cur;
  }
  return 2 * mx;
}

cudaError_t eval_grid(const EvalLayout& L, const double* coef, const long long* k, const double* const* E,
                      double* out, double* work, long long work_elems, cudaStream_t stream) {
  const int J = L.J;
  long long dense = 1;
  for (int d = 0; d < J; ++d) dense *= L.n[d];
  const long long need = eval_grid_work_elems(L, k);
  if (work_elems < need) return cudaErrorInvalidValue;
  double* bufA = work;
  double* bufB = work + need / 2;
  const double* cur = coef;
  const bool fuse = grid_fuse_last_two(L, k);
  long long total = dense;
  if (fuse && L.q == 2) {
    // the eval layout's trailing K = n_{J-2} * n_{J-1} (padded to Kp) is exactly the fused pair:
    // the single passes carry the padded rows along and the fused kernel ignores rows >= n^2
    total = dense / L.K * L.Kp;
  } else if (L.Kp != L.K) {
    cudaError_t err = cudaMemcpy2DAsync(bufA, sizeof(double) * L.K, coef, sizeof(double) * L.Kp,
                                        sizeof(double) * L.K, L.R, cudaMemcpyDeviceToDevice, stream);
    if (err != cudaSuccess) return err;
    cur = bufA;
  }
  // pass plan, left to right: a pair of equal modes with an instantiated fused kernel goes in one
  // fused pass (rotating layout in (n, n, R) -> out (R, k, k)), any other mode in a single
  // rotating pass; the final pair is fused only when grid_fuse_last_two (padding carried, q = 2)
  const bool padded = fuse && L.q == 2;  // modes J-2, J-1 travel as one padded Kp axis
  auto pairable = [&](int d) {
    if (d + 1 >= J || L.n[d] != L.n[d + 1] || k[d] != k[d + 1]) return false;
    if (d + 2 == J) return fuse;
    if (padded && d + 1 >= J - 2) return false;
    return (L.n[d] == 13 && k[d] == 25) || (L.n[d] == 5 && k[d] == 4);
  };
  auto const_ok = [&](int d) { return L.n[d] == 13 && k[d] == 25; };
  ConstSlotGuard guard(stream);
  if (guard.err != cudaSuccess) return guard.err;
  // uniform 13 -> 25 grid: every matrix into its constant offset up front (one copy when the J
  // matrices are contiguous, as cb_eval_grid_targets lays them out)
  bool uniform = J * 13 * 25 <= kCETotal;
  for (int j = 0; j < J; ++j) uniform = uniform && const_ok(j);
  if (uniform) {
    bool contiguous = true;
    for (int j = 1; j < J; ++j) contiguous = contiguous && E[j] == E[0] + j * 13 * 25;
    cudaError_t err = contiguous ? cudaMemcpyToSymbolAsync(cGridE, E[0], sizeof(double) * J * 13 * 25, 0,
                                                           cudaMemcpyDeviceToDevice, stream)
                                 : cudaSuccess;
    for (int j = 0; !contiguous && j < J && err == cudaSuccess; ++j) err = upload_const<13, 25>(j, E[j], stream);
    if (err != cudaSuccess) return err;
  }
  int d = 0;
  while (d < J) {
    const bool pair = pairable(d);
    const int last = pair ? d + 1 : d;
    double* dst = (last == J - 1) ? out : ((cur == bufA) ? bufB : bufA);
    cudaError_t err;
    if (pair) {
      const long long n = L.n[d], kk = k[d];
      const long long R = total / ((last == J - 1 && L.q == 2) ? L.Kp : n * n);
      // CB_GRID_MODE=ws selects the DMMA (FP64 tensor core) form of the 13 -> 25 pair: correct
      // (tested), but slower than the DFMA form so far (0.85 vs 0.63 ms per 25^6 grid), so opt-in
      static const bool ws = [] {
        const char* m = std::getenv("CB_GRID_MODE");
        return m && m[0] == 'w';
      }();
      if (n == 13 && kk == 25 && ws) err = launch_fused2_dmma_ws(E[d], E[d + 1], cur, dst, R, stream);
      else if (n == 13 && kk == 25) err = launch_fused2<13, 25>(d, E[d], E[d + 1], uniform, cur, dst, R, stream);
      else err = launch_fused2<5, 4>(d, E[d], E[d + 1], false, cur, dst, R, stream);
      total = R * kk * kk;
    } else {
      const long long R = total / L.n[d];
      err = const_ok(d) ? launch_rotate_const<13, 25>(d, E[d], uniform, cur, dst, R, stream)
                        : contract_axis(1, static_cast<int>(L.n[d]), R, 1, static_cast<int>(k[d]), E[d], cur, dst, 0, 1,
                                        k[d], stream);
      total = R * k[d];
    }
    if (err != cudaSuccess) return err;
    cur = dst;
    d = last + 1;
  }
  return cudaSuccess;
}

}  // namespace cb
