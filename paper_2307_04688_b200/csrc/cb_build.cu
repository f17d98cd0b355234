// K1: Chebyshev interpolant build (node values -> coefficient tensor) on sm_100a, fp64.
//
// Reference: tensor_coeffs S/chebnd.py:162-190 applies the 1-D DCT-I (cheb_transform,
// S/cheb1d.py:138-170, an rfft of the even extension) along every mode, rotating the axes
// in between.  Mathematically that is J mode-n products with the n x n matrix
// M0 = diag(s) B^T diag(w) of S/solver.py:162-171.  Every path below applies those products with
// the even/odd fold M0[l, N-k] = (-1)^l M0[l, k] (n/2 FMA per element per mode) and the same
// per-fiber FMA order, so all paths give bitwise-identical coefficients.  Paths, by shape:
//   * <= 6,144 entries, every mode n <= 34: ONE single-CTA launch (small_build_kernel) — the
//     whole tensor in shared memory (config 1, the solver's fields, most test shapes);
//   * full builds with every mode the same n in {5, 9, 13, 17, 33} (the BASELINE tensors 33^3,
//     17^4, 17^5, 13^6): mode-GROUP passes (group_pass_kernel), 2 launches — the trailing <= 3
//     modes on contiguous slabs read once from the dense samples and written to the eval layout,
//     then the leading modes in place on column tiles; the tensor crosses the L2 <-> SM boundary
//     twice instead of J times;
//   * any other shape with modes n <= 34: one fiber pass per mode (fiber_pass_kernel /
//     fiber_inner_kernel, thread per fiber, L2-resident between passes), in place on the output;
//   * modes n > 34: smem group passes with runtime sizes (build_pass_kernel).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "cb_common.cuh"
#include "cb_kernels.h"

namespace cb {

namespace {

constexpr int kBuildThreads = 256;
constexpr int kMaxGroup = 4;
constexpr int kMaxTemplN = 34;   // fiber sizes with a fully unrolled register path
constexpr int kMaxGenericN = 128;   // degree <= 127 on the smem group path (build_pass_kernel)
constexpr int kMaxTransformN = 1 << 16;   // larger modes: large_fiber_kernel (per-mode passes)

struct PassParams {
  const double* in;
  double* out;
  Status* st;
  int check_finite;
  int contiguous;
  int k;                      // modes in the group
  int n[kMaxGroup];           // their sizes, outer -> inner
  int sm_stride[kMaxGroup];   // smem stride of each mode
  int sm_outer[kMaxGroup];    // smem stride of the dim before each mode (ext_i * stride_i)
  FastDiv fd_inner[kMaxGroup];  // divisor = real element count after mode i (incl. ct)
  int fibers[kMaxGroup];      // number of fibers for each mode
  int moff[kMaxGroup];        // offset of each mode's folded matrix in smem
  int mat_total;              // doubles of folded matrices
  int tile_elems;             // real elements per tile (incl. ct)
  int tile_smem;              // smem doubles of the tile (with padding)
  long long tiles;
  // contiguous flavour
  int nlast, nls;             // last mode size and its padded smem extent
  FastDiv fd_nlast, fd_K;
  int K, Kp;
  long long in_tile_stride, out_tile_stride;
  // strided flavour
  long long Cn;               // inner extent (contiguous elements per group row)
  int ct;                     // inner tile width (power of two)
  int ct_shift;
  long long ctiles;           // column tiles per outer index
};

// Folded matrix for a mode of size n: Mf[l][j] for j in [0, H] (H = n/2), row pitch H+1.
__device__ void fill_folded(double* Mf, int n, int tid, int nthreads) {
  int N = n - 1, H = n / 2, pitch = H + 1;
  for (int e = tid; e < n * pitch; e += nthreads) {
    int l = e / pitch, j = e - l * pitch;
    Mf[e] = (j <= N) ? transform_entry(l, j, N) : 0.0;
  }
}

template <int TN>
__device__ __forceinline__ void fiber_fixed(double* s, int stride, const double* Mf) {
  if constexpr (TN == 1) {
    return;  // degree 0: cheb_transform returns a copy (S/cheb1d.py:163-164)
  } else {
    constexpr int N = TN - 1;
    constexpr int H = TN / 2;
    constexpr int P = H + 1;
    double e[H], o[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      double a = s[k * stride];
      double b = s[(N - k) * stride];
      e[k] = a + b;
      o[k] = a - b;
    }
    double mid = 0.0;
    if constexpr (TN & 1) mid = s[H * stride];
#pragma unroll
    for (int l = 0; l <= N; ++l) {
      const double* row = Mf + l * P;
      double acc = 0.0;
      if ((l & 1) == 0) {
#pragma unroll
        for (int k = 0; k < H; ++k) acc = fma(row[k], e[k], acc);
        if constexpr (TN & 1) acc = fma(row[H], mid, acc);
      } else {
#pragma unroll
        for (int k = 0; k < H; ++k) acc = fma(row[k], o[k], acc);
      }
      s[l * stride] = acc;
    }
  }
}

__device__ void fiber_generic(double* s, int stride, const double* Mf, int n) {
  if (n == 1) return;
  int N = n - 1, H = n / 2, P = H + 1;
  double e[kMaxGenericN / 2], o[kMaxGenericN / 2];
  for (int k = 0; k < H; ++k) {
    double a = s[k * stride], b = s[(N - k) * stride];
    e[k] = a + b;
    o[k] = a - b;
  }
  double mid = (n & 1) ? s[H * stride] : 0.0;
  for (int l = 0; l <= N; ++l) {
    const double* row = Mf + l * P;
    double acc = 0.0;
    if ((l & 1) == 0) {
      for (int k = 0; k < H; ++k) acc = fma(row[k], e[k], acc);
      if (n & 1) acc = fma(row[H], mid, acc);
    } else {
      for (int k = 0; k < H; ++k) acc = fma(row[k], o[k], acc);
    }
    s[l * stride] = acc;
  }
}

template <int TN>
__device__ __forceinline__ void mode_loop_fixed(double* sm, const PassParams& p, int i, const double* Mf) {
  const int stride = p.sm_stride[i];
  const int outer = p.sm_outer[i];
  const bool inner_pad = p.contiguous && (i < p.k - 1);
  for (int f = threadIdx.x; f < p.fibers[i]; f += blockDim.x) {
    uint32_t fo, fi;
    p.fd_inner[i].divmod(static_cast<uint32_t>(f), fo, fi);
    uint32_t off = fi;
    if (inner_pad) {
      uint32_t q, r;
      p.fd_nlast.divmod(fi, q, r);
      off = q * p.nls + r;
    }
    fiber_fixed<TN>(sm + fo * outer + off, stride, Mf);
  }
}

__device__ void mode_loop_generic(double* sm, const PassParams& p, int i, const double* Mf) {
  const int stride = p.sm_stride[i];
  const int outer = p.sm_outer[i];
  const bool inner_pad = p.contiguous && (i < p.k - 1);
  for (int f = threadIdx.x; f < p.fibers[i]; f += blockDim.x) {
    uint32_t fo, fi;
    p.fd_inner[i].divmod(static_cast<uint32_t>(f), fo, fi);
    uint32_t off = fi;
    if (inner_pad) {
      uint32_t q, r;
      p.fd_nlast.divmod(fi, q, r);
      off = q * p.nls + r;
    }
    fiber_generic(sm + fo * outer + off, stride, Mf, p.n[i]);
  }
}

template <int TN>
struct ModeTag { static constexpr int value = TN; };

template <typename F>
__device__ __forceinline__ bool dispatch_n(int n, F&& f) {
  switch (n) {
#define CB_CASE(v) case v: f(ModeTag<v>{}); return true;
    CB_CASE(1) CB_CASE(2) CB_CASE(3) CB_CASE(4) CB_CASE(5) CB_CASE(6) CB_CASE(7) CB_CASE(8)
    CB_CASE(9) CB_CASE(10) CB_CASE(11) CB_CASE(12) CB_CASE(13) CB_CASE(14) CB_CASE(15) CB_CASE(16)
    CB_CASE(17) CB_CASE(18) CB_CASE(19) CB_CASE(20) CB_CASE(21) CB_CASE(22) CB_CASE(23) CB_CASE(24)
    CB_CASE(25) CB_CASE(26) CB_CASE(27) CB_CASE(28) CB_CASE(29) CB_CASE(30) CB_CASE(31) CB_CASE(32)
    CB_CASE(33) CB_CASE(34)
#undef CB_CASE
    default: return false;
  }
}

__global__ void __launch_bounds__(kBuildThreads) build_pass_kernel(PassParams p) {
  extern __shared__ __align__(16) double smem[];
  double* mats = smem;
  double* tile = smem + ((p.mat_total + 1) & ~1);

  for (int i = 0; i < p.k; ++i) fill_folded(mats + p.moff[i], p.n[i], threadIdx.x, blockDim.x);

  for (long long t = blockIdx.x; t < p.tiles; t += gridDim.x) {
    __syncthreads();  // previous tile fully stored (and matrices ready on the first tile)
    // ---------------- load ----------------
    if (p.contiguous) {
      const double* src = p.in + t * p.in_tile_stride;
      for (int e = threadIdx.x; e < p.tile_elems; e += blockDim.x) {
        double v = __ldg(src + e);
        if (p.check_finite && !isfinite(v)) atomicAdd(&p.st->nonfinite, 1u);
        uint32_t q, r;
        p.fd_nlast.divmod(static_cast<uint32_t>(e), q, r);
        tile[q * p.nls + r] = v;
      }
    } else {
      long long a = t / p.ctiles;
      long long c0 = (t - a * p.ctiles) * p.ct;
      const double* src = p.in + a * (p.tile_elems / p.ct) * p.Cn + c0;
      for (int e = threadIdx.x; e < p.tile_elems; e += blockDim.x) {
        int b = e >> p.ct_shift, c = e & (p.ct - 1);
        double v = 0.0;
        if (c0 + c < p.Cn) {
          v = src[static_cast<long long>(b) * p.Cn + c];
          if (p.check_finite && !isfinite(v)) atomicAdd(&p.st->nonfinite, 1u);
        }
        tile[e] = v;
      }
    }
    // ---------------- mode products in shared memory ----------------
    for (int i = 0; i < p.k; ++i) {
      __syncthreads();
      const double* Mf = mats + p.moff[i];
      bool done = dispatch_n(p.n[i], [&](auto tag) {
        mode_loop_fixed<decltype(tag)::value>(tile, p, i, Mf);
      });
      if (!done) mode_loop_generic(tile, p, i, Mf);
    }
    __syncthreads();
    // ---------------- store ----------------
    if (p.contiguous) {
      double* dst = p.out + t * p.out_tile_stride;
      for (int e = threadIdx.x; e < p.tile_elems; e += blockDim.x) {
        uint32_t q, r;
        p.fd_nlast.divmod(static_cast<uint32_t>(e), q, r);
        double v = tile[q * p.nls + r];
        uint32_t row, col;
        p.fd_K.divmod(static_cast<uint32_t>(e), row, col);
        dst[static_cast<long long>(row) * p.Kp + col] = v;
      }
      if (p.Kp > p.K) {
        int padw = p.Kp - p.K;
        int rows = p.tile_elems / p.K;
        for (int z = threadIdx.x; z < rows * padw; z += blockDim.x) {
          int row = z / padw, col = p.K + (z - row * padw);
          dst[static_cast<long long>(row) * p.Kp + col] = 0.0;
        }
      }
    } else {
      long long a = t / p.ctiles;
      long long c0 = (t - a * p.ctiles) * p.ct;
      double* dst = p.out + a * (p.tile_elems / p.ct) * p.Cn + c0;
      for (int e = threadIdx.x; e < p.tile_elems; e += blockDim.x) {
        int b = e >> p.ct_shift, c = e & (p.ct - 1);
        if (c0 + c < p.Cn) dst[static_cast<long long>(b) * p.Cn + c] = tile[e];
      }
    }
  }
}

// Smem budget per tile (doubles).  96 KB keeps two CTAs per SM.
constexpr int kTileBudget = 12288;

// Fill the group-dependent smem geometry of a pass.
void finish_geometry(PassParams& p) {
  // smem extents: contiguous -> dims (n_0..n_{k-1}) with the last padded to odd;
  //               strided    -> dims (n_0..n_{k-1}, ct) dense.
  int ext_last_stride;
  if (p.contiguous) {
    p.nlast = p.n[p.k - 1];
    p.nls = (p.nlast % 2 == 0) ? p.nlast + 1 : p.nlast;
    p.sm_stride[p.k - 1] = 1;
    p.sm_outer[p.k - 1] = p.nls;
    ext_last_stride = p.nls;
  } else {
    p.nlast = p.n[p.k - 1];
    p.nls = p.nlast;
    p.sm_stride[p.k - 1] = p.ct;
    p.sm_outer[p.k - 1] = p.ct * p.nlast;
    ext_last_stride = p.ct * p.nlast;
  }
  for (int i = p.k - 2; i >= 0; --i) {
    p.sm_stride[i] = ext_last_stride;
    p.sm_outer[i] = ext_last_stride * p.n[i];
    ext_last_stride *= p.n[i];
  }
  p.tile_smem = ext_last_stride;
  long long real = p.contiguous ? 1 : p.ct;
  for (int i = 0; i < p.k; ++i) real *= p.n[i];
  p.tile_elems = static_cast<int>(real);
  for (int i = 0; i < p.k; ++i) {
    long long inner = p.contiguous ? 1 : p.ct;
    for (int m = i + 1; m < p.k; ++m) inner *= p.n[m];
    p.fd_inner[i] = FastDiv(static_cast<uint32_t>(inner));
    p.fibers[i] = static_cast<int>(real / p.n[i]);
  }
  p.fd_nlast = FastDiv(static_cast<uint32_t>(p.nlast));
  int off = 0;
  for (int i = 0; i < p.k; ++i) {
    p.moff[i] = off;
    off += p.n[i] * (p.n[i] / 2 + 1);
  }
  p.mat_total = off;
}

cudaError_t launch_pass(PassParams& p, cudaStream_t stream) {
  size_t smem = sizeof(double) * (static_cast<size_t>((p.mat_total + 1) & ~1) + p.tile_smem);
  ensure_smem_attr(reinterpret_cast<const void*>(build_pass_kernel), 200 * 1024);
  long long grid = p.tiles;
  long long cap = static_cast<long long>(num_sms()) * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  build_pass_kernel<<<static_cast<unsigned>(grid), kBuildThreads, smem, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}


// ------------------------------------------------------------------------------------------
// Fiber-parallel mode pass (one launch per transformed mode): thread = one fiber along the mode,
// i.e. one (n)-vector of the tensor with every other index fixed.  Fibers are enumerated with the
// innermost remaining index fastest, so a warp's loads/stores are coalesced whenever the mode is
// not the innermost one.  Any strided layout works for input and output (dense C-order tensors,
// the pitched eval layout, stacks with a trailing member axis), so the first pass can read the
// dense samples and write the eval layout while later passes run in place.  The folded matrix
// rides in the kernel parameters and unrolled FMAs take it as constant-bank operands.
// ------------------------------------------------------------------------------------------
constexpr int kFiberThreads = 128;
constexpr long long kFiberMinFibers = 1;  // fiber passes whenever every mode has n <= 34
constexpr int kFMat = 34 * 18;

struct FiberParams {
  const double* in;
  double* out;
  Status* st;
  int check_finite;
  int nother;                          // number of other (non-transformed) dims
  int nd[kMaxDims + 1];                // their sizes, enumeration order (last = fastest)
  FastDiv fd[kMaxDims + 1];
  long long sin[kMaxDims + 1], sout[kMaxDims + 1];  // their strides (elements)
  long long kin, kout;                 // stride of the transformed mode
  long long fibers;
  double M[kFMat];                     // folded matrix, row pitch n/2 + 1 (n <= 34)
};

template <int TN>
__global__ void __launch_bounds__(kFiberThreads) fiber_pass_kernel(const __grid_constant__ FiberParams p) {
  const long long f = static_cast<long long>(blockIdx.x) * kFiberThreads + threadIdx.x;
  if (f >= p.fibers) return;
  long long oin = 0, oout = 0;
  uint32_t rem = static_cast<uint32_t>(f);
#pragma unroll
  for (int i = kMaxDims; i >= 0; --i) {
    if (i < p.nother) {
      uint32_t q, r;
      p.fd[i].divmod(rem, q, r);
      oin += static_cast<long long>(r) * p.sin[i];
      oout += static_cast<long long>(r) * p.sout[i];
      rem = q;
    }
  }
  const double* src = p.in + oin;
  double* dst = p.out + oout;
  if constexpr (TN == 1) {
    dst[0] = src[0];
    if (p.check_finite && !isfinite(src[0])) atomicAdd(&p.st->nonfinite, 1u);
  } else {
    constexpr int N = TN - 1, H = TN / 2, P = H + 1;
    double v[TN];
#pragma unroll
    for (int k = 0; k < TN; ++k) v[k] = src[k * p.kin];
    if (p.check_finite) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < TN; ++k) ok &= isfinite(v[k]);
      if (!ok) atomicAdd(&p.st->nonfinite, 1u);
    }
    double e[H], o[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      e[k] = v[k] + v[N - k];
      o[k] = v[k] - v[N - k];
    }
#pragma unroll
    for (int l = 0; l <= N; ++l) {
      double acc = 0.0;
      if ((l & 1) == 0) {
#pragma unroll
        for (int k = 0; k < H; ++k) acc = fma(p.M[l * P + k], e[k], acc);
        if constexpr (TN & 1) acc = fma(p.M[l * P + H], v[H], acc);
      } else {
#pragma unroll
        for (int k = 0; k < H; ++k) acc = fma(p.M[l * P + k], o[k], acc);
      }
      dst[l * p.kout] = acc;
    }
  }
}


// Innermost-mode fiber pass (unit stride in and out): a block stages 128 consecutive fibers
// (contiguous 128*TN doubles of the dense input) through shared memory, so global loads and the
// row stores are coalesced instead of each lane walking its own TN-element fiber.
template <int TN>
__global__ void __launch_bounds__(kFiberThreads) fiber_inner_kernel(const __grid_constant__ FiberParams p) {
  __shared__ double buf[kFiberThreads * TN];
  __shared__ long long ooff[kFiberThreads];
  const long long f0 = static_cast<long long>(blockIdx.x) * kFiberThreads;
  const int nf = static_cast<int>(min(static_cast<long long>(kFiberThreads), p.fibers - f0));
  // fiber f's input offset is f*TN (dense, innermost mode); output offset via the other-dim strides
  {
    const long long f = f0 + threadIdx.x;
    long long oout = 0;
    if (threadIdx.x < nf) {
      uint32_t rem = static_cast<uint32_t>(f);
#pragma unroll
      for (int i = kMaxDims; i >= 0; --i) {
        if (i < p.nother) {
          uint32_t q, r;
          p.fd[i].divmod(rem, q, r);
          oout += static_cast<long long>(r) * p.sout[i];
          rem = q;
        }
      }
    }
    ooff[threadIdx.x] = oout;
  }
  const double* src = p.in + f0 * TN;
  for (int e = threadIdx.x; e < nf * TN; e += kFiberThreads) buf[e] = src[e];
  __syncthreads();
  if (threadIdx.x < nf) {
    constexpr int N = TN - 1, H = TN / 2, P = H + 1;
    double v[TN];
    double* row = buf + threadIdx.x * TN;
#pragma unroll
    for (int k = 0; k < TN; ++k) v[k] = row[k];
    if (p.check_finite) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < TN; ++k) ok &= isfinite(v[k]);
      if (!ok) atomicAdd(&p.st->nonfinite, 1u);
    }
    double e[H > 0 ? H : 1], o[H > 0 ? H : 1];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      e[k] = v[k] + v[N - k];
      o[k] = v[k] - v[N - k];
    }
#pragma unroll
    for (int l = 0; l <= N; ++l) {
      double acc = 0.0;
      if ((l & 1) == 0) {
#pragma unroll
        for (int k = 0; k < H; ++k) acc = fma(p.M[l * P + k], e[k], acc);
        if constexpr (TN & 1) acc = fma(p.M[l * P + H], v[H], acc);
      } else {
#pragma unroll
        for (int k = 0; k < H; ++k) acc = fma(p.M[l * P + k], o[k], acc);
      }
      row[l] = acc;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nf * TN; e += kFiberThreads) {
    const int fl = e / TN, l = e - (e / TN) * TN;
    p.out[ooff[fl] + l] = buf[e];
  }
}

template <int TN>
struct FTag { static constexpr int value = TN; };

template <typename F>
bool dispatch_fiber(int n, F&& f) {
  switch (n) {
#define CB_CASE(v) case v: f(FTag<v>{}); return true;
    CB_CASE(1) CB_CASE(2) CB_CASE(3) CB_CASE(4) CB_CASE(5) CB_CASE(6) CB_CASE(7) CB_CASE(8)
    CB_CASE(9) CB_CASE(10) CB_CASE(11) CB_CASE(12) CB_CASE(13) CB_CASE(14) CB_CASE(15) CB_CASE(16)
    CB_CASE(17) CB_CASE(18) CB_CASE(19) CB_CASE(20) CB_CASE(21) CB_CASE(22) CB_CASE(23) CB_CASE(24)
    CB_CASE(25) CB_CASE(26) CB_CASE(27) CB_CASE(28) CB_CASE(29) CB_CASE(30) CB_CASE(31) CB_CASE(32)
    CB_CASE(33) CB_CASE(34)
#undef CB_CASE
    default: return false;
  }
}

// One mode pass over a strided tensor: dims (sizes) with input strides `sin` and output strides
// `sout`; mode `d` is transformed.  Returns false when n is outside the unrolled range.
bool launch_fiber_pass(int nd, const long long* sizes, const long long* sin, const long long* sout, int d,
                       const double* in, double* out, Status* st, int check_finite, cudaStream_t stream,
                       cudaError_t* err) {
  FiberParams p{};
  p.in = in;
  p.out = out;
  p.st = st;
  p.check_finite = check_finite;
  long long fibers = 1;
  int j = 0;
  for (int i = 0; i < nd; ++i) {
    if (i == d) continue;
    p.nd[j] = static_cast<int>(sizes[i]);
    p.fd[j] = FastDiv(static_cast<uint32_t>(sizes[i]));
    p.sin[j] = sin[i];
    p.sout[j] = sout[i];
    fibers *= sizes[i];
    ++j;
  }
  p.nother = j;
  p.kin = sin[d];
  p.kout = sout[d];
  p.fibers = fibers;
  const int n = static_cast<int>(sizes[d]);
  const int N = n - 1, P = n / 2 + 1;
  if (n > 34) return false;
  for (int l = 0; l < n; ++l)
    for (int c = 0; c < P; ++c) p.M[l * P + c] = (c <= N) ? transform_entry(l, c, N) : 0.0;
  const long long grid = (fibers + kFiberThreads - 1) / kFiberThreads;
  *err = cudaSuccess;
  if (grid <= 0) return true;
  // innermost mode with a dense input and unit output stride: shared-memory staged variant
  bool dense_in = p.kin == 1 && p.kout == 1 && n >= 2;
  if (dense_in) {
    long long expect = n;  // input strides of the other dims must be those of a dense C array
    for (int i = j - 1; i >= 0; --i) {
      dense_in = dense_in && p.sin[i] == expect;
      expect *= p.nd[i];
    }
  }
  dispatch_fiber(n, [&](auto tag) {
    constexpr int TN = decltype(tag)::value;
    if (dense_in && TN >= 2) fiber_inner_kernel<TN><<<static_cast<unsigned>(grid), kFiberThreads, 0, stream>>>(p);
    else fiber_pass_kernel<TN><<<static_cast<unsigned>(grid), kFiberThreads, 0, stream>>>(p);
  });
  count_launch();
  *err = cudaGetLastError();
  return true;
}


// ------------------------------------------------------------------------------------------
// Large modes (n > 34, any size up to the C-ABI limit): one CTA per fiber (grid-stride), the
// fiber's folded halves e/o staged in shared memory, each thread producing outputs l with the
// folded matrix read k-major from a device scratch table (coalesced across l).  The entries come
// from the same transform_entry (exact integer angle reduction) and every output sums k
// ascending then the middle sample, like fiber_fixed/fiber_generic: the same numerics at any n.
// ------------------------------------------------------------------------------------------
constexpr int kLargeThreads = 256;

__global__ void fold_matrix_kernel(double* Mt, int n) {
  const int N = n - 1, H = n / 2;
  const long long total = static_cast<long long>(H + 1) * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e / n), l = static_cast<int>(e % n);
    Mt[e] = (k <= N) ? transform_entry(l, k, N) : 0.0;
  }
}

struct LargeParams {
  const double* in;
  double* out;
  const double* Mt;       // [H+1][n] folded matrix, k-major
  Status* st;
  int check_finite;
  int n;
  int nother;
  int nd[kMaxDims + 1];
  long long sin[kMaxDims + 1], sout[kMaxDims + 1];
  long long kin, kout;
  long long fibers;
};

__global__ void __launch_bounds__(kLargeThreads) large_fiber_kernel(const __grid_constant__ LargeParams p) {
  extern __shared__ __align__(16) double lsm[];   // e[H+1], o[H]
  const int n = p.n, N = n - 1, H = n / 2;
  double* e = lsm;
  double* o = lsm + H + 1;
  bool ok = true;
  for (long long f = blockIdx.x; f < p.fibers; f += gridDim.x) {
    long long oin = 0, oout = 0, rem = f;
    for (int i = p.nother - 1; i >= 0; --i) {
      const long long q = rem / p.nd[i], r = rem - q * p.nd[i];
      oin += r * p.sin[i];
      oout += r * p.sout[i];
      rem = q;
    }
    __syncthreads();   // the previous fiber's outputs are written (in place) before new loads
    for (int k = threadIdx.x; k < H; k += blockDim.x) {
      const double a = p.in[oin + k * p.kin], b = p.in[oin + (N - k) * p.kin];
      ok &= isfinite(a) && isfinite(b);
      e[k] = a + b;
      o[k] = a - b;
    }
    if ((n & 1) && threadIdx.x == 0) {
      const double m = p.in[oin + H * p.kin];
      ok &= isfinite(m);
      e[H] = m;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < n; l += blockDim.x) {
      double acc = 0.0;
      if ((l & 1) == 0) {
        for (int k = 0; k < H; ++k) acc = fma(p.Mt[static_cast<long long>(k) * n + l], e[k], acc);
        if (n & 1) acc = fma(p.Mt[static_cast<long long>(H) * n + l], e[H], acc);
      } else {
        for (int k = 0; k < H; ++k) acc = fma(p.Mt[static_cast<long long>(k) * n + l], o[k], acc);
      }
      p.out[oout + l * p.kout] = acc;
    }
  }
  if (p.check_finite && !ok) atomicAdd(&p.st->nonfinite, 1u);
}

// One large-mode pass (mode d of a strided tensor, folded matrix Mt prepared for sizes[d]).
cudaError_t launch_large_pass(int nd, const long long* sizes, const long long* sin, const long long* sout, int d,
                              const double* in, double* out, const double* Mt, Status* st, int check_finite,
                              cudaStream_t stream) {
  LargeParams p{};
  p.in = in;
  p.out = out;
  p.Mt = Mt;
  p.st = st;
  p.check_finite = check_finite;
  p.n = static_cast<int>(sizes[d]);
  long long fibers = 1;
  int j = 0;
  for (int i = 0; i < nd; ++i) {
    if (i == d) continue;
    p.nd[j] = static_cast<int>(sizes[i]);
    p.sin[j] = sin[i];
    p.sout[j] = sout[i];
    fibers *= sizes[i];
    ++j;
  }
  p.nother = j;
  p.kin = sin[d];
  p.kout = sout[d];
  p.fibers = fibers;
  if (fibers <= 0) return cudaSuccess;
  long long grid = std::min<long long>(fibers, static_cast<long long>(num_sms()) * 8);
  const size_t bytes = sizeof(double) * (2 * static_cast<size_t>(p.n / 2) + 1);
  if (bytes > 48 * 1024) ensure_smem_attr(reinterpret_cast<const void*>(large_fiber_kernel), static_cast<int>(bytes));
  large_fiber_kernel<<<static_cast<unsigned>(grid), kLargeThreads, bytes, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

// Small tensors (<= kSmallBuild doubles, every mode n <= 34): the whole build in ONE launch of one
// CTA — samples staged in shared memory, every mode transformed there (last mode first, the same
// folded-matrix arithmetic as the fiber passes, so the result is bitwise identical to the
// multi-launch path), then scattered into the output layout with its zero padding written in the
// same kernel.  Replaces 3-7 launches (one per mode + pad zeroing) whose fixed cost dominates
// at these sizes (config 1, 17 x 17: 15.8 us -> one launch).
constexpr int kSmallBuild = 6144;     // doubles staged in shared memory (48 KB)
constexpr int kSmallMat = 2048;       // folded matrices of all modes (kernel parameters)
constexpr int kSmallThreads = 256;

struct SmallBuildParams {
  const double* in;
  double* out;
  Status* st;
  int check_finite;
  int nd;
  int n[kMaxDims + 1];
  int moff[kMaxDims + 1];               // offset of mode d's folded matrix in M
  long long sout[kMaxDims + 1];         // output strides (dense C-order or the eval layout)
  long long total;
  int evl;                              // write the eval layout's zero padding
  long long R, R8, K, Kp;
  double M[kSmallMat];
};

__global__ void __launch_bounds__(kSmallThreads) small_build_kernel(const __grid_constant__ SmallBuildParams p) {
  __shared__ double s[kSmallBuild];
  const int tid = threadIdx.x;
  const int total = static_cast<int>(p.total);
  for (int e = tid; e < total; e += kSmallThreads) {
    const double v = p.in[e];
    if (p.check_finite && !isfinite(v)) atomicAdd(&p.st->nonfinite, 1u);
    s[e] = v;
  }
  int stride = 1;
  for (int d = p.nd - 1; d >= 0; --d) {
    const int n = p.n[d];
    __syncthreads();
    if (n > 1) {
      const int fibers = total / n;
      for (int f = tid; f < fibers; f += kSmallThreads) {
        const int inner = f % stride, outer = f / stride;
        fiber_generic(s + outer * n * stride + inner, stride, p.M + p.moff[d], n);
      }
    }
    stride *= n;
  }
  __syncthreads();
  for (int e = tid; e < total; e += kSmallThreads) {
    long long off = 0;
    int rem = e;
    for (int d = p.nd - 1; d >= 0; --d) {
      const int q = rem / p.n[d];
      off += static_cast<long long>(rem - q * p.n[d]) * p.sout[d];
      rem = q;
    }
    p.out[off] = s[e];
  }
  if (p.evl) {
    const long long pc = p.Kp - p.K;
    for (long long i = tid; i < p.R * pc; i += kSmallThreads) p.out[(i / pc) * p.Kp + p.K + i % pc] = 0.0;
    for (long long i = p.R * p.Kp + tid; i < p.R8 * p.Kp; i += kSmallThreads) p.out[i] = 0.0;
  }
}

// Zero the pad columns [K, Kp) of rows [0, R) and the pad rows [R, R8) of an eval-layout tensor
// (one launch instead of a 2-D memset with a 3-column width plus a row memset).
__global__ void zero_pad_kernel(double* out, long long R, long long R8, long long K, long long Kp) {
  const long long pc = Kp - K;
  const long long n1 = R * pc, n2 = (R8 - R) * Kp;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n1 + n2;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (e < n1) out[(e / pc) * Kp + K + (e % pc)] = 0.0;
    else out[R * Kp + (e - n1)] = 0.0;
  }
}

}  // namespace

// Transform the consecutive axes [a0, a1) of a dense C-order array `shape` (ndim dims).
// When `evl` is non-null the call is a full tensor build (a0 = 0, a1 = ndim) and the output is
// written in the eval layout described by evl.
// ------------------------------------------------------------------------------------------
// Mode-group passes for full builds of equal-size modes (every BASELINE tensor above the
// single-CTA size): the J mode products are applied in 2 launches instead of J, each CTA holding
// one tile that spans a GROUP of up to 3 modes in shared memory, so the tensor crosses the
// L2 <-> SM boundary twice instead of J times (the intermediate stays in the 126 MB L2).
//   pass 1 (contiguous): the trailing group — a tile is S whole slabs of N^G contiguous samples,
//                        read once from the dense input (non-finite check), written to the eval
//                        layout with its pad columns (and, by block 0, the pad rows);
//   pass 2+ (strided)  : a group of leading modes in place on the eval layout — a tile is N^G rows
//                        x CW contiguous inner columns (32-128 B row segments).
// Per fiber the arithmetic is exactly the fiber passes' (same folded constant-bank matrix, same
// FMA order), so the result is bitwise identical to the per-mode path.
// ------------------------------------------------------------------------------------------
constexpr int kGroupMaxTile = 9216;        // doubles of one tile (72 KB: 2-3 CTAs per SM)
constexpr int kGroupMaxSlab = 6144;        // contiguous flavour: N^G per slab
constexpr int kGroupMaxG = 3;
// fibers per thread per mode: 2 measured faster for n = 13 (13^6: 51 -> 43 us), 1 for 17 and 33
#ifndef CB_FPT13
#define CB_FPT13 2
#endif
template <int TN>
constexpr int group_fpt() { return TN == 13 ? CB_FPT13 : 1; }

// One thread per fiber per mode (nf = E / N threads): straight-line code like the fiber passes
// (a loop over fibers lets the compiler hoist the ~N^2/2 matrix constants into registers and
// spill).  Each mode of the group reads its own copy of the folded matrix so the constants are
// not shared (and kept live) across the modes either.  Group size G and tile width CW are
// template parameters, so every fiber stride is a compile-time constant (immediate smem offsets,
// division by constants) — the kernel was issue-bound on index arithmetic before.
template <int TN>
constexpr int group_threads_max() { return TN > 24 ? 256 : 512; }

constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

template <int TN>
struct GroupParams {
  const double* in;
  double* out;
  Status* st;
  int check_finite;
  int vec;                  // 16-byte aligned rows: cp.async / stores two doubles at a time
  // contiguous flavour (CW = 1): tile t = slabs [t*S, t*S+S) of A, written in the output layout
  // (rows of K values at pitch Kp)
  int S;
  long long A;
  int K, Kp;
  FastDiv fd_Kp;
  long long R, R8;          // pad rows [R, R8) zeroed by block 0 (eval layout only)
  // strided flavour: tile t = (a, column tile), a < A, rows N^G x CW columns of inner extent Cn
  long long Cn, ctiles;
  double M[kGroupMaxG][TN * (TN / 2 + 1)];   // folded matrix per mode, row pitch N/2 + 1
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int TN, int STRIDE, bool CHECK>
__device__ __forceinline__ void group_fiber(double* s, const double* M, bool& ok, double* dst, long long step) {
  constexpr int N = TN - 1, H = TN / 2, P = H + 1;
  double v[TN];
#pragma unroll
  for (int k = 0; k < TN; ++k) v[k] = s[k * STRIDE];
  if constexpr (CHECK) {
#pragma unroll
    for (int k = 0; k < TN; ++k) ok &= isfinite(v[k]);
  }
  double e[H > 0 ? H : 1], o[H > 0 ? H : 1];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    e[k] = v[k] + v[N - k];
    o[k] = v[k] - v[N - k];
  }
#pragma unroll
  for (int l = 0; l <= N; ++l) {
    double acc = 0.0;
    if ((l & 1) == 0) {
#pragma unroll
      for (int k = 0; k < H; ++k) acc = fma(M[l * P + k], e[k], acc);
      if constexpr (TN & 1) acc = fma(M[l * P + H], v[H], acc);
    } else {
#pragma unroll
      for (int k = 0; k < H; ++k) acc = fma(M[l * P + k], o[k], acc);
    }
    if (dst) dst[l * step] = acc;   // the group's last mode: straight to the output
    else s[l * STRIDE] = acc;
  }
}

// The group's last mode writes its outputs straight to global memory (no final barrier and store
// loop) for the big tiles — three-mode groups or 16-column tiles: 13^6 42.5 -> 37.8 us, 17^5 16.8
// -> 15.0 us; the small tiles of 17^4 and 33^3 (few CTAs, latency-bound) measured faster through
// the tile and a row-wise store loop, which they keep.
template <int TN, int G, int CW>
constexpr bool group_direct() { return G == 3 || CW == 16; }

// where a tile's output goes (the group's last mode writes to global memory directly)
struct GroupOut {
  long long a0;       // contiguous flavour: first slab of the tile
  long long gbase;    // strided flavour: the tile's first element in the output
  long long c0;       // strided flavour: the tile's first column
};

template <int TN, int G, int CW, int g>
__device__ __forceinline__ void group_mode(double* tile, int nf, const GroupParams<TN>& p, bool& ok,
                                           const GroupOut& go) {
  constexpr int STRIDE = ipow(TN, G - 1 - g) * CW;
  constexpr int PG = ipow(TN, G);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < group_fpt<TN>(); ++j) {
    const int f = threadIdx.x + j * blockDim.x;
    if (f < nf) {
      const int o = f / STRIDE, i = f - (f / STRIDE) * STRIDE;
      double* dst = nullptr;
      long long step = 0;
      if constexpr (g == 0 && group_direct<TN, G, CW>()) {
        if constexpr (CW == 1) {
          const long long a = go.a0 + o;          // slab
          if (p.K == PG) {                        // one output row per slab
            dst = p.out + a * p.Kp + i;
            step = STRIDE;
          } else {                                // K divides STRIDE
            dst = p.out + (a * (PG / p.K) + i / p.K) * p.Kp + (i % p.K);
            step = static_cast<long long>(STRIDE / p.K) * p.Kp;
          }
        } else {
          const int cc = i % CW;
          if (go.c0 + cc >= p.Cn) continue;       // column past the end
          dst = p.out + go.gbase + static_cast<long long>(i / CW) * p.Cn + cc;
          step = static_cast<long long>(ipow(TN, G - 1)) * p.Cn;
        }
      }
      group_fiber<TN, STRIDE, g == G - 1 && CW == 1>(tile + o * TN * STRIDE + i, p.M[g], ok, dst, step);
    }
  }
  if constexpr (g > 0) group_mode<TN, G, CW, (g > 0 ? g - 1 : 0)>(tile, nf, p, ok, go);
}

template <int TN, int G, int CW>
__global__ void __launch_bounds__(group_threads_max<TN>()) group_pass_kernel(const __grid_constant__ GroupParams<TN> p) {
  constexpr int P = ipow(TN, G);
  extern __shared__ __align__(16) double tile[];
  const int tid = threadIdx.x, nth = blockDim.x;
  const long long t = blockIdx.x;
  bool ok = true;
  GroupOut go{};
  if constexpr (CW == 1) {
    // ---------------- contiguous flavour: S whole slabs of the dense input ----------------
    const long long a0 = t * p.S;
    const int valid = static_cast<int>(min(static_cast<long long>(p.S), p.A - a0)) * P;
    const double* src = p.in + a0 * P;
    if (p.vec) {
      const int vend = valid & ~1;   // a last tile of an odd number of odd slabs: one tail element
      for (int e = 2 * tid; e < vend; e += 2 * nth) cp_async16(tile + e, src + e);
      if (tid == 0 && vend < valid) cp_async8(tile + vend, src + vend);
    } else {
      for (int e = tid; e < valid; e += nth) cp_async8(tile + e, src + e);
    }
    cp_async_wait_all();
    go.a0 = a0;
    // innermost mode first (the per-mode passes' order: bitwise-identical results); the last
    // mode writes the output rows (pitch Kp) directly
    group_mode<TN, G, CW, G - 1>(tile, valid / TN, p, ok, go);
    if (p.check_finite && !ok) atomicAdd(&p.st->nonfinite, 1u);   // first mode's loads checked
    if constexpr (!group_direct<TN, G, CW>()) {
      // rows of K values -> output rows of pitch Kp (pad columns written as zeros)
      __syncthreads();
      const int rows = valid / p.K;
      double* dst = p.out + (a0 * P / p.K) * p.Kp;
      const int n_out = rows * p.Kp;
      if (p.vec) {
        for (int z = 2 * tid; z < n_out; z += 2 * nth) {
          uint32_t row, col;
          p.fd_Kp.divmod(static_cast<uint32_t>(z), row, col);
          const double* srow = tile + row * p.K;
          double2 v;
          v.x = (static_cast<int>(col) < p.K) ? srow[col] : 0.0;
          v.y = (static_cast<int>(col) + 1 < p.K) ? srow[col + 1] : 0.0;
          *reinterpret_cast<double2*>(dst + z) = v;
        }
      } else {
        for (int z = tid; z < n_out; z += nth) {
          uint32_t row, col;
          p.fd_Kp.divmod(static_cast<uint32_t>(z), row, col);
          dst[z] = (static_cast<int>(col) < p.K) ? tile[row * p.K + col] : 0.0;
        }
      }
    }
    // pad columns of this tile's output rows
    const int padw = p.Kp - p.K;
    if (group_direct<TN, G, CW>() && padw > 0) {
      const int rows = valid / p.K;
      double* prow = p.out + (a0 * P / p.K) * p.Kp + p.K;
      for (int z = tid; z < rows * padw; z += nth) prow[static_cast<long long>(z / padw) * p.Kp + z % padw] = 0.0;
    }
    if (t == 0 && p.R8 > p.R) {
      double* pad = p.out + p.R * p.Kp;
      const long long n = (p.R8 - p.R) * p.Kp;
      for (long long z = tid; z < n; z += nth) pad[z] = 0.0;
    }
  } else {
    // ---------------- strided flavour: N^G rows x CW columns, in place ----------------
    constexpr int E = P * CW;
    const long long a = t / p.ctiles;
    const long long c0 = (t - a * p.ctiles) * CW;
    const long long gbase = a * P * p.Cn + c0;
    const bool full = c0 + CW <= p.Cn;
    const double* src = p.in + gbase;
    if (full && p.vec) {
      for (int e = 2 * tid; e < E; e += 2 * nth) {
        const int r = e / CW, cc = e % CW;
        cp_async16(tile + e, src + static_cast<long long>(r) * p.Cn + cc);
      }
    } else {
      for (int e = tid; e < E; e += nth) {
        const int r = e / CW, cc = e % CW;
        if (c0 + cc < p.Cn) cp_async8(tile + e, src + static_cast<long long>(r) * p.Cn + cc);
        else tile[e] = 0.0;
      }
    }
    cp_async_wait_all();
    go.gbase = gbase;
    go.c0 = c0;
    // in place: the tile's inputs are all in shared memory before the last mode stores anything
    group_mode<TN, G, CW, G - 1>(tile, E / TN, p, ok, go);
    if constexpr (!group_direct<TN, G, CW>()) {
      __syncthreads();
      double* dst = p.out + gbase;
      if (full && p.vec) {
        for (int e = 2 * tid; e < E; e += 2 * nth) {
          const int r = e / CW, cc = e % CW;
          *reinterpret_cast<double2*>(dst + static_cast<long long>(r) * p.Cn + cc) =
              *reinterpret_cast<const double2*>(tile + e);
        }
      } else {
        for (int e = tid; e < E; e += nth) {
          const int r = e / CW, cc = e % CW;
          if (c0 + cc < p.Cn) dst[static_cast<long long>(r) * p.Cn + cc] = tile[e];
        }
      }
    }
  }
}

// Host-side description of one group pass (independent of the template size).
struct GroupPass {
  int contiguous, G, P, E, S, K, Kp, CW, vec;
  long long A, R, R8, Cn, tiles;
};

template <int TN>
constexpr bool group_templated() { return TN == 5 || TN == 9 || TN == 13 || TN == 17 || TN == 33; }

template <int TN, int G>
void launch_group_g(const GroupParams<TN>& p, const GroupPass& g, int threads, int bytes, cudaStream_t stream) {
  auto go = [&](auto kern) {
    ensure_smem_attr(reinterpret_cast<const void*>(kern), kGroupMaxTile * 8, true);
    kern<<<static_cast<unsigned>(g.tiles), threads, bytes, stream>>>(p);
  };
  switch (g.CW) {
    case 1: go(group_pass_kernel<TN, G, 1>); break;
    case 4: go(group_pass_kernel<TN, G, 4>); break;
    case 8: go(group_pass_kernel<TN, G, 8>); break;
    case 16: go(group_pass_kernel<TN, G, 16>); break;
    default: break;   // not planned
  }
}

template <int TN>
void launch_group(const GroupPass& g, const double* in, double* out, Status* st, int check_finite,
                  cudaStream_t stream) {
  if constexpr (group_templated<TN>()) {
    GroupParams<TN> p{};
    p.in = in;
    p.out = out;
    p.st = st;
    p.check_finite = check_finite;
    p.vec = g.vec;
    p.S = g.S;
    p.A = g.A;
    p.K = g.K;
    p.Kp = g.Kp;
    if (g.Kp > 0) p.fd_Kp = FastDiv(static_cast<uint32_t>(g.Kp));
    p.R = g.R;
    p.R8 = g.R8;
    p.Cn = g.Cn;
    p.ctiles = g.contiguous ? 0 : (g.Cn + g.CW - 1) / g.CW;
    constexpr int N = TN - 1, P = TN / 2 + 1;
    for (int l = 0; l < TN; ++l)
      for (int c = 0; c < P; ++c) {
        const double v = (c <= N) ? transform_entry(l, c, N) : 0.0;
        for (int k = 0; k < kGroupMaxG; ++k) p.M[k][l * P + c] = v;
      }
    const int nf = g.E / TN;
    int threads = ((nf + group_fpt<TN>() - 1) / group_fpt<TN>() + 31) & ~31;
    if (threads < 64) threads = 64;
    const int bytes = g.E * static_cast<int>(sizeof(double));
    if (g.G == 1) launch_group_g<TN, 1>(p, g, threads, bytes, stream);
    else if (g.G == 2) launch_group_g<TN, 2>(p, g, threads, bytes, stream);
    else launch_group_g<TN, 3>(p, g, threads, bytes, stream);
    count_launch();
  }
}

// Full build of a tensor whose modes all have size n (2 <= n <= 34) in 2-3 mode-group passes.
// Returns false (nothing launched) when the shape does not fit the plan.
bool group_build(int ndim, const long long* shape, const double* in, double* out, Status* st, int check_finite,
                 const EvalLayout* evl, cudaStream_t stream, cudaError_t* err) {
  *err = cudaSuccess;
  if (ndim < 2 || ndim > kMaxDims) return false;
  const int n = static_cast<int>(shape[0]);
  if (n != 5 && n != 9 && n != 13 && n != 17 && n != 33) return false;   // group_templated<>
  for (int d = 1; d < ndim; ++d)
    if (shape[d] != n) return false;
  long long pw[kMaxDims + 1];
  pw[0] = 1;
  for (int d = 1; d <= ndim; ++d) pw[d] = pw[d - 1] * n;
  const long long total = pw[ndim];
  const int q = evl ? evl->q : 0;
  const long long K = evl ? evl->K : 1, Kp = evl ? evl->Kp : 1;
  const long long outsz = evl ? evl->R8 * evl->Kp : total;
  if (outsz >= (1LL << 31) || total >= (1LL << 31)) return false;
  const int max_threads = (n > 24 ? 256 : 512) * (n == 13 ? CB_FPT13 : 1);   // fibers per tile and mode
  const long long max_tile = std::min<long long>(kGroupMaxTile, static_cast<long long>(max_threads) * n);
  const int sms = num_sms();
  GroupPass plan[3];
  int np = 0;
  // trailing group (pass 1): the largest g (>= q, < ndim) whose slab fits, preferring >= one
  // slab per SM
  int gt = 0;
  // CB_GROUP_MAXG=<1..3> (experiments only): cap the modes per group
  static const int gmax = [] {
    const char* e = std::getenv("CB_GROUP_MAXG");
    const int v = e ? std::atoi(e) : kGroupMaxG;
    return v < 1 || v > kGroupMaxG ? kGroupMaxG : v;
  }();
  for (int g = std::min(ndim - 1, gmax); g >= 1; --g) {
    if (g < q || pw[g] > std::min<long long>(kGroupMaxSlab, max_tile)) continue;
    if (gt == 0) gt = g;
    if (pw[ndim - g] >= sms) { gt = g; break; }
  }
  if (gt == 0) return false;
  {
    GroupPass& g = plan[np++];
    g = GroupPass{};
    g.contiguous = 1;
    g.CW = 1;
    g.G = gt;
    g.P = static_cast<int>(pw[gt]);
    g.A = pw[ndim - gt];
    int S = 1;
    // CB_GROUP_SMAX=<n> (experiments only): cap the slabs per CTA of the contiguous pass
    static const int smax = [] {
      const char* e = std::getenv("CB_GROUP_SMAX");
      const int v = e ? std::atoi(e) : 0;
      return v >= 1 ? v : 1 << 20;
    }();
    while (2 * S <= smax && 2LL * S * g.P <= max_tile && (g.A + 2 * S - 1) / (2 * S) >= 2 * sms && S * g.P / n < 256) S *= 2;
    if ((g.P & 1) && (S & 1) && S > 1) --S;
    g.S = S;
    g.E = S * g.P;
    g.K = evl ? static_cast<int>(K) : g.P;
    g.Kp = evl ? static_cast<int>(Kp) : g.P;
    g.R = evl ? evl->R : 0;
    g.R8 = evl ? evl->R8 : 0;
    g.tiles = (g.A + S - 1) / S;
    // 16-byte vectors: every tile's slab start and every output row 16-byte aligned
    g.vec = (reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
             (static_cast<long long>(S) * g.P) % 2 == 0 && g.Kp % 2 == 0 && (g.P % 2 == 0 || S % 2 == 0))
                ? 1 : 0;
  }
  // leading modes [0, ndim - gt): strided groups, innermost first, in place on the output
  for (int hi = ndim - gt; hi > 0;) {
    int G = 0;
    while (G < gmax && hi - G - 1 >= 0 && pw[G + 1] * 4 <= max_tile) ++G;
    if (G == 0 || np == 3) return false;   // more passes than the plan is worth: per-mode path
    GroupPass& g = plan[np++];
    g = GroupPass{};
    g.contiguous = 0;
    g.G = G;
    g.P = static_cast<int>(pw[G]);
    long long Cn = 1;
    if (evl) {
      for (int d = hi; d < ndim - q; ++d) Cn *= n;
      Cn *= Kp;
    } else {
      Cn = pw[ndim - hi];
    }
    g.A = pw[hi - G];
    int CW = 16;
    while (CW > 4 && (g.P * CW > max_tile || g.A * ((Cn + CW - 1) / CW) < 2 * sms)) CW >>= 1;
    if (g.P * CW > max_tile) return false;
    g.CW = CW;
    g.Cn = Cn;
    g.E = g.P * CW;
    g.tiles = g.A * ((Cn + CW - 1) / CW);
    g.vec = (reinterpret_cast<uintptr_t>(out) % 16 == 0 && Cn % 2 == 0) ? 1 : 0;
    hi -= G;
  }
  for (int i = 0; i < np; ++i) {
    const bool ok = dispatch_fiber(n, [&](auto tag) {
      launch_group<decltype(tag)::value>(plan[i], i == 0 ? in : out, out, st, i == 0 ? check_finite : 0, stream);
    });
    if (!ok) return i > 0;
    *err = cudaGetLastError();
    if (*err != cudaSuccess) return true;
  }
  return true;
}

cudaError_t transform_axes(int ndim, const long long* shape, int a0, int a1, const double* in, double* out,
                           Status* st, int check_finite, const EvalLayout* evl, cudaStream_t stream) {
  // the status block is optional (header): without one there is nowhere to report a non-finite
  // sample, so the kernels must not touch it
  if (st == nullptr) check_finite = 0;
  if (a0 >= a1) {
    // nothing to transform: plain copy
    long long total = 1;
    for (int d = 0; d < ndim; ++d) total *= shape[d];
    if (in != out) return cudaMemcpyAsync(out, in, sizeof(double) * total, cudaMemcpyDeviceToDevice, stream);
    return cudaSuccess;
  }
  bool large_modes = false;
  for (int d = a0; d < a1; ++d) {
    if (shape[d] < 1 || shape[d] > kMaxTransformN) return cudaErrorInvalidValue;
    if (shape[d] > kMaxGenericN) large_modes = true;
  }
  {
    long long total = 1;
    bool small_modes = true;
    long long min_fibers = -1;
    for (int d = 0; d < ndim; ++d) total *= shape[d];
    for (int d = a0; d < a1; ++d) {
      if (shape[d] > 34) small_modes = false;
      const long long fb = total / shape[d];
      if (min_fibers < 0 || fb < min_fibers) min_fibers = fb;
    }
    // CB_BUILD_PERMODE=1 (experiments only): keep the per-mode fiber passes for A/B timing
    static const bool permode = [] {
      const char* e = std::getenv("CB_BUILD_PERMODE");
      return e && e[0] == '1';
    }();
    if (a0 == 0 && a1 == ndim && total > kSmallBuild && !permode) {
      cudaError_t gerr = cudaSuccess;
      if (group_build(ndim, shape, in, out, st, check_finite, evl, stream, &gerr)) return gerr;
    }
    if ((small_modes || large_modes) && min_fibers >= kFiberMinFibers && ndim <= kMaxDims + 1) {
      // strides: input dense C-order; output dense or the eval layout (leading rows x Kp pitch)
      long long sin[kMaxDims + 1], sout[kMaxDims + 1];
      long long acc = 1;
      for (int d = ndim - 1; d >= 0; --d) {
        sin[d] = acc;
        acc *= shape[d];
      }
      if (evl) {
        long long a2 = 1;
        for (int d = ndim - 1; d >= ndim - evl->q; --d) {
          sout[d] = a2;
          a2 *= shape[d];
        }
        long long a3 = evl->Kp;
        for (int d = ndim - evl->q - 1; d >= 0; --d) {
          sout[d] = a3;
          a3 *= shape[d];
        }
      } else {
        for (int d = 0; d < ndim; ++d) sout[d] = sin[d];
      }
      // small tensor, all modes: one single-CTA launch (small_build_kernel)
      long long mat = 0;
      for (int d = 0; d < ndim; ++d) mat += shape[d] * (shape[d] / 2 + 1);
      if (small_modes && a0 == 0 && a1 == ndim && total <= kSmallBuild && mat <= kSmallMat) {
        SmallBuildParams sp{};
        sp.in = in;
        sp.out = out;
        sp.st = st;
        sp.check_finite = check_finite;
        sp.nd = ndim;
        sp.total = total;
        int mo = 0;
        for (int d = 0; d < ndim; ++d) {
          const int n = static_cast<int>(shape[d]), N = n - 1, P = n / 2 + 1;
          sp.n[d] = n;
          sp.sout[d] = sout[d];
          sp.moff[d] = mo;
          for (int l = 0; l < n; ++l)
            for (int c = 0; c < P; ++c) sp.M[mo + l * P + c] = (c <= N) ? transform_entry(l, c, N) : 0.0;
          mo += n * P;
        }
        if (evl) {
          sp.evl = 1;
          sp.R = evl->R;
          sp.R8 = evl->R8;
          sp.K = evl->K;
          sp.Kp = evl->Kp;
        }
        small_build_kernel<<<1, kSmallThreads, 0, stream>>>(sp);
        count_launch();
        return cudaGetLastError();
      }
      if (evl) {
        // zero the pad columns / rows (never written by the passes)
        if (evl->Kp > evl->K || evl->R8 > evl->R) {
          const long long n = evl->R * (evl->Kp - evl->K) + (evl->R8 - evl->R) * evl->Kp;
          long long g = (n + 255) / 256;
          if (g > num_sms() * 4LL) g = num_sms() * 4LL;
          zero_pad_kernel<<<static_cast<unsigned>(g), 256, 0, stream>>>(out, evl->R, evl->R8, evl->K, evl->Kp);
          count_launch();
          cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) return e;
        }
      } else {
        for (int d = 0; d < ndim; ++d) sout[d] = sin[d];
      }
      // folded matrices of the large modes: device scratch (stream-ordered pool), one per size
      double* mats[kMaxDims + 1] = {};
      cudaError_t err = cudaSuccess;
      for (int d = a0; d < a1 && err == cudaSuccess; ++d) {
        if (shape[d] <= 34) continue;
        for (int d2 = a0; d2 < d; ++d2)
          if (shape[d2] == shape[d]) mats[d] = mats[d2];
        if (mats[d]) continue;
        const long long n = shape[d], cnt = (n / 2 + 1) * n;
        err = cudaMallocAsync(reinterpret_cast<void**>(&mats[d]), sizeof(double) * cnt, stream);
        if (err != cudaSuccess) {
          mats[d] = nullptr;
          break;
        }
        fold_matrix_kernel<<<static_cast<unsigned>(std::min<long long>((cnt + 255) / 256, 1024)), 256, 0, stream>>>(
            mats[d], static_cast<int>(n));
        count_launch();
        err = cudaGetLastError();
      }
      const double* cur = in;
      bool first = true;
      for (int d = a1 - 1; d >= a0 && err == cudaSuccess; --d) {
        if (shape[d] <= 34) {
          if (!launch_fiber_pass(ndim, shape, first ? sin : sout, sout, d, cur, out, st, first ? check_finite : 0,
                                 stream, &err))
            err = cudaErrorInvalidValue;
        } else {
          err = launch_large_pass(ndim, shape, first ? sin : sout, sout, d, cur, out, mats[d], st,
                                  first ? check_finite : 0, stream);
        }
        cur = out;
        first = false;
      }
      for (int d = a0; d < a1; ++d) {
        if (!mats[d]) continue;
        bool shared = false;
        for (int d2 = d + 1; d2 < a1; ++d2) shared = shared || mats[d2] == mats[d];
        if (!shared) cudaFreeAsync(mats[d], stream);
      }
      return err;
    }
  }
  long long inner = 1;
  for (int d = a1; d < ndim; ++d) inner *= shape[d];
  long long outer = 1;
  for (int d = 0; d < a0; ++d) outer *= shape[d];

  const double* cur_in = in;
  int hi = a1;  // modes [a0, hi) still to do
  bool first = true;

  // Pass 1 (contiguous) when the transformed modes are innermost.
  if (inner == 1) {
    int g = 0;
    long long prod = 1;
    while (hi - g - 1 >= a0) {
      long long next = prod * shape[hi - g - 1];
      long long padded = (next / shape[hi - 1]) * (shape[hi - 1] + 1);
      if (padded > kTileBudget || g >= kMaxGroup) break;
      prod = next;
      ++g;
    }
    if (evl) {
      // the contiguous group must cover the q merged modes
      if (g < evl->q) return cudaErrorInvalidValue;
    }
    if (g >= 1) {
      PassParams p{};
      p.in = cur_in;
      p.out = out;
      p.st = st;
      p.check_finite = check_finite;
      p.contiguous = 1;
      p.k = g;
      for (int i = 0; i < g; ++i) p.n[i] = static_cast<int>(shape[hi - g + i]);
      p.ct = 1;
      finish_geometry(p);
      long long rest = outer;
      for (int d = a0; d < hi - g; ++d) rest *= shape[d];
      p.tiles = rest;
      p.in_tile_stride = prod;
      if (evl) {
        p.K = static_cast<int>(evl->K);
        p.Kp = static_cast<int>(evl->Kp);
        p.out_tile_stride = (prod / evl->K) * evl->Kp;
      } else {
        p.K = static_cast<int>(prod);
        p.Kp = p.K;
        p.out_tile_stride = prod;
      }
      p.fd_K = FastDiv(static_cast<uint32_t>(p.K));
      cudaError_t err = launch_pass(p, stream);
      if (err != cudaSuccess) return err;
      cur_in = out;
      first = false;
      hi -= g;
    }
  } else if (evl) {
    return cudaErrorInvalidValue;
  }

  // Remaining modes: strided groups, innermost first, in place on `out`.
  while (hi > a0) {
    // inner extent (in the output layout) of the modes after `hi`
    long long Cn = 1;
    if (evl) {
      for (int d = hi; d < ndim - evl->q; ++d) Cn *= shape[d];
      Cn *= evl->Kp;
    } else {
      for (int d = hi; d < ndim; ++d) Cn *= shape[d];
    }
    int g = 0;
    long long prod = 1;
    while (hi - g - 1 >= a0 && g < kMaxGroup) {
      long long next = prod * shape[hi - g - 1];
      if (next * 4 > kTileBudget && g >= 1) break;
      prod = next;
      ++g;
    }
    int ct = 32;
    while (ct > 1 && (prod * ct > kTileBudget || ct / 2 >= Cn)) ct >>= 1;
    PassParams p{};
    p.in = cur_in;
    p.out = out;
    p.st = st;
    p.check_finite = first ? check_finite : 0;
    p.contiguous = 0;
    p.k = g;
    for (int i = 0; i < g; ++i) p.n[i] = static_cast<int>(shape[hi - g + i]);
    p.ct = ct;
    p.ct_shift = 0;
    while ((1 << p.ct_shift) < ct) ++p.ct_shift;
    p.Cn = Cn;
    finish_geometry(p);
    long long A = outer;
    for (int d = a0; d < hi - g; ++d) A *= shape[d];
    p.ctiles = (Cn + ct - 1) / ct;
    p.tiles = A * p.ctiles;
    cudaError_t err = launch_pass(p, stream);
    if (err != cudaSuccess) return err;
    cur_in = out;
    first = false;
    hi -= g;
  }
  if (evl && evl->R8 > evl->R) {
    return cudaMemsetAsync(out + evl->R * evl->Kp, 0, sizeof(double) * (evl->R8 - evl->R) * evl->Kp, stream);
  }
  return cudaSuccess;
}

}  // namespace cb
