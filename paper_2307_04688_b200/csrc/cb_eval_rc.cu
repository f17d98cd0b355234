// K2 row-contraction evaluator (q == 1, K <= 48): see the kernel comment below; launched by
// eval_points() in cb_eval.cu.  Separate translation unit so its instantiations compile in
// parallel with the k-contraction kernels.
#include <cuda.h>
#include "cb_common.cuh"
#include "cb_eval_dev.cuh"
#include "cb_kernels.h"

namespace cb {
namespace evk {
namespace {

// ------------------------------------------------------------------------------------------
// Row-contraction form for small K (q == 1, K <= 48), e.g. BASELINE config 2 (33^3):
//   U'[k][p] = sum_r A[r][k] W[r][p]   (DMMA: M = k (padded to 8*MTK), K-dim = rows, N = points)
//   v[p]     = sum_k U'[k][p] T_k(x_{J-1,p})   (once per tile)
// W[r][p] = prod_{leading d} T_{l_d(r)}(x_{d,p}) is formed on the fly as the B operand, so the
// per-row weighting rides inside the tensor-core reduction and the accumulators are consumed
// only once per tile (no per-stage epilogue / DMMA drain).
// ------------------------------------------------------------------------------------------
template <int NL, int MTK, int KT>
__global__ void __launch_bounds__(kRcThreads, 1)
    eval_rc_kernel(const __grid_constant__ EvalParams p, const __grid_constant__ DmmaSmem sm,
                   const __grid_constant__ CUtensorMap amap) {
  constexpr int NCW = kRcConsumers, NT = kRcNT, kRows = kRcRows, RG = kRcRG, KS = kRows / RG / 4;  // KS k-steps per warp per stage
  constexpr int NGR = 8 / NT;   // point groups (8*NT points each) per row group
  constexpr int J = NL + 1;
  constexpr int KTMAX = (KT < 0) ? 3 : KT;        // DFMA tail columns (compile-time when KT >= 0)
  const int ktail = (KT < 0) ? p.ktail : KT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* bar_empty = bar_full + kMaxStages;
  uint64_t* tab_full = bar_empty + kMaxStages;
  uint64_t* tab_empty = tab_full + 2;
  uint64_t* red_full = tab_empty + 2;   // [2] per-warp tile partials written (NCW arrivals)
  uint64_t* red_empty = red_full + 2;   // [2] partials consumed by the finisher
  double* Src = reinterpret_cast<double*>(smem_raw + sm.src);        // [ntab][P]
  double* Red = reinterpret_cast<double*>(smem_raw + sm.red);        // [2][4][P]
  double* Ts = reinterpret_cast<double*>(smem_raw + sm.ts);          // [ntab][ts_stride]
  double* As = reinterpret_cast<double*>(smem_raw + sm.as);          // [stages][64][kc]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const long long ntiles = (p.M + kP - 1) / kP;
  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], NCW);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tab_full[s], 1);
      mbar_init(&tab_empty[s], NCW + 1);  // consumers + finisher (reads Src)
      mbar_init(&red_full[s], NCW);
      mbar_init(&red_empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {  // producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
      const unsigned stage_bytes = static_cast<unsigned>(kRows * p.kc * 8);
      int slot = 0;
      unsigned phase = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int blk = 0; blk < p.nstage_blocks; ++blk) {
          mbar_wait(&bar_empty[slot], phase ^ 1);
          mbar_arrive_expect_tx(&bar_full[slot], stage_bytes);
          tma_load_2d(As + static_cast<size_t>(slot) * kRows * p.kc, &amap, 0, blk * kRows, &bar_full[slot]);
          if (++slot == p.stages) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }
  if (warp == NCW + 1) {  // builder: per-tile point tables
    int it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ts = it % sm.ntab;
      mbar_wait(&tab_empty[ts], ((it / sm.ntab) & 1) ^ 1);
      double* Tsb = Ts + ts * sm.ts_stride;
      for (int pp = lane; pp < kP; pp += 32) {
        const long long g = tile * kP + pp;
        double t[kMaxDims];
        double src = 0.0;
        if (g < p.M) {
          point_coords(p, g, t, &src);
        } else {
#pragma unroll
          for (int d = 0; d < kMaxDims; ++d) t[d] = 0.0;
        }
        Src[ts * kP + pp] = src;
#pragma unroll
        for (int d = 0; d < J; ++d) {
          double* col = Tsb + p.toff[d] + pp;
          cheb_row(t[d], p.n[d], col, kTP);
          for (int l = p.n[d]; l < p.trows[d]; ++l) col[l * kTP] = 0.0;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tab_full[ts]);
    }
    return;
  }

  if (warp == NCW + 2) {  // finisher: sums the warps' tile partials and writes the results
    int it = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ts = it % sm.ntab;
      const int rb = it & 1;
      mbar_wait(&red_full[rb], (it >> 1) & 1);
      const double* Rb = Red + rb * 2 * RG * kP;
      for (int pp = lane; pp < kP; pp += 32) {
        const long long g = tile * kP + pp;
        if (g < p.M) {
          double v = Rb[pp];
#pragma unroll
          for (int q = 1; q < RG; ++q) v += Rb[q * kP + pp];
          if (KTMAX > 0 && ktail) {
            double t = Rb[RG * kP + pp];
#pragma unroll
            for (int q = 1; q < RG; ++q) t += Rb[(RG + q) * kP + pp];
            v += t;
          }
          emit(p, g, v - Src[ts * kP + pp]);
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&red_empty[rb]);
        mbar_arrive(&tab_empty[ts]);
      }
    }
    return;
  }

  // consumers: warp = (row group rg: kRows/4 rows of each stage) x (point group ng: 16 points)
  const int rg = warp / NGR, ng = warp % NGR;
  const int gq = lane >> 2, tq = lane & 3;
  const int pcol = ng * 8 * NT + gq;  // B-fragment column (point) of this lane (+ nt*8)
  int slot = 0, it = 0;
  unsigned phase = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int ts = it % sm.ntab;
    mbar_wait(&tab_full[ts], (it / sm.ntab) & 1);
    const double* Tsb = Ts + ts * sm.ts_stride;
    double acc[MTK][NT][2];
#pragma unroll
    for (int m = 0; m < MTK; ++m)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[m][nt][0] = acc[m][nt][1] = 0.0;
    double tacc[KTMAX > 0 ? KTMAX : 1][NT];
#pragma unroll
    for (int t = 0; t < KTMAX; ++t)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) tacc[t][nt] = 0.0;

    for (int blk = 0; blk < p.nstage_blocks; ++blk) {
      mbar_wait(&bar_full[slot], phase);
      const double* Ast = As + static_cast<size_t>(slot) * kRows * p.kc + (rg * (kRows / RG) + tq) * p.kc + gq;
      const int rbase = blk * kRows + rg * (kRows / RG) + tq;   // this lane's row at k-step ks: rbase + 4*ks
      // one k-step: 4 rows of the stage; the row digits come straight from FastDiv (no carries),
      // so the fully-valid case below is straight-line code the scheduler can software-pipeline
      // B fragments W[r][p] of k-step ks for this lane's row r and points pcol + 8*nt (zero past R)
      auto wfrag = [&](int ks, double* w) {
        const int r = rbase + 4 * ks;
        int dig[NL];
        {
          uint32_t rem = static_cast<uint32_t>(r);
#pragma unroll
          for (int d = NL - 1; d >= 1; --d) {
            uint32_t qd, l;
            p.fdn[d].divmod(rem, qd, l);
            dig[d] = static_cast<int>(l);
            rem = qd;
          }
          dig[0] = min(static_cast<int>(rem), p.n[0] - 1);  // r >= R: clamp the lookup (A is zero on those rows)
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          double v = Tsb[p.toff[0] + dig[0] * kTP + pcol + nt * 8];
#pragma unroll
          for (int d = 1; d < NL; ++d) v *= Tsb[p.toff[d] + dig[d] * kTP + pcol + nt * 8];
          w[nt] = v;   // rows >= R: A is zero there (layout padding / TMA zero fill), the digits are clamped
        }
      };
      // one k-step: 4 rows of the stage, DMMAs on the DMMA m-tiles + DFMA tail columns
      auto kstep = [&](int ks, const double* w) {
        double a[MTK];
#pragma unroll
        for (int m = 0; m < MTK; ++m) a[m] = Ast[ks * 4 * p.kc + m * 8];
        // issue order: no two consecutive DMMAs share an A or B register (a shared operand in
        // back-to-back DMMAs costs the warp an issue bubble)
#pragma unroll
        for (int h = 0; h < NT; ++h)
#pragma unroll
          for (int m = 0; m < MTK; ++m) {
            const int nt = (m + h) % NT;
            dmma884(acc[m][nt][0], acc[m][nt][1], a[m], w[nt]);
          }
        // tail columns k = 8*MTK + t (t < ktail) on DFMA: lane-partial sums over its rows
#pragma unroll
        for (int t = 0; t < KTMAX; ++t) {
          if (t < ktail) {
            const double at = Ast[ks * 4 * p.kc + MTK * 8 + t - gq];  // A[r][8*MTK + t] (broadcast in tq)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) tacc[t][nt] = fma(at, w[nt], tacc[t][nt]);
          }
        }
      };
      const int kvalid = min(KS, (static_cast<int>(p.R8) - (blk * kRows + rg * (kRows / RG)) + 3) / 4);  // k-steps with rows < R8
      if (kvalid == KS) {
        // software-pipelined: the next k-step's W products are formed (and pinned in program
        // order by the volatile asm) before this k-step's DMMAs, hiding the DMUL latency
        double wc[NT], wn[NT];
        wfrag(0, wc);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          if (ks + 1 < KS) {
            wfrag(ks + 1, wn);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) asm volatile("" : "+d"(wn[nt]));
          }
          kstep(ks, wc);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) wc[nt] = wn[nt];
        }
      } else {
#pragma unroll 1
        for (int ks = 0; ks < kvalid; ++ks) {
          double w[NT];
          wfrag(ks, w);
          kstep(ks, w);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_empty[slot]);
      if (++slot == p.stages) {
        slot = 0;
        phase ^= 1;
      }
    }
    // tile end: contract k with T_k(x_{J-1}):  lane holds U'[k = m*8 + gq][p = ng*8*NT + nt*8 + 2tq + i]
    double vp[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int pp = ng * 8 * NT + nt * 8 + 2 * tq + i;
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < MTK; ++m) v = fma(acc[m][nt][i], Tsb[p.toff[J - 1] + (m * 8 + gq) * kTP + pp], v);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        vp[nt][i] = v;
      }
    // tail columns: reduce the row-partials over the 4 tq lanes -> U'[8*MTK + t][p = pcol + 8*nt]
    double tv[NT] = {};
#pragma unroll
    for (int t = 0; t < KTMAX; ++t) {
      if (t < ktail) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          double u = tacc[t][nt];
          u += __shfl_xor_sync(0xffffffffu, u, 1);
          u += __shfl_xor_sync(0xffffffffu, u, 2);
          tv[nt] = fma(u, Tsb[p.toff[J - 1] + (MTK * 8 + t) * kTP + pcol + nt * 8], tv[nt]);
        }
      }
    }
    // hand the tile's partials to the finisher warp (no consumer-wide barrier at the tile end)
    const int rb = it & 1;
    if (it >= 2) mbar_wait(&red_empty[rb], ((it >> 1) & 1) ^ 1);
    double* Rb = Red + rb * 2 * RG * kP;  // [2][rg: RG main + RG tail][P]
    if (gq == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) Rb[rg * kP + ng * 8 * NT + nt * 8 + 2 * tq + i] = vp[nt][i];
    }
    if (tq == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) Rb[(RG + rg) * kP + pcol + nt * 8] = tv[nt];
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&red_full[rb]);
      mbar_arrive(&tab_empty[ts]);
    }
  }
}

}  // namespace

bool launch_eval_rc(int NL, int MTK, int KT, unsigned grid, size_t bytes, cudaStream_t stream, const EvalParams& p,
                    const DmmaSmem& sm, const CUtensorMap& amap) {
  // exact tail instantiations for J <= 4 (the common shapes); runtime tail above
  const int kt = (NL <= 3) ? KT : -1;
  switch ((NL * 8 + MTK) * 8 + (kt + 1)) {
#define CB_RC(v, m, t)                                                                                    \
  case (v * 8 + m) * 8 + (t + 1):                                                                         \
    ensure_smem_attr(reinterpret_cast<const void*>(eval_rc_kernel<v, m, t>), 227 * 1024);                 \
    eval_rc_kernel<v, m, t><<<grid, kRcThreads, bytes, stream>>>(p, sm, amap);                    \
    return true;
#define CB_RCT(v, m) CB_RC(v, m, 0) CB_RC(v, m, 1) CB_RC(v, m, 2) CB_RC(v, m, 3)
#define CB_RCM(v, X) X(v, 1) X(v, 2) X(v, 3) X(v, 4) X(v, 5) X(v, 6)
#define CB_RCR(v, m) CB_RC(v, m, -1)
    CB_RCM(1, CB_RCT) CB_RCM(2, CB_RCT) CB_RCM(3, CB_RCT)
    CB_RCM(4, CB_RCR) CB_RCM(5, CB_RCR) CB_RCM(6, CB_RCR) CB_RCM(7, CB_RCR)
#undef CB_RCR
#undef CB_RCM
#undef CB_RCT
#undef CB_RC
    default:
      return false;
  }
}

}  // namespace evk
}  // namespace cb
