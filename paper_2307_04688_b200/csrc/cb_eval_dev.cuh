// Shared device-side pieces of the K2 evaluators (cb_eval.cu, cb_eval_rc.cu): parameter block,
// mbarrier / TMA / DMMA wrappers, point coordinates, warp roles.
#pragma once
#include <cstdint>
#include <cuda.h>
#include "cb_common.cuh"

namespace cb {
namespace evk {

constexpr int kP = 64;                 // points per CTA
constexpr int kBP = kP + 4;            // smem pitch of the B table (bank-conflict free fragments)
constexpr int kTP = kP + 4;            // smem pitch of the per-dim T tables (8 rows per warp lookup)
#ifndef CB_MAX_STAGES
#define CB_MAX_STAGES 4
#endif
constexpr int kMaxStages = CB_MAX_STAGES;
constexpr int kMaxNodeTab = 64;        // nodes per dim carried in the kernel params (advection)
constexpr int kMaxPeers = 8;           // GPUs one evaluation can store its results into

struct EvalParams {
  const double* coef;   // eval layout [R8][Kp]
  const double* pts;    // (M, J) row-major reference coordinates (nullptr when advecting)
  double* out;
  Status* st;
  long long M;
  int J, q;
  int n[kMaxDims];
  FastDiv fdn[kMaxDims];
  long long R, R8;
  int K, Kp;
  int kc, kcs, nchunks, stages;
  int ktail;             // row-contraction kernel: trailing k columns done on DFMA (0..3)
  int nstage_blocks;     // ceil(R8 / rows per stage)
  int toff[kMaxDims];    // offsets of per-dim T tables in smem (doubles); -1 if not stored
  int tsm_total;
  int trows[kMaxDims];   // rows allocated per T table (>= n_d; zero padded)
  // advection (K4 loop)
  int advect;
  int dbg;               // experiment switches (bit0: no epilogue, bit1: no TMA wait, bit2: no TMA)
  long long node_begin;
  double A[kMaxDims * kMaxDims];
  double dt;
  double lo[kMaxDims], hi[kMaxDims];
  int source;
  double nodes[kMaxDims][kMaxNodeTab];
  const double* node_tab;   // modes above kMaxNodeTab nodes: device table [J][node_pitch] instead
  int node_pitch;
  // fused exchange (multi-GPU loop): results go to every rank's node-value buffer through
  // NVLink peer stores instead of `out` (peers[r] already offset to this launch's first node)
  int npeers;
  double* peers[kMaxPeers];
};

// Result store of every evaluator: `out`, or all peers' buffers (the all-gather fused into the
// evaluation: each rank writes its slab straight into every rank's copy of the node values).
__device__ __forceinline__ void emit(const EvalParams& p, long long g, double v) {
  if (p.npeers == 0) {
    p.out[g] = v;
    return;
  }
#pragma unroll 1
  for (int r = 0; r < p.npeers; ++r) p.peers[r][g] = v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Reference coordinate of point p (global index g) along dim d, plus the source term.
__device__ __forceinline__ void point_coords(const EvalParams& p, long long g, double* t, double* src) {
  if (!p.advect) {
    const double* row = p.pts + g * p.J;
#pragma unroll
    for (int d = 0; d < kMaxDims; ++d) t[d] = (d < p.J) ? clamp_ref(row[d], p.st) : 0.0;
    *src = 0.0;
    return;
  }
  // advected node: digits of the flat C-order node index, Euler step, clip to the box
  // (the BASELINE loop skeleton, S/solver.py:383-386 with fixed control).
  long long idx = p.node_begin + g;
  double x[kMaxDims];
#pragma unroll
  for (int d = kMaxDims - 1; d >= 0; --d) {
    x[d] = 0.0;
    if (d < p.J) {
      const long long qd = idx / p.n[d];
      const int kd = static_cast<int>(idx - qd * p.n[d]);
      idx = qd;
      x[d] = p.node_tab ? p.node_tab[d * p.node_pitch + kd] : p.nodes[d][kd];
    }
  }
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < kMaxDims; ++d)
    if (d < p.J) s = fma(x[d], x[d], s);
#pragma unroll
  for (int i = 0; i < kMaxDims; ++i) {
    t[i] = 0.0;
    if (i < p.J) {
      double gi = 0.0;
#pragma unroll
      for (int j = 0; j < kMaxDims; ++j)
        if (j < p.J) gi = fma(p.A[i * p.J + j], x[j], gi);
      double y = fma(p.dt, gi, x[i]);
      y = fmin(p.hi[i], fmax(p.lo[i], y));
      t[i] = fmin(1.0, fmax(-1.0, (2.0 * y - (p.lo[i] + p.hi[i])) / (p.hi[i] - p.lo[i])));
    }
  }
  *src = p.source ? p.dt * s : 0.0;
}

// Smem carve-up of the persistent kernel (byte offsets computed on the host, see eval_points()).
struct DmmaSmem {
  int src, red, ts, as;   // byte offsets
  int ts_stride;          // doubles per point-table buffer
  int ntab;               // point-table buffers (1 or 2)
  int tail;               // byte offset of the resident last m-tile (0: none), k-contraction kernel
  int tail_pitch;         // its row pitch in doubles
};

// Warp roles (NCW consumer warps + producer + builder):
//   consumers  : NCW/(8/NT) m-groups x (8/NT) n-groups; each warp owns MT x NT DMMA tiles
//                (8 rows x 8 points each) of every stage.  NCW = 16 -> NT = 2, one CTA per SM;
//                NCW = 8 -> NT = 4, two CTAs per SM (out of phase with each other).
//   producer   : one TMA 2-D box per stage into the stage ring.
//   builder    : per-tile point tables (coordinates, per-dim T_l rows) in 1-2 buffers.
// The B operand B[k][p] = prod_{trailing j} T_{l_j(k)}(x_{j,p}) is formed on the fly from the
// T tables while loading fragments (Q = 1: a plain table read; Q = 2: one DMUL per fragment),
// so no per-chunk B table has to be built or stored and the smem goes to wide k chunks.
// Shape codes W (consumer warps, m-tiles x n-tiles per warp):
//   16 -> 16 warps, 2 x 2, rows 64;   8 -> 8 warps, 2 x 4, two CTAs per SM;
//   12 -> 8 warps, 4 x 2, rows 64;   28 -> 12 warps, 4 x 2, rows 96;
//   one accumulator set (epilogue right after its row block) for the rest:
//   20 -> 8 warps, 4 x 4, rows 128;  24 -> 16 warps, 4 x 2, rows 128;
//   32 -> 8 warps, 8 x 2, rows 128;  36 -> 12 warps, 8 x 2, rows 192.
template <int W>
struct Roles {
  static constexpr int NCW = (W == 16 || W == 24) ? 16 : (W == 28 || W == 36) ? 12 : 8;   // consumer warps
  static constexpr int NT = (W == 8 || W == 20) ? 4 : 2;
  static constexpr int NGROUPS = 8 / NT;           // n-groups over the 64 points
  static constexpr int MGROUPS = NCW / NGROUPS;    // m-groups over the stage rows
  static constexpr int MT = (W == 16 || W == 8) ? 2 : (W == 32 || W == 36) ? 8 : 4;
  static constexpr int ROWS = MGROUPS * MT * 8;    // coefficient rows per stage
  static constexpr bool PINGPONG = (W == 16 || W == 8 || W == 12 || W == 28);
  static constexpr int PRODUCER = NCW;
  static constexpr int BUILDER = NCW + 1;
  static constexpr int THREADS = (NCW + 2) * 32;
  static constexpr int MIN_BLOCKS = (W == 8) ? 2 : 1;
};
inline int roles_rows(int w) {
  switch (w) {
    case 20: case 24: case 32: return 128;
    case 28: return 96;
    case 36: return 192;
    default: return 64;
  }
}

__device__ __forceinline__ void consumer_sync_n(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}


// Row-contraction evaluator shape: 16 consumer warps + producer + builder + finisher, stages of
// kRcRows coefficient rows.
#ifndef CB_RC_NT
#define CB_RC_NT 4
#endif
constexpr int kRcNT = CB_RC_NT;                       // n-tiles (8 points) per consumer warp
#ifndef CB_RC_RG
#define CB_RC_RG 4
#endif
constexpr int kRcRG = CB_RC_RG;                       // row groups (each kRcRows / kRcRG rows of a stage)
constexpr int kRcConsumers = kRcRG * (8 / kRcNT);     // row groups x (64 / (8 NT)) point groups
constexpr int kRcThreads = (kRcConsumers + 3) * 32;
#ifndef CB_RC_ROWS
#define CB_RC_ROWS (32 * CB_RC_RG)
#endif
constexpr int kRcRows = CB_RC_ROWS;

// Row-contraction evaluator launch (cb_eval_rc.cu): NL leading modes, MTK DMMA m-tiles over k,
// KT exact DFMA tail columns (-1: runtime p.ktail).  Returns false if not instantiated.
bool launch_eval_rc(int NL, int MTK, int KT, unsigned grid, size_t bytes, cudaStream_t stream, const EvalParams& p,
                    const DmmaSmem& sm, const CUtensorMap& amap);

}  // namespace evk
}  // namespace cb
