// C ABI (include/chebnash_b200.h): argument validation, layout planning, stream plumbing and
// the device-resident time loop.  All numerics run in the kernels of cb_build.cu, cb_eval.cu and
// cb_axis.cu.
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include "../../include/chebnash_b200.h"
#include "cb_common.cuh"
#include "cb_kernels.h"

namespace cb {

namespace {
thread_local std::string g_last_error;
std::mutex g_attr_mutex;
constexpr int kMaxDevices = 64;
struct AttrEntry {
  const void* func;
  int bytes;
};
AttrEntry g_attr[kMaxDevices][64];
int g_attr_n[kMaxDevices];
int g_sms[kMaxDevices];
}  // namespace

void ensure_smem_attr(const void* func, int bytes, bool max_carveout) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return;
  std::lock_guard<std::mutex> lock(g_attr_mutex);
  for (int i = 0; i < g_attr_n[dev]; ++i)
    if (g_attr[dev][i].func == func && g_attr[dev][i].bytes >= bytes) return;
  cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  // several smem-tiled CTAs per SM: ask for the whole unified L1/smem as shared memory (the
  // driver's default carveout left room for only 1-3 such CTAs)
  if (max_carveout)
    cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (g_attr_n[dev] < 64) g_attr[dev][g_attr_n[dev]++] = {func, bytes};
}

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return 148;
  if (!g_sms[dev]) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = sms > 0 ? sms : 148;
  }
  return g_sms[dev];
}

}  // namespace cb

using namespace cb;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static int cuda_fail(cudaError_t err, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorName(err) + ": " + cudaGetErrorString(err);
  return fail(CB_ECUDA, m);
}

#define CB_CUDA(call, where)                      \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

static int check_dims(int J, const int64_t* n, const char* fn) {
  if (J < 1 || J > kMaxDims) return fail(CB_EINVAL, std::string(fn) + ": number of modes must be in [1, 12]");
  if (!n) return fail(CB_EINVAL, std::string(fn) + ": null size array");
  long long total = 1;
  for (int d = 0; d < J; ++d) {
    if (n[d] < 1) return fail(CB_EINVAL, std::string(fn) + ": mode sizes must be >= 1");
    if (n[d] > kMaxModeSize)
      return fail(CB_EINVAL, std::string(fn) + ": mode size above 4096 (degree 4095) is not supported");
    total *= n[d];
    if (total > (1LL << 31)) return fail(CB_EINVAL, std::string(fn) + ": tensor larger than 2^31 elements");
  }
  return CB_OK;
}

static EvalLayout layout_of(int J, const int64_t* n) {
  long long nn[kMaxDims];
  for (int d = 0; d < J; ++d) nn[d] = n[d];
  return make_eval_layout(J, nn);
}

extern "C" {

int cb_abi_version(void) { return CB_ABI_VERSION; }

const char* cb_last_error(void) { return g_last_error.c_str(); }

int64_t cb_kernel_launches(void) { return launch_count(); }

const char* cb_last_eval_plan(void) { return last_eval_plan(); }

int cb_runtime_info(int* device_count, int* sm_count, int* cc_major, int* cc_minor) {
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess) {
    cudaGetLastError();
    cnt = 0;
  }
  if (device_count) *device_count = cnt;
  if (sm_count) *sm_count = 0;
  if (cc_major) *cc_major = 0;
  if (cc_minor) *cc_minor = 0;
  if (cnt > 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (sm_count) cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  }
  return CB_OK;
}

int cb_eval_layout(int J, const int64_t* n, int64_t* out6) {
  int rc = check_dims(J, n, "cb_eval_layout");
  if (rc) return rc;
  EvalLayout L = layout_of(J, n);
  out6[0] = L.q;
  out6[1] = L.R;
  out6[2] = L.R8;
  out6[3] = L.K;
  out6[4] = L.Kp;
  out6[5] = L.elems();
  return CB_OK;
}

int cb_pack_eval(int J, const int64_t* n, const double* d_dense, double* d_eval, void* stream) {
  int rc = check_dims(J, n, "cb_pack_eval");
  if (rc) return rc;
  EvalLayout L = layout_of(J, n);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (L.Kp != L.K || L.R8 != L.R) CB_CUDA(cudaMemsetAsync(d_eval, 0, sizeof(double) * L.elems(), s), "cb_pack_eval");
  CB_CUDA(cudaMemcpy2DAsync(d_eval, sizeof(double) * L.Kp, d_dense, sizeof(double) * L.K, sizeof(double) * L.K, L.R,
                            cudaMemcpyDeviceToDevice, s),
          "cb_pack_eval");
  return CB_OK;
}

int cb_unpack_eval(int J, const int64_t* n, const double* d_eval, double* d_dense, void* stream) {
  int rc = check_dims(J, n, "cb_unpack_eval");
  if (rc) return rc;
  EvalLayout L = layout_of(J, n);
  CB_CUDA(cudaMemcpy2DAsync(d_dense, sizeof(double) * L.K, d_eval, sizeof(double) * L.Kp, sizeof(double) * L.K, L.R,
                            cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)),
          "cb_unpack_eval");
  return CB_OK;
}

int cb_tensor_coeffs(int J, const int64_t* n, const double* d_samples, double* d_coef, void* d_status, void* stream) {
  int rc = check_dims(J, n, "cb_tensor_coeffs");
  if (rc) return rc;
  EvalLayout L = layout_of(J, n);
  long long shape[kMaxDims];
  for (int d = 0; d < J; ++d) shape[d] = n[d];
  CB_CUDA(transform_axes(J, shape, 0, J, d_samples, d_coef, static_cast<Status*>(d_status), 1, &L,
                         static_cast<cudaStream_t>(stream)),
          "cb_tensor_coeffs");
  return CB_OK;
}

int cb_transform_axes(int ndim, const int64_t* shape, int a0, int a1, const double* d_in, double* d_out,
                      void* d_status, int check_finite, void* stream) {
  if (ndim < 1 || ndim > 16 || a0 < 0 || a1 > ndim || a0 > a1)
    return fail(CB_EINVAL, "cb_transform_axes: bad axes");
  long long shp[16];
  long long total = 1;
  for (int d = 0; d < ndim; ++d) {
    if (shape[d] < 1) return fail(CB_EINVAL, "cb_transform_axes: empty axis");
    shp[d] = shape[d];
    total *= shape[d];
    if (total > (1LL << 31)) return fail(CB_EINVAL, "cb_transform_axes: array larger than 2^31 elements");
  }
  for (int d = a0; d < a1; ++d)
    if (shape[d] > kMaxModeSize)
      return fail(CB_EINVAL, "cb_transform_axes: axis longer than 4096 (degree 4095) not supported");
  CB_CUDA(transform_axes(ndim, shp, a0, a1, d_in, d_out, static_cast<Status*>(d_status), check_finite, nullptr,
                         static_cast<cudaStream_t>(stream)),
          "cb_transform_axes");
  return CB_OK;
}

int cb_eval_points(int J, const int64_t* n, const double* d_coef, int64_t M, const double* d_points, double* d_out,
                   void* d_status, int flags, void* stream) {
  int rc = check_dims(J, n, "cb_eval_points");
  if (rc) return rc;
  if (M < 0) return fail(CB_EINVAL, "cb_eval_points: negative point count");
  EvalLayout L = layout_of(J, n);
  CB_CUDA(eval_points(L, d_coef, M, d_points, nullptr, d_out, static_cast<Status*>(d_status), flags & 0xffff,
                      static_cast<cudaStream_t>(stream)),
          "cb_eval_points");
  return CB_OK;
}

int cb_build_eval_points(int J, const int64_t* n, const double* d_values, int64_t M, const double* d_points,
                         double* d_out, double* d_coef, void* d_status, void* stream) {
  int rc = check_dims(J, n, "cb_build_eval_points");
  if (rc) return rc;
  if (M < 0) return fail(CB_EINVAL, "cb_build_eval_points: negative point count");
  if (!d_values || !d_coef) return fail(CB_EINVAL, "cb_build_eval_points: null values / coefficient buffer");
  EvalLayout L = layout_of(J, n);
  long long shape[kMaxDims];
  for (int d = 0; d < J; ++d) shape[d] = n[d];
  CB_CUDA(build_eval_points(L, shape, d_values, M, d_points, d_out, d_coef, static_cast<Status*>(d_status),
                            static_cast<cudaStream_t>(stream)),
          "cb_build_eval_points");
  return CB_OK;
}

// Copy streams + events for the host-buffer pipeline (one set per device, created on first use).
namespace {
constexpr int kPipeMaxChunks = 16;
struct Pipe {
  cudaStream_t up = nullptr, down = nullptr;
  cudaEvent_t start = nullptr, done = nullptr;
  cudaEvent_t landed[kPipeMaxChunks] = {}, evaluated[kPipeMaxChunks] = {};
};
Pipe g_pipe[kMaxDevices];
std::mutex g_pipe_mutex;

cudaError_t pipe_for_device(Pipe** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  Pipe& p = g_pipe[dev];
  if (!p.up) {
    e = cudaStreamCreateWithFlags(&p.up, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p.down, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming);
    for (int i = 0; i < kPipeMaxChunks && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&p.landed[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.evaluated[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return e;
  }
  *out = &p;
  return cudaSuccess;
}
}  // namespace

int cb_eval_points_host(int J, const int64_t* n, const double* d_coef, int64_t M, const double* h_points,
                        double* h_out, double* d_points_ws, double* d_out_ws, void* d_status, int flags,
                        void* stream) {
  int rc = check_dims(J, n, "cb_eval_points_host");
  if (rc) return rc;
  if (M < 0) return fail(CB_EINVAL, "cb_eval_points_host: negative point count");
  if (M == 0) return CB_OK;
  EvalLayout L = layout_of(J, n);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::lock_guard<std::mutex> lock(g_pipe_mutex);
  Pipe* p = nullptr;
  CB_CUDA(pipe_for_device(&p), "cb_eval_points_host");
  // chunk plan: ramp up ~2^15, 2^16, 2^17 and down ~2^17, 2^16 (the first upload and the last
  // download are the only exposed transfers), equal middle chunks of about 2^18 points (several
  // evaluator waves each); at most 16 chunks.  Every chunk but the last is a whole number of
  // evaluator waves (64-point tiles x SMs), so no chunk ends in a partly idle wave.
  long long bounds[kPipeMaxChunks + 1];
  int nch = 0;
  {
    const long long W = 64LL * num_sms();
    auto waves = [&](long long v) { return (v + W - 1) / W * W; };
    long long sizes[kPipeMaxChunks];
    long long rem = M;
    int nh = 0, nt = 0;
    long long head[3], tail[2];
    for (long long s0 : {1LL << 15, 1LL << 16, 1LL << 17}) {
      if (rem <= 0) break;
      head[nh] = rem < waves(s0) ? rem : waves(s0);
      rem -= head[nh++];
    }
    for (long long s0 : {1LL << 16, 1LL << 17}) {
      if (rem <= (1LL << 18)) break;
      tail[nt++] = waves(s0);
      rem -= waves(s0);
    }
    long long nmid = rem > 0 ? (rem + (1LL << 18) - 1) >> 18 : 0;
    if (nmid > kPipeMaxChunks - nh - nt) nmid = kPipeMaxChunks - nh - nt;
    for (int i = 0; i < nh; ++i) sizes[nch++] = head[i];
    {
      const long long each = nmid > 0 ? waves((rem + nmid - 1) / nmid) : 0;
      long long left = rem;
      for (long long i = 0; i < nmid && left > 0; ++i) {
        const long long sz = (i + 1 == nmid || left < each) ? left : each;
        sizes[nch++] = sz;
        left -= sz;
      }
    }
    for (int i = nt - 1; i >= 0; --i) sizes[nch++] = tail[i];
    bounds[0] = 0;
    for (int c = 0; c < nch; ++c) bounds[c + 1] = bounds[c] + sizes[c];
  }
  CB_CUDA(cudaEventRecord(p->start, s), "cb_eval_points_host");  // inputs (coefficients) ready
  CB_CUDA(cudaStreamWaitEvent(p->up, p->start, 0), "cb_eval_points_host");
  CB_CUDA(cudaStreamWaitEvent(p->down, p->start, 0), "cb_eval_points_host");
  for (int c = 0; c < nch; ++c) {
    const long long b = bounds[c], m = bounds[c + 1] - bounds[c];
    CB_CUDA(cudaMemcpyAsync(d_points_ws + b * J, h_points + b * J, sizeof(double) * m * J, cudaMemcpyHostToDevice,
                            p->up),
            "cb_eval_points_host");
    CB_CUDA(cudaEventRecord(p->landed[c], p->up), "cb_eval_points_host");
    CB_CUDA(cudaStreamWaitEvent(s, p->landed[c], 0), "cb_eval_points_host");
    CB_CUDA(eval_points(L, d_coef, m, d_points_ws + b * J, nullptr, d_out_ws + b, static_cast<Status*>(d_status),
                        flags & 0xffff, s),
            "cb_eval_points_host");
    CB_CUDA(cudaEventRecord(p->evaluated[c], s), "cb_eval_points_host");
    CB_CUDA(cudaStreamWaitEvent(p->down, p->evaluated[c], 0), "cb_eval_points_host");
    CB_CUDA(cudaMemcpyAsync(h_out + b, d_out_ws + b, sizeof(double) * m, cudaMemcpyDeviceToHost, p->down),
            "cb_eval_points_host");
  }
  CB_CUDA(cudaEventRecord(p->done, p->down), "cb_eval_points_host");
  CB_CUDA(cudaStreamWaitEvent(s, p->done, 0), "cb_eval_points_host");  // completion is ordered on `stream`
  return CB_OK;
}

// Device node tables for advected evaluations whose modes have more nodes than the kernel
// parameters carry (kMaxNodeTab): make_basis nodes (S/cheb1d.py:97-103, descending, ends pinned;
// the same host arithmetic as the parameter tables) uploaded once per (device, shape, box) and
// cached for the life of the process (a few KB each; the graph cache and in-flight launches may
// hold the pointer, so entries are never freed).  Created synchronously: not inside a capture.
struct NodeTable {
  int device, J;
  long long n[kMaxDims];
  double lo[kMaxDims], hi[kMaxDims];
  double* d_tab;
  int pitch;
};
std::mutex g_node_mutex;
std::vector<NodeTable> g_node_tables;
constexpr size_t kMaxNodeTables = 1024;

static int advect_node_table(int J, const int64_t* n, AdvectSpec& adv, cudaStream_t stream, const char* who) {
  bool big = false;
  for (int d = 0; d < J; ++d) big = big || n[d] > 64;
  if (!big) return CB_OK;
  int dev = 0;
  CB_CUDA(cudaGetDevice(&dev), who);
  std::lock_guard<std::mutex> lock(g_node_mutex);
  for (const NodeTable& t : g_node_tables) {
    bool same = t.device == dev && t.J == J;
    for (int d = 0; same && d < J; ++d) same = t.n[d] == n[d] && t.lo[d] == adv.lo[d] && t.hi[d] == adv.hi[d];
    if (same) {
      adv.node_tab = t.d_tab;
      adv.node_pitch = t.pitch;
      return CB_OK;
    }
  }
  if (g_node_tables.size() >= kMaxNodeTables) return fail(CB_EINVAL, std::string(who) + ": too many distinct grids");
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CB_CUDA(cudaStreamIsCapturing(stream, &cs), who);
  if (cs != cudaStreamCaptureStatusNone)
    return fail(CB_EINVAL, std::string(who) + ": first evaluation of a grid with > 64 nodes per mode inside a capture");
  NodeTable t{};
  t.device = dev;
  t.J = J;
  int pitch = 0;
  for (int d = 0; d < J; ++d) {
    t.n[d] = n[d];
    t.lo[d] = adv.lo[d];
    t.hi[d] = adv.hi[d];
    pitch = std::max(pitch, static_cast<int>(n[d]));
  }
  t.pitch = pitch;
  std::vector<double> h(static_cast<size_t>(J) * pitch, 0.0);
  for (int d = 0; d < J; ++d) make_nodes(adv.lo[d], adv.hi[d], n[d], h.data() + static_cast<size_t>(d) * pitch);
  CB_CUDA(cudaMalloc(reinterpret_cast<void**>(&t.d_tab), sizeof(double) * h.size()), who);
  CB_CUDA(cudaMemcpy(t.d_tab, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice), who);
  g_node_tables.push_back(t);
  adv.node_tab = t.d_tab;
  adv.node_pitch = pitch;
  return CB_OK;
}

static int fill_advect(int J, const double* A, double dt, const double* lo, const double* hi, int source,
                       AdvectSpec& adv) {
  std::memset(&adv, 0, sizeof(adv));
  for (int i = 0; i < J * J; ++i) adv.A[i] = A[i];
  adv.dt = dt;
  for (int d = 0; d < J; ++d) {
    if (!(hi[d] > lo[d])) return fail(CB_EINVAL, "interval must satisfy a < b");
    adv.lo[d] = lo[d];
    adv.hi[d] = hi[d];
  }
  adv.source = source;
  return CB_OK;
}

static int check_node_range(int J, const int64_t* n, int64_t node_begin, int64_t count, const char* who) {
  long long N = 1;
  for (int d = 0; d < J; ++d) N *= n[d];
  if (node_begin < 0 || count < 0 || node_begin > N || count > N - node_begin)
    return fail(CB_EINVAL, std::string(who) + ": node range [node_begin, node_begin + count) outside the grid");
  return CB_OK;
}

int cb_eval_advected(int J, const int64_t* n, const double* d_coef, int64_t node_begin, int64_t count,
                     const double* A, double dt, const double* lo, const double* hi, int source, double* d_out,
                     void* stream) {
  int rc = check_dims(J, n, "cb_eval_advected");
  if (rc) return rc;
  rc = check_node_range(J, n, node_begin, count, "cb_eval_advected");
  if (rc) return rc;
  EvalLayout L = layout_of(J, n);
  AdvectSpec adv;
  rc = fill_advect(J, A, dt, lo, hi, source, adv);
  if (rc) return rc;
  rc = advect_node_table(J, n, adv, static_cast<cudaStream_t>(stream), "cb_eval_advected");
  if (rc) return rc;
  adv.node_begin = node_begin;
  CB_CUDA(eval_points(L, d_coef, count, nullptr, &adv, d_out, nullptr, 0, static_cast<cudaStream_t>(stream)),
          "cb_eval_advected");
  return CB_OK;
}

int cb_eval_advected_peers(int J, const int64_t* n, const double* d_coef, int64_t node_begin, int64_t count,
                           const double* A, double dt, const double* lo, const double* hi, int source,
                           double* const* d_full, int G, void* stream) {
  int rc = check_dims(J, n, "cb_eval_advected_peers");
  if (rc) return rc;
  if (G < 1 || G > 8 || !d_full) return fail(CB_EINVAL, "cb_eval_advected_peers: need 1..8 destination buffers");
  for (int r = 0; r < G; ++r)
    if (!d_full[r]) return fail(CB_EINVAL, "cb_eval_advected_peers: null destination buffer");
  rc = check_node_range(J, n, node_begin, count, "cb_eval_advected_peers");
  if (rc) return rc;
  EvalLayout L = layout_of(J, n);
  AdvectSpec adv;
  rc = fill_advect(J, A, dt, lo, hi, source, adv);
  if (rc) return rc;
  rc = advect_node_table(J, n, adv, static_cast<cudaStream_t>(stream), "cb_eval_advected_peers");
  if (rc) return rc;
  adv.node_begin = node_begin;
  adv.npeers = G;
  for (int r = 0; r < G; ++r) adv.peers[r] = d_full[r];
  CB_CUDA(eval_points(L, d_coef, count, nullptr, &adv, d_full[0] + node_begin, nullptr, 0,
                      static_cast<cudaStream_t>(stream)),
          "cb_eval_advected_peers");
  return CB_OK;
}

// cuMemGetAddressRange through the runtime's driver entry point (the library links no libcuda)
typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_getAddressRange address_range_fn() {
  static PFN_getAddressRange fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      ptr = nullptr;
    return reinterpret_cast<PFN_getAddressRange>(ptr);
  }();
  return fn;
}

int cb_ipc_export(const void* d_ptr, void* record72) {
  if (!d_ptr || !record72) return fail(CB_EINVAL, "cb_ipc_export: null pointer");
  PFN_getAddressRange range = address_range_fn();
  if (!range) return fail(CB_ECUDA, "cb_ipc_export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
    return fail(CB_ECUDA, "cb_ipc_export: pointer is not device memory");
  cudaIpcMemHandle_t h;
  CB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cb_ipc_export");
  const uint64_t off = static_cast<uint64_t>(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
  std::memcpy(record72, &h, 64);
  std::memcpy(static_cast<char*>(record72) + 64, &off, 8);
  return CB_OK;
}

int cb_ipc_import(const void* record72, void** d_ptr_out, void** d_base_out) {
  if (!record72 || !d_ptr_out || !d_base_out) return fail(CB_EINVAL, "cb_ipc_import: null pointer");
  cudaIpcMemHandle_t h;
  uint64_t off = 0;
  std::memcpy(&h, record72, 64);
  std::memcpy(&off, static_cast<const char*>(record72) + 64, 8);
  void* base = nullptr;
  CB_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cb_ipc_import");
  *d_base_out = base;
  *d_ptr_out = static_cast<char*>(base) + off;
  return CB_OK;
}

int cb_ipc_close(void* d_base) {
  if (!d_base) return CB_OK;
  CB_CUDA(cudaIpcCloseMemHandle(d_base), "cb_ipc_close");
  return CB_OK;
}

static cudaError_t loop_step(const EvalLayout& L, const long long* shape, const AdvectSpec& adv, const double* vin,
                             double* vout, double* coef, Status* st, long long N, cudaStream_t s) {
  cudaError_t e = transform_axes(L.J, shape, 0, L.J, vin, coef, st, 1, &L, s);
  if (e != cudaSuccess) return e;
  return eval_points(L, coef, N, nullptr, &adv, vout, nullptr, 0, s);
}

// Instantiated step-pair graphs of cb_advect_loop, cached per (device, shape, buffers, drift):
// the graph bakes in its buffer pointers and the advection parameters, so a repeated call with the
// same arguments replays the executable graph instead of re-capturing it.  Each entry owns the
// private capture/replay stream (the caller's stream may be the legacy default stream, which
// cannot be captured) and the event ordering it after / before the caller's stream.  Guarded by
// g_loop_mutex (the one per-device context cache the header allows).
struct LoopGraphKey {
  int device, J;
  long long shape[kMaxDims];
  const void* ptrs[4];
  AdvectSpec adv;
  bool operator==(const LoopGraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};
struct LoopGraph {
  LoopGraphKey key;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  cudaGraphExec_t exec = nullptr;
  long long kernels = 0;   // kernel launches captured in the step pair (counted per replay)
  unsigned long long last_use = 0;
};
constexpr int kLoopGraphCache = 8;
std::mutex g_loop_mutex;
LoopGraph g_loop_graphs[kLoopGraphCache];
unsigned long long g_loop_clock = 0;

static void loop_graph_release(LoopGraph& g) {
  if (g.cs) cudaStreamSynchronize(g.cs);  // an in-flight replay finishes before its exec goes
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.ev) cudaEventDestroy(g.ev);
  if (g.cs) cudaStreamDestroy(g.cs);
  g = LoopGraph{};
}

static cudaError_t loop_graph_build(LoopGraph& g, const EvalLayout& L, const long long* shape, const AdvectSpec& adv,
                                    double* v, double* tmp, double* coef, Status* st, long long N) {
  cudaError_t e = cudaStreamCreateWithFlags(&g.cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming);
  cudaGraph_t graph = nullptr;
  if (e == cudaSuccess) e = cudaStreamBeginCapture(g.cs, cudaStreamCaptureModeThreadLocal);
  const long long launches0 = launch_count();
  if (e == cudaSuccess) {
    cudaError_t e1 = loop_step(L, shape, adv, v, tmp, coef, st, N, g.cs);
    cudaError_t e2 = e1 == cudaSuccess ? loop_step(L, shape, adv, tmp, v, coef, st, N, g.cs) : e1;
    cudaError_t e3 = cudaStreamEndCapture(g.cs, &graph);
    e = e1 != cudaSuccess ? e1 : e2 != cudaSuccess ? e2 : e3;
  }
  // the captured launches did not run: they count once per replay instead (loop_graph_run)
  g.kernels = launch_count() - launches0;
  g_launches.fetch_sub(g.kernels, std::memory_order_relaxed);
  if (e == cudaSuccess) e = cudaGraphInstantiate(&g.exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    cudaGetLastError();
    loop_graph_release(g);
  }
  return e;
}

static cudaError_t loop_graph_run(const EvalLayout& L, const long long* shape, const AdvectSpec& adv, double* v,
                                  double* tmp, double* coef, Status* st, long long N, int pairs, cudaStream_t user) {
  LoopGraphKey key;
  std::memset(&key, 0, sizeof(key));
  cudaError_t e = cudaGetDevice(&key.device);
  if (e != cudaSuccess) return e;
  key.J = L.J;
  for (int d = 0; d < L.J; ++d) key.shape[d] = shape[d];
  key.ptrs[0] = v;
  key.ptrs[1] = tmp;
  key.ptrs[2] = coef;
  key.ptrs[3] = st;
  key.adv = adv;
  std::lock_guard<std::mutex> lock(g_loop_mutex);
  LoopGraph* g = nullptr;
  for (auto& c : g_loop_graphs)
    if (c.exec && c.key == key) g = &c;
  if (!g) {
    g = &g_loop_graphs[0];
    for (auto& c : g_loop_graphs)
      if (!c.exec || c.last_use < g->last_use) g = &c;
    if (g->exec) loop_graph_release(*g);
    g->key = key;
    e = loop_graph_build(*g, L, shape, adv, v, tmp, coef, st, N);
    if (e != cudaSuccess) return e;
  }
  g->last_use = ++g_loop_clock;
  e = cudaEventRecord(g->ev, user);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(g->cs, g->ev, 0);
  for (int s = 0; s < pairs && e == cudaSuccess; ++s) {
    e = cudaGraphLaunch(g->exec, g->cs);
    if (e == cudaSuccess) g_launches.fetch_add(g->kernels, std::memory_order_relaxed);
  }
  if (e == cudaSuccess) e = cudaEventRecord(g->ev, g->cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(user, g->ev, 0);
  return e;
}

int cb_advect_loop(int J, const int64_t* n, double* d_values, double* d_tmp, double* d_coef, int steps,
                   const double* A, double dt, const double* lo, const double* hi, void* d_status, int use_graph,
                   void* stream) {
  int rc = check_dims(J, n, "cb_advect_loop");
  if (rc) return rc;
  if (steps < 0) return fail(CB_EINVAL, "cb_advect_loop: negative step count");
  EvalLayout L = layout_of(J, n);
  AdvectSpec adv;
  rc = fill_advect(J, A, dt, lo, hi, 1, adv);
  if (rc) return rc;
  rc = advect_node_table(J, n, adv, static_cast<cudaStream_t>(stream), "cb_advect_loop");
  if (rc) return rc;
  adv.node_begin = 0;
  long long shape[kMaxDims];
  long long N = 1;
  for (int d = 0; d < J; ++d) {
    shape[d] = n[d];
    N *= n[d];
  }
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  Status* st = static_cast<Status*>(d_status);
  if (steps == 0) return CB_OK;
  const int pairs = steps / 2;
  if (!use_graph || pairs < 2) {
    for (int s = 0; s < pairs; ++s) {
      CB_CUDA(loop_step(L, shape, adv, d_values, d_tmp, d_coef, st, N, user), "cb_advect_loop");
      CB_CUDA(loop_step(L, shape, adv, d_tmp, d_values, d_coef, st, N, user), "cb_advect_loop");
    }
  } else {
    CB_CUDA(loop_graph_run(L, shape, adv, d_values, d_tmp, d_coef, st, N, pairs, user), "cb_advect_loop");
  }
  if (steps & 1) {
    CB_CUDA(loop_step(L, shape, adv, d_values, d_tmp, d_coef, st, N, user), "cb_advect_loop");
    CB_CUDA(cudaMemcpyAsync(d_values, d_tmp, sizeof(double) * N, cudaMemcpyDeviceToDevice, user),
            "cb_advect_loop: copy");
  }
  return CB_OK;
}

int cb_contract_axis(int64_t A, int n, int64_t R, int64_t Q, int k, const double* d_E, const double* d_in,
                     double* d_out, int64_t oA, int64_t oJ, int64_t oR, void* stream) {
  if (A < 0 || n < 1 || R < 0 || Q < 0 || k < 0) return fail(CB_EINVAL, "cb_contract_axis: bad sizes");
  CB_CUDA(contract_axis(A, n, R, Q, k, d_E, d_in, d_out, oA, oJ, oR, static_cast<cudaStream_t>(stream)),
          "cb_contract_axis");
  return CB_OK;
}

int cb_contract_diagonal(int64_t M, int n, int64_t R, const double* d_x, const double* d_W, int clamp,
                         const double* d_in, int64_t sM, int64_t sL, int64_t sR, double* d_out, int64_t oM, int64_t oR,
                         void* d_status, void* stream) {
  if (M < 0 || n < 1 || R < 0) return fail(CB_EINVAL, "cb_contract_diagonal: bad sizes");
  if (!d_x && !d_W) return fail(CB_EINVAL, "cb_contract_diagonal: need points or weights");
  CB_CUDA(contract_diagonal(M, n, R, d_x, d_W, clamp, d_in, sM, sL, sR, d_out, oM, oR, static_cast<Status*>(d_status),
                            static_cast<cudaStream_t>(stream)),
          "cb_contract_diagonal");
  return CB_OK;
}

int cb_derivative(int64_t rows, int L, const double* d_in, double* d_out, void* stream) {
  if (rows < 0 || L < 2) return fail(CB_EINVAL, "need degree >= 1 to differentiate");
  CB_CUDA(derivative(rows, L, d_in, d_out, static_cast<cudaStream_t>(stream)), "cb_derivative");
  return CB_OK;
}

int cb_basis_matrix(int64_t k, const double* d_x, int size, double* d_out, void* d_status, int clamp, void* stream) {
  if (k < 0 || size < 1) return fail(CB_EINVAL, "cb_basis_matrix: bad sizes");
  CB_CUDA(basis_matrix(k, d_x, size, d_out, static_cast<Status*>(d_status), clamp, static_cast<cudaStream_t>(stream)),
          "cb_basis_matrix");
  return CB_OK;
}

int cb_gather_index(int64_t rest, int64_t count, int64_t* d_flat, void* stream) {
  if (rest < 1 || count < 1) return fail(CB_EINVAL, "cb_gather_index: bad sizes");
  CB_CUDA(gather_index(rest, count, reinterpret_cast<long long*>(d_flat), static_cast<cudaStream_t>(stream)),
          "cb_gather_index");
  return CB_OK;
}

int cb_gather_take(int ndim_in, const int64_t* shape_in, const double* d_in, int64_t nsel, const int64_t* d_flat,
                   int ndim_out, const int64_t* shape_out, double* d_out, void* stream) {
  if (ndim_in < 1 || ndim_out < 1) return fail(CB_EINVAL, "cb_gather_take: bad ranks");
  long long si[16], so[16];
  if (ndim_in > 12 || ndim_out > 12) return fail(CB_EINVAL, "cb_gather_take: rank above 12");
  for (int d = 0; d < ndim_in; ++d) si[d] = shape_in[d];
  for (int d = 0; d < ndim_out; ++d) so[d] = shape_out[d];
  CB_CUDA(gather_take_f(ndim_in, si, d_in, nsel, reinterpret_cast<const long long*>(d_flat), ndim_out, so, d_out,
                        static_cast<cudaStream_t>(stream)),
          "cb_gather_take");
  return CB_OK;
}

int64_t cb_eval_grid_workspace(int J, const int64_t* n, const int64_t* k) {
  if (check_dims(J, n, "cb_eval_grid_workspace")) return -1;
  EvalLayout L = layout_of(J, n);
  long long kk[kMaxDims];
  for (int d = 0; d < J; ++d) kk[d] = k[d];
  return eval_grid_work_elems(L, kk);
}

int cb_eval_grid(int J, const int64_t* n, const double* d_coef, const int64_t* k, const double* const* d_E,
                 double* d_out, double* d_work, int64_t work_elems, void* stream) {
  int rc = check_dims(J, n, "cb_eval_grid");
  if (rc) return rc;
  long long kk[kMaxDims];
  for (int d = 0; d < J; ++d) {
    if (k[d] < 1) return fail(CB_EINVAL, "cb_eval_grid: empty target axis");
    kk[d] = k[d];
  }
  EvalLayout L = layout_of(J, n);
  if (work_elems < eval_grid_work_elems(L, kk)) return fail(CB_EINVAL, "cb_eval_grid: workspace too small");
  CB_CUDA(eval_grid(L, d_coef, kk, d_E, d_out, d_work, work_elems, static_cast<cudaStream_t>(stream)),
          "cb_eval_grid");
  return CB_OK;
}

int cb_eval_grid_targets(int J, const int64_t* n, const double* d_coef, const int64_t* k,
                         const double* const* d_targets, double* d_E_ws, void* d_status, double* d_out,
                         double* d_work, int64_t work_elems, void* stream) {
  int rc = check_dims(J, n, "cb_eval_grid_targets");
  if (rc) return rc;
  long long kk[kMaxDims], nn[kMaxDims];
  const double* E[kMaxDims];
  long long off = 0;
  for (int d = 0; d < J; ++d) {
    if (k[d] < 1) return fail(CB_EINVAL, "cb_eval_grid_targets: empty target axis");
    if (!d_targets || !d_targets[d]) return fail(CB_EINVAL, "cb_eval_grid_targets: null target vector");
    kk[d] = k[d];
    nn[d] = n[d];
    E[d] = d_E_ws + off;
    off += k[d] * n[d];
  }
  EvalLayout L = layout_of(J, n);
  if (work_elems < eval_grid_work_elems(L, kk)) return fail(CB_EINVAL, "cb_eval_grid_targets: workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CB_CUDA(basis_matrices(J, kk, d_targets, nn, d_E_ws, static_cast<Status*>(d_status), s), "cb_eval_grid_targets");
  CB_CUDA(eval_grid(L, d_coef, kk, E, d_out, d_work, work_elems, s), "cb_eval_grid_targets");
  return CB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// collocation solver (cb_solver.cu)
// ---------------------------------------------------------------------------------------------
static int check_game(const cb_game_t* g, const char* fn) {
  if (!g) return fail(CB_EINVAL, std::string(fn) + ": null game");
  if (g->J < 2 || g->J > CB_MAX_PLAYERS) return fail(CB_EINVAL, std::string(fn) + ": need 2..8 players");
  long long nodes = 1;
  for (int d = 0; d < g->J; ++d) {
    if (g->np[d] < 2 || g->np[d] > 64) return fail(CB_EINVAL, std::string(fn) + ": state degree must be 1..63");
    if (g->nu[d] < 2 || g->nu[d] > CB_MAX_CONTROL_NODES)
      return fail(CB_EINVAL, std::string(fn) + ": control degree must be 1..31");
    nodes *= g->np[d];
    if (nodes > (1LL << 31)) return fail(CB_EINVAL, std::string(fn) + ": state grid too large");
  }
  if (!(g->P_max > 0) || !(g->U_max > 0) || !(g->h > 0))
    return fail(CB_EINVAL, std::string(fn) + ": boxes and step must be positive");
  return CB_OK;
}

int64_t cb_solver_drift_elems(const cb_game_t* game) {
  if (check_game(game, "cb_solver_drift_elems")) return -1;
  return drift_elems(*game);
}

int cb_solver_drift_layout(const cb_game_t* game, const double* d_stacks, double* d_drift, void* stream) {
  int rc = check_game(game, "cb_solver_drift_layout");
  if (rc) return rc;
  CB_CUDA(drift_layout(*game, d_stacks, d_drift, static_cast<cudaStream_t>(stream)), "cb_solver_drift_layout");
  return CB_OK;
}

int cb_bellman_sweep(const cb_game_t* game, const double* d_nodes, const double* d_drift, const double* d_coef,
                     const double* d_v, const double* d_u, double* d_v_out, double* d_u_out, uint64_t* d_clamped,
                     void* d_status, void* stream) {
  int rc = check_game(game, "cb_bellman_sweep");
  if (rc) return rc;
  CB_CUDA(bellman_sweep(*game, d_nodes, d_drift, d_coef, d_v, d_u, d_v_out, d_u_out,
                        reinterpret_cast<unsigned long long*>(d_clamped), static_cast<Status*>(d_status),
                        static_cast<cudaStream_t>(stream)),
          "cb_bellman_sweep");
  return CB_OK;
}

int64_t cb_solve_work_bytes(const cb_game_t* game, int64_t max_iters) {
  if (check_game(game, "cb_solve_work_bytes") || max_iters < 1) return -1;
  return solve_work_bytes(*game, max_iters);
}

int cb_solve(const cb_game_t* game, const double* d_nodes, const double* d_drift, double* d_v, double* d_u,
             double* d_coef, void* d_work, int64_t max_iters, int64_t* iterations, int* converged, void* stream) {
  int rc = check_game(game, "cb_solve");
  if (rc) return rc;
  if (max_iters < 1) return fail(CB_EINVAL, "max_iters must be positive");
  long long its = 0;
  int conv = 0, nonfinite = 0;
  CB_CUDA(solve(*game, d_nodes, d_drift, d_v, d_u, d_coef, d_work, max_iters, &its, &conv, &nonfinite,
                static_cast<cudaStream_t>(stream)),
          "cb_solve");
  *iterations = its;
  *converged = conv;
  if (nonfinite) return fail(CB_ENONFINITE, "non-finite objective sample in sweep");
  return CB_OK;
}

int cb_maximise_rows(int64_t m, int L, const double* d_coef, const double* d_x0, double* d_x, double* d_f,
                     int always_scan, void* stream) {
  if (m < 0 || L < 1 || L > CB_MAX_CONTROL_NODES) return fail(CB_EINVAL, "cb_maximise_rows: need 1 <= L <= 32");
  CB_CUDA(maximise_rows(m, L, d_coef, d_x0, d_x, d_f, always_scan, static_cast<cudaStream_t>(stream)),
          "cb_maximise_rows");
  return CB_OK;
}

int cb_simulate(const cb_game_t* game, int64_t batch, const double* d_policies, const double* d_p0, int64_t n_steps,
                double* d_states, double* d_controls, void* stream) {
  int rc = check_game(game, "cb_simulate");
  if (rc) return rc;
  if (batch < 0 || n_steps < 0) return fail(CB_EINVAL, "cb_simulate: negative batch or step count");
  CB_CUDA(simulate(*game, batch, d_policies, d_p0, n_steps, d_states, d_controls, static_cast<cudaStream_t>(stream)),
          "cb_simulate");
  return CB_OK;
}

int cb_lq(const cb_game_t* game, double* d_state, double* d_work, int64_t max_iters, double tol, int mode,
          int64_t* iterations, void* stream) {
  int rc = check_game(game, "cb_lq");
  if (rc) return rc;
  long long its = 0;
  int status = 0;
  CB_CUDA(lq(*game, d_state, d_work, max_iters, tol, mode, &its, &status, static_cast<cudaStream_t>(stream)), "cb_lq");
  *iterations = its;
  if (status == 1) return fail(CB_ENONFINITE, "interior maximisation is not concave");
  if (status == 2) return fail(CB_ENOFIX, "quadratic fixed point not reached in " + std::to_string(max_iters) +
                                             " iterations");
  return CB_OK;
}
