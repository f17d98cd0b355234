// DMMA throughput with shared-memory operand traffic: each warp streams A/B fragments from smem
// (LDS.64) at a given loads-per-DMMA ratio.  Calibrates how much LDS traffic the DMMA pipe hides.
#include <cstdio>
#include <cuda_runtime.h>

template <int MT, int NT, bool LOADS>
__global__ void __launch_bounds__(512, 1) k_dmma(double* out, int iters) {
  __shared__ double sm[64 * 68 + 256];
  for (int i = threadIdx.x; i < 64 * 68 + 256; i += blockDim.x) sm[i] = 1.0 + i * 1e-7;
  __syncthreads();
  const int lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  double acc[MT][NT][2];
  for (int m = 0; m < MT; ++m)
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  const double* ap = sm + gq * 36 + tq;
  const double* bp = sm + 2304 + tq * 68 + gq;
  double a[MT], b[NT];
  for (int m = 0; m < MT; ++m) a[m] = ap[m * 288];
  for (int n = 0; n < NT; ++n) b[n] = bp[n * 8];
  for (int it = 0; it < iters; ++it) {
    const int ks = it & 7;
    double na[MT], nb[NT];
    if (LOADS) {
#pragma unroll
      for (int m = 0; m < MT; ++m) na[m] = ap[m * 288 + ks * 4];
#pragma unroll
      for (int n = 0; n < NT; ++n) nb[n] = bp[ks * 4 * 68 + n * 8];
    }
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[m][n][0]), "+d"(acc[m][n][1]) : "d"(a[m]), "d"(b[n]));
    if (LOADS) {
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = na[m];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = nb[n];
    }
  }
  double s = 0;
  for (int m = 0; m < MT; ++m)
    for (int n = 0; n < NT; ++n) s += acc[m][n][0] + acc[m][n][1];
  if (s == 1.2345) out[0] = s;
}

template <int MT, int NT, bool LOADS>
void run(const char* name, int warps, double* out) {
  const int iters = 4096;
  int sms = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dmma<MT, NT, LOADS><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e0);
  k_dmma<MT, NT, LOADS><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * MT * NT * double(iters) * warps * sms;
  printf("\"%s_w%d\": %.2f, ", name, warps, flops / (ms * 1e-3) / 1e12);
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  printf("{");
  run<2, 2, false>("noload_m2n2", 16, out);
  run<2, 2, true>("lds_m2n2", 16, out);
  run<4, 2, true>("lds_m4n2", 16, out);
  run<2, 4, true>("lds_m2n4", 8, out);
  run<2, 4, true>("lds_m2n4", 16, out);
  run<4, 4, true>("lds_m4n4", 8, out);
  run<4, 4, true>("lds_m4n4", 16, out);
  run<1, 4, true>("lds_m1n4", 16, out);
  run<2, 2, true>("lds_m2n2", 8, out);
  printf("\"ok\": 1}\n");
  return 0;
}
