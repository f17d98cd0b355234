// FP64 peak microbenchmark for the roofline denominator (DFMA vs DMMA) on sm_100a.
// Register-resident, no memory traffic; results printed as one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m8n8k4 f64: A 8x4 (1 reg/thread), B 4x8 (1 reg), C/D 8x8 (2 regs)
template <int CHAINS>
__global__ void dmma884_kernel(double* out, int iters, double a0, double b0) {
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k16 f64: A 16x16 (8 regs), B 16x8 (4 regs), C 16x8 (4 regs)
template <int CHAINS>
__global__ void dmma16816_kernel(double* out, int iters, double a0, double b0) {
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0; }
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = b0 - (threadIdx.x + i) * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
static float time_kernel(K kern, dim3 grid, dim3 block, double* out, int iters, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<grid, block>>>(out, iters, 1.0000001, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int iters = 1 << 14;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", p.name, sms, clk_khz);
  // DFMA: 8 independent chains, grid = sms*8 blocks of 256 threads (16 warps/SM... 64 warps/SM max)
  for (int bps : {4, 8}) {
    dim3 g(sms * bps), b(256);
    float ms = time_kernel(dfma_kernel<8>, g, b, out, iters, 5);
    double flops = 2.0 * 8 * iters * (double)g.x * b.x;
    printf(", \"dfma8_bps%d_tflops\": %.3f", bps, flops / (ms * 1e-3) / 1e12);
  }
  {
    dim3 g(sms * 8), b(256);
    float ms = time_kernel(dfma_kernel<4>, g, b, out, iters, 5);
    double flops = 2.0 * 4 * iters * (double)g.x * b.x;
    printf(", \"dfma4_bps8_tflops\": %.3f", flops / (ms * 1e-3) / 1e12);
  }
  for (int bps : {2, 4, 8}) {
    dim3 g(sms * bps), b(256);
    float ms = time_kernel(dmma884_kernel<4>, g, b, out, iters / 4, 5);
    double flops = 2.0 * 8 * 8 * 4 * 4 * (iters / 4) * (double)g.x * (b.x / 32);
    printf(", \"dmma884_c4_bps%d_tflops\": %.3f", bps, flops / (ms * 1e-3) / 1e12);
  }
  for (int bps : {2, 4, 8}) {
    dim3 g(sms * bps), b(256);
    float ms = time_kernel(dmma16816_kernel<2>, g, b, out, iters / 16, 5);
    double flops = 2.0 * 16 * 8 * 16 * 2 * (iters / 16) * (double)g.x * (b.x / 32);
    printf(", \"dmma16816_c2_bps%d_tflops\": %.3f", bps, flops / (ms * 1e-3) / 1e12);
  }
  // sustained DFMA: ~3 s loop for the power-capped figure
  {
    dim3 g(sms * 8), b(256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = 0; float total = 0;
    cudaEventRecord(e0);
    while (total < 3000.f) {
      for (int r = 0; r < 20; ++r) dfma_kernel<8><<<g, b>>>(out, iters, 1.0000001, 1e-7);
      reps += 20;
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&total, e0, e1);
    }
    double flops = 2.0 * 8 * iters * (double)g.x * b.x * reps;
    printf(", \"dfma8_sustained_tflops\": %.3f, \"sustained_ms\": %.0f", flops / (total * 1e-3) / 1e12, total);
  }
  {
    dim3 g(sms * 4), b(256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = 0; float total = 0;
    cudaEventRecord(e0);
    while (total < 3000.f) {
      for (int r = 0; r < 20; ++r) dmma884_kernel<4><<<g, b>>>(out, iters / 4, 1.0000001, 1e-7);
      reps += 20;
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&total, e0, e1);
    }
    double flops = 2.0 * 8 * 8 * 4 * 4 * (iters / 4) * (double)g.x * (b.x / 32) * reps;
    printf(", \"dmma884_sustained_tflops\": %.3f", flops / (total * 1e-3) / 1e12);
  }
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
