// Stage-loop microbenchmark mirroring the K2 consumer: per "stage" each warp loads A/B fragments
// from smem (LDS), issues MT x NT x KS DMMAs, then runs an epilogue that consumes the accumulators.
// Variants isolate the cost of consuming DMMA results.
#include <cstdio>
#include <cuda_runtime.h>

// EPI: 0 none (results folded only at the end), 1 epilogue after each stage,
//      2 deferred: epilogue of stage s-1 after issuing the first k-step of stage s (two sets)
template <int MT, int NT, int KS, int EPI>
__global__ void __launch_bounds__(512, 1) k_stage(double* out, int stages) {
  __shared__ double sm[64 * 40 + 40 * 72 + 64];
  for (int i = threadIdx.x; i < 64 * 40 + 40 * 72 + 64; i += blockDim.x) sm[i] = 1.0 + (i % 97) * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const double* A = sm + (warp & 1) * 8 * 40 + gq * 40 + tq;
  const double* B = sm + 64 * 40 + tq * 72 + gq;
  const double* W = sm + 64 * 40 + 2;
  double v[NT][2];
  for (int n = 0; n < NT; ++n) v[n][0] = v[n][1] = 0.0;
  double acc[MT][NT][2], accp[MT][NT][2];
  for (int m = 0; m < MT; ++m)
    for (int n = 0; n < NT; ++n) accp[m][n][0] = accp[m][n][1] = 0.0;
  for (int s = 0; s < stages; ++s) {
    const int off = (s & 7);
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double a[MT], b[NT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = A[(m & 1) * 16 * 40 + ks * 4 + off];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = B[ks * 4 * 72 + n * 8 + off];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[m][n][0]), "+d"(acc[m][n][1]) : "d"(a[m]), "d"(b[n]));
      if (EPI == 2 && ks == 0) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int i = 0; i < 2; ++i) v[n][i] = fma(W[(m * 8 + gq + off) * 2 + n], accp[m][n][i], v[n][i]);
      }
    }
    if (EPI == 1) {
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int i = 0; i < 2; ++i) v[n][i] = fma(W[(m * 8 + gq + off) * 2 + n], acc[m][n][i], v[n][i]);
    }
    if (EPI == 2 || EPI == 0) {
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          if (EPI == 2) {
            accp[m][n][0] = acc[m][n][0];
            accp[m][n][1] = acc[m][n][1];
          } else if (s == stages - 1) {
            v[n][0] += acc[m][n][0];
            v[n][1] += acc[m][n][1];
          }
        }
    }
  }
  double t = 0;
  for (int n = 0; n < NT; ++n) t += v[n][0] + v[n][1];
  if (t == 1.2345) out[0] = t;
}

template <int MT, int NT, int KS, int EPI>
void run(const char* name, double* out) {
  const int stages = 2048, sms = 148, warps = 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_stage<MT, NT, KS, EPI><<<sms, warps * 32>>>(out, stages);
  cudaEventRecord(e0);
  k_stage<MT, NT, KS, EPI><<<sms, warps * 32>>>(out, stages);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double tf = 2.0 * 256 * MT * NT * KS * double(stages) * warps * sms / (ms * 1e-3) / 1e12;
  printf("\"%s\": %.2f, ", name, tf);
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  printf("{");
  run<2, 2, 9, 0>("m2n2k9_noepi", out);
  run<2, 2, 9, 1>("m2n2k9_epi", out);
  run<2, 2, 9, 2>("m2n2k9_deferred", out);
  run<2, 2, 18, 1>("m2n2k18_epi", out);
  run<4, 2, 9, 1>("m4n2k9_epi", out);
  run<2, 4, 9, 1>("m2n4k9_epi", out);
  run<2, 2, 8, 1>("m2n2k8_epi", out);
  printf("\"ok\": 1}\n");
  return 0;
}
