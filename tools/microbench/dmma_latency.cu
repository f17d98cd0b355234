// DMMA.8x8x4 latency / per-warp issue microbenchmark (one CTA, W warps per SM-subpartition).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void chain_kernel(double* out, long long* cycles, int iters) {
  double c[CHAINS][2];
  for (int k = 0; k < CHAINS; ++k) c[k][0] = c[k][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

template <int CHAINS>
void run(int warps, double* out, long long* cyc) {
  const int iters = 4096;
  chain_kernel<CHAINS><<<1, 32 * warps>>>(out, cyc, iters);
  chain_kernel<CHAINS><<<1, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double per = double(h) / (iters * CHAINS);
  // per-SMSP DMMA rate: warps spread over 4 SMSPs
  double smsp_warps = warps < 4 ? 1.0 : warps / 4.0;
  printf("\"c%d_w%d\": {\"cyc_per_dmma_per_warp\": %.2f, \"cyc_per_dmma_per_smsp\": %.2f}, ", CHAINS, warps, per,
         per / smsp_warps);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64);
  cudaMalloc(&cyc, 64);
  printf("{");
  run<1>(1, out, cyc);
  run<2>(1, out, cyc);
  run<4>(1, out, cyc);
  run<8>(1, out, cyc);
  run<16>(1, out, cyc);
  run<1>(4, out, cyc);
  run<2>(4, out, cyc);
  run<4>(4, out, cyc);
  run<1>(8, out, cyc);
  run<2>(8, out, cyc);
  run<4>(8, out, cyc);
  run<4>(16, out, cyc);
  run<8>(16, out, cyc);
  run<2>(16, out, cyc);
  printf("\"ok\": 1}\n");
  return 0;
}
