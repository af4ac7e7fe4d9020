// Microbenchmark: FP64 FMA peak of the B200 SM (calibrates the FP64 roofline
// used for the tile kernel).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
void run(int blocks_per_sm, int threads) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096;
  k_dfma<CHAINS><<<sms * blocks_per_sm, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_dfma<CHAINS><<<sms * blocks_per_sm, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fmas = (double)sms * blocks_per_sm * threads * iters * CHAINS;
  printf("chains=%d warps/SM=%d: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.965 GHz)\n", CHAINS,
         blocks_per_sm * threads / 32, 2 * fmas / (ms * 1e-3) / 1e12,
         fmas / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(out);
}

int main() {
  run<8>(1, 256);
  run<8>(2, 256);
  run<8>(4, 256);
  run<16>(1, 256);
  run<16>(2, 256);
  run<4>(8, 256);
  return 0;
}
