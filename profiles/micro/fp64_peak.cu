// Microbenchmark: FP64 FMA peak of the B200 SM, burst (2 ms) and sustained
// (~2 s, under the power cap), to calibrate the FP64 roofline of the tile
// kernel.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdlib>
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

double run(int blocks_per_sm, int iters, int reps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  k_dfma<8><<<sms * blocks_per_sm, 256>>>(out, 64, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_dfma<8><<<sms * blocks_per_sm, 256>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  const double fmas = (double)sms * blocks_per_sm * 256 * iters * 8 * reps;
  return 2 * fmas / (ms * 1e-3) / 1e12;
}

int main() {
  const double burst = run(4, 4096, 1);
  const double sustained = run(4, 4096, 1500);
  printf("{\"fp64_tflops_burst\": %.2f, \"fp64_tflops_sustained\": %.2f, "
         "\"how\": \"profiles/micro/fp64_peak.cu: 8 independent DFMA chains/thread, 4x256 "
         "threads/SM; burst = one 2 ms launch, sustained = 1500 back-to-back launches\"}\n",
         burst, sustained);
  return 0;
}
