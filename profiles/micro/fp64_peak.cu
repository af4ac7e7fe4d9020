// Microbenchmark: FP64 peak of the B200 SM on its two FP64 paths, to
// calibrate the FP64 roofline of the tile kernel and to decide whether the
// FP64 tensor cores (DMMA, mma.sync .f64) can beat the DFMA pipe for the
// contraction-shaped work (5-target fused blocks; reference zgemm path
// kernels.py:100-106).
//   * DFMA: 8 independent fma chains per thread, 4 x 256 threads per SM;
//   * DMMA m8n8k4 and m16n8k16 (.f64): 4 independent accumulators per warp.
// burst = one ~2 ms launch, sustained = back-to-back launches for ~2 s (under
// the power cap).  Output: one JSON line (profiles/fp64_peak.py adds clocks).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak
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

// m8n8k4: A 1 double, B 1 double, C/D 2 doubles per thread; 256 FMA per warp op
__global__ void __launch_bounds__(256) k_dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double d[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = c * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
          : "+d"(d[c][0]), "+d"(d[c][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

// m16n8k16 (sm_90+ shape): A 8 doubles, B 4, C/D 4 per thread; 2048 FMA per warp op
__global__ void __launch_bounds__(256) k_dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + (threadIdx.x + j) * 1e-9;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 0.999999 - j * 1e-9;
  double d[2][4];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int j = 0; j < 4; ++j) d[c][j] = c * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
            "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += d[c][j];
  if (s == 12345.678) out[0] = s;
}

enum Kind { DFMA, DMMA884, DMMA16816 };

double run(Kind kind, int blocks_per_sm, int iters, int reps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  auto launch = [&](int it) {
    if (kind == DFMA) k_dfma<8><<<sms * blocks_per_sm, 256>>>(out, it, 0.999999, 1e-7);
    else if (kind == DMMA884) k_dmma_m8n8k4<<<sms * blocks_per_sm, 256>>>(out, it);
    else k_dmma_m16n8k16<<<sms * blocks_per_sm, 256>>>(out, it);
  };
  launch(64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch(iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  const double threads = (double)sms * blocks_per_sm * 256;
  double fmas;
  if (kind == DFMA) fmas = threads * iters * 8 * reps;
  else if (kind == DMMA884) fmas = threads / 32 * iters * 4 * 256.0 * reps;
  else fmas = threads / 32 * iters * 2 * 2048.0 * reps;
  return 2 * fmas / (ms * 1e-3) / 1e12;
}

int main() {
  const double burst = run(DFMA, 4, 4096, 1);
  const double sustained = run(DFMA, 4, 4096, 1500);
  const double m884_b = run(DMMA884, 4, 2048, 1);
  const double m884_s = run(DMMA884, 4, 2048, 600);
  const double m16_b = run(DMMA16816, 4, 512, 1);
  const double m16_s = run(DMMA16816, 4, 512, 600);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"fp64_tflops_burst\": %.2f, \"fp64_tflops_sustained\": %.2f, "
         "\"dmma_m8n8k4_tflops_burst\": %.2f, \"dmma_m8n8k4_tflops_sustained\": %.2f, "
         "\"dmma_m16n8k16_tflops_burst\": %.2f, \"dmma_m16n8k16_tflops_sustained\": %.2f, "
         "\"cuda_status\": \"%s\", "
         "\"how\": \"profiles/micro/fp64_peak.cu: DFMA = 8 independent chains/thread, 4x256 "
         "threads/SM; DMMA = mma.sync .f64 with 4 (m8n8k4) / 2 (m16n8k16) independent "
         "accumulators per warp; burst = one launch, sustained = back-to-back launches\"}\n",
         burst, sustained, m884_b, m884_s, m16_b, m16_s, cudaGetErrorString(e));
  return 0;
}
