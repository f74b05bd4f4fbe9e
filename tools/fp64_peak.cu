// fp64 FMA peak of this B200 (the ALU roofline of the C4 right-hand side, k_rhs_c4).
// Every thread runs NACC independent DFMA chains of ITER steps (no memory traffic in the loop); all SMs, 4
// resident CTAs of 256 threads each; CUDA events, best of 5. Prints one JSON line: TFLOP/s (2 flops per DFMA).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NACC = 8, ITER = 4096;

__global__ void __launch_bounds__(256) k_dfma(double* out, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITER; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;   // keeps the chains live
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, 256>>>(out, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, 256>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * NACC * ITER * 256.0 * blocks;
  const double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"blocks\": %d, \"threads\": 256, \"chains_per_thread\": %d, "
         "\"clock_rate_khz\": %d, \"per_sm_per_clk_fma\": %.2f}\n",
         tf, best, sms, blocks, NACC, clk, flops / 2.0 / (best * 1e-3) / sms / (clk * 1e3));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
