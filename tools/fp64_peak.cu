// fp64_peak.cu -- measured FP64 FMA throughput of this B200 (the "alu" roofline denominator of the
// control search).  8 independent DFMA chains per thread, 148 x 8 CTAs of 256 threads, timed with
// CUDA events after warm-up; prints one JSON line {"tflops": ..., ...}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x] = s;  // never true; keeps the chains live
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  const double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
         "\"dfma_per_clk_per_sm_at_max_clock\": %.1f, \"how\": \"8 independent DFMA chains/thread, "
         "%d CTAs x 256 threads, best of 10 after 3 warm-ups (tools/fp64_peak.cu)\"}\n",
         tf, best, sms, clk / 1e3, tf * 1e12 / 2.0 / sms / (clk * 1e3), blocks);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
