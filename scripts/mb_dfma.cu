// Microbenchmark: FP64 FMA throughput of this GPU (SURVEY Appendix B "FP64 ~37 TF/s, assumed; verify
// with a DFMA microbenchmark").  Every thread runs 8 independent DFMA chains; the
// grid fills every SM with 32 warps.  Reports TFLOP/s (2 flops per DFMA, CUDA-event time) and DFMA per SM per clock at the
// device's maximum SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_dfma scripts/mb_dfma.cu && /tmp/mb_dfma
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int kChains = 8;

__global__ void __launch_bounds__(1024) dfma_stream(int iters, double seed, double* out) {
  double x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = seed + threadIdx.x * 1e-9 + k;
  const double m = 0.999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < kChains; ++k) x[k] = fma(x[k], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += x[k];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, ctas = 2 * sms, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_stream<<<ctas, threads>>>(iters, 1.0, out);  // warm-up
  cudaEventRecord(e0);
  dfma_stream<<<ctas, threads>>>(iters, 1.0, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double dfma = (double)ctas * threads * iters * 16.0 * kChains;
  // per SM and clock at the device's maximum SM clock (a lower bound on the per-clock rate if
  // the clock sagged during the run); TFLOP/s counts 2 flops per DFMA over the event time
  printf("{\"tflops\": %.2f, \"ms\": %.3f, \"dfma_per_clk_per_sm_at_max_clock\": %.1f, \"max_mhz\": %d, \"err\": \"%s\"}\n",
         2.0 * dfma / (ms * 1e-3) / 1e12, ms, dfma / sms / (ms * 1e-3) / (khz * 1e3), khz / 1000,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
