// Microbenchmark: peak register-side shared-memory bandwidth of LDS.128 on this GPU (bytes per SM
// clock), the denominator of the bench line's `cache_roofline`.  Every warp
// streams 16-B loads of 32 distinct consecutive words (conflict-free, one 128-B wavefront per
// quarter warp) with ILP independent loads in flight per thread and minimal ALU work; the best over
// CTA shapes and ILP is the peak.  Prints one JSON line per configuration and a final "peak" line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_lds_peak scripts/mb_lds_peak.cu && /tmp/mb_lds_peak
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int ILP>
__global__ void __launch_bounds__(1024) lds_stream(int iters, unsigned* out, long long* clk) {
  __shared__ uint4 sm[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_uint4(i, 3 * i, 5 * i, 7 * i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned acc = 0;
  unsigned idx = (unsigned)(warp * 32 + lane) & 2047u;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint4 v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = sm[(idx + 32u * (unsigned)k) & 2047u];
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    idx = (idx + 32u * ILP) & 2047u;
  }
  const long long t1 = clock64();
  if (acc == 0x12345678u) out[0] = acc;
  if (lane == 0) clk[blockIdx.x * 32 + warp] = t1 - t0;
}

template <int ILP>
double run(int sms, int ctas_per_sm, int warps, int iters, unsigned* out, long long* clk) {
  const int grid = sms * ctas_per_sm;
  lds_stream<ILP><<<grid, 32 * warps>>>(iters, out, clk);
  lds_stream<ILP><<<grid, 32 * warps>>>(iters, out, clk);
  cudaDeviceSynchronize();
  long long c[64];
  cudaMemcpy(c, clk, sizeof(long long) * 32 * ctas_per_sm, cudaMemcpyDeviceToHost);  // the CTAs on SM 0 first
  long long cmax = 1;
  for (int w = 0; w < warps * ctas_per_sm && w < 64; ++w) cmax = c[w] > cmax ? c[w] : cmax;
  // bytes one SM's warps delivered to registers / the slowest warp's cycles (CTAs co-resident)
  return (double)ctas_per_sm * warps * 32 * 16.0 * ILP * iters / (double)cmax;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  long long* clk;
  cudaMalloc(&out, 16);
  cudaMalloc(&clk, sizeof(long long) * sms * 64);
  double best = 0;
  for (int ctas : {1, 2}) {
    for (int warps : {16, 32}) {
      if (ctas * warps > 64) continue;
      double b8 = run<8>(sms, ctas, warps, 2048, out, clk);
      double b16 = run<16>(sms, ctas, warps, 1024, out, clk);
      printf("{\"ctas_per_sm\": %d, \"warps\": %d, \"ilp8_B_per_clk\": %.1f, \"ilp16_B_per_clk\": %.1f}\n", ctas, warps,
             b8, b16);
      best = b8 > best ? b8 : best;
      best = b16 > best ? b16 : best;
    }
  }
  printf("{\"peak_lds128_B_per_clk_per_sm\": %.1f, \"err\": \"%s\"}\n", best, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
