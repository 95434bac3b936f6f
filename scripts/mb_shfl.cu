// Microbenchmark: does SHFL run beside LDS.128 on sm_100a, and what does a broadcast LDS cost?
// Decides whether the R = 32 sweep's matrix-value broadcast (8 lanes of a row read the same 16-B
// value: LDS.128 with 4 distinct addresses per warp) can move to shuffles.
// Every mode runs one CTA of W warps per SM, each warp issuing a fixed instruction mix per
// iteration with independent operands; reports SM clocks per iteration per warp-instruction kind.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_shfl scripts/mb_shfl.cu && /tmp/mb_shfl
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

// NL distinct-address LDS.128, NB broadcast LDS.128 (address = lane / 8), NS 32-bit SHFL.idx
template <int NL, int NB, int NS, int NB1>
__global__ void __launch_bounds__(1024) mix(int iters, unsigned* out, long long* clk) {
  __shared__ uint4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_uint4(i, 3 * i, 5 * i, 7 * i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned acc = lane, acc2 = 0;
  unsigned idx = (unsigned)(warp * 32 + lane) & 2047u;
  unsigned bidx = (unsigned)(warp * 4 + (lane >> 3)) & 2047u;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint4 v[NL > 0 ? NL : 1], b[NB > 0 ? NB : 1], b1[NB1 > 0 ? NB1 : 1];
    unsigned s[NS > 0 ? NS : 1];
#pragma unroll
    for (int k = 0; k < NL; ++k) v[k] = sm[(idx + 32u * (unsigned)k) & 2047u];
#pragma unroll
    for (int k = 0; k < NB; ++k) b[k] = sm[(bidx + 128u * (unsigned)k) & 2047u];
#pragma unroll
    for (int k = 0; k < NB1; ++k) b1[k] = sm[(unsigned)(warp + 64 * k) & 2047u];
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = __shfl_sync(0xffffffffu, acc + k, (lane & 24) | (k & 7));
#pragma unroll
    for (int k = 0; k < NL; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
#pragma unroll
    for (int k = 0; k < NB; ++k) acc ^= b[k].x ^ b[k].y ^ b[k].z ^ b[k].w;
#pragma unroll
    for (int k = 0; k < NB1; ++k) acc ^= b1[k].x ^ b1[k].y ^ b1[k].z ^ b1[k].w;
#pragma unroll
    for (int k = 0; k < NS; ++k) acc2 += s[k];
    idx = (idx + 32u * 8u) & 2047u;
    bidx = (bidx + 4u) & 2047u;
    acc += acc2 & 1u;
  }
  const long long t1 = clock64();
  if ((acc ^ acc2) == 0x12345678u) out[0] = acc;
  if (lane == 0) clk[blockIdx.x * 32 + warp] = t1 - t0;
}

template <int NL, int NB, int NS, int NB1>
void run(const char* name, int sms, int warps, int iters, unsigned* out, long long* clk) {
  mix<NL, NB, NS, NB1><<<sms, 32 * warps>>>(iters, out, clk);
  mix<NL, NB, NS, NB1><<<sms, 32 * warps>>>(iters, out, clk);
  cudaDeviceSynchronize();
  long long c[32];
  cudaMemcpy(c, clk, sizeof(long long) * 32, cudaMemcpyDeviceToHost);
  long long cmax = 1;
  for (int w = 0; w < warps; ++w) cmax = c[w] > cmax ? c[w] : cmax;
  const double per_it = (double)cmax / iters;  // SM clocks per iteration (all W warps)
  printf("{\"mode\": \"%s\", \"warps\": %d, \"lds128\": %d, \"lds128_bcast8\": %d, \"shfl32\": %d, "
         "\"lds128_bcast32\": %d, \"clk_per_iter_per_warp\": %.3f, \"err\": \"%s\"}\n",
         name, warps, NL, NB, NS, NB1, per_it / warps, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  long long* clk;
  cudaMalloc(&out, 16);
  cudaMalloc(&clk, sizeof(long long) * sms * 32);
  for (int warps : {8, 16, 32}) {
    const int it = 4096;
    run<8, 0, 0, 0>("lds128 x8", sms, warps, it, out, clk);                   // expect 32 clk (4 wavefronts each)
    run<0, 8, 0, 0>("lds128 bcast8 x8", sms, warps, it, out, clk);            // 4 addresses per warp
    run<0, 0, 0, 8>("lds128 bcast32 x8", sms, warps, it, out, clk);           // one address per warp
    run<0, 0, 8, 0>("shfl32 x8", sms, warps, it, out, clk);
    run<0, 0, 32, 0>("shfl32 x32", sms, warps, it, out, clk);
    run<8, 0, 8, 0>("lds128 x8 + shfl32 x8", sms, warps, it, out, clk);       // additive = 40 clk
    run<8, 0, 16, 0>("lds128 x8 + shfl32 x16", sms, warps, it, out, clk);
    run<8, 2, 0, 0>("lds128 x8 + bcast8 x2", sms, warps, it, out, clk);       // the R = 32 kernel's mix
    run<8, 0, 8, 0>("lds128 x8 + shfl32 x8 (again)", sms, warps, it, out, clk);
  }
  return 0;
}
