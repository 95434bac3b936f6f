// Microbenchmark (round 2): do texture fetches and shared-memory loads share the
// register-side data path of the SM?  Warps either stream LDS.128 from shared memory, or fetch
// 16-B texels (tex1Dfetch<int4>) of a small L1-resident buffer, or both kinds side by side in
// one CTA; bytes delivered to registers per SM clock for each mix.  Build and run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_pipes scripts/mb_pipes.cu && /tmp/mb_pipes
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kIters = 4096;

// mode 0: all warps LDS; 1: all warps TEX; 2: even warps LDS, odd warps TEX; 3: all warps LDG.nc
__global__ void __launch_bounds__(512) mix(cudaTextureObject_t tex, const int4* __restrict__ g, int n_tex, int mode,
                                          int4* out, long long* clk) {
  __shared__ int4 sm[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_int4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool use_tex = mode == 1 || (mode == 2 && (warp & 1));
  const bool use_ldg = mode == 3;
  int4 acc = make_int4(0, 0, 0, 0);
  unsigned idx = (threadIdx.x * 7u) & 2047u;
  const long long t0 = clock64();
#pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    int4 v;
    if (use_tex)
      v = tex1Dfetch<int4>(tex, (int)(idx & (unsigned)(n_tex - 1)));
    else if (use_ldg)
      v = __ldg(g + (idx & (unsigned)(n_tex - 1)));
    else
      v = sm[idx];
    acc.x += v.x;
    acc.y ^= v.y;
    acc.z += v.z;
    acc.w ^= v.w;
    idx = (idx + 32u) & 2047u;  // independent of the loaded data: loads overlap (throughput, not latency)
  }
  const long long t1 = clock64();
  if (acc.x == 0x7fffffff) out[0] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  (void)lane;
}

int main() {
  const int n_tex = 1024;  // 16 KB of texels: L1-resident
  int4* g;
  cudaMalloc(&g, n_tex * sizeof(int4));
  cudaMemset(g, 1, n_tex * sizeof(int4));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = g;
  rd.res.linear.desc = cudaCreateChannelDesc<int4>();
  rd.res.linear.sizeInBytes = n_tex * sizeof(int4);
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int4* out;
  long long* clk;
  cudaMalloc(&out, 16);
  cudaMalloc(&clk, sizeof(long long) * sms);
  const char* names[] = {"LDS.128 only", "TEX (tex1Dfetch int4) only", "LDS + TEX (half the warps each)",
                         "LDG.nc (L1 hits) only"};
  for (int warps : {8, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      mix<<<sms, 32 * warps>>>(tex, g, n_tex, mode, out, clk);  // warm-up
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      mix<<<sms, 32 * warps>>>(tex, g, n_tex, mode, out, clk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      long long c = 0;
      cudaMemcpy(&c, clk, sizeof(long long), cudaMemcpyDeviceToHost);
      const double bytes_per_sm = 32.0 * warps * 16.0 * kIters;
      printf("{\"warps\": %d, \"mode\": \"%s\", \"cycles\": %lld, \"bytes_per_clk_per_sm\": %.1f, \"ms\": %.4f}\n", warps,
             names[mode], c, bytes_per_sm / (double)c, ms);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
