// Optimisation-stage ladder: the paper's stage-0 "naive" KPM-DOS of
// Fig. 3 `alg:kpm_naive` on the GPU, one BLAS-1 kernel per line of the
// algorithm -- spmv(), axpy(), scal(), axpy(), nrm2(), dot() -- run column by column.  It exists to
// measure what the fusion of Fig. 4 and the blocking of Fig. 5 buy on a B200 (the paper's
// Fig. 11 / Table III comparison), not as a production path.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kpm_internal.h"

namespace kpm {
namespace {

constexpr int kNaiveBlock = 256;

// u = H v   (SELL-32, one thread per row, stored order)
__global__ void spmv_kernel(const double2* __restrict__ val, const int* __restrict__ col, const int64_t* __restrict__ cptr,
                            const double2* __restrict__ v, double2* __restrict__ u, int64_t n_pad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_pad; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = p >> 5;
    const int k = (int)(p & 31);
    const int64_t s0 = cptr[c];
    const int L = (int)((cptr[c + 1] - s0) >> 5);
    double2 s = make_double2(0.0, 0.0);
    for (int j = 0; j < L; ++j) {
      const double2 h = val[s0 + (int64_t)j * kC + k];
      const double2 x = v[col[s0 + (int64_t)j * kC + k]];
      s.x = fma(h.x, x.x, s.x);
      s.x = fma(-h.y, x.y, s.x);
      s.y = fma(h.x, x.y, s.y);
      s.y = fma(h.y, x.x, s.y);
    }
    u[p] = s;
  }
}

// y = y + alpha x  (real alpha)
__global__ void axpy_kernel(double2* __restrict__ y, const double2* __restrict__ x, double alpha, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 a = y[i];
    const double2 b = x[i];
    a.x = fma(alpha, b.x, a.x);
    a.y = fma(alpha, b.y, a.y);
    y[i] = a;
  }
}

// y = alpha y
__global__ void scal_kernel(double2* __restrict__ y, double alpha, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 a = y[i];
    y[i] = make_double2(alpha * a.x, alpha * a.y);
  }
}

// y = alpha x
__global__ void scale_copy_kernel(double2* __restrict__ y, const double2* __restrict__ x, double alpha, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 b = x[i];
    y[i] = make_double2(alpha * b.x, alpha * b.y);
  }
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
  __syncthreads();
  return s;
}

// nrm2(): partial[0][block] = sum |v|^2 ;  dot(): partial[1..2][block] = sum conj(w) v
__global__ void nrm2_kernel(const double2* __restrict__ v, int64_t n, double* __restrict__ part, int64_t pstride) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = v[i];
    s = fma(a.x, a.x, fma(a.y, a.y, s));
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  (void)pstride;
}

__global__ void dot_kernel(const double2* __restrict__ w, const double2* __restrict__ v, int64_t n,
                           double* __restrict__ part, int64_t pstride) {
  __shared__ double sh[32];
  double re = 0.0, im = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = w[i], b = v[i];
    re = fma(a.x, b.x, fma(a.y, b.y, re));
    im = fma(a.x, b.y, fma(-a.y, b.x, im));
  }
  re = block_sum(re, sh);
  im = block_sum(im, sh);
  if (threadIdx.x == 0) {
    part[pstride + blockIdx.x] = re;
    part[2 * pstride + blockIdx.x] = im;
  }
}

}  // namespace

int naive_grid() { return 148 * 8; }

// One naive sweep of one column (Fig. 3): for init, w = a (H v - b v); else swap is implicit
// (caller passes v, w), u = Hv; u = u - b v; w = -w; w = w + 2a u; then nrm2, dot.
cudaError_t naive_sweep(const DevSell& s, const double2* v, double2* w, double2* u, double a, double b, bool init,
                        double* part, cudaStream_t st) {
  const int g = naive_grid();
  const int64_t n = s.n_loc;  // padding rows stay zero and never enter the sums
  spmv_kernel<<<g, kNaiveBlock, 0, st>>>(s.val, s.col, s.cptr, v, u, s.n_pad);                   // spmv()
  axpy_kernel<<<g, kNaiveBlock, 0, st>>>(u, v, -b, n);                                            // axpy()
  if (init) {
    scale_copy_kernel<<<g, kNaiveBlock, 0, st>>>(w, u, a, n);                                     // nu_1 = a u
  } else {
    scal_kernel<<<g, kNaiveBlock, 0, st>>>(w, -1.0, n);                                           // scal()
    axpy_kernel<<<g, kNaiveBlock, 0, st>>>(w, u, 2.0 * a, n);                                     // axpy()
  }
  nrm2_kernel<<<g, kNaiveBlock, 0, st>>>(v, n, part, g);                                          // nrm2()
  dot_kernel<<<g, kNaiveBlock, 0, st>>>(w, v, n, part, g);                                        // dot()
  return cudaGetLastError();
}

}  // namespace kpm
