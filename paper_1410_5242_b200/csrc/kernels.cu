// sm_100a kernels of the KPM-DOS hot path (arXiv:1410.5242, Fig. 5 `alg:kpm_improved_blocked`,
// PAPER.md P:388-406).  See DESIGN.md "Kernels" for the mapping and its roofline.
//
//   z4_init      |rand()> start block: Z4 phases from Philox4x32-10.
//   aug_spmmv    W <- scale*(H V - b V) [- W]  and the per-CTA partial column sums of
//                <V|V> and <W|V> (Eq. (3); eta definitions).
//   eta_finalize per-sweep grid reduction of the partials in a fixed order (deterministic),
//                done once for all sweeps after the loop (the "single reduction at the end"
//                of P:301-302 applied inside the device as well).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kpm_internal.h"

namespace kpm {
namespace {

// ------------------------------------------------------------------ Philox4x32-10 --
// Salmon et al., SC'11.  Device copy; the oracle has its own independent copy.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    if (i) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ double2 z4_phase(uint64_t seed, uint64_t row, uint32_t colg) {
  const uint4 w = philox4x32_10(make_uint4((uint32_t)row, (uint32_t)(row >> 32), colg, 0u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint32_t q = w.x >> 30;  // {1, i, -1, -i}
  return make_double2(q == 0 ? 1.0 : (q == 2 ? -1.0 : 0.0), q == 1 ? 1.0 : (q == 3 ? -1.0 : 0.0));
}

__global__ void z4_init_kernel(double2* __restrict__ V, double2* __restrict__ W, const int* __restrict__ perm,
                               int64_t n_loc, int64_t n_total, int R, int64_t row_begin, int64_t col_begin,
                               int r_valid, uint64_t seed) {
  const int64_t n_el = n_total * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / R;
    const int r = (int)(e - p * R);
    double2 v = make_double2(0.0, 0.0);
    if (p < n_loc && r < r_valid) {
      const int64_t row = row_begin + (perm ? (int64_t)perm[p] : p);
      v = z4_phase(seed, (uint64_t)row, (uint32_t)(col_begin + r));
    }
    V[e] = v;
    W[e] = make_double2(0.0, 0.0);
  }
}

__global__ void v0_permute_kernel(double2* __restrict__ V, double2* __restrict__ W, const double2* __restrict__ v0,
                                  const int* __restrict__ perm, int64_t n_loc, int64_t n_total, int R,
                                  int r_valid) {
  const int64_t n_el = n_total * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / R;
    const int r = (int)(e - p * R);
    double2 v = make_double2(0.0, 0.0);
    if (p < n_loc && r < r_valid) {
      const int64_t row = perm ? (int64_t)perm[p] : p;
      v = v0[row * r_valid + r];
    }
    V[e] = v;
    W[e] = make_double2(0.0, 0.0);
  }
}

// ------------------------------------------------------------- memory helpers ------
// Matrix entries and the old W are streamed once per sweep: bypass L1 and mark them
// evict-first in L2 so that L1/L2 keep the gathered V rows.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_stream_nc(const double2* ptr, uint64_t pol) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
      : "=d"(r.x), "=d"(r.y)
      : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ int ld_stream_nc(const int* ptr, uint64_t pol) {
  int r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* ptr, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_stream(double2* ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(ptr), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
}

// u += h * x  (complex multiply-add, 4 DFMA)
__device__ __forceinline__ void cmac(double2& u, const double2 h, const double2 x) {
  u.x = fma(h.x, x.x, u.x);
  u.x = fma(-h.y, x.y, u.x);
  u.y = fma(h.x, x.y, u.y);
  u.y = fma(h.y, x.x, u.y);
}

template <int R>
struct Map {
  static constexpr int LPR = R < 8 ? R : 8;  // lanes per row: LPR*16 B contiguous per row segment
  static constexpr int CPL = R / LPR;        // block columns per lane
  static constexpr int RW = 32 / LPR;        // rows per warp (= per row group)
  static constexpr int U = (CPL >= 4) ? 2 : (CPL == 2 ? 4 : 4);  // j-unroll (loads in flight)
};

// ------------------------------------------------------------------ aug_spmmv ------
// Thread mapping: a warp owns a row group of RW consecutive SELL
// positions inside one chunk; lane = (q, t): q = row in the group, t = lane in the row.
// Lane t of row q handles block columns r = cc*LPR + t, cc < CPL, so every gathered
// V row segment is LPR*16 contiguous bytes (a full 128-B line for R >= 8) and each
// SELL sub-column load of val/col serves RW rows.
template <int R, bool INIT>
__global__ void __launch_bounds__(kThreads) aug_spmmv_kernel(const SweepArgs a) {
  using Mp = Map<R>;
  constexpr int LPR = Mp::LPR, CPL = Mp::CPL, RW = Mp::RW, U = Mp::U;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int q = lane / LPR;
  const int t = lane - q * LPR;
  const uint64_t pol = policy_evict_first();

  double ee[CPL], eor[CPL], eoi[CPL];
#pragma unroll
  for (int cc = 0; cc < CPL; ++cc) ee[cc] = eor[cc] = eoi[cc] = 0.0;

  const int64_t n_groups = a.group_end - a.group_begin;
  const int64_t seg_groups = (int64_t)a.segment * (kThreads / 32);
  const int64_t n_segs = (n_groups + seg_groups - 1) / seg_groups;
  for (int64_t sg = blockIdx.x; sg < n_segs; sg += gridDim.x) {
    const int64_t g_end = min(n_groups, (sg + 1) * seg_groups);
    for (int64_t gl = sg * seg_groups + warp; gl < g_end; gl += kThreads / 32) {
      const int64_t g = a.group_begin + gl;
      const int64_t p = g * RW + q;       // SELL position of this lane's row
      const int64_t c = (g * RW) >> 5;    // chunk
      const int k = (int)(p & 31);
      const int64_t s0 = __ldg(a.cptr + c);
      const int len = (int)((__ldg(a.cptr + c + 1) - s0) >> 5);
      const double2* vp = a.val + s0 + k;
      const int* cp = a.col + s0 + k;
      const double2* Vt = a.V + t;

      double2 u[CPL];
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) u[cc] = make_double2(0.0, 0.0);

      int j = 0;
      for (; j + U <= len; j += U) {
        double2 h[U];
        int cj[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          h[uu] = ld_stream_nc(vp + (j + uu) * kC, pol);
          cj[uu] = ld_stream_nc(cp + (j + uu) * kC, pol);
        }
        double2 x[U][CPL];
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) x[uu][cc] = __ldg(Vt + (int64_t)cj[uu] * R + cc * LPR);
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) cmac(u[cc], h[uu], x[uu][cc]);
      }
      for (; j < len; ++j) {
        const double2 h = ld_stream_nc(vp + j * kC, pol);
        const int cj = ld_stream_nc(cp + j * kC, pol);
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) cmac(u[cc], h, __ldg(Vt + (int64_t)cj * R + cc * LPR));
      }

      // epilogue: shift, scale, -W, store, fused dot products (Fig. 5 "&" chain)
      if (p < a.n_loc) {
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
          const int64_t e = p * R + cc * LPR + t;
          const double2 vi = __ldg(a.V + e);
          double2 uu = u[cc];
          uu.x = fma(-a.b, vi.x, uu.x);
          uu.y = fma(-a.b, vi.y, uu.y);
          double2 w;
          if (INIT) {
            w = make_double2(a.scale * uu.x, a.scale * uu.y);
          } else {
            const double2 wo = ld_stream(a.W + e, pol);
            w = make_double2(fma(a.scale, uu.x, -wo.x), fma(a.scale, uu.y, -wo.y));
          }
          st_stream(a.W + e, w, pol);
          ee[cc] = fma(vi.x, vi.x, fma(vi.y, vi.y, ee[cc]));
          // conj(w) * v = (wr vr + wi vi) + i (wr vi - wi vr)
          eor[cc] = fma(w.x, vi.x, fma(w.y, vi.y, eor[cc]));
          eoi[cc] = fma(w.x, vi.y, fma(-w.y, vi.x, eoi[cc]));
        }
      }
    }
  }

  // ---- CTA reduction (fixed order => deterministic) --------------------------------
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
      ee[cc] += __shfl_xor_sync(0xffffffffu, ee[cc], off);
      eor[cc] += __shfl_xor_sync(0xffffffffu, eor[cc], off);
      eoi[cc] += __shfl_xor_sync(0xffffffffu, eoi[cc], off);
    }
  }
  __shared__ double red[kThreads / 32][3 * R];
  if (lane < LPR) {
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
      const int r = cc * LPR + lane;
      red[warp][r] = ee[cc];
      red[warp][R + r] = eor[cc];
      red[warp][2 * R + r] = eoi[cc];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * R; i += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) s += red[w][i];
    a.partials[(int64_t)i * gridDim.x + blockIdx.x] = s;
  }
}

// One warp per (sweep, component, column): sum the grid partials in a fixed order.
__global__ void eta_finalize_kernel(const double* __restrict__ partials, int n_sweeps, int R, int grid,
                                    double2* __restrict__ eta_even, double2* __restrict__ eta_odd) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_out = (int64_t)n_sweeps * 3 * R;
  if (wid >= n_out) return;
  const int64_t m = wid / (3 * R);
  const int i = (int)(wid - m * 3 * R);
  const double* src = partials + (m * 3 * R + i) * (int64_t)grid;
  double s = 0.0;
  for (int bq = lane; bq < grid; bq += 32) s += src[bq];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) {
    const int comp = i / R, r = i - comp * R;
    if (comp == 0) {
      eta_even[m * R + r] = make_double2(s, 0.0);
    } else if (comp == 1) {
      eta_odd[m * R + r].x = s;
    } else {
      eta_odd[m * R + r].y = s;
    }
  }
}

template <int R>
cudaError_t launch_r(bool init, const SweepArgs& a, int grid, cudaStream_t s) {
  if (init)
    aug_spmmv_kernel<R, true><<<grid, kThreads, 0, s>>>(a);
  else
    aug_spmmv_kernel<R, false><<<grid, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

template <int R>
int occupancy_r(bool init) {
  int n = 0;
  if (init)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, aug_spmmv_kernel<R, true>, kThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, aug_spmmv_kernel<R, false>, kThreads, 0);
  return n;
}

}  // namespace

int rows_per_group(int R) {
  switch (R) {
    case 1: return Map<1>::RW;
    case 2: return Map<2>::RW;
    case 4: return Map<4>::RW;
    case 8: return Map<8>::RW;
    case 16: return Map<16>::RW;
    case 32: return Map<32>::RW;
  }
  return 0;
}

int sweep_occupancy(int R, bool init) {
  switch (R) {
    case 1: return occupancy_r<1>(init);
    case 2: return occupancy_r<2>(init);
    case 4: return occupancy_r<4>(init);
    case 8: return occupancy_r<8>(init);
    case 16: return occupancy_r<16>(init);
    case 32: return occupancy_r<32>(init);
  }
  return 0;
}

cudaError_t launch_aug_spmmv(int R, bool init, const SweepArgs& a, int grid, cudaStream_t s) {
  switch (R) {
    case 1: return launch_r<1>(init, a, grid, s);
    case 2: return launch_r<2>(init, a, grid, s);
    case 4: return launch_r<4>(init, a, grid, s);
    case 8: return launch_r<8>(init, a, grid, s);
    case 16: return launch_r<16>(init, a, grid, s);
    case 32: return launch_r<32>(init, a, grid, s);
  }
  return cudaErrorInvalidValue;
}

static int elementwise_grid(int64_t n_el) {
  int64_t g = (n_el + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_z4_init(double2* V, double2* W, const int* perm, int64_t n_loc, int64_t n_rows_total, int R,
                           int64_t row_begin, int64_t col_begin, int r_valid, uint64_t seed, cudaStream_t s) {
  z4_init_kernel<<<elementwise_grid(n_rows_total * R), 256, 0, s>>>(V, W, perm, n_loc, n_rows_total, R, row_begin,
                                                                     col_begin, r_valid, seed);
  return cudaGetLastError();
}

cudaError_t launch_v0_upload_permute(double2* V, double2* W, const double2* v0_dev, const int* perm, int64_t n_loc,
                                     int64_t n_rows_total, int R, int r_valid, cudaStream_t s) {
  v0_permute_kernel<<<elementwise_grid(n_rows_total * R), 256, 0, s>>>(V, W, v0_dev, perm, n_loc, n_rows_total, R,
                                                                        r_valid);
  return cudaGetLastError();
}

cudaError_t launch_eta_finalize(const double* partials, int n_sweeps, int R, int grid, double2* eta_even,
                                double2* eta_odd, cudaStream_t s) {
  const int64_t n_threads = (int64_t)n_sweeps * 3 * R * 32;
  const int blocks = (int)((n_threads + 255) / 256);
  eta_finalize_kernel<<<blocks, 256, 0, s>>>(partials, n_sweeps, R, grid, eta_even, eta_odd);
  return cudaGetLastError();
}

}  // namespace kpm
