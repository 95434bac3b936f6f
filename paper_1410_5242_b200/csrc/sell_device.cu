// Device-side setup: CSR (device) -> SELL-32 (sigma = 1) + the tiled feed's
// gather plan, for matrices too large to stage through host memory (config C5: 1.5e9
// nonzeros per GPU).  Produces exactly the layout of the host builder (sell_build.cpp,
// DESIGN.md "SELL-C-sigma"; tests compare both with oracle/sell_ref.py), plus the
// fixed-capacity per-chunk run lists from which the per-R copy records are built
// (build_records_kernel, used by both build paths).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "kpm_internal.h"

namespace kpm {
namespace {

constexpr int kTileCap = 2048;  // slots of one chunk the device tile planner handles (L <= 64)

__global__ void validate_kernel(const int64_t* __restrict__ rp, const int64_t* __restrict__ col,
                                const double2* __restrict__ val, int64_t n_loc, int64_t n_global, int* flags) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < n_loc; i += stride)
    if (rp[i + 1] < rp[i]) atomicOr(flags, 1);
  const int64_t nnz = rp[n_loc];
  for (int64_t k = i0; k < nnz; k += stride) {
    if (col[k] < 0 || col[k] >= n_global) atomicOr(flags, 2);
    const double2 v = val[k];
    if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(flags, 4);
  }
}

__global__ void width_kernel(const int64_t* __restrict__ rp, int64_t n_loc, int64_t n_chunks, int64_t* __restrict__ w,
                             int64_t* __restrict__ slots) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = 0;
    for (int k = 0; k < kC; ++k) {
      const int64_t p = c * kC + k;
      if (p < n_loc) m = max(m, rp[p + 1] - rp[p]);
    }
    w[c] = m;
    slots[c] = m * kC;
  }
}

struct IsRemote {
  int64_t b, e;
  __host__ __device__ bool operator()(const int64_t g) const { return g < b || g >= e; }
};

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t g) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < g)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// one warp per chunk, lane = row of the chunk
__global__ void scatter_kernel(const int64_t* __restrict__ rp, const int64_t* __restrict__ col,
                               const double2* __restrict__ val, int64_t n_loc, int64_t n_chunks, int64_t row_begin,
                               int64_t row_end, int64_t n_pad, const int64_t* __restrict__ halo, int64_t n_halo,
                               const int64_t* __restrict__ cptr, double2* __restrict__ sval, int* __restrict__ scol) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < n_chunks; c += warps) {
    const int64_t s0 = cptr[c];
    const int L = (int)((cptr[c + 1] - s0) >> 5);
    const int64_t p = c * kC + lane;
    const int64_t base = p < n_loc ? rp[p] : 0;
    const int len = p < n_loc ? (int)(rp[p + 1] - base) : 0;
    // own-position (diagonal) entry first, then the others in stored order (R18)
    int jd = len;
    for (int j = 0; j < len; ++j)
      if (col[base + j] == row_begin + p) {
        jd = j;
        break;
      }
    for (int j = 0; j < L; ++j) {
      const int64_t d = s0 + (int64_t)j * kC + lane;
      if (j < len) {
        const int js = jd == len ? j : (j == 0 ? jd : (j <= jd ? j - 1 : j));  // source entry
        const int64_t g = col[base + js];
        scol[d] = (int)(g >= row_begin && g < row_end ? g - row_begin : n_pad + lower_bound_i64(halo, n_halo, g));
        sval[d] = val[base + js];
      } else {
        scol[d] = (int)p;
        sval[d] = make_double2(0.0, 0.0);
      }
    }
  }
}

// exclusive block scan of one int per thread (blockDim = 256)
__device__ __forceinline__ int block_excl_scan(int v, int* tmp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += n;
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int y = lane < (int)(blockDim.x >> 5) ? tmp[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) y += n;
    }
    tmp[lane] = y;  // inclusive warp totals
  }
  __syncthreads();
  const int excl = x - v + (warp ? tmp[warp - 1] : 0);
  *total = tmp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return excl;
}

// Tile plan of one chunk per CTA (256 threads): distinct other columns (sorted, unique),
// their runs, and each slot's tile-row index (uint16).
__global__ void __launch_bounds__(256) tiles_kernel(const int* __restrict__ scol, const int64_t* __restrict__ cptr,
                                                    int64_t n_chunks, uint16_t* __restrict__ lcol,
                                                    int* __restrict__ nruns, int* __restrict__ runs,
                                                    int* __restrict__ nother, int* __restrict__ flags) {
  __shared__ int key[kTileCap];
  __shared__ int uni[kTileCap];
  __shared__ int tmp[32];
  for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int64_t s0 = cptr[c];
    const int n = (int)(cptr[c + 1] - s0);
    const int own0 = (int)(c * kC);
    if (n > kTileCap) {
      if (threadIdx.x == 0) {
        atomicOr(flags, 8);
        nruns[c] = 0;
        nother[c] = 0;
      }
      continue;
    }
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
      int k = INT32_MAX;
      if (i < n) {
        const int g = scol[s0 + i];
        if (g < own0 || g >= own0 + kC) k = g;
      }
      key[i] = k;
    }
    __syncthreads();
    // bitonic sort, ascending
    for (int size = 2; size <= np2; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < np2; i += blockDim.x) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            const int a = key[i], b = key[j];
            if ((a > b) == up) {
              key[i] = b;
              key[j] = a;
            }
          }
        }
        __syncthreads();
      }
    // unique (each thread owns a contiguous segment of up to 8 entries)
    const int per = (np2 + blockDim.x - 1) / blockDim.x;
    const int i0 = threadIdx.x * per;
    int cnt = 0;
    for (int i = i0; i < min(i0 + per, np2); ++i)
      if (key[i] != INT32_MAX && (i == 0 || key[i] != key[i - 1])) ++cnt;
    int n_other;
    int o = block_excl_scan(cnt, tmp, &n_other);
    for (int i = i0; i < min(i0 + per, np2); ++i)
      if (key[i] != INT32_MAX && (i == 0 || key[i] != key[i - 1])) uni[o++] = key[i];
    __syncthreads();
    // runs of consecutive rows
    const int per2 = (n_other + blockDim.x - 1) / blockDim.x;
    const int j0 = threadIdx.x * per2;
    int rc = 0;
    for (int i = j0; i < min(j0 + per2, n_other); ++i)
      if (i == 0 || uni[i] != uni[i - 1] + 1) ++rc;
    int n_runs;
    int r = block_excl_scan(rc, tmp, &n_runs);
    if (n_runs > kMaxRuns) {
      if (threadIdx.x == 0) atomicOr(flags, 16);
    } else {
      for (int i = j0; i < min(j0 + per2, n_other); ++i)
        if (i == 0 || uni[i] != uni[i - 1] + 1) {
          int e = i + 1;
          while (e < n_other && uni[e] == uni[e - 1] + 1) ++e;
          runs[c * 2 * kMaxRuns + 2 * r] = uni[i];
          runs[c * 2 * kMaxRuns + 2 * r + 1] = e - i;
          ++r;
        }
    }
    if (threadIdx.x == 0) {
      nruns[c] = n_runs;
      nother[c] = n_other;
      if (n_other + kC > 65535) atomicOr(flags, 8);
    }
    // tile-row index of every slot
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int g = scol[s0 + i];
      int idx;
      if (g >= own0 && g < own0 + kC) {
        idx = g - own0;
      } else {
        int lo = 0, hi = n_other;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (uni[mid] < g)
            lo = mid + 1;
          else
            hi = mid;
        }
        idx = min(kC + lo, 65535);
      }
      lcol[s0 + i] = (uint16_t)idx;
    }
    __syncthreads();
  }
}

__global__ void reads_halo_kernel(const int* __restrict__ scol, const int64_t* __restrict__ cptr, int64_t n_chunks,
                                  int64_t n_pad, char* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < n_chunks; c += warps) {
    bool any = false;
    for (int64_t k = cptr[c] + lane; k < cptr[c + 1]; k += 32) any |= scol[k] >= n_pad;
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) out[c] = any ? 1 : 0;
  }
}

// Copy records (sell_build.h, kRecSlots x 16 B per chunk) for block width R.
__global__ void build_records_kernel(const int64_t* __restrict__ cptr, const int* __restrict__ nruns,
                                     const int* __restrict__ runs, int64_t n_chunks, int R, int off_w, int off_val,
                                     int off_lcol, uint4* __restrict__ rec) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowb = (int64_t)R * 16;
    uint4* r = rec + c * kRecSlots;
    int n = 0;
    int64_t total = 0;
    auto cmd = [&](uint32_t base, int64_t src, int64_t dst, int64_t bytes) {
      ++n;
      r[n] = make_uint4((uint32_t)src, (uint32_t)((uint64_t)src >> 32), (uint32_t)dst, (uint32_t)bytes | (base << 28));
      total += bytes;
    };
    const int64_t s0 = cptr[c], nslot = cptr[c + 1] - cptr[c];
    cmd(0, c * kC * rowb, 0, kC * rowb);
    cmd(1, c * kC * rowb, off_w, kC * rowb);
    const int64_t wbytes = kC * rowb;
    if (nslot) {
      cmd(2, s0 * 16, off_val, nslot * 16);
      cmd(3, s0 * 2, off_lcol, nslot * 2);
    }
    int64_t dst_row = kC;
    for (int k = 0; k < nruns[c]; ++k) {
      const int64_t first = runs[c * 2 * kMaxRuns + 2 * k], cnt = runs[c * 2 * kMaxRuns + 2 * k + 1];
      cmd(0, first * rowb, dst_row * rowb, cnt * rowb);
      dst_row += cnt;
    }
    for (int k = n + 1; k < kRecSlots; ++k) r[k] = make_uint4(0u, 0u, 0u, 0u);
    r[0] = make_uint4((uint32_t)total, (uint32_t)(total - wbytes), (uint32_t)(nslot / kC), (uint32_t)n);
  }
}

// Block-cache records: one thread per CTA simulates that CTA's pool of 32-row V blocks over its
// tile sequence (list positions b, b + G, b + 2G, ...).  A tile needs its own block and every
// block-aligned full 32-row run of its other rows (pool), the remaining rows are copied per
// stage (extra rows).  A slot may be refilled for tile k only if its last user is tile k - S or
// older: the producer refills stage k % S after all warps released tile k - S (ring order).
__global__ void bc_plan_kernel(const int64_t* __restrict__ cptr, const int* __restrict__ nruns,
                               const int* __restrict__ runs, const int64_t* __restrict__ list, int64_t n_chunks, int G,
                               int R, int with_w, TileLayout tl, uint4* __restrict__ rec, int* __restrict__ map,
                               int* __restrict__ fail) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= G) return;
  int sblk[kBcMaxSlots];
  int64_t slast[kBcMaxSlots];
  for (int i = 0; i < kBcMaxSlots; ++i) {
    sblk[i] = -1;
    slast[i] = -(1ll << 40);
  }
  const int64_t rowb = 16ll * R, blkb = 32 * rowb;
  const int S = tl.stages, P = tl.pool_slots;
  for (int64_t k = 0; b + k * G < n_chunks; ++k) {
    const int64_t pos = b + k * G;
    const int64_t c = list ? list[pos] : pos;
    const int64_t stage = tl.pool_bytes + (k % S) * (int64_t)tl.stage_bytes;
    uint4* r = rec + pos * kRecSlots;
    int* m = map + pos * kBcMapInts;
    bool ok = true;
    int n = 0;
    int64_t total = 0, wbytes = 0;
    auto cmd = [&](uint32_t base, int64_t src, int64_t dst, int64_t bytes) {
      if (n + 1 >= kRecSlots) {
        ok = false;
        return;
      }
      ++n;
      r[n] = make_uint4((uint32_t)src, (uint32_t)((uint64_t)src >> 32), (uint32_t)dst, (uint32_t)bytes | (base << 28));
      total += bytes;
    };
    int need[7], nneed = 0, xs[8], xc[8], nx = 0;
    need[nneed++] = (int)c;  // own rows = block c
    for (int q = 0; q < nruns[c]; ++q) {
      int first = runs[c * 2 * kMaxRuns + 2 * q], cnt = runs[c * 2 * kMaxRuns + 2 * q + 1];
      while (cnt > 0) {
        if ((first & 31) == 0 && cnt >= 32) {
          if (nneed < 7) need[nneed++] = first >> 5; else ok = false;
          first += 32;
          cnt -= 32;
        } else {
          const int piece = min(cnt, 32 - (first & 31));
          if (nx < 8) {
            xs[nx] = first;
            xc[nx] = piece;
            ++nx;
          } else {
            ok = false;
          }
          first += piece;
          cnt -= piece;
        }
      }
    }
    m[0] = nneed;
    for (int i = 0; i < nneed && ok; ++i) {
      int slot = -1;
      for (int p = 0; p < P; ++p)
        if (sblk[p] == need[i]) slot = p;
      if (slot < 0) {
        int64_t best = 1ll << 62;
        for (int p = 0; p < P; ++p)
          if (slast[p] <= k - S && slast[p] < best) {
            best = slast[p];
            slot = p;
          }
        if (slot < 0) {
          ok = false;
          break;
        }
        sblk[slot] = need[i];
        cmd(0, (int64_t)need[i] * blkb, (int64_t)slot * blkb, blkb);
      }
      slast[slot] = k;
      m[1 + 2 * i] = need[i];
      m[2 + 2 * i] = slot * 32;
    }
    m[15] = nx;
    int64_t erow = 0;
    for (int i = 0; i < nx && ok; ++i) {
      if (erow + xc[i] > tl.extra_rows) {
        ok = false;
        break;
      }
      const int64_t dst = stage + erow * rowb;
      cmd(0, (int64_t)xs[i] * rowb, dst, xc[i] * rowb);
      m[16 + 3 * i] = xs[i];
      m[17 + 3 * i] = xc[i];
      m[18 + 3 * i] = (int)(dst / rowb);
      erow += xc[i];
    }
    const int64_t s0 = cptr[c], nslot = cptr[c + 1] - s0;
    if (with_w) {
      cmd(1, c * blkb, stage + tl.off_w, blkb);
      wbytes = blkb;
    }
    if (nslot) {
      cmd(2, s0 * 16, stage + tl.off_val, nslot * 16);
      if (tl.lt_stride)  // row-major tile indices: fixed-size block per chunk
        cmd(3, c * kC * tl.lt_stride * 2, stage + tl.off_lcol, (int64_t)kC * tl.lt_stride * 2);
      else
        cmd(3, s0 * 2, stage + tl.off_lcol, nslot * 2);
    }
    for (int q = n + 1; q < kRecSlots; ++q) r[q] = make_uint4(0u, 0u, 0u, 0u);
    r[0] = make_uint4((uint32_t)total, (uint32_t)(total - wbytes), (uint32_t)(nslot / kC),
                      (uint32_t)n | ((uint32_t)m[2] << 8));
    if (!ok) atomicOr(fail, 1);
  }
}

// Tile-row index (absolute shared-memory V row) of every SELL slot, one warp per tile.
__global__ void bc_lcol_kernel(const int* __restrict__ scol, const int64_t* __restrict__ cptr,
                               const int64_t* __restrict__ list, int64_t n_chunks, const int* __restrict__ map,
                               uint16_t* __restrict__ lcol, int* __restrict__ fail, int lts, int R) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t pos = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); pos < n_chunks; pos += warps) {
    const int64_t c = list ? list[pos] : pos;
    const int* m = map + pos * kBcMapInts;
    const int nb = min(m[0], 7), nx = min(m[15], 8);
    for (int64_t e = cptr[c] + lane; e < cptr[c + 1]; e += 32) {
      const int g = scol[e];
      int row = -1;
      for (int i = 0; i < nb; ++i)
        if (m[1 + 2 * i] == (g >> 5)) row = m[2 + 2 * i] + (g & 31);
      for (int i = 0; i < nx && row < 0; ++i)
        if (g >= m[16 + 3 * i] && g < m[16 + 3 * i] + m[17 + 3 * i]) row = m[18 + 3 * i] + g - m[16 + 3 * i];
      // stored as row * R (the V row's offset in double2 units, < 227 KB / 16): the sweep adds it to
      // its lane's base address without a multiply
      row = row < 0 ? -1 : row * R;
      if (row < 0 || row > 65535) atomicOr(fail, 2);
      if (lts) {  // row-major: entries 1.. at k*lts + j - 1, entry 0 at k*lts + lts - 4
        const int64_t off = e - cptr[c];
        const int j = (int)(off / kC), k = (int)(off % kC);
        lcol[(c * kC + k) * lts + (j == 0 ? lts - 4 : j - 1)] = (uint16_t)max(row, 0);
      } else {
        lcol[e] = (uint16_t)max(row, 0);
      }
    }
  }
}

int grid_for(int64_t n, int block) {
  const int64_t g = (n + block - 1) / block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

}  // namespace

cudaError_t launch_build_bc(const int64_t* cptr, const int* nruns, const int* runs, const int* scol,
                            const int64_t* list, int64_t n_chunks, int grid, int R, bool with_w,
                            const TileLayout& tl, uint4* rec, int* map, uint16_t* lcol_bc, int* fail,
                            cudaStream_t s) {
  bc_plan_kernel<<<(grid + 63) / 64, 64, 0, s>>>(cptr, nruns, runs, list, n_chunks, grid, R, with_w ? 1 : 0, tl, rec,
                                                  map, fail);
  bc_lcol_kernel<<<grid_for(n_chunks * 32, 256), 256, 0, s>>>(scol, cptr, list, n_chunks, map, lcol_bc, fail,
                                                               tl.lt_stride, R);
  return cudaGetLastError();
}

cudaError_t launch_build_records(const int64_t* cptr, const int* nruns, const int* runs, int64_t n_chunks, int R,
                                 int off_w, int off_val, int off_lcol, uint4* rec, cudaStream_t s) {
  build_records_kernel<<<grid_for(n_chunks, 256), 256, 0, s>>>(cptr, nruns, runs, n_chunks, R, off_w, off_val, off_lcol,
                                                               rec);
  return cudaGetLastError();
}

#define DB_CUDA(call)                                         \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) {                                  \
      err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      return 5;                                               \
    }                                                         \
  } while (0)

int build_sell_device(const int64_t* rp, const int64_t* col, const double2* val, int64_t n_loc, int64_t row_begin,
                      int64_t row_end, int64_t n_global, DevSell& d, DeviceBuild& out, BuildScratch& ws,
                      std::string& err, cudaStream_t s) {
  out = DeviceBuild();
  int* flags = nullptr;
  DB_CUDA(ws.get(BuildScratch::kFlags, 1, &flags));
  DB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), s));
  validate_kernel<<<grid_for(n_loc, 256), 256, 0, s>>>(rp, col, val, n_loc, n_global, flags);
  DB_CUDA(cudaGetLastError());
  int64_t rp0 = 0, nnz = 0;
  DB_CUDA(cudaMemcpyAsync(&rp0, rp, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DB_CUDA(cudaMemcpyAsync(&nnz, rp + n_loc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  int hflags = 0;
  DB_CUDA(cudaMemcpyAsync(&hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  DB_CUDA(cudaStreamSynchronize(s));
  if (rp0 != 0 || (hflags & 1)) {
    err = "malformed row_ptr";
    return 1;
  }
  if (hflags & 2) {
    err = "column outside [0, n_global)";
    return 3;
  }
  if (hflags & 4) {
    err = "non-finite value";
    return 1;
  }
  const int64_t n_chunks = (n_loc + kC - 1) / kC, n_pad = n_chunks * kC;
  d.n_loc = n_loc;
  d.n_pad = n_pad;
  d.n_chunks = n_chunks;

  // chunk widths, cptr
  int64_t *w = nullptr, *slots = nullptr;
  DB_CUDA(ws.get(BuildScratch::kWidth, n_chunks, &w));
  DB_CUDA(ws.get(BuildScratch::kSlots, n_chunks, &slots));
  DB_CUDA(reserve((void**)&d.cptr, &d.cptr_cap, sizeof(int64_t) * (n_chunks + 1)));
  width_kernel<<<grid_for(n_chunks, 256), 256, 0, s>>>(rp, n_loc, n_chunks, w, slots);
  DB_CUDA(cudaGetLastError());
  DB_CUDA(cudaMemsetAsync(d.cptr, 0, sizeof(int64_t), s));
  unsigned char* tmp = nullptr;
  size_t need = 0;
  auto ensure_tmp = [&](size_t b) -> cudaError_t { return ws.get(BuildScratch::kTmp, b, &tmp); };
  DB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, need, slots, d.cptr + 1, n_chunks, s));
  DB_CUDA(ensure_tmp(need));
  DB_CUDA(cub::DeviceScan::InclusiveSum(tmp, need, slots, d.cptr + 1, n_chunks, s));
  int64_t* maxw = nullptr;
  DB_CUDA(ws.get(BuildScratch::kMaxW, 1, &maxw));
  DB_CUDA(cub::DeviceReduce::Max(nullptr, need, w, maxw, n_chunks, s));
  DB_CUDA(ensure_tmp(need));
  DB_CUDA(cub::DeviceReduce::Max(tmp, need, w, maxw, n_chunks, s));
  DB_CUDA(cudaMemcpyAsync(&d.max_width, maxw, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DB_CUDA(cudaMemcpyAsync(&d.n_slots, d.cptr + n_chunks, sizeof(int64_t), cudaMemcpyDeviceToHost, s));

  // halo: distinct remote columns, ascending (selected on the device in pieces, sorted on
  // the host: a slab's remote entries are its boundary planes, a small fraction of nnz)
  int64_t* halo = nullptr;
  int64_t n_halo = 0;
  {
    const int64_t piece = std::min<int64_t>(std::max<int64_t>(nnz, 1), (int64_t)1 << 26);
    int64_t *sel = nullptr, *nsel = nullptr;
    DB_CUDA(ws.get(BuildScratch::kSel, piece, &sel));
    DB_CUDA(ws.get(BuildScratch::kNsel, 1, &nsel));
    const IsRemote pred{row_begin, row_end};
    std::vector<int64_t> acc;
    for (int64_t b0 = 0; b0 < nnz; b0 += piece) {
      const int64_t len = std::min(piece, nnz - b0);
      size_t nb = 0;
      DB_CUDA(cub::DeviceSelect::If(nullptr, nb, col + b0, sel, nsel, len, pred, s));
      DB_CUDA(ensure_tmp(nb));
      DB_CUDA(cub::DeviceSelect::If(tmp, nb, col + b0, sel, nsel, len, pred, s));
      int64_t k = 0;
      DB_CUDA(cudaMemcpyAsync(&k, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      DB_CUDA(cudaStreamSynchronize(s));
      if (k) {
        const size_t o = acc.size();
        acc.resize(o + k);
        DB_CUDA(cudaMemcpy(acc.data() + o, sel, sizeof(int64_t) * k, cudaMemcpyDeviceToHost));
      }
    }
    std::sort(acc.begin(), acc.end());
    acc.erase(std::unique(acc.begin(), acc.end()), acc.end());
    out.halo = acc;
    n_halo = (int64_t)out.halo.size();
    DB_CUDA(ws.get(BuildScratch::kHalo, n_halo, &halo));
    if (n_halo) DB_CUDA(cudaMemcpyAsync(halo, out.halo.data(), sizeof(int64_t) * n_halo, cudaMemcpyHostToDevice, s));
  }
  d.n_halo = n_halo;
  if (n_pad + n_halo > (int64_t)INT32_MAX) {
    err = "local rows + halo rows exceed the int32 kernel index range";
    return 3;
  }
  DB_CUDA(cudaStreamSynchronize(s));

  // scatter
  DB_CUDA(reserve((void**)&d.val, &d.val_cap, sizeof(double2) * d.n_slots));
  DB_CUDA(reserve((void**)&d.col, &d.col_cap, sizeof(int) * d.n_slots));
  scatter_kernel<<<grid_for(n_chunks * 32, 256), 256, 0, s>>>(rp, col, val, n_loc, n_chunks, row_begin, row_end,
                                                               n_pad, halo, n_halo, d.cptr, d.val, d.col);
  DB_CUDA(cudaGetLastError());

  // tile plan
  DB_CUDA(reserve((void**)&d.lcol, &d.lcol_cap, sizeof(uint16_t) * d.n_slots));
  DB_CUDA(reserve((void**)&d.nruns, &d.nruns_cap, sizeof(int) * n_chunks));
  DB_CUDA(reserve((void**)&d.runs, &d.runs_cap, sizeof(int) * 2 * kMaxRuns * n_chunks));
  int* nother = nullptr;
  DB_CUDA(ws.get(BuildScratch::kNother, n_chunks, &nother));
  DB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), s));
  tiles_kernel<<<(int)std::min<int64_t>(n_chunks, 148 * 16), 256, 0, s>>>(d.col, d.cptr, n_chunks, d.lcol, d.nruns,
                                                                          d.runs, nother, flags);
  DB_CUDA(cudaGetLastError());
  int* maxo = nullptr;
  DB_CUDA(ws.get(BuildScratch::kMaxO, 1, &maxo));
  DB_CUDA(cub::DeviceReduce::Max(nullptr, need, nother, maxo, n_chunks, s));
  DB_CUDA(ensure_tmp(need));
  DB_CUDA(cub::DeviceReduce::Max(tmp, need, nother, maxo, n_chunks, s));
  int hmaxo = 0;
  DB_CUDA(cudaMemcpyAsync(&hmaxo, maxo, sizeof(int), cudaMemcpyDeviceToHost, s));
  DB_CUDA(cudaMemcpyAsync(&hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  // per-chunk "reads a halo slot" flags and the host copy of cptr (multi-rank planning)
  out.cptr.resize(n_chunks + 1);
  DB_CUDA(cudaMemcpyAsync(out.cptr.data(), d.cptr, sizeof(int64_t) * (n_chunks + 1), cudaMemcpyDeviceToHost, s));
  if (n_halo) {
    char* rh = nullptr;
    DB_CUDA(ws.get(BuildScratch::kReadsHalo, n_chunks, &rh));
    reads_halo_kernel<<<grid_for(n_chunks * 32, 256), 256, 0, s>>>(d.col, d.cptr, n_chunks, n_pad, rh);
    DB_CUDA(cudaGetLastError());
    out.reads_halo.resize(n_chunks);
    DB_CUDA(cudaMemcpyAsync(out.reads_halo.data(), rh, n_chunks, cudaMemcpyDeviceToHost, s));
    DB_CUDA(cudaStreamSynchronize(s));
  }
  DB_CUDA(cudaStreamSynchronize(s));
  d.max_other = hmaxo;
  d.tiles_ok = (hflags & (8 | 16)) == 0;
  return 0;
}

}  // namespace kpm
