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

#include <algorithm>

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
                               int64_t n_loc, int64_t n_pad, const int64_t* __restrict__ halo_rows, int64_t n_total,
                               int R, int64_t row_begin, int64_t col_begin, int r_valid, uint64_t seed) {
  const int64_t n_el = n_total * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / R;
    const int r = (int)(e - p * R);
    double2 v = make_double2(0.0, 0.0);
    if (r < r_valid && (p < n_loc || p >= n_pad)) {
      const int64_t row = p < n_loc ? row_begin + (perm ? (int64_t)perm[p] : p) : halo_rows[p - n_pad];
      v = z4_phase(seed, (uint64_t)row, (uint32_t)(col_begin + r));
    }
    V[e] = v;
    // W's halo slots are left alone: with the fused exchange the neighbours' init sweep may
    // already be storing nu_1 into them.
    if (p < n_pad) W[e] = make_double2(0.0, 0.0);
  }
}

__global__ void v0_permute_kernel(double2* __restrict__ V, double2* __restrict__ W, const double2* __restrict__ v0,
                                  const int* __restrict__ perm, int64_t n_loc, int64_t n_pad, int64_t n_total, int R,
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
    if (p < n_pad) W[e] = make_double2(0.0, 0.0);  // halo slots: see z4_init_kernel
  }
}

// ------------------------------------------------------------- memory helpers ------
// Matrix entries and the old W are streamed once per sweep: bypass L1 and mark them
// evict-first in L2 so that L1/L2 keep the gathered V rows.
// Gathered V rows are reused across ~2 x-planes of the sweep (the x-neighbour window, 65 MB
// at C4, R = 32): keep them in L2 ahead of the streamed matrix / W lines.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
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
  // no "memory" clobber: nothing in a sweep reads back a W row it stored (the old W rows are read
  // before, by the TMA fill of the same tile), and the clobber made the compiler reload every
  // kernel parameter after each store
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(ptr), "d"(v.x), "d"(v.y),
               "l"(pol));
}

// Fused halo exchange: a boundary row's new value also goes straight into the neighbour's
// halo slot (peer memory over NVLink); made visible by the stream-ordered system-scope
// fence of the flag write that follows the launch (kpm_abi.cu).
template <int R>
__device__ __forceinline__ void store_peers(const SweepArgs& a, int64_t p, int col, double2 w) {
  for (int i = 0; i < a.n_peer; ++i) {
    const PeerRun& pr = a.peer[i];
    if (p >= pr.pos && p < pr.pos + pr.count) pr.dst[(p - pr.pos) * R + col] = w;
  }
}

// u += h * x  (complex multiply-add, 4 DFMA)
__device__ __forceinline__ void cmac(double2& u, const double2 h, const double2 x) {
  u.x = fma(h.x, x.x, u.x);
  u.x = fma(-h.y, x.y, u.x);
  u.y = fma(h.x, x.y, u.y);
  u.y = fma(h.y, x.x, u.y);
}


// ------------------------------------------------------------------ aug_spmmv ------
// Thread mapping: a warp owns a row group of RW = 32/LPR
// consecutive SELL positions inside one chunk; lane = (q, t): q = row in the group,
// t = lane in the row.  Lane t of row q handles block columns r = cc*LPR + t, cc < CPL,
// so every gathered V row segment is LPR*16 contiguous bytes (a full 128-B line for
// LPR >= 8) and each SELL sub-column read of val/col serves RW rows.
//
// Two matrix feeds:
//   direct  -- val/col loaded from global (L1 bypass, L2 evict-first); used for R <= 4.
//   staged  -- one chunk (32 rows) per CTA tile; an elected thread streams the chunk's
//              val/col block into a 4-stage shared-memory ring with cp.async.bulk (TMA
//              bulk copy, mbarrier complete_tx), so the only latency left on the
//              critical path is the V gather.  Used when every chunk fits a stage
//              (width <= kLcap); otherwise the host selects the direct feed.

constexpr int kStages = 4;
constexpr int kLcap = 16;                                  // max chunk width staged
constexpr int kStageValBytes = kC * kLcap * 16;            // 8 KB
constexpr int kStageColBytes = kC * kLcap * 4;             // 2 KB
constexpr int kStageBytes = kStageValBytes + kStageColBytes;
constexpr int kStagedSmem = kStages * kStageBytes;         // 40 KB dynamic

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}


// i-th chunk of the launch's work list (a contiguous range, or a host-built list such as the
// edge / interior chunks of the multi-GPU split).
__device__ __forceinline__ int64_t chunk_at(const SweepArgs& a, int64_t i) {
  return a.chunk_list ? __ldg(a.chunk_list + a.chunk_begin + i) : a.chunk_begin + i;
}

template <int R, int LPR, int U>
struct Cfg {
  static_assert(R % LPR == 0 && 32 % LPR == 0, "bad lane mapping");
  static constexpr int CPL = R / LPR;  // block columns per lane
  static constexpr int RW = 32 / LPR;  // rows per warp (row group)
};

// Accumulators of the fused dot products of one lane: sum |V|^2, sum conj(W) V.
template <int CPL>
struct Dots {
  double ee[CPL], eor[CPL], eoi[CPL];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) ee[cc] = eor[cc] = eoi[cc] = 0.0;
  }
};

// One row group: u = sum_j H_pj V_j over the chunk's L entries (stored order), then
// the shift/scale/-W epilogue and the fused dot products (Fig. 5 "&" chain).
// vp/cp point at entry 0 of this lane's row (stride 32 between entries).
template <int R, int LPR, int U, bool INIT, bool SMEM>
__device__ __forceinline__ void row_group(const SweepArgs& a, const double2* vp, const int* cp, int L, int64_t p,
                                          int t, uint64_t pol, Dots<R / LPR>& d) {
  using Cf = Cfg<R, LPR, U>;
  constexpr int CPL = Cf::CPL;
  const bool live = p < a.n_loc;
  double2 wo[CPL];
  if (!INIT && live) {  // old W is streamed from HBM: issue it first so it lands under the gathers
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) wo[cc] = ld_stream(a.W + p * R + cc * LPR + t, pol);
  }
  double2 u[CPL];
#pragma unroll
  for (int cc = 0; cc < CPL; ++cc) u[cc] = make_double2(0.0, 0.0);
  const double2* Vt = a.V + t;
  for (int j = 0; j < L; j += U) {
    const int nb = min(U, L - j);
    double2 h[U];
    int cj[U];
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      if (uu < nb) {
        if (SMEM) {
          h[uu] = vp[(j + uu) * kC];
          cj[uu] = cp[(j + uu) * kC];
        } else {
          h[uu] = ld_stream_nc(vp + (j + uu) * kC, pol);
          cj[uu] = ld_stream_nc(cp + (j + uu) * kC, pol);
        }
      }
    }
    double2 x[U][CPL];
#pragma unroll
    for (int uu = 0; uu < U; ++uu)
      if (uu < nb)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) x[uu][cc] = __ldg(Vt + (int64_t)cj[uu] * R + cc * LPR);
#pragma unroll
    for (int uu = 0; uu < U; ++uu)
      if (uu < nb)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) cmac(u[cc], h[uu], x[uu][cc]);
  }
  if (live) {
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
      const int64_t e = p * R + cc * LPR + t;
      const double2 vi = __ldg(a.V + e);
      double2 uu = u[cc];
      uu.x = fma(-a.b, vi.x, uu.x);
      uu.y = fma(-a.b, vi.y, uu.y);
      double2 w;
      if (INIT)
        w = make_double2(a.scale * uu.x, a.scale * uu.y);
      else
        w = make_double2(fma(a.scale, uu.x, -wo[cc].x), fma(a.scale, uu.y, -wo[cc].y));
      st_stream(a.W + e, w, pol);
      store_peers<R>(a, p, cc * LPR + t, w);
      d.ee[cc] = fma(vi.x, vi.x, fma(vi.y, vi.y, d.ee[cc]));
      // conj(w) * v = (wr vr + wi vi) + i (wr vi - wi vr)
      d.eor[cc] = fma(w.x, vi.x, fma(w.y, vi.y, d.eor[cc]));
      d.eoi[cc] = fma(w.x, vi.y, fma(-w.y, vi.x, d.eoi[cc]));
    }
  }
}

// Warp shuffles over the rows of a warp, then a fixed-order CTA sum -> partials.
template <int R, int LPR>
__device__ __forceinline__ void cta_reduce(const SweepArgs& a, Dots<R / LPR>& d, double* red /* [8][3R] */) {
  constexpr int CPL = R / LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
      d.ee[cc] += __shfl_xor_sync(0xffffffffu, d.ee[cc], off);
      d.eor[cc] += __shfl_xor_sync(0xffffffffu, d.eor[cc], off);
      d.eoi[cc] += __shfl_xor_sync(0xffffffffu, d.eoi[cc], off);
    }
  }
  if (lane < LPR) {
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
      const int r = cc * LPR + lane;
      red[warp * 3 * R + r] = d.ee[cc];
      red[warp * 3 * R + R + r] = d.eor[cc];
      red[warp * 3 * R + 2 * R + r] = d.eoi[cc];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * R; i += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) s += red[w * 3 * R + i];
    a.partials[(int64_t)i * a.pstride + blockIdx.x] = s;
  }
}

// Direct feed: grid-stride over row groups.
template <int R, int LPR, int U, bool INIT>
__global__ void __launch_bounds__(kThreads) aug_spmmv_direct(const SweepArgs a) {
  using Cf = Cfg<R, LPR, U>;
  constexpr int RW = Cf::RW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane / LPR, t = lane - q * LPR;
  const uint64_t pol = policy_evict_first();
  Dots<Cf::CPL> d;
  d.zero();
  constexpr int G = kC / RW;
  const int64_t g1 = (a.chunk_end - a.chunk_begin) * G;
  for (int64_t g = blockIdx.x * (int64_t)(kThreads / 32) + warp; g < g1; g += (int64_t)gridDim.x * (kThreads / 32)) {
    const int64_t c = chunk_at(a, g / G);
    const int k = (int)((g % G) * RW) + q;
    const int64_t p = c * kC + k;
    const int64_t s0 = __ldg(a.cptr + c);
    const int L = (int)((__ldg(a.cptr + c + 1) - s0) >> 5);
    row_group<R, LPR, U, INIT, false>(a, a.val + s0 + k, a.col + s0 + k, L, p, t, pol, d);
  }
  __shared__ double red[(kThreads / 32) * 3 * R];
  cta_reduce<R, LPR>(a, d, red);
}

// Staged feed: grid-stride over chunks, TMA bulk copies into a kStages-deep ring.
template <int R, int LPR, int U, bool INIT>
__global__ void __launch_bounds__(kThreads, 2) aug_spmmv_staged(const SweepArgs a) {
  using Cf = Cfg<R, LPR, U>;
  constexpr int RW = Cf::RW, G = kC / RW;  // row groups per chunk
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ double red[(kThreads / 32) * 3 * R];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane / LPR, t = lane - q * LPR;
  const uint64_t pol = policy_evict_first();
  const int64_t n_chunks = a.chunk_end - a.chunk_begin;
  const int64_t my_tiles = n_chunks > blockIdx.x ? (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  auto issue = [&](int64_t k) {  // producer: stage tile k (one elected thread)
    const int s = (int)(k % kStages);
    const int64_t c = chunk_at(a, blockIdx.x + k * gridDim.x);
    const int64_t s0 = a.cptr[c];
    const int L = (int)((a.cptr[c + 1] - s0) >> 5);
    const uint32_t bar = smem_u32(&full[s]);
    const uint32_t vb = (uint32_t)(kC * L * 16), cb = (uint32_t)(kC * L * 4);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(bar, vb + cb);
    if (vb) {
      bulk_g2s(smem_u32(ring + s * kStageBytes), a.val + s0, vb, bar, pol);
      bulk_g2s(smem_u32(ring + s * kStageBytes + kStageValBytes), a.col + s0, cb, bar, pol);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(smem_u32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int64_t k = 0; k < kStages && k < my_tiles; ++k) issue(k);

  Dots<Cf::CPL> d;
  d.zero();
  for (int64_t k = 0; k < my_tiles; ++k) {
    const int s = (int)(k % kStages);
    const int64_t c = chunk_at(a, blockIdx.x + k * gridDim.x);
    const int L = (int)((__ldg(a.cptr + c + 1) - __ldg(a.cptr + c)) >> 5);
    mbar_wait(smem_u32(&full[s]), (uint32_t)((k / kStages) & 1));
    const double2* sv = reinterpret_cast<const double2*>(ring + s * kStageBytes);
    const int* sc = reinterpret_cast<const int*>(ring + s * kStageBytes + kStageValBytes);
    for (int gq = warp; gq < G; gq += kThreads / 32) {
      const int kr = gq * RW + q;
      row_group<R, LPR, U, INIT, true>(a, sv + kr, sc + kr, L, c * kC + kr, t, pol, d);
    }
    __syncthreads();  // stage s consumed by every warp
    if (tid == 0 && k + kStages < my_tiles) issue(k + kStages);
  }
  cta_reduce<R, LPR>(a, d, red);
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

// ------------------------------------------------------------- tiled feed --------
// One chunk (32 rows) per CTA tile.  Warp 0 streams the whole working set of the tile into
// a shared-memory ring with cp.async.bulk (TMA bulk copies, one mbarrier per stage):
//   [V rows of the tile: own 32 rows | the chunk's other distinct columns, as runs]
//   [W of the 32 own rows (main sweep)] [val block] [lcol block (uint16 tile-row index)]
// so every gathered V row is fetched from L2/HBM once per chunk and no gather occupies a
// register while in flight.  All warps then compute from shared memory.
constexpr int kMaxTileStages = 4;
enum SweepKind { kAug = 0, kAugNoDot = 1, kSpmmv = 2 };  // = KPM_SWEEP_* in kpm.h
constexpr int kTileBudget = 232448 - 8192;  // minus static smem (reduction buffer, barriers)  // 227 KB dynamic shared memory minus margin

// CS = column split: CS consumer warps share a row group, each owning CPL/CS of the lane's
// block columns (more warps in flight for the same registers; val/lcol reads repeat CS times).
// Consumer warps per column part: one per row group of a chunk, at most 8 (so R < 8 uses
// small CTAs: G = LPR row groups of 32/LPR rows each).
template <int LPR>
__host__ __device__ constexpr int tiled_ncwg() { return LPR < 8 ? LPR : (LPR == 16 ? 16 : 8); }
template <int LPR, int CS>
__host__ __device__ constexpr int tiled_threads() { return 32 * (tiled_ncwg<LPR>() * CS + 1); }

// WS: the old W rows travel in the tile (TMA) or, WS = false, straight into registers (LDG,
// streaming) -- a smaller stage, so more CTAs fit per SM.
// KIND: the paper's three kernels of the bottleneck analysis (Fig. 9):
//   kAug       the fully augmented SpMMV of Fig. 5 (the hot path),
//   kAugNoDot  the same without the on-the-fly dot products,
//   kSpmmv     the plain SpMMV W = H V (no shift/scale, no old W).
// MINB: CTAs per SM the register allocation must leave room for (2 for the variants whose
// smaller ring is meant to fit two CTAs per SM).
// BC: block-cache feed: records per list position, V rows of a tile live in a
// pool of 32-row blocks kept across the CTA's tiles (plus per-stage extra rows), lcol holds
// absolute shared-memory V rows (times R), the header carries the own block's first row.
template <int R, int LPR, int U, int CS, bool WS, bool INIT, int KIND = kAug, int MINB = 1, bool BC = false>
__global__ void __launch_bounds__(tiled_threads<LPR, CS>(), MINB) aug_spmmv_tiled(const SweepArgs a) {
  using Cf = Cfg<R, LPR, U>;
  constexpr int RW = Cf::RW, G = kC / RW;
  static_assert(Cf::CPL % CS == 0, "column split must divide the columns per lane");
  constexpr int CPL = Cf::CPL / CS;       // block columns per lane in this warp
  constexpr int NCWG = tiled_ncwg<LPR>(); // consumer warps per column part
  constexpr int NCW = NCWG * CS;          // consumer warps
  constexpr int kTiledThreads = tiled_threads<LPR, CS>();
  constexpr bool NEED_W = !INIT && KIND != kSpmmv;  // the recurrence's "- W" term
  constexpr bool W_TILE = NEED_W && WS;             // old W rows staged in the tile
  extern __shared__ __align__(128) unsigned char tsm[];
  __shared__ __align__(8) uint64_t full[kMaxTileStages], empty[kMaxTileStages];
  __shared__ int tile_len[kMaxTileStages], tile_own[kMaxTileStages];
  __shared__ int64_t tile_chunk[kMaxTileStages];
  __shared__ double red[NCWG * 3 * R];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const TileLayout tl = a.tl;
  const int64_t n_chunks = a.chunk_end - a.chunk_begin;
  const int64_t my_tiles = n_chunks > blockIdx.x ? (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint64_t pol = policy_evict_first();

  if (tid == 0) {
    for (int s = 0; s < tl.stages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  Dots<CPL> d;
  d.zero();
  const uint32_t full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);  // barrier s at +8 s
  if (warp == NCW) {
    // ---------------- producer warp: TMA bulk copies of tile k into stage k % S ----------
    // Lane i < 16 holds slot i of the chunk's copy record (header + up to 15 bulk copies);
    // the record of tile k+1 is loaded while tile k is issued, so no metadata load sits on
    // the producer's critical path.
    const uint64_t pol_v = a.v_evict_last ? policy_evict_last() : 0ull;
    int64_t c_nxt = my_tiles > 0 ? chunk_at(a, blockIdx.x) : 0;
    uint4 nxt = my_tiles > 0 && lane < 16 ? __ldg(a.rec + (BC ? (int64_t)blockIdx.x : c_nxt) * 16 + lane)
                                          : make_uint4(0u, 0u, 0u, 0u);
    // ring stage s = k mod S and its round r = k div S, kept incrementally (a runtime 64-bit
    // division per tile cost ~27 instructions per warp and tile)
    int s = 0;
    uint32_t rnd = 0;
    for (int64_t k = 0; k < my_tiles; ++k, s = (s + 1 == tl.stages) ? 0 : s + 1, rnd += (s == 0)) {
      const uint4 cur = nxt;
      const int64_t c_cur = c_nxt;
      if (k + 1 < my_tiles) {
        c_nxt = chunk_at(a, blockIdx.x + (k + 1) * gridDim.x);
        const int64_t ri = BC ? blockIdx.x + (k + 1) * gridDim.x : c_nxt;
        nxt = lane < 16 ? __ldg(a.rec + ri * 16 + lane) : make_uint4(0u, 0u, 0u, 0u);
      }
      const uint32_t total = __shfl_sync(0xffffffffu, W_TILE ? cur.x : cur.y, 0);
      const uint32_t L = __shfl_sync(0xffffffffu, cur.z, 0);
      const uint32_t hw = __shfl_sync(0xffffffffu, cur.w, 0);
      const uint32_t ncmd = BC ? (hw & 0xFFu) : hw;
      if (rnd > 0) mbar_wait(empty0 + 8 * s, (rnd - 1) & 1u);
      unsigned char* st = BC ? tsm : tsm + (size_t)s * tl.stage_bytes;  // BC records: absolute offsets
      const uint32_t bar = full0 + 8 * s;
      if (lane == 0) {
        tile_len[s] = (int)L;
        tile_own[s] = BC ? (int)(hw >> 8) : 0;
        tile_chunk[s] = c_cur;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(bar, total);
      }
      __syncwarp();
      if (lane >= 1 && (uint32_t)lane <= ncmd) {
        const uint32_t base = cur.w >> 28, bytes = cur.w & 0x0FFFFFFFu;
        const int64_t off = (int64_t)(((uint64_t)cur.y << 32) | cur.x);
        if (W_TILE || base != 1) {
          const unsigned char* src = base == 0   ? reinterpret_cast<const unsigned char*>(a.V)
                                     : base == 1 ? reinterpret_cast<const unsigned char*>(a.W)
                                     : base == 2 ? reinterpret_cast<const unsigned char*>(a.val)
                                                 : reinterpret_cast<const unsigned char*>(a.lcol);
          bulk_g2s(smem_u32(st + cur.z), src + off, bytes, bar, base == 0 ? pol_v : pol);
        }
      }
    }
  } else {
    // ---------------- consumer warps ---------------------------------------------------
    const int q = lane / LPR;
    const int g0 = warp % NCWG, part = warp / NCWG;
    const int t = lane - q * LPR + part * CPL * LPR;  // first block column of this lane
    // Bank-conflict swizzle for LPR < 8: the 8 lanes of one shared-memory phase span 8/LPR
    // rows whose LPR*16-byte segments would sit on the same banks; row q visits its column
    // blocks in the order cc ^ (q mod 8/LPR), so the rows of a phase cover one 128-B window.
    constexpr int SWR = (LPR < 8 && CPL * LPR >= 8) ? 8 / LPR : 1;
    const int sw = q % SWR;
    const bool peers = a.n_peer > 0;  // fused halo stores of this launch (edge chunks only)
    int s = 0;
    uint32_t rnd = 0;
    for (int64_t k = 0; k < my_tiles; ++k, s = (s + 1 == tl.stages) ? 0 : s + 1, rnd += (s == 0)) {
      const unsigned char* st = tsm + (size_t)tl.pool_bytes + (size_t)s * tl.stage_bytes;
      const double2* sV = reinterpret_cast<const double2*>(BC ? tsm : st);
      const double2* sW = reinterpret_cast<const double2*>(st + tl.off_w);
      const double2* sval = reinterpret_cast<const double2*>(st + tl.off_val);
      const uint16_t* slc = reinterpret_cast<const uint16_t*>(st + tl.off_lcol);
      mbar_wait(full0 + 8 * s, rnd & 1u);
      const int L = tile_len[s];
      const int own_row = tile_own[s];  // 0 unless BC
      const int64_t c = tile_chunk[s];
      for (int gq = g0; gq < G; gq += NCWG) {
        const int kr = gq * RW + q;
        const int64_t p = c * kC + kr;
        double2 wreg[CPL];
        if (NEED_W && !WS && p < a.n_loc) {  // old W straight from HBM, lands under the gathers
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) wreg[cc] = ld_stream(a.W + p * R + (cc ^ sw) * LPR + t, pol);
        }
        double2 u[CPL];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) u[cc] = make_double2(0.0, 0.0);
        const double2* sv = sval + kr;
        const int lts = BC ? tl.lt_stride : 0;  // row-major tile indices (TileLayout::lt_stride)
        // RMC: the row-major tile-index path fixed at compile time (block-cache kernels without a
        // multi-CTA register cap: -2 % at R = 32; at R = 16 the runtime test measured faster)
        constexpr bool RMC = BC && MINB == 1;
        const uint16_t* sl = (RMC || lts) ? slc + kr * lts : slc + kr;
        constexpr int LM = BC ? 1 : R;  // block-cache tile indices are stored pre-multiplied by R
        const double2* sVt = sV + t;
        // gather address = this lane's base + 16 * index (one IMAD per gathered row; written this way
        // the compiler stops folding t into every index)
        const uint32_t vbase = smem_u32(sVt);
        auto vat = [&](int li, int cc) -> double2 {
          double2 r;
          asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y)
                       : "r"(vbase + (uint32_t)(li + (cc ^ sw) * LPR) * 16u));
          return r;
        };
        int j = 0;
        // The SELL order puts a row's own-position (diagonal) entry first, if stored (DESIGN.md
        // R18): then entry 0's gather is the own row V_i, which the epilogue needs as well, so
        // it is kept in registers instead of being read from shared memory a second time.
        // (Only without a multi-CTA register cap: there x0's live range costs more than the
        // saved read, measured at R = 8 and 16; entry 0 is still peeled, keeping the batches
        // of the TI's 13-entry rows full.)
        constexpr bool PEEL = MINB == 1;
        double2 x0[CPL];
        int li0 = -1;
        if (L > 0) {  // uniform per tile
          const double2 h0 = sv[0];
          li0 = ((RMC || lts) ? sl[lts - 4] : sl[0]) * LM;
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) {
            x0[cc] = vat(li0, cc);
            cmac(u[cc], h0, x0[cc]);
          }
          j = 1;
        }
        if (PEEL && li0 != (own_row + kr) * R) {  // entry 0 is not the diagonal: x0 <- V_i
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) x0[cc] = sV[(own_row + kr) * R + (cc ^ sw) * LPR + t];
        }
        for (; j + U <= L; j += U) {  // full batches: no predication
          double2 h[U];
          int li[U];
#pragma unroll
          for (int uu = 0; uu < U; ++uu) h[uu] = sv[(j + uu) * kC];
          if (U == 4 && (RMC || (lts && ((j - 1) & 3) == 0))) {  // one 8-byte load: entries j..j+3
            const uint2 q4 = *reinterpret_cast<const uint2*>(sl + (j - 1));
            li[0] = (int)(q4.x & 0xFFFFu) * LM;
            li[1 % U] = (int)(q4.x >> 16) * LM;
            li[2 % U] = (int)(q4.y & 0xFFFFu) * LM;
            li[3 % U] = (int)(q4.y >> 16) * LM;
          } else {
#pragma unroll
            for (int uu = 0; uu < U; ++uu) li[uu] = ((RMC || lts) ? sl[j + uu - 1] : sl[(j + uu) * kC]) * LM;
          }
          double2 x[U][CPL];
#pragma unroll
          for (int uu = 0; uu < U; ++uu)
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) x[uu][cc] = vat(li[uu], cc);
#pragma unroll
          for (int uu = 0; uu < U; ++uu)
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) cmac(u[cc], h[uu], x[uu][cc]);
        }
        for (; j < L; ++j) {
          const double2 h = sv[j * kC];
          const int li = ((RMC || lts) ? sl[j - 1] : sl[j * kC]) * LM;
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) cmac(u[cc], h, vat(li, cc));
        }
        if (p < a.n_loc) {
          double2* const wrow = a.W + p * R;
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) {
            const int col = (cc ^ sw) * LPR + t;
            if (KIND == kSpmmv) {
              st_stream(wrow + col, u[cc], pol);
              continue;
            }
            const double2 vi_c = PEEL ? x0[cc] : sV[(own_row + kr) * R + col];
            double2 uu = u[cc];
            uu.x = fma(-a.b, vi_c.x, uu.x);
            uu.y = fma(-a.b, vi_c.y, uu.y);
            double2 w;
            if (INIT) {
              w = make_double2(a.scale * uu.x, a.scale * uu.y);
            } else {
              const double2 wo = WS ? sW[kr * R + col] : wreg[cc];
              w = make_double2(fma(a.scale, uu.x, -wo.x), fma(a.scale, uu.y, -wo.y));
            }
            st_stream(wrow + col, w, pol);
            if (peers) store_peers<R>(a, p, col, w);
            if (KIND == kAug) {
              d.ee[cc] = fma(vi_c.x, vi_c.x, fma(vi_c.y, vi_c.y, d.ee[cc]));
              d.eor[cc] = fma(w.x, vi_c.x, fma(w.y, vi_c.y, d.eor[cc]));
              d.eoi[cc] = fma(w.x, vi_c.y, fma(-w.y, vi_c.x, d.eoi[cc]));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s);  // stage s released by this warp
    }
    // undo the swizzle so that accumulator cc holds column block cc on every lane
    if (SWR > 1 && KIND == kAug) {
      Dots<CPL> e = d;
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
        for (int k2 = 0; k2 < CPL; ++k2)
          if ((k2 ^ sw) == cc) {
            d.ee[cc] = e.ee[k2];
            d.eor[cc] = e.eor[k2];
            d.eoi[cc] = e.eoi[k2];
          }
    }
    // warp-level part of the dot-product reduction
#pragma unroll
    for (int off = LPR; off < (KIND == kAug ? 32 : 0); off <<= 1) {
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        d.ee[cc] += __shfl_xor_sync(0xffffffffu, d.ee[cc], off);
        d.eor[cc] += __shfl_xor_sync(0xffffffffu, d.eor[cc], off);
        d.eoi[cc] += __shfl_xor_sync(0xffffffffu, d.eoi[cc], off);
      }
    }
    if (KIND == kAug && lane < LPR) {
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        const int r = cc * LPR + t;
        red[g0 * 3 * R + r] = d.ee[cc];
        red[g0 * 3 * R + R + r] = d.eor[cc];
        red[g0 * 3 * R + 2 * R + r] = d.eoi[cc];
      }
    }
  }
  if (KIND != kAug) return;
  __syncthreads();
  for (int i = tid; i < 3 * R; i += kTiledThreads) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < NCWG; ++w) sum += red[w * 3 * R + i];
    a.partials[(int64_t)i * a.pstride + blockIdx.x] = sum;
  }
}

enum Feed { kDirect = 0, kStaged = 1, kTiled = 2 };

template <int R, int LPR, int U, int FEED, int CS = 1, bool WS = true, int MINB = 1, bool BC = false>
struct Variant {
  static cudaError_t launch(bool init, const SweepArgs& a, int grid, cudaStream_t s) {
    if constexpr (FEED == kStaged) {
      if (init)
        aug_spmmv_staged<R, LPR, U, true><<<grid, kThreads, kStagedSmem, s>>>(a);
      else
        aug_spmmv_staged<R, LPR, U, false><<<grid, kThreads, kStagedSmem, s>>>(a);
    } else if constexpr (FEED == kTiled) {
      const int smem = a.tl.pool_bytes + a.tl.stages * a.tl.stage_bytes;
      auto k_init = aug_spmmv_tiled<R, LPR, U, CS, WS, true, kAug, MINB, BC>;
      auto k_main = aug_spmmv_tiled<R, LPR, U, CS, WS, false, kAug, MINB, BC>;
      cudaFuncSetAttribute(k_init, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_main, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      (init ? k_init : k_main)<<<grid, tiled_threads<LPR, CS>(), smem, s>>>(a);
    } else {
      if (init)
        aug_spmmv_direct<R, LPR, U, true><<<grid, kThreads, 0, s>>>(a);
      else
        aug_spmmv_direct<R, LPR, U, false><<<grid, kThreads, 0, s>>>(a);
    }
    return cudaGetLastError();
  }
  // Also loads both the init and the main kernel (CUDA 12 loads modules lazily, and a load can
  // synchronize the device: it must not happen inside the sweep loop, where another rank's stream
  // of the same process may wait on a flag this thread has yet to enqueue -- virtual ranks).
  static int occupancy(int dyn_smem) {
    int n = 0;
    cudaFuncAttributes fa;
    if constexpr (FEED == kStaged) {
      cudaFuncGetAttributes(&fa, aug_spmmv_staged<R, LPR, U, true>);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, aug_spmmv_staged<R, LPR, U, false>, kThreads, kStagedSmem);
    } else if constexpr (FEED == kTiled) {
      auto k_init = aug_spmmv_tiled<R, LPR, U, CS, WS, true, kAug, MINB, BC>;
      auto k_main = aug_spmmv_tiled<R, LPR, U, CS, WS, false, kAug, MINB, BC>;
      cudaFuncSetAttribute(k_init, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem);
      cudaFuncSetAttribute(k_main, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_main, tiled_threads<LPR, CS>(), dyn_smem);
    } else {
      cudaFuncGetAttributes(&fa, aug_spmmv_direct<R, LPR, U, true>);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, aug_spmmv_direct<R, LPR, U, false>, kThreads, 0);
    }
    return n;
  }
};

typedef cudaError_t (*LaunchFn)(bool, const SweepArgs&, int, cudaStream_t);
typedef int (*OccFn)(int);
struct Entry {
  int R;
  const char* name;
  int feed;
  bool wstage;
  LaunchFn launch;
  OccFn occ;
  int stages = 0;  // tiled feed: preferred ring depth (0 = plan_tiles default)
  int bc_ctas = 0;  // block-cache feed: CTAs per SM its shared-memory plan is sized for (0: not BC)
  int strip = 1;    // chunk-order width the library's line walk uses for it (chunk_order.cpp)
};
#define KPM_VARIANT(R, LPR, U, F, NAME) {R, NAME, F, true, Variant<R, LPR, U, F>::launch, Variant<R, LPR, U, F>::occupancy}
#define KPM_VARIANT_CS(R, LPR, U, CS, NAME) \
  {R, NAME, kTiled, true, Variant<R, LPR, U, kTiled, CS>::launch, Variant<R, LPR, U, kTiled, CS>::occupancy}
// S-deep ring, W via registers; registers capped so that the CTAs the smaller ring is meant
// for fit per SM (3 for R <= 8, 2 above)
#define KPM_VARIANT_WR_S(R, LPR, U, S, NAME)                                                                 \
  {R, NAME, kTiled, false, Variant<R, LPR, U, kTiled, 1, false, (R <= 8 ? 3 : 2)>::launch,                     \
   Variant<R, LPR, U, kTiled, 1, false, (R <= 8 ? 3 : 2)>::occupancy, S}
#define KPM_VARIANT_WR(R, LPR, U, NAME) \
  {R, NAME, kTiled, false, Variant<R, LPR, U, kTiled, 1, false>::launch, Variant<R, LPR, U, kTiled, 1, false>::occupancy}
// First entry of each width is the default (chosen from the B200 measurements in DESIGN.md); at
// R = 16 and 32 that is the block-cache feed (on one rank: one plan for the chunk order; on several
// ranks: one plan per edge / interior list).  Where its plan does not fit the matrix on some rank,
// every rank falls back together to the next variant in table order that fits (select_variant in
// kpm_abi.cu); the last entry of each width, the direct feed, always does.
const Entry kTable[] = {
    KPM_VARIANT(1, 1, 4, kTiled, "tiled.lpr1.u4"),
    KPM_VARIANT(1, 1, 4, kDirect, "direct.lpr1.u4"),
    KPM_VARIANT(1, 1, 8, kDirect, "direct.lpr1.u8"),
    KPM_VARIANT(2, 2, 4, kTiled, "tiled.lpr2.u4"),
    KPM_VARIANT(2, 2, 4, kDirect, "direct.lpr2.u4"),
    KPM_VARIANT(2, 2, 8, kDirect, "direct.lpr2.u8"),
    KPM_VARIANT_WR(4, 4, 4, "tiled.lpr4.u4.wr"),
    KPM_VARIANT(4, 4, 4, kTiled, "tiled.lpr4.u4"),
    KPM_VARIANT_WR_S(4, 4, 4, 2, "tiled.lpr4.u4.wr.s2"),
    KPM_VARIANT(4, 2, 4, kTiled, "tiled.lpr2.u4"),
    KPM_VARIANT(4, 4, 2, kTiled, "tiled.lpr4.u2"),
    KPM_VARIANT(4, 4, 4, kDirect, "direct.lpr4.u4"),
    KPM_VARIANT(4, 4, 8, kDirect, "direct.lpr4.u8"),
    KPM_VARIANT_WR_S(8, 4, 4, 2, "tiled.lpr4.u4.wr.s2"),
    // block cache at R = 8: -1.4 % power-capped, +3 % at full clock (profiles/r01_bc/bc8.jsonl)
    {8, "tiled.bc.lpr4.u4.wr", kTiled, false, Variant<8, 4, 4, kTiled, 1, false, 3, true>::launch,
     Variant<8, 4, 4, kTiled, 1, false, 3, true>::occupancy, 2, 3},
    KPM_VARIANT(8, 4, 4, kTiled, "tiled.lpr4.u4"),
    KPM_VARIANT(8, 8, 4, kTiled, "tiled.lpr8.u4"),
    KPM_VARIANT(8, 8, 4, kStaged, "staged.lpr8.u4"),
    KPM_VARIANT(8, 8, 4, kDirect, "direct.lpr8.u4"),
    // R = 16: 8 lanes per row, 2 block columns per lane, 2 CTAs per SM (18 warps): -7.5 % vs the
    // 4-lane map under the power cap (profiles/r02_variants/)
    {16, "tiled.bc.lpr8.u4.wr", kTiled, false, Variant<16, 8, 4, kTiled, 1, false, 2, true>::launch,
     Variant<16, 8, 4, kTiled, 1, false, 2, true>::occupancy, 2, 2},
    {16, "tiled.bc.lpr4.u4.wr", kTiled, false, Variant<16, 4, 4, kTiled, 1, false, 2, true>::launch,
     Variant<16, 4, 4, kTiled, 1, false, 2, true>::occupancy, 2, 2},
    KPM_VARIANT_WR_S(16, 4, 4, 2, "tiled.lpr4.u4.wr.s2"),
    KPM_VARIANT(16, 8, 4, kTiled, "tiled.lpr8.u4"),
    KPM_VARIANT(16, 4, 2, kTiled, "tiled.lpr4.u2"),
    KPM_VARIANT_WR(16, 8, 4, "tiled.lpr8.u4.wr"),
    KPM_VARIANT_WR(16, 4, 4, "tiled.lpr4.u4.wr"),
    KPM_VARIANT_WR_S(16, 8, 4, 2, "tiled.lpr8.u4.wr.s2"),
    KPM_VARIANT_CS(16, 8, 4, 2, "tiled.lpr8.u4.cs2"),
    KPM_VARIANT(16, 8, 4, kStaged, "staged.lpr8.u4"),
    KPM_VARIANT(16, 8, 4, kDirect, "direct.lpr8.u4"),
    // R = 32: walked in strips of two lines (-2 % under the power cap, profiles/r02_variants/)
    {32, "tiled.bc.lpr8.u4", kTiled, true, Variant<32, 8, 4, kTiled, 1, true, 1, true>::launch,
     Variant<32, 8, 4, kTiled, 1, true, 1, true>::occupancy, 2, 1, 2},
    KPM_VARIANT(32, 8, 4, kTiled, "tiled.lpr8.u4"),
    KPM_VARIANT_WR(32, 8, 4, "tiled.lpr8.u4.wr"),
    KPM_VARIANT_CS(32, 8, 4, 2, "tiled.lpr8.u4.cs2"),
    KPM_VARIANT(32, 8, 2, kTiled, "tiled.lpr8.u2"),
    KPM_VARIANT(32, 16, 4, kStaged, "staged.lpr16.u4"),
    KPM_VARIANT(32, 8, 2, kDirect, "direct.lpr8.u2"),
};

const Entry* find(int R, int variant) {
  int i = 0;
  for (const Entry& e : kTable)
    if (e.R == R && i++ == variant) return &e;
  return nullptr;
}

}  // namespace

int variant_count(int R) {
  int n = 0;
  for (const Entry& e : kTable) n += (e.R == R);
  return n;
}

const char* variant_name(int R, int variant) {
  const Entry* e = find(R, variant);
  return e ? e->name : nullptr;
}

bool variant_staged(int R, int variant) {
  const Entry* e = find(R, variant);
  return e && e->feed == kStaged;
}

bool variant_tiled(int R, int variant) {
  const Entry* e = find(R, variant);
  return e && e->feed == kTiled;
}

int variant_stages(int R, int variant) {
  const Entry* e = find(R, variant);
  return e ? e->stages : 0;
}

int base_variant(int R) {
  int i = 0;
  for (const Entry& e : kTable)
    if (e.R == R) {
      if (!e.bc_ctas) return i;
      ++i;
    }
  return 0;
}

int variant_strip(int R, int variant) {
  const Entry* e = find(R, variant);
  return e ? e->strip : 1;
}

int variant_bc(int R, int variant) {
  const Entry* e = find(R, variant);
  return e ? e->bc_ctas : 0;
}

bool variant_wstage(int R, int variant) {
  const Entry* e = find(R, variant);
  return e && e->wstage;
}

static int round128(int64_t b) { return (int)((b + 127) / 128 * 128); }

TileLayout plan_tiles(int R, int64_t max_other, int64_t max_width, int stages, bool with_w) {
  TileLayout tl;
  const int64_t v = round128((kC + max_other) * R * 16);
  const int64_t w = with_w ? round128(kC * R * 16) : 0;
  const int64_t val = round128(kC * max_width * 16);
  const int64_t lc = round128(kC * max_width * 2);
  const int64_t stage = v + w + val + lc;
  // Three stages by default, fewer if they do not fit (R = 32: two): measured on B200 against
  // 1, 2 and 4 stages; `stages` (env KPM_TILE_STAGES) overrides.
  int n = (int)std::min<int64_t>(stages > 0 ? stages : 3, kTileBudget / std::max<int64_t>(stage, 1));
  if (n < 1) return tl;
  tl.stages = n;
  tl.stage_bytes = (int)stage;
  tl.off_w = (int)v;
  tl.off_val = (int)(v + w);
  tl.off_lcol = (int)(v + w + val);
  return tl;
}

// Block-cache layout: a stage = [kBcExtraRows V rows | W | val | lcol], rounded to V rows; the
// pool takes the rest of the budget in 32-row blocks: at least 5 S, so that S tiles without
// any reuse (TI: own + 4 neighbour blocks each) can be in flight.
constexpr int kBcExtraRows = 8;
TileLayout plan_tiles_bc(int R, int64_t max_width, bool with_w, int stages, int ctas, bool lcol_t) {
  TileLayout tl;
  const int64_t rowb = 16ll * R;
  const int S = stages > 0 ? stages : 2;
  auto up = [&](int64_t b) { return (b + rowb - 1) / rowb * rowb; };
  const int64_t extra = kBcExtraRows * rowb;
  const int64_t w = with_w ? kC * rowb : 0;
  const int64_t lt = lcol_t ? ((std::max<int64_t>(max_width, 1) - 1 + 3) / 4) * 4 + 4 : 0;
  const int64_t val = round128(kC * max_width * 16), lc = round128(kC * (lcol_t ? lt : max_width) * 2);
  const int64_t stage = up(extra + w + val + lc);
  const int64_t pool = kTileBudget / std::max(ctas, 1) - (ctas > 1 ? 4096 : 0) - S * stage;
  const int P = (int)std::min<int64_t>(kBcMaxSlots, pool / (kC * rowb));
  if (P < 5 * S) return tl;
  tl.stages = S;
  tl.stage_bytes = (int)stage;
  tl.off_w = (int)extra;
  tl.off_val = (int)(extra + w);
  tl.off_lcol = (int)(extra + w + val);
  tl.pool_slots = P;
  tl.pool_bytes = (int)(P * kC * rowb);
  tl.extra_rows = kBcExtraRows;
  tl.lt_stride = (int)lt;
  return tl;
}

int staged_max_width() { return kLcap; }

int sweep_occupancy(int R, int variant, int dyn_smem) {
  const Entry* e = find(R, variant);
  return e ? e->occ(dyn_smem) : 0;
}

cudaError_t launch_aug_spmmv(int R, int variant, bool init, const SweepArgs& a, int grid, cudaStream_t s) {
  const Entry* e = find(R, variant);
  if (!e) return cudaErrorInvalidValue;
  return e->launch(init, a, grid, s);
}

// Bottleneck-analysis kernels (KPM_SWEEP_AUG_NODOT / KPM_SWEEP_SPMMV): the default tiled
// variant of each width (first kTable entry) with the dots, or also the shift/scale/-W, removed.
namespace {
template <int R, int LPR, bool WS, int KIND>
cudaError_t launch_kind(const SweepArgs& a, int grid, cudaStream_t s) {
  const int smem = a.tl.stages * a.tl.stage_bytes;
  cudaFuncSetAttribute(aug_spmmv_tiled<R, LPR, 4, 1, WS, false, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  aug_spmmv_tiled<R, LPR, 4, 1, WS, false, KIND><<<grid, tiled_threads<LPR, 1>(), smem, s>>>(a);
  return cudaGetLastError();
}
typedef cudaError_t (*KindFn)(const SweepArgs&, int, cudaStream_t);
struct KindEntry {
  int R;
  KindFn nodot, spmmv;
};
// keep in step with base_variant(R) of each width in kTable
const KindEntry kKinds[] = {
    {1, launch_kind<1, 1, true, kAugNoDot>, launch_kind<1, 1, true, kSpmmv>},
    {2, launch_kind<2, 2, true, kAugNoDot>, launch_kind<2, 2, true, kSpmmv>},
    {4, launch_kind<4, 4, false, kAugNoDot>, launch_kind<4, 4, false, kSpmmv>},
    {8, launch_kind<8, 4, false, kAugNoDot>, launch_kind<8, 4, false, kSpmmv>},
    {16, launch_kind<16, 4, false, kAugNoDot>, launch_kind<16, 4, false, kSpmmv>},
    {32, launch_kind<32, 8, true, kAugNoDot>, launch_kind<32, 8, true, kSpmmv>},
};
}  // namespace

cudaError_t launch_sweep_kind(int R, int kind, const SweepArgs& a, int grid, cudaStream_t s) {
  const int bv = base_variant(R);
  if (kind == kAug) return launch_aug_spmmv(R, bv, false, a, grid, s);
  if (!variant_tiled(R, bv)) return cudaErrorInvalidValue;
  for (const KindEntry& e : kKinds)
    if (e.R == R) return kind == kAugNoDot ? e.nodot(a, grid, s) : kind == kSpmmv ? e.spmmv(a, grid, s) : cudaErrorInvalidValue;
  return cudaErrorInvalidValue;
}

cudaError_t preload_aux_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, z4_init_kernel);
  cudaFuncGetAttributes(&fa, v0_permute_kernel);
  cudaFuncGetAttributes(&fa, eta_finalize_kernel);
  return cudaGetLastError();
}

static int elementwise_grid(int64_t n_el) {
  int64_t g = (n_el + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_z4_init(double2* V, double2* W, const int* perm, int64_t n_loc, int64_t n_pad, const int64_t* halo_rows,
                           int64_t n_rows_total, int R, int64_t row_begin, int64_t col_begin, int r_valid,
                           uint64_t seed, cudaStream_t s) {
  z4_init_kernel<<<elementwise_grid(n_rows_total * R), 256, 0, s>>>(V, W, perm, n_loc, n_pad, halo_rows, n_rows_total, R,
                                                                     row_begin, col_begin, r_valid, seed);
  return cudaGetLastError();
}

cudaError_t launch_v0_upload_permute(double2* V, double2* W, const double2* v0_dev, const int* perm, int64_t n_loc,
                                     int64_t n_pad, int64_t n_rows_total, int R, int r_valid, cudaStream_t s) {
  v0_permute_kernel<<<elementwise_grid(n_rows_total * R), 256, 0, s>>>(V, W, v0_dev, perm, n_loc, n_pad, n_rows_total,
                                                                        R, r_valid);
  return cudaGetLastError();
}

cudaError_t launch_eta_finalize(const double* partials, int n_sweeps, int R, int width, double2* eta_even,
                                double2* eta_odd, cudaStream_t s) {
  const int64_t n_threads = (int64_t)n_sweeps * 3 * R * 32;
  const int blocks = (int)((n_threads + 255) / 256);
  eta_finalize_kernel<<<blocks, 256, 0, s>>>(partials, n_sweeps, R, width, eta_even, eta_odd);
  return cudaGetLastError();
}

}  // namespace kpm
