// Internal declarations of the B200 KPM library (not part of the ABI; see include/kpm.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace kpm {

constexpr int kC = 32;             // SELL chunk height = warpSize (north_star subsystem 1)
constexpr int kThreads = 256;      // threads per CTA of the sweep kernels (8 warps)
constexpr int kMaxBlockWidth = 32; // widest specialised block (R per batch)
constexpr int kRecSlots = 16;      // copy-record slots per chunk (header + 15 bulk copies)
constexpr int kMaxRuns = kRecSlots - 5;  // row runs per chunk (besides own rows, W, val, lcol)

// Grow-only device allocation: reuse *p if it holds `bytes`, else reallocate (kpm_set_matrix is
// called once per step in the e2e loop; large cudaFree/cudaMalloc pairs would dominate it).
inline cudaError_t reserve(void** p, size_t* cap, size_t bytes) {
  bytes = bytes < 16 ? 16 : bytes;
  if (*p && *cap >= bytes) return cudaSuccess;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) *cap = bytes;
  return e;
}

// Device-side SELL-C-sigma matrix ("Data layout in HBM").
struct DevSell {
  double2* val = nullptr;  // n_slots, chunk-column-major: entry j of row k of chunk c at cptr[c]+j*32+k
  int* col = nullptr;      // n_slots, int32 local column (position in the local+halo vector)
  int64_t* cptr = nullptr; // n_chunks+1
  int* perm = nullptr;     // n_loc: local row stored at position p (NULL: identity, sigma = 1)
  int* perm_buf = nullptr; // grow-only storage behind perm
  int64_t n_loc = 0, n_pad = 0, n_chunks = 0, n_slots = 0, n_halo = 0;
  int64_t max_width = 0;   // widest chunk (entries per row)
  // tiled feed (TMA gather plan, see sell_build.h HostTiles)
  bool tiles_ok = false;
  uint16_t* lcol = nullptr;    // n_slots: column as index into the chunk's shared-memory tile
  int* nruns = nullptr;        // n_chunks: runs of other rows per chunk
  int* runs = nullptr;         // n_chunks x kMaxRuns x (first row, count)
  int64_t max_other = 0, max_runs = 0;
  uint4* rec[12] = {};        // copy records per (log2(R), W staged)
  size_t rec_cap[12] = {};
  bool rec_valid[12] = {};     // built for the current matrix
  bool rec_failed[12] = {};
  // capacities (bytes) of the grow-only buffers above
  size_t val_cap = 0, col_cap = 0, cptr_cap = 0, perm_cap = 0, lcol_cap = 0, nruns_cap = 0, runs_cap = 0;
};

// Shared-memory layout of one stage of the tiled feed (bytes, 128-B aligned sections).
struct TileLayout {
  int stages = 0;
  int stage_bytes = 0;
  int off_w = 0, off_val = 0, off_lcol = 0;  // V tile rows start at 0
  // block-cache feed only: dynamic shared memory = [pool of pool_slots blocks of
  // 32 V rows][stage 0]..[stage S-1]; a stage holds [extra_rows V rows | W | val | lcol] and
  // starts at pool_bytes + s * stage_bytes; all offsets are multiples of one V row (16 R bytes)
  int pool_bytes = 0, pool_slots = 0, extra_rows = 0;
  // block-cache feed with row-major tile indices (lt_stride > 0): in a chunk's lcol block row k's
  // entries 1..L-1 sit at k*lt_stride + 0..L-2 (padded to a multiple of 4) and entry 0 at
  // k*lt_stride + lt_stride - 4, so one 8-byte load gives a batch of 4 entries (kernels.cu)
  int lt_stride = 0;
};
constexpr int kBcMaxSlots = 16;  // block-cache pool slots (max)
constexpr int kBcMapInts = 40;   // per tile: [n_blocks, (block, smem row) x 7, -, n_extra, (row, count, smem row) x 8]

// Fused halo exchange: rows [pos, pos+count) of the new W are also stored to dst (a peer
// GPU's halo slots, mapped over NVLink with CUDA IPC) by the sweep kernel's epilogue.
constexpr int kMaxPeerRuns = 8;
struct PeerRun {
  int64_t pos, count;
  double2* dst;
};

// One aug_spmmv sweep over a chunk range / chunk list.
struct SweepArgs {
  const double2* val;
  const int* col;
  const int64_t* cptr;
  const double2* V;    // nu_m   (read only)
  double2* W;          // nu_{m-1} in, nu_{m+1} out
  int64_t n_loc;
  const int64_t* chunk_list;       // NULL: chunks [chunk_begin, chunk_end); else chunk_list[chunk_begin .. chunk_end)
  int64_t chunk_begin, chunk_end;
  double scale;        // 2a for the main sweep, a for the init sweep
  double b;
  double* partials;    // [3R][pstride]: per-CTA (eta_even, Re eta_odd, Im eta_odd) of this launch at [i*pstride + cta]
  int64_t pstride;
  // tiled feed only
  const uint4* rec;      // kRecSlots per chunk (sell_build.h)
  const uint16_t* lcol;
  TileLayout tl;
  int v_evict_last;    // tiled feed: L2 evict-last hint on the gathered V rows (env KPM_V_EVICT_LAST, default 1)
  // fused halo exchange (edge launches only; n_peer = 0 otherwise)
  int n_peer;
  PeerRun peer[kMaxPeerRuns];
};

// Launch helpers (kernels.cu).  All return cudaGetLastError() of the launch.
// V = Z4 start block for the local rows (global row row_begin + perm[p]) and the halo slots
// (global row halo_rows[h], h = p - n_pad); padding rows and W = 0.
cudaError_t launch_z4_init(double2* V, double2* W, const int* perm, int64_t n_loc, int64_t n_pad, const int64_t* halo_rows,
                           int64_t n_rows_total, int R, int64_t row_begin, int64_t col_begin, int r_valid,
                           uint64_t seed, cudaStream_t s);
cudaError_t launch_v0_upload_permute(double2* V, double2* W, const double2* v0_dev, const int* perm,
                                     int64_t n_loc, int64_t n_pad, int64_t n_rows_total, int R, int r_valid,
                                     cudaStream_t s);
// Kernel variants per block width R (feed x lanes-per-row x unroll); variant 0 is the default.
int variant_count(int R);
const char* variant_name(int R, int variant);
int sweep_occupancy(int R, int variant, int dyn_smem);
bool variant_staged(int R, int variant);
int staged_max_width();  // widest chunk (entries per row) the staged feed accepts
bool variant_tiled(int R, int variant);
// Shared-memory plan of the tiled feed for block width R, or stages == 0 if it does not fit.
TileLayout plan_tiles(int R, int64_t max_other, int64_t max_width, int stages, bool with_w);  // stages 0 = default
bool variant_wstage(int R, int variant);  // tiled feed: old W staged in shared memory
int variant_stages(int R, int variant);   // tiled feed: preferred ring depth (0 = default)
cudaError_t launch_aug_spmmv(int R, int variant, bool init, const SweepArgs& a, int grid, cudaStream_t s);
// kind = KPM_SWEEP_*: the default variant (aug), or it without dots / as a plain SpMMV (main sweep form)
int check_hermitian(const int64_t* rp, const int64_t* col, const double* val, int64_t n_loc, int64_t row_begin,
                    int64_t row_end, int64_t n_global, double rtol, std::string& msg);  // hermitian.cpp
cudaError_t launch_sweep_kind(int R, int kind, const SweepArgs& a, int grid, cudaStream_t s);
// Load the start-block and eta kernels now (lazy module loading may synchronize the device).
cudaError_t preload_aux_kernels();
// eta[m][r] (double2) for m in [0, n_sweeps) from partials[m][3R][width] (width = launches x grid)
cudaError_t launch_eta_finalize(const double* partials, int n_sweeps, int R, int width, double2* eta_even,
                                double2* eta_odd, cudaStream_t s);

// Naive stage-0 sweep of one column (naive.cu): separate spmv/axpy/scal/axpy/nrm2/dot kernels.
int naive_grid();
cudaError_t naive_sweep(const DevSell& s, const double2* v, double2* w, double2* u, double a, double b, bool init,
                        double* part, cudaStream_t st);

// Device-side setup (sell_device.cu): CSR on the device -> SELL-32 (sigma = 1) + tile plan.
struct DeviceBuild {
  std::vector<int64_t> halo;     // global ids of the halo slots (host copy)
  std::vector<int64_t> cptr;     // host copy of cptr
  std::vector<char> reads_halo;  // per chunk (empty if no halo)
};
// Grow-only device temporaries of build_sell_device, owned by the context (a per-call
// cudaMalloc/cudaFree of the ~0.3 GB selection buffer cost up to a second per call).
struct BuildScratch {
  enum { kFlags, kWidth, kSlots, kTmp, kMaxW, kSel, kNsel, kHalo, kNother, kMaxO, kReadsHalo, kCount };
  void* p[kCount] = {};
  size_t cap[kCount] = {};
  template <class T>
  cudaError_t get(int i, size_t n, T** out) {
    const cudaError_t e = reserve(&p[i], &cap[i], n * sizeof(T));
    *out = static_cast<T*>(p[i]);
    return e;
  }
  void release() {
    for (int i = 0; i < kCount; ++i) cudaFree(p[i]);
    *this = BuildScratch();
  }
};
int build_sell_device(const int64_t* rp, const int64_t* col, const double2* val, int64_t n_loc, int64_t row_begin,
                      int64_t row_end, int64_t n_global, DevSell& d, DeviceBuild& out, BuildScratch& ws,
                      std::string& err, cudaStream_t s);
// Copy records of the tiled feed for block width R from the per-chunk run lists.
// Block-cache feed: per-position copy records (kRecSlots uint4, list position b + G k = CTA b's
// k-th tile) from a simulation of each CTA's pool of 32-row V blocks, and the tile-row index (times R)
// of every SELL slot pointing into that CTA's shared memory.  *fail != 0 if some tile does not fit.
cudaError_t launch_build_bc(const int64_t* cptr, const int* nruns, const int* runs, const int* scol,
                            const int64_t* list, int64_t n_chunks, int grid, int R, bool with_w,
                            const TileLayout& tl, uint4* rec, int* map, uint16_t* lcol_bc, int* fail,
                            cudaStream_t s);
TileLayout plan_tiles_bc(int R, int64_t max_width, bool with_w, int stages, int ctas, bool lcol_t = false);
int variant_bc(int R, int variant);  // block-cache feed: CTAs per SM it is planned for, 0 = other feed
int base_variant(int R);             // first variant of width R that is not a block-cache feed
int variant_strip(int R, int variant);  // width (1, 2) of the library's line walk for this variant
cudaError_t launch_build_records(const int64_t* cptr, const int* nruns, const int* runs, int64_t n_chunks, int R,
                                 int off_w, int off_val, int off_lcol, uint4* rec, cudaStream_t s);

}  // namespace kpm
