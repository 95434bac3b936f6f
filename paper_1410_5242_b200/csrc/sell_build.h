#pragma once
#include <stdint.h>

#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace kpm {

// Allocator that leaves new elements uninitialised (the builders write every element), so
// resizing the multi-GB SELL arrays does not zero-fill them first.
template <class T>
struct NoInit : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInit<U>;
  };
  NoInit() = default;
  template <class U>
  NoInit(const NoInit<U>&) {}
  template <class U>
  void construct(U* p) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using raw_vector = std::vector<T, NoInit<T>>;

struct HostSell {
  int64_t n_loc = 0, n_pad = 0, n_chunks = 0, n_halo = 0;
  int C = 32, sigma = 1;
  raw_vector<double> val;      // 2*n_slots (re, im)
  raw_vector<int32_t> col;     // n_slots
  std::vector<int64_t> cptr;   // n_chunks+1
  std::vector<int32_t> perm;   // n_loc
  std::vector<int64_t> halo;   // n_halo global ids, ascending
};

// Per-chunk gather plan of the TMA-fed ("tiled") sweep kernel: the distinct columns a chunk
// reads that are not its own 32 rows, as maximal runs of consecutive rows (ascending), and
// every SELL slot's column re-expressed as an index into the chunk's shared-memory tile
// [own rows 0..31 | run rows in order].
struct HostTiles {
  bool ok = false;                 // false: some chunk needs > 65535 tile rows
  std::vector<int64_t> run_ptr;    // n_chunks+1, into runs
  std::vector<int32_t> runs;       // 2 per run: first row, row count
  raw_vector<uint16_t> lcol;       // n_slots
  int64_t max_other = 0;           // max rows outside the own block, over chunks
  int64_t max_runs = 0;
};
void build_tiles_host(const HostSell& s, HostTiles& out);

// Copy-command records of the tiled feed (built on the device, sell_device.cu): kRecSlots x
// 16-byte slots per chunk.  Slot 0 = {bytes (main sweep), bytes (init sweep, no W), chunk
// width L, n_cmd}; slots 1..n_cmd = {src byte offset lo, hi, dst byte offset in the stage,
// bytes | base << 28} with base 0 = V, 1 = W, 2 = val, 3 = lcol.

// Returns 0 or a kpm_status code (err filled).
int build_sell_host(const int64_t* row_ptr, const int64_t* col, const double* val, int64_t n_loc,
                    int64_t row_begin, int64_t row_end, int C, int sigma, HostSell& out, std::string& err);

}  // namespace kpm
