// Host-side planning of the row-distribution halo exchange.
//
// The data-parallel row distribution of PAPER.md P:849-854 (equal weights): rank p owns the
// global rows [row_begins[p], row_begins[p+1]).  A rank's halo is every distinct remote
// column its rows read, ordered by (owner rank, global id) -- the order of the halo slots
// appended after n_pad in its vectors.  The exchange moves, after every sweep, the owners'
// freshly written rows into those slots.  Pure host code: no CUDA, no NCCL, so the index
// logic is testable on a CPU (tests/test_halo_plan.py, gloo world size 2).
#pragma once
#include <stdint.h>

#include <vector>

namespace kpm {

// Receive run: halo slots [slot, slot+count) <- global rows [gfirst, gfirst+count) of `peer`.
struct RecvRun {
  int peer;
  int64_t gfirst, count, slot;
};
// Send run: my local positions [pos, pos+count) -> `peer` (matched in order with its RecvRun).
struct SendRun {
  int peer;
  int64_t pos, count;
  int64_t peer_slot = -1;  // first halo slot of the run in the peer's vectors (fused exchange)
};

// Maximal runs of consecutive global ids in the (sorted) halo list, split at owner changes.
std::vector<RecvRun> plan_recv_runs(const std::vector<int64_t>& halo, const std::vector<int64_t>& row_begins);

// Send runs for the runs `req` (gfirst, count pairs, in the requester's order) that `peer`
// asked of this rank.  pos = invperm[g - row_begin] (perm empty = identity); every requested
// run must map to consecutive positions (true for sigma = 1), otherwise returns false.
bool plan_send_runs(int peer, const std::vector<int64_t>& req, int64_t row_begin, int64_t row_end,
                    const std::vector<int32_t>& perm, std::vector<SendRun>& out);

// Chunks that must be computed before the exchange (they hold rows that are sent) or that
// read halo slots (reads_halo[c], empty = none); the rest are interior.  Both ascending.
void plan_edge_chunks(int64_t n_chunks, const std::vector<char>& reads_halo, int C, const std::vector<SendRun>& sends,
                      std::vector<int64_t>& edge, std::vector<int64_t>& interior);

}  // namespace kpm
