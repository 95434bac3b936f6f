// Locality order of the SELL chunks (chunk_order.cpp; DESIGN.md §7 "Chunk order").  Host only.
#pragma once
#include <stdint.h>

#include <vector>

namespace kpm {

// Block-neighbour lists (CSR: ptr n_chunks+1, nbr) from the tiled feed's per-chunk row runs
// (nruns[c] runs of (first row, count) at runs[(c * max_runs + k) * 2]): chunk b is a block
// neighbour of c if c reads all C rows of b.
void block_neighbours(int64_t n_chunks, const int* nruns, const int* runs, int max_runs, int C,
                      std::vector<int64_t>& ptr, std::vector<int64_t>& nbr);

// Line walk in rounds of G lines (width 1) or strips of two lines (width 2) (see chunk_order.cpp);
// skip (empty or n_chunks flags): chunks kept out of the lines and appended last.  Returns a
// permutation of 0..n_chunks-1.
std::vector<int64_t> line_order(int64_t n_chunks, const std::vector<int64_t>& ptr, const std::vector<int64_t>& nbr,
                                int64_t G, const std::vector<char>& skip, int width = 1);

// 90th percentile over the chunks of the largest |b - c| to a block neighbour: the reuse distance
// (in chunks) of a storage-order sweep, periodic wraps aside.
int64_t typical_block_offset(int64_t n_chunks, const std::vector<int64_t>& ptr, const std::vector<int64_t>& nbr);

}  // namespace kpm
