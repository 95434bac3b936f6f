// Locality order of the SELL chunks, derived inside the library from the matrix itself
// (DESIGN.md §7 "Chunk order"; the paper's cache-blocking outlook, and the effect of
// the gathered-vector reuse factor Omega).  Host code, no CUDA: testable on a CPU
// through kpm_plan_chunk_order (plan_abi.cpp).
//
// Chunk b is a *block neighbour* of chunk c when c's entries reference all 32 rows of b (for a
// stencil such as the TI lattice: the chunks one step away along a periodic/open direction whose
// sites line up with c's).  The line direction d is the smallest positive chunk offset that at
// least half of the chunks have as a block neighbour (TI, x slowest: d = Nz/8, one step in y).
// A line is a maximal chain c, c + d, c + 2d, ... of mutual block neighbours.  Lines of equal
// length are taken in rounds of G (the sweep grid, one line per CTA, list position b + G k =
// CTA b's k-th tile), interleaved so that all CTAs are at the same step: consecutive tiles of a
// CTA then share their line-direction neighbour blocks (the block-cache feed keeps them in shared
// memory) and the other neighbours are the current tiles of other CTAs (L2 hits).  Lines left
// over after the last full round, then chunks in no line, are cut into G balanced contiguous
// segments, one per CTA, also walked in lock step.  Chunks with
// skip[c] != 0 (the edge chunks of a multi-rank split) are kept out of the lines and go last.
// width = 2 walks strips of two adjacent lines step by step (c, c', c + d, c' + d, ... with c' =
// c + d2, d2 the next frequent offset: TI x): a tile's neighbour on the strip's inside is then a
// block its CTA already holds.  Measured on C3: -2 % sweep time for the R = 32 block-cache
// kernel (1 CTA per SM, 10-block pool), +2 % for the R = 16 ones (2 CTAs per SM), so the kernel
// table chooses the width per variant.
#include <stdint.h>

#include <algorithm>
#include <array>
#include <map>
#include <vector>

#include "chunk_order.h"

namespace kpm {

void block_neighbours(int64_t n_chunks, const int* nruns, const int* runs, int max_runs, int C,
                      std::vector<int64_t>& ptr, std::vector<int64_t>& nbr) {
  ptr.assign(n_chunks + 1, 0);
  nbr.clear();
  for (int64_t c = 0; c < n_chunks; ++c) {
    for (int k = 0; k < nruns[c]; ++k) {
      const int64_t first = runs[(c * max_runs + k) * 2], cnt = runs[(c * max_runs + k) * 2 + 1];
      for (int64_t b = (first + C - 1) / C; (b + 1) * C <= first + cnt; ++b)
        if (b != c && b < n_chunks) nbr.push_back(b);
    }
    ptr[c + 1] = (int64_t)nbr.size();
  }
}

std::vector<int64_t> line_order(int64_t n_chunks, const std::vector<int64_t>& ptr, const std::vector<int64_t>& nbr,
                                int64_t G, const std::vector<char>& skip, int width) {
  auto in = [&](int64_t c) { return c >= 0 && c < n_chunks && (skip.empty() || !skip[c]); };
  auto is_nbr = [&](int64_t c, int64_t b) {
    for (int64_t i = ptr[c]; i < ptr[c + 1]; ++i)
      if (nbr[i] == b) return true;
    return false;
  };
  // line direction: the smallest positive offset that at least half of the chunks have
  std::map<int64_t, int64_t> freq;
  int64_t n_in = 0;
  for (int64_t c = 0; c < n_chunks; ++c) {
    if (!in(c)) continue;
    ++n_in;
    for (int64_t i = ptr[c]; i < ptr[c + 1]; ++i)
      if (nbr[i] > c && in(nbr[i])) ++freq[nbr[i] - c];
  }
  int64_t d = 0, d2 = 0;  // line direction; the next frequent offset (strips of width 2)
  for (const auto& kv : freq)
    if (2 * kv.second >= n_in) {
      if (!d)
        d = kv.first;
      else if (!d2)
        d2 = kv.first;
    }
  std::vector<int64_t> order;
  order.reserve(n_chunks);
  std::vector<char> used(n_chunks, 0);
  if (d > 0 && G > 0) {
    auto linked = [&](int64_t c) { return in(c + d) && is_nbr(c, c + d) && is_nbr(c + d, c); };
    std::vector<std::pair<int64_t, int64_t>> lines;  // (start, length), starts ascending
    for (int64_t c = 0; c < n_chunks; ++c) {
      if (!in(c) || (c - d >= 0 && in(c - d) && linked(c - d))) continue;
      int64_t len = 1;
      for (int64_t x = c; linked(x); x += d) ++len;
      lines.push_back({c, len});
    }
    // width 2: pair each line (ascending start) with the unpaired equal-length line d2 further on
    // whose chunks are block neighbours of its own; a unit = a line or a pair of lines
    std::vector<std::array<int64_t, 3>> units;  // (start, length, partner start or -1)
    if (width == 2 && d2 > 0) {
      std::map<int64_t, size_t> at;
      for (size_t l = 0; l < lines.size(); ++l) at[lines[l].first] = l;
      std::vector<char> paired(lines.size(), 0);
      for (size_t l = 0; l < lines.size(); ++l) {
        if (paired[l]) continue;
        const auto it = at.find(lines[l].first + d2);
        if (it != at.end() && !paired[it->second] && lines[it->second].second == lines[l].second) {
          bool adj = true;
          for (int64_t k = 0; k < lines[l].second && adj; ++k)
            adj = is_nbr(lines[l].first + k * d, lines[l].first + k * d + d2);
          if (adj) {
            paired[l] = paired[it->second] = 1;
            units.push_back({lines[l].first, lines[l].second, lines[it->second].first});
          }
        }
      }
    } else {
      for (const auto& ln : lines) units.push_back({ln.first, ln.second, -1});
    }
    // rounds of G units of equal length and kind (longest first, starts ascending inside a
    // length), all CTAs at the same step; a pair advances both of its lines per step
    std::stable_sort(units.begin(), units.end(), [](const auto& a, const auto& b) { return a[1] > b[1]; });
    std::vector<int64_t> rest;  // walks of the units left over after the full rounds, in unit order
    size_t i = 0;
    while (i < units.size()) {
      size_t j = i;
      while (j < units.size() && units[j][1] == units[i][1]) ++j;
      const size_t full = (j - i) / (size_t)G * (size_t)G;
      for (size_t r = i; r < i + full; r += (size_t)G)
        for (int64_t step = 0; step < units[i][1]; ++step)
          for (int lane = 0; lane < (units[i][2] >= 0 ? 2 : 1); ++lane)
            for (size_t l = r; l < r + (size_t)G; ++l) {
              const int64_t c = (lane ? units[l][2] : units[l][0]) + step * d;
              order.push_back(c);
              used[c] = 1;
            }
      for (size_t l = i + full; l < j; ++l)
        for (int64_t step = 0; step < units[l][1]; ++step)
          for (int lane = 0; lane < (units[l][2] >= 0 ? 2 : 1); ++lane) {
            const int64_t c = (lane ? units[l][2] : units[l][0]) + step * d;
            rest.push_back(c);
            used[c] = 1;
          }
      i = j;
    }
    for (int64_t c = 0; c < n_chunks; ++c)  // chunks in no line
      if (!used[c] && in(c)) rest.push_back(c);
    // The rest in G balanced contiguous segments, one per CTA, walked in lock step (position
    // base + k G + b = step k of CTA b): a CTA keeps walking its strip(s) instead of jumping
    // through storage order (at 4 GPUs half of a C4 slab's strips are left over).
    const int64_t n_left = (int64_t)rest.size(), K = n_left / G, rem = n_left % G;
    std::vector<int64_t> seg(n_left);
    for (int64_t b = 0; b < G; ++b) {
      const int64_t start = b * K + std::min(b, rem), len = K + (b < rem ? 1 : 0);
      for (int64_t k = 0; k < len; ++k) seg[k * G + b] = rest[start + k];
    }
    order.insert(order.end(), seg.begin(), seg.end());
  } else {
    for (int64_t c = 0; c < n_chunks; ++c)  // no line direction: storage order
      if (in(c)) order.push_back(c);
  }
  for (int64_t c = 0; c < n_chunks; ++c)  // skipped chunks last
    if (!in(c)) order.push_back(c);
  return order;
}

int64_t typical_block_offset(int64_t n_chunks, const std::vector<int64_t>& ptr, const std::vector<int64_t>& nbr) {
  std::vector<int64_t> per;  // largest |b - c| of every chunk that has block neighbours
  for (int64_t c = 0; c < n_chunks; ++c) {
    int64_t m = -1;
    for (int64_t i = ptr[c]; i < ptr[c + 1]; ++i) m = std::max(m, nbr[i] > c ? nbr[i] - c : c - nbr[i]);
    if (m >= 0) per.push_back(m);
  }
  if (per.empty()) return 0;
  // the 90th percentile: a periodic wrap (the first plane's neighbours in the last) is rare
  std::nth_element(per.begin(), per.begin() + (int64_t)(per.size() * 9 / 10), per.end());
  return per[per.size() * 9 / 10];
}

}  // namespace kpm
