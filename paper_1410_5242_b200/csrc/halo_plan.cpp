#include "halo_plan.h"

#include <algorithm>

namespace kpm {

static int owner_of(int64_t g, const std::vector<int64_t>& row_begins) {
  return (int)(std::upper_bound(row_begins.begin(), row_begins.end(), g) - row_begins.begin()) - 1;
}

std::vector<RecvRun> plan_recv_runs(const std::vector<int64_t>& halo, const std::vector<int64_t>& row_begins) {
  std::vector<RecvRun> runs;
  for (size_t h = 0; h < halo.size(); ++h) {
    const int q = owner_of(halo[h], row_begins);
    if (!runs.empty() && runs.back().peer == q && runs.back().gfirst + runs.back().count == halo[h]) {
      ++runs.back().count;
    } else {
      runs.push_back(RecvRun{q, halo[h], 1, (int64_t)h});
    }
  }
  return runs;
}

bool plan_send_runs(int peer, const std::vector<int64_t>& req, int64_t row_begin, int64_t row_end,
                    const std::vector<int32_t>& perm, std::vector<SendRun>& out) {
  std::vector<int64_t> invperm;
  if (!perm.empty()) {
    invperm.resize(perm.size());
    for (size_t p = 0; p < perm.size(); ++p) invperm[perm[p]] = (int64_t)p;
  }
  auto pos = [&](int64_t g) { return invperm.empty() ? g - row_begin : invperm[g - row_begin]; };
  for (size_t i = 0; i + 1 < req.size(); i += 2) {
    const int64_t g0 = req[i], cnt = req[i + 1];
    if (cnt < 1 || g0 < row_begin || g0 + cnt > row_end) return false;
    const int64_t p0 = pos(g0);
    for (int64_t k = 1; k < cnt; ++k)
      if (pos(g0 + k) != p0 + k) return false;
    out.push_back(SendRun{peer, p0, cnt, -1});
  }
  return true;
}

void plan_edge_chunks(int64_t n_chunks, const std::vector<char>& reads_halo, int C, const std::vector<SendRun>& sends,
                      std::vector<int64_t>& edge, std::vector<int64_t>& interior) {
  std::vector<char> is_edge(n_chunks, 0);
  for (const SendRun& s : sends)
    for (int64_t c = s.pos / C; c <= (s.pos + s.count - 1) / C; ++c) is_edge[c] = 1;
  for (int64_t c = 0; c < n_chunks && c < (int64_t)reads_halo.size(); ++c)
    if (reads_halo[c]) is_edge[c] = 1;
  edge.clear();
  interior.clear();
  for (int64_t c = 0; c < n_chunks; ++c) (is_edge[c] ? edge : interior).push_back(c);
}

}  // namespace kpm
