// Host-side SELL-C-sigma builder and row-distribution halo list.
//
// SELL-C-sigma: Kreutzer et al., cited at PAPER.md P:126-128; C = 32 = warpSize; sigma-window
// descending-length sort; "the CRS format (similar to SELL-1) can be used".
// Layout contract: DESIGN.md "SELL-C-sigma" (the tests compare this builder bit for bit
// with the independent numpy reference in oracle/sell_ref.py).
#include "sell_build.h"

#include <algorithm>
#include <numeric>
#include <stdexcept>
#include <thread>

namespace kpm {

// Static block partition of [0, n) over the host's cores (the build is one-off setup work,
// but it sits inside the e2e path, so it uses every core).  f(begin, end, thread index).
template <class F>
static void parallel_for(int64_t n, F f) {
  int T = (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 64u);
  if (n < 4096) T = 1;
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    const int64_t b = n * t / T, e = n * (t + 1) / T;
    if (t == T - 1)
      f(b, e, t);
    else
      th.emplace_back(f, b, e, t);
  }
  for (auto& x : th) x.join();
}

static int n_threads_for(int64_t n) {
  return n < 4096 ? 1 : (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 64u);
}

int build_sell_host(const int64_t* row_ptr, const int64_t* col, const double* val, int64_t n_loc,
                    int64_t row_begin, int64_t row_end, int C, int sigma, HostSell& out, std::string& err) {
  out = HostSell();
  out.n_loc = n_loc;
  out.C = C;
  out.sigma = sigma;
  std::vector<int64_t> len(n_loc);
  for (int64_t i = 0; i < n_loc; ++i) len[i] = row_ptr[i + 1] - row_ptr[i];

  // sigma-window stable sort by descending row length
  out.perm.resize(n_loc);
  std::iota(out.perm.begin(), out.perm.end(), 0);
  if (sigma > 1) {
    for (int64_t w0 = 0; w0 < n_loc; w0 += sigma) {
      const int64_t w1 = std::min<int64_t>(w0 + sigma, n_loc);
      std::stable_sort(out.perm.begin() + w0, out.perm.begin() + w1,
                       [&](int a, int b) { return len[a] > len[b]; });
    }
  }
  std::vector<int64_t> invperm(n_loc);
  for (int64_t p = 0; p < n_loc; ++p) invperm[out.perm[p]] = p;

  out.n_chunks = (n_loc + C - 1) / C;
  out.n_pad = out.n_chunks * C;

  // halo: distinct remote columns, ascending global id (== by owner rank, then id)
  std::vector<int64_t>& halo = out.halo;
  {
    const int64_t nnz = row_ptr[n_loc];
    std::vector<std::vector<int64_t>> part(n_threads_for(nnz));
    parallel_for(nnz, [&](int64_t b, int64_t e, int t) {
      for (int64_t k = b; k < e; ++k)
        if (col[k] < row_begin || col[k] >= row_end) part[t].push_back(col[k]);
      std::sort(part[t].begin(), part[t].end());
      part[t].erase(std::unique(part[t].begin(), part[t].end()), part[t].end());
    });
    for (auto& v : part) halo.insert(halo.end(), v.begin(), v.end());
    std::sort(halo.begin(), halo.end());
    halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  }
  out.n_halo = (int64_t)halo.size();
  if (out.n_pad + out.n_halo > (int64_t)INT32_MAX) {
    err = "local rows + halo rows exceed the int32 kernel index range";
    return 3;
  }

  out.cptr.assign(out.n_chunks + 1, 0);
  for (int64_t c = 0; c < out.n_chunks; ++c) {
    int64_t m = 0;
    for (int64_t k = 0; k < C; ++k) {
      const int64_t p = c * C + k;
      if (p < n_loc) m = std::max(m, len[out.perm[p]]);
    }
    out.cptr[c + 1] = out.cptr[c] + C * m;
  }
  const int64_t n_slots = out.cptr[out.n_chunks];
  out.val.resize(2 * n_slots);
  out.col.resize(n_slots);
  parallel_for(out.n_chunks, [&](int64_t cb, int64_t ce, int) {
  for (int64_t c = cb; c < ce; ++c) {
    const int64_t L = (out.cptr[c + 1] - out.cptr[c]) / C;
    for (int64_t k = 0; k < C; ++k) {
      const int64_t p = c * C + k;
      const int64_t nrow = (p < n_loc) ? len[out.perm[p]] : 0;
      const int64_t src = (p < n_loc) ? row_ptr[out.perm[p]] : 0;
      // own-position (diagonal) entry first, then the others in stored order (R18)
      const int64_t gdiag = row_begin + ((p < n_loc) ? (int64_t)out.perm[p] : 0);
      int64_t jd = nrow;
      for (int64_t j = 0; j < nrow; ++j)
        if (col[src + j] == gdiag) {
          jd = j;
          break;
        }
      for (int64_t j = 0; j < L; ++j) {
        const int64_t d = out.cptr[c] + j * C + k;
        if (j < nrow) {
          const int64_t js = jd == nrow ? j : (j == 0 ? jd : (j <= jd ? j - 1 : j));  // source entry
          const int64_t g = col[src + js];
          int64_t lc;
          if (g >= row_begin && g < row_end) {
            lc = invperm[g - row_begin];
          } else {
            lc = out.n_pad + (std::lower_bound(halo.begin(), halo.end(), g) - halo.begin());
          }
          out.col[d] = (int32_t)lc;
          out.val[2 * d] = val[2 * (src + js)];
          out.val[2 * d + 1] = val[2 * (src + js) + 1];
        } else {
          out.col[d] = (int32_t)p;  // padding: value 0, column = own position
          out.val[2 * d] = 0.0;
          out.val[2 * d + 1] = 0.0;
        }
      }
    }
  }
  });
  return 0;
}

void build_tiles_host(const HostSell& s, HostTiles& out) {
  out = HostTiles();
  const int C = s.C;
  const int64_t n_slots = s.cptr[s.n_chunks];
  out.run_ptr.assign(s.n_chunks + 1, 0);
  out.lcol.resize(n_slots);
  out.ok = true;
  // pass 1 (parallel over chunks): lcol, per-chunk runs; pass 2: concatenate the runs
  const int T = n_threads_for(s.n_chunks);
  std::vector<std::vector<int32_t>> runs_t(T);
  std::vector<int64_t> max_other_t(T, 0), max_runs_t(T, 0);
  std::vector<char> ok_t(T, 1);
  parallel_for(s.n_chunks, [&](int64_t cb, int64_t ce, int tt) {
  std::vector<int32_t> other;
  std::vector<int32_t>& runs = runs_t[tt];
  for (int64_t c = cb; c < ce; ++c) {
    const int64_t a = s.cptr[c], b = s.cptr[c + 1];
    const int64_t own0 = c * C, own1 = own0 + C;
    other.clear();
    for (int64_t k = a; k < b; ++k)
      if (s.col[k] < own0 || s.col[k] >= own1) other.push_back(s.col[k]);
    std::sort(other.begin(), other.end());
    other.erase(std::unique(other.begin(), other.end()), other.end());
    if ((int64_t)other.size() + C > 65535) ok_t[tt] = 0;
    max_other_t[tt] = std::max<int64_t>(max_other_t[tt], (int64_t)other.size());
    int64_t nr = 0;
    for (size_t i = 0; i < other.size(); ++i) {
      if (i == 0 || other[i] != other[i - 1] + 1) {
        runs.push_back(other[i]);
        runs.push_back(1);
        ++nr;
      } else {
        ++runs.back();
      }
    }
    max_runs_t[tt] = std::max(max_runs_t[tt], nr);
    out.run_ptr[c + 1] = nr;  // count for now, prefix-summed below
    for (int64_t k = a; k < b; ++k) {
      const int32_t g = s.col[k];
      if (g >= own0 && g < own1) {
        out.lcol[k] = (uint16_t)(g - own0);
      } else {
        const int64_t idx = std::lower_bound(other.begin(), other.end(), g) - other.begin();
        out.lcol[k] = (uint16_t)std::min<int64_t>(C + idx, 65535);
      }
    }
  }
  });
  for (int64_t c = 0; c < s.n_chunks; ++c) out.run_ptr[c + 1] += out.run_ptr[c];
  for (int t = 0; t < T; ++t) {
    out.runs.insert(out.runs.end(), runs_t[t].begin(), runs_t[t].end());
    out.ok = out.ok && ok_t[t];
    out.max_other = std::max(out.max_other, max_other_t[t]);
    out.max_runs = std::max(out.max_runs, max_runs_t[t]);
  }
}

}  // namespace kpm
