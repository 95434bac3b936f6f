// Optional debug check of kpm_set_matrix (kpm_options.flags & KPM_CHECK_HERMITIAN): the
// method needs a Hermitian H (the doubling identities of P:258-260, R4, hold
// only then), which the library otherwise does not verify (an O(nnz log nnz) transpose).
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/kpm.h"

namespace kpm {

namespace {
struct Entry {
  int64_t i, j;
  double re, im;
};
bool key_less(const Entry& x, const Entry& y) { return x.i < y.i || (x.i == y.i && x.j < y.j); }
}  // namespace

// Entries whose row and column are both in [row_begin, row_end) (global ids); duplicates
// are summed first.  |H_ij - conj(H_ji)| <= rtol * max |H_kl| for every such pair, a missing
// partner counting as 0.  Returns KPM_OK, or KPM_EINVAL / KPM_ERANGE with msg.
int check_hermitian(const int64_t* rp, const int64_t* col, const double* val, int64_t n_loc, int64_t row_begin,
                    int64_t row_end, int64_t n_global, double rtol, std::string& msg) {
  if (rp[0] != 0) {
    msg = "row_ptr[0] != 0";
    return KPM_EINVAL;
  }
  std::vector<Entry> e;
  e.reserve((size_t)rp[n_loc]);
  for (int64_t r = 0; r < n_loc; ++r) {
    if (rp[r + 1] < rp[r]) {
      msg = "row_ptr not non-decreasing";
      return KPM_EINVAL;
    }
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      if (col[k] < 0 || col[k] >= n_global) {
        msg = "column outside [0, n_global)";
        return KPM_ERANGE;
      }
      if (col[k] >= row_begin && col[k] < row_end) e.push_back({row_begin + r, col[k], val[2 * k], val[2 * k + 1]});
    }
  }
  std::sort(e.begin(), e.end(), key_less);
  size_t m = 0;  // sum duplicates
  for (size_t k = 0; k < e.size(); ++k) {
    if (m > 0 && e[m - 1].i == e[k].i && e[m - 1].j == e[k].j) {
      e[m - 1].re += e[k].re;
      e[m - 1].im += e[k].im;
    } else {
      e[m++] = e[k];
    }
  }
  e.resize(m);
  double hmax = 0.0;
  for (const Entry& x : e) hmax = std::max(hmax, std::hypot(x.re, x.im));
  const double tol = rtol * hmax;
  for (const Entry& x : e) {
    const Entry key{x.j, x.i, 0.0, 0.0};
    auto it = std::lower_bound(e.begin(), e.end(), key, key_less);
    const bool found = it != e.end() && it->i == x.j && it->j == x.i;
    const double dre = x.re - (found ? it->re : 0.0), dim = x.im + (found ? it->im : 0.0);
    if (std::hypot(dre, dim) > tol) {
      char buf[256];
      snprintf(buf, sizeof buf, "matrix is not Hermitian: H[%lld][%lld] = (%.17g, %.17g) but H[%lld][%lld] = (%.17g, %.17g)",
               (long long)x.i, (long long)x.j, x.re, x.im, (long long)x.j, (long long)x.i, found ? it->re : 0.0,
               found ? it->im : 0.0);
      msg = buf;
      return KPM_EINVAL;
    }
  }
  return KPM_OK;
}

}  // namespace kpm
