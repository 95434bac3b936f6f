// Row-pair entry order of the SELL-32 copy (R18b, §7 "Row-pair feed").
//
// The paper fixes neither the order of a row's entries nor how rows are grouped inside a
// chunk (SELL-C-sigma is only cited); the summation order it prescribes is that
// of the SpMV itself.  This pass permutes the entries *within* each row
// of a chunk so that two rows a and b = a ^ m of the chunk (m: one XOR mask per chunk) list
// the columns they have in common at the same positions 1..Ls; the row-pair sweep kernel
// (kernels.cu, aug_spmmv_pair) then loads each shared V row once for both rows.  For the
// TI Hamiltonian (Eq. (1)) the orbitals {0, 3} and {1, 2} of a site share their 8
// x/y-hopping columns (m = 3, Ls = 8 of 13 entries).
//
// Rule (oracle/sell_ref.py `pair_order` is the independent numpy reference):
//   * eligible chunk: 2 <= L <= 32 and every one of its 32 rows holds its own position at
//     entry 0 (the R18 diagonal-first order; padding rows qualify, their value is 0);
//   * for a mask m in 1..31 the rows a with bit lowbit(m) clear are paired with b = a ^ m;
//     s(a) = number of distinct columns other than the two own positions that both rows
//     list at entries >= 1; Ls(m) = min over the 16 pairs;
//   * m_c = the m with the largest Ls (smallest m on ties); Ls_c = Ls(m_c); if Ls_c = 0 the
//     chunk keeps the R18 order (pinfo = 0);
//   * otherwise every row keeps entry 0, then lists at entries 1..Ls_c the Ls_c smallest
//     shared columns in ascending order (each at its first occurrence in the row), then the
//     remaining entries in their R18 order (padding last).  pinfo[c] = m_c | Ls_c << 8.
// Values, columns and tile-row indices (lcol) move together; nothing else changes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kpm_internal.h"

namespace kpm {
namespace {

constexpr int kPairMaxL = 32;

__global__ void __launch_bounds__(32) pair_order_kernel(const int64_t* __restrict__ cptr, int64_t n_chunks,
                                                        double2* __restrict__ val, int* __restrict__ col,
                                                        uint16_t* __restrict__ lcol, int* __restrict__ pinfo) {
  __shared__ int sc[kPairMaxL][32];
  __shared__ double2 sv[kPairMaxL][32];
  __shared__ uint16_t sl[kPairMaxL][32];
  __shared__ unsigned char ord[32][kPairMaxL + 1];
  const int k = threadIdx.x;
  for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int64_t s0 = cptr[c];
    const int L = (int)((cptr[c + 1] - s0) >> 5);
    const int own = (int)(c * kC + k);
    __syncwarp();
    if (L < 2 || L > kPairMaxL) {  // uniform per chunk
      if (k == 0) pinfo[c] = 0;
      continue;
    }
    for (int j = 0; j < L; ++j) sc[j][k] = col[s0 + (int64_t)j * kC + k];
    __syncwarp();
    if (!__all_sync(0xffffffffu, sc[0][k] == own)) {
      if (k == 0) pinfo[c] = 0;
      continue;
    }
    auto is_shared = [&](int g, int p, int ownp) {  // g listed by row p at an entry >= 1
      if (g == own || g == ownp) return false;
      for (int j2 = 1; j2 < L; ++j2)
        if (sc[j2][p] == g) return true;
      return false;
    };
    int best_m = 0, best_ls = 0;
    for (int m = 1; m < 32; ++m) {
      const int lb = __ffs(m) - 1;
      int cnt = 0x7fffffff;
      if (((k >> lb) & 1) == 0) {
        const int p = k ^ m, ownp = (int)(c * kC + p);
        cnt = 0;
        for (int j = 1; j < L; ++j) {
          const int g = sc[j][k];
          bool first = true;
          for (int j2 = 1; j2 < j; ++j2)
            if (sc[j2][k] == g) first = false;
          if (first && is_shared(g, p, ownp)) ++cnt;
        }
      }
      const int ls = __reduce_min_sync(0xffffffffu, cnt);
      if (ls > best_ls) {
        best_ls = ls;
        best_m = m;
      }
    }
    if (best_ls == 0) {
      if (k == 0) pinfo[c] = 0;
      continue;
    }
    // new order of this lane's row: entry 0, the best_ls smallest shared columns, the rest
    const int p = k ^ best_m, ownp = (int)(c * kC + p);
    uint32_t used = 1u;
    ord[k][0] = 0;
    int n = 1;
    int last = INT32_MIN;
    bool have_last = false;
    for (int i = 0; i < best_ls; ++i) {
      int gmin = 0, jmin = -1;
      for (int j = 1; j < L; ++j) {
        const int g = sc[j][k];
        if ((have_last && g <= last) || (jmin >= 0 && g >= gmin)) continue;
        if (is_shared(g, p, ownp)) {
          gmin = g;
          jmin = j;  // first occurrence: later equal columns fail g >= gmin
        }
      }
      last = gmin;
      have_last = true;
      used |= 1u << jmin;
      ord[k][n++] = (unsigned char)jmin;
    }
    for (int j = 1; j < L; ++j)
      if (!(used >> j & 1u)) ord[k][n++] = (unsigned char)j;
    for (int j = 0; j < L; ++j) {
      sv[j][k] = val[s0 + (int64_t)j * kC + k];
      if (lcol) sl[j][k] = lcol[s0 + (int64_t)j * kC + k];
    }
    __syncwarp();
    for (int j = 0; j < L; ++j) {
      const int o = ord[k][j];
      const int64_t d = s0 + (int64_t)j * kC + k;
      val[d] = sv[o][k];
      col[d] = sc[o][k];
      if (lcol) lcol[d] = sl[o][k];
    }
    if (k == 0) pinfo[c] = best_m | (best_ls << 8);
  }
}

}  // namespace

cudaError_t launch_pair_order(const int64_t* cptr, int64_t n_chunks, double2* val, int* col, uint16_t* lcol,
                              int* pinfo, cudaStream_t s) {
  if (n_chunks <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>(n_chunks, 148 * 16);
  pair_order_kernel<<<grid, 32, 0, s>>>(cptr, n_chunks, val, col, lcol, pinfo);
  return cudaGetLastError();
}

}  // namespace kpm
