// Host-only diagnostic exports of the halo-exchange planning and the chunk order (include/kpm.h,
// kpm_plan_*).
// They run the same functions kpm_set_matrix uses (halo_plan.cpp) without CUDA or NCCL, so
// the multi-rank index logic is testable on a CPU (tests/test_halo_plan.py).
#include <algorithm>
#include <vector>

#include "../../include/kpm.h"
#include "chunk_order.h"
#include "halo_plan.h"

using namespace kpm;

extern "C" kpm_status kpm_plan_recv(int nranks, const int64_t* row_begins, int rank, const int64_t* row_ptr,
                                    const int64_t* col, int64_t* n_runs, int64_t* runs) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !row_begins || !row_ptr || !col || !n_runs) return KPM_EINVAL;
  std::vector<int64_t> rb(row_begins, row_begins + nranks + 1);
  for (int q = 0; q < nranks; ++q)
    if (rb[q + 1] < rb[q]) return KPM_EINVAL;
  const int64_t b = rb[rank], e = rb[rank + 1], n_loc = e - b;
  std::vector<int64_t> halo;
  for (int64_t k = 0; k < row_ptr[n_loc]; ++k) {
    if (col[k] < 0 || col[k] >= rb[nranks]) return KPM_ERANGE;
    if (col[k] < b || col[k] >= e) halo.push_back(col[k]);
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  const std::vector<RecvRun> rr = plan_recv_runs(halo, rb);
  if (runs) {
    if (*n_runs < (int64_t)rr.size()) return KPM_EINVAL;
    for (size_t i = 0; i < rr.size(); ++i) {
      runs[4 * i] = rr[i].peer;
      runs[4 * i + 1] = rr[i].gfirst;
      runs[4 * i + 2] = rr[i].count;
      runs[4 * i + 3] = rr[i].slot;
    }
  }
  *n_runs = (int64_t)rr.size();
  return KPM_OK;
}

extern "C" kpm_status kpm_plan_send(int64_t row_begin, int64_t row_end, int peer, int64_t n_req, const int64_t* req,
                                    int64_t* n_runs, int64_t* runs) {
  if (row_end < row_begin || n_req < 0 || (n_req && !req) || !n_runs) return KPM_EINVAL;
  const std::vector<int32_t> perm;  // sigma = 1: identity
  std::vector<int64_t> rq(req, req + 2 * n_req);
  std::vector<SendRun> out;
  if (!plan_send_runs(peer, rq, row_begin, row_end, perm, out)) return KPM_ERANGE;
  if (runs) {
    if (*n_runs < (int64_t)out.size()) return KPM_EINVAL;
    for (size_t i = 0; i < out.size(); ++i) {
      runs[3 * i] = out[i].peer;
      runs[3 * i + 1] = out[i].pos;
      runs[3 * i + 2] = out[i].count;
    }
  }
  *n_runs = (int64_t)out.size();
  return KPM_OK;
}

extern "C" kpm_status kpm_plan_chunk_order(int64_t n_chunks, const int64_t* nbr_ptr, const int64_t* nbr, int64_t grid,
                                           int width, const int8_t* skip, int64_t* order) {
  if (n_chunks < 0 || !nbr_ptr || (nbr_ptr[n_chunks] > 0 && !nbr) || grid < 1 || !order || width < 1 || width > 2)
    return KPM_EINVAL;
  std::vector<int64_t> ptr(nbr_ptr, nbr_ptr + n_chunks + 1), nb(nbr, nbr + nbr_ptr[n_chunks]);
  for (int64_t c = 0; c < n_chunks; ++c)
    if (ptr[c + 1] < ptr[c]) return KPM_EINVAL;
  for (int64_t b : nb)
    if (b < 0 || b >= n_chunks) return KPM_ERANGE;
  std::vector<char> sk;
  if (skip) sk.assign(skip, skip + n_chunks);
  const std::vector<int64_t> o = line_order(n_chunks, ptr, nb, grid, sk, width);
  std::copy(o.begin(), o.end(), order);
  return KPM_OK;
}
