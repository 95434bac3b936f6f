#pragma once
#include <stdint.h>

#include <string>
#include <vector>

namespace kpm {

struct HostSell {
  int64_t n_loc = 0, n_pad = 0, n_chunks = 0, n_halo = 0;
  int C = 32, sigma = 1;
  std::vector<double> val;     // 2*n_slots (re, im)
  std::vector<int32_t> col;    // n_slots
  std::vector<int64_t> cptr;   // n_chunks+1
  std::vector<int32_t> perm;   // n_loc
  std::vector<int64_t> halo;   // n_halo global ids, ascending
};

// Returns 0 or a kpm_status code (err filled).
int build_sell_host(const int64_t* row_ptr, const int64_t* col, const double* val, int64_t n_loc,
                    int64_t row_begin, int64_t row_end, int C, int sigma, HostSell& out, std::string& err);

}  // namespace kpm
