/* Plain-C caller of libkpm.so (the boundary is a C ABI).  Reads a CSR matrix
 * from a binary file, runs kpm_create / kpm_set_matrix / kpm_moments / kpm_destroy and prints
 * the moments, one per line.  Used by tests/test_abi.py (no GPU: kpm_create must fail with a
 * message, exit 2) and tests/test_gpu_parity.py (C1 moments vs the oracle).
 *
 * usage: kpm_c_demo FILE a b M R seed
 * FILE: int64 n, int64 nnz, int64 row_ptr[n+1], int64 col[nnz], double val[2*nnz] (re, im). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "kpm.h"

static void* read_n(FILE* f, size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p || fread(p, 1, bytes, f) != bytes) {
    fprintf(stderr, "short read\n");
    exit(3);
  }
  return p;
}

int main(int argc, char** argv) {
  if (argc != 7) {
    fprintf(stderr, "usage: %s FILE a b M R seed\n", argv[0]);
    return 1;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  int64_t hdr[2];
  if (fread(hdr, sizeof(int64_t), 2, f) != 2) return 3;
  const int64_t n = hdr[0], nnz = hdr[1];
  int64_t* rp = (int64_t*)read_n(f, sizeof(int64_t) * (size_t)(n + 1));
  int64_t* col = (int64_t*)read_n(f, sizeof(int64_t) * (size_t)nnz);
  double* val = (double*)read_n(f, sizeof(double) * 2 * (size_t)nnz);
  fclose(f);
  const double a = atof(argv[2]), b = atof(argv[3]);
  const int M = atoi(argv[4]), R = atoi(argv[5]);
  const uint64_t seed = strtoull(argv[6], NULL, 0);

  kpm_options opt = {0};
  opt.nranks = 1;
  kpm_ctx* ctx = NULL;
  kpm_status st = kpm_create(&ctx, &opt);
  if (st != KPM_OK) {
    fprintf(stderr, "kpm_create: status %d: %s\n", (int)st, kpm_last_error(NULL));
    return 2;
  }
  kpm_csr H;
  H.n_global = n;
  H.row_begin = 0;
  H.row_end = n;
  H.row_ptr = rp;
  H.col = col;
  H.val = val;
  H.mem = KPM_MEM_HOST;
  double* mu = (double*)malloc(sizeof(double) * (size_t)M);
  st = kpm_set_matrix(ctx, &H, a, b);
  if (st == KPM_OK) st = kpm_moments(ctx, M, R, seed, mu, NULL);
  if (st != KPM_OK && st != KPM_WDIVERGED) {
    fprintf(stderr, "kpm: status %d: %s\n", (int)st, kpm_last_error(ctx));
    kpm_destroy(ctx);
    return 4;
  }
  for (int i = 0; i < M; ++i) printf("%.17g\n", mu[i]);
  kpm_destroy(ctx);
  free(mu);
  free(rp);
  free(col);
  free(val);
  return 0;
}
