// ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously correct CPU implementation of what the KPM-DOS hot path
// computes (arXiv:1410.5242, PAPER.md).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load this library.  It shares no
// code, header, table or constant generator with the CUDA path under
// paper_1410_5242_b200/csrc/, and it does not include anything from there.
//
// What it follows, step by step (PAPER.md line numbers, "P:n"):
//   * Chebyshev recurrence, Eq. (3) `eq:kpm_iter`:
//       |nu_1> = H~|nu_0>,  |nu_{m+1}> = 2 H~|nu_m> - |nu_{m-1}>,  H~ = a(H - b 1).
//   * scalar products eta_2m = <nu_m|nu_m>, eta_2m+1 = <nu_{m+1}|nu_m>,
//     <x|y> = sum_i conj(x_i) y_i.
//   * Fig. 3 `alg:kpm_naive`: outer loop over r, swap(w, v), then the BLAS-1
//     chain  u = H v ; u = u - b v ; w = -w ; w = w + 2a u ; eta_2m = <v|v> ; eta_2m+1 = <w|v>
//     (mode ORA_CHAINED), and Fig. 4 `alg:kpm_improved`, the same
//     operations fused per row w_i = 2a(sum_j H_ij v_j - b v_i) - w_i (mode ORA_FUSED).
//   * "Initialization steps and computation of eta_0, eta_1" read as
//     nu_1 = H~ nu_0 (Eq. 3), eta_0 = <nu_0|nu_0>, eta_1 = <nu_1|nu_0>   (R2).
//   * loop bound: M/2 matrix sweeps in total = the init sweep + (M/2 - 1) loop sweeps,
//     giving eta_0 .. eta_{M-1} ("the matrix only has to be read M/2 times", P:408;
//     Table I "RM/2" spmv calls)                                  (R1).
//   * eta -> mu (formula not printed; standard KPM doubling
//     T_m T_n = (T_{m+n} + T_|m-n|)/2):  m_0 = eta_0, m_1 = eta_1,
//     m_2k = 2 eta_2k - m_0, m_2k+1 = 2 eta_2k+1 - m_1;  stochastic trace
//     mu_n = (1/R) sum_r Re m_n^(r)                         (R4, R5).
//   * |rand()>: Z4 phases {1, i, -1, -i} chosen by the top two bits of word 0 of
//     Philox4x32-10 (Salmon et al., SC'11) with counter (row lo, row hi, column, 0) and
//     key (seed lo, seed hi)                                            (R6).
//
// Arithmetic: IEEE double, compiled with -ffp-contract=off (no FMA contraction), rows
// summed in stored CSR order, dot products summed in row order with Neumaier
// compensation.  OpenMP splits only element-wise loops (each row computed by one thread
// in the same order), so results are bitwise independent of the thread count.
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef std::complex<double> cplx;

enum { ORA_OK = 0, ORA_EINVAL = 1 };
enum { ORA_CHAINED = 0, ORA_FUSED = 1 };

// ---------------------------------------------------------------- Philox4x32-10 ----
// Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3", SC'11:
// round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
//        c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);  key bump k += (W0, W1) between rounds.
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  const uint32_t n0 = hi1 ^ c[1] ^ k[0];
  const uint32_t n2 = hi0 ^ c[3] ^ k[1];
  c[0] = n0;
  c[1] = lo1;
  c[2] = n2;
  c[3] = lo0;
}

extern "C" void ora_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k[0] += 0x9E3779B9u;
      k[1] += 0xBB67AE85u;
    }
    philox_round(c, k);
  }
  for (int i = 0; i < 4; ++i) out[i] = c[i];
}

// Z4 start-vector entry for global row i, global column r (R6).
static cplx z4_entry(uint64_t seed, int64_t i, int64_t r) {
  const uint64_t ui = (uint64_t)i;
  const uint32_t ctr[4] = {(uint32_t)ui, (uint32_t)(ui >> 32), (uint32_t)r, 0u};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  ora_philox4x32_10(ctr, key, out);
  switch (out[0] >> 30) {
    case 0: return cplx(1.0, 0.0);
    case 1: return cplx(0.0, 1.0);
    case 2: return cplx(-1.0, 0.0);
    default: return cplx(0.0, -1.0);
  }
}

// out[(i*R + r)*2 + {0,1}] = Z4(row_begin + i, col_begin + r)
extern "C" void ora_z4_block(int64_t row_begin, int64_t n_rows, int64_t col_begin, int R,
                             uint64_t seed, double* out) {
  for (int64_t i = 0; i < n_rows; ++i)
    for (int r = 0; r < R; ++r) {
      const cplx z = z4_entry(seed, row_begin + i, col_begin + r);
      out[(i * R + r) * 2 + 0] = z.real();
      out[(i * R + r) * 2 + 1] = z.imag();
    }
}

// ---------------------------------------------------------------- small helpers ----
static inline cplx cmul(cplx x, cplx y) {  // (xr + i xi)(yr + i yi), written out
  return cplx(x.real() * y.real() - x.imag() * y.imag(), x.real() * y.imag() + x.imag() * y.real());
}

// Neumaier-compensated running sum of one real component.
struct NSum {
  double s = 0.0, c = 0.0;
  void add(double x) {
    const double t = s + x;
    if (std::fabs(s) >= std::fabs(x))
      c += (s - t) + x;
    else
      c += (x - t) + s;
    s = t;
  }
  double value() const { return s + c; }
};

// <x|y> = sum_i conj(x_i) y_i, summed in row order.
static cplx dot(const std::vector<cplx>& x, const std::vector<cplx>& y) {
  NSum re, im;
  for (size_t i = 0; i < x.size(); ++i) {
    const cplx p = cmul(std::conj(x[i]), y[i]);
    re.add(p.real());
    im.add(p.imag());
  }
  return cplx(re.value(), im.value());
}

struct Csr {
  int64_t n;
  const int64_t* row_ptr;
  const int64_t* col;
  const cplx* val;
};

// u = H v   (spmv(), Table I; each row summed in stored order)
static void spmv(const Csr& H, const std::vector<cplx>& v, std::vector<cplx>& u) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < H.n; ++i) {
    cplx s(0.0, 0.0);
    for (int64_t k = H.row_ptr[i]; k < H.row_ptr[i + 1]; ++k) s += cmul(H.val[k], v[H.col[k]]);
    u[i] = s;
  }
}

// One column of Fig. 3 / Fig. 4: eta[0..M-1] for start vector v0.
static void kpm_column(const Csr& H, double a, double b, int M, const std::vector<cplx>& v0,
                       int mode, cplx* eta) {
  const int64_t n = H.n;
  std::vector<cplx> v(v0), w(n), u(n);
  // Initialization steps (Eq. 3): w = nu_1 = a (H v - b v); eta_0, eta_1.
  spmv(H, v, u);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    u[i] = u[i] - b * v[i];
    w[i] = a * u[i];
  }
  eta[0] = dot(v, v);
  eta[1] = dot(w, v);
  const double two_a = 2.0 * a;
  for (int m = 1; m < M / 2; ++m) {
    std::swap(v, w);  // swap(|w>, |v>)  ("not performed explicitly")
    if (mode == ORA_CHAINED) {
      spmv(H, v, u);  // u = H v                 spmv()
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) u[i] = u[i] - b * v[i];  // u = u - b v    axpy()
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) w[i] = -w[i];  // w = -w          scal()
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) w[i] = w[i] + two_a * u[i];  // w = w + 2a u   axpy()
    } else {
      // aug_spmv(): w = 2a(H - b 1) v - w  (Fig. 4), one pass over the rows
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        cplx s(0.0, 0.0);
        for (int64_t k = H.row_ptr[i]; k < H.row_ptr[i + 1]; ++k) s += cmul(H.val[k], v[H.col[k]]);
        s = s - b * v[i];
        w[i] = two_a * s - w[i];
      }
    }
    eta[2 * m] = dot(v, v);          // nrm2()
    eta[2 * m + 1] = dot(w, v);      // dot()
  }
}

static int check_args(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                      double a, double b, int M, int R) {
  if (n < 1 || !row_ptr || !col || !val) return ORA_EINVAL;
  if (M < 2 || (M % 2) != 0 || R < 1) return ORA_EINVAL;
  if (!(a > 0.0) || !std::isfinite(a) || !std::isfinite(b)) return ORA_EINVAL;
  if (row_ptr[0] != 0) return ORA_EINVAL;
  for (int64_t i = 0; i < n; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return ORA_EINVAL;
  for (int64_t k = 0; k < row_ptr[n]; ++k)
    if (col[k] < 0 || col[k] >= n) return ORA_EINVAL;
  return ORA_OK;
}

// eta for R explicit start vectors v0[(i*R + r)*2 + {re,im}] (row-major block).
// eta_out[(r*M + n)*2 + {re,im}] = eta_n of column r.
extern "C" int ora_kpm_eta_v0(int64_t n, const int64_t* row_ptr, const int64_t* col,
                              const double* val, double a, double b, int M, int R,
                              const double* v0, int mode, int nthreads, double* eta_out) {
  int st = check_args(n, row_ptr, col, val, a, b, M, R);
  if (st != ORA_OK || !v0 || !eta_out) return ORA_EINVAL;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  Csr H{n, row_ptr, col, reinterpret_cast<const cplx*>(val)};
  std::vector<cplx> v(n);
  for (int r = 0; r < R; ++r) {  // outer loop over random vectors (Fig. 3)
    for (int64_t i = 0; i < n; ++i) v[i] = cplx(v0[(i * R + r) * 2], v0[(i * R + r) * 2 + 1]);
    kpm_column(H, a, b, M, v, mode, reinterpret_cast<cplx*>(eta_out) + (size_t)r * M);
  }
  return ORA_OK;
}

// Same with |rand()> = Z4 Philox start vectors for global columns col_begin .. col_begin+R-1.
extern "C" int ora_kpm_eta(int64_t n, const int64_t* row_ptr, const int64_t* col,
                           const double* val, double a, double b, int M, int R, uint64_t seed,
                           int64_t col_begin, int mode, int nthreads, double* eta_out) {
  int st = check_args(n, row_ptr, col, val, a, b, M, R);
  if (st != ORA_OK || !eta_out) return ORA_EINVAL;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  Csr H{n, row_ptr, col, reinterpret_cast<const cplx*>(val)};
  std::vector<cplx> v(n);
  for (int r = 0; r < R; ++r) {
    for (int64_t i = 0; i < n; ++i) v[i] = z4_entry(seed, i, col_begin + r);  // |rand()>
    kpm_column(H, a, b, M, v, mode, reinterpret_cast<cplx*>(eta_out) + (size_t)r * M);
  }
  return ORA_OK;
}

// Per-column moments m_n^(r) from eta (doubling identities) and the stochastic trace
// mu_n = (1/R) sum_r Re m_n^(r).  m_out may be NULL.
extern "C" void ora_eta_to_mu(int M, int R, const double* eta, double* mu, double* m_out) {
  const cplx* e = reinterpret_cast<const cplx*>(eta);
  std::vector<cplx> m(M);
  for (int n = 0; n < M; ++n) mu[n] = 0.0;
  for (int r = 0; r < R; ++r) {
    const cplx* er = e + (size_t)r * M;
    m[0] = er[0];
    m[1] = er[1];
    for (int k = 1; 2 * k < M; ++k) {
      m[2 * k] = 2.0 * er[2 * k] - m[0];
      m[2 * k + 1] = 2.0 * er[2 * k + 1] - m[1];
    }
    for (int n = 0; n < M; ++n) {
      mu[n] += m[n].real();
      if (m_out) {
        m_out[((size_t)r * M + n) * 2] = m[n].real();
        m_out[((size_t)r * M + n) * 2 + 1] = m[n].imag();
      }
    }
  }
  for (int n = 0; n < M; ++n) mu[n] /= (double)R;
}

extern "C" int ora_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
