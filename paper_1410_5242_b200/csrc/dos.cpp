// Moment -> density-of-states reconstruction with the Jackson kernel (north_star subsystem 5;
// SURVEY §8(f) NEXT #1).  The paper calls this "a second computationally inexpensive step"
// and defines the DOS in Eq. (2) `DOS`; the kernel and the
// reconstruction formula are those of the KPM review it cites ([Weisse06]):
//   g_n = [(M-n+1) cos(pi n/(M+1)) + sin(pi n/(M+1)) cot(pi/(M+1))] / (M+1),
//   rho~(x) = [g_0 mu_0 + 2 sum_{n>=1} g_n mu_n T_n(x)] / (pi sqrt(1-x^2)),  x = a(E-b),
//   rho(E) = a rho~(x).
// O(M K) host work (Clenshaw summation per point), off the hot path.
#include <cmath>
#include <vector>

#include "../../include/kpm.h"

extern "C" kpm_status kpm_dos(int M, const double* mu, double a, double b, int K, const double* energies, int kernel,
                              double* E_out, double* rho_out) {
  if (M < 1 || !mu || K < 1 || !E_out || !rho_out || !(a > 0.0) || !std::isfinite(a) || !std::isfinite(b))
    return KPM_EINVAL;
  if (kernel != KPM_KERNEL_NONE && kernel != KPM_KERNEL_JACKSON) return KPM_EINVAL;
  const double pi = 3.14159265358979323846;
  std::vector<double> c(M);
  const double q = pi / (M + 1);
  for (int n = 0; n < M; ++n) {
    const double g = kernel == KPM_KERNEL_JACKSON
                         ? ((M - n + 1) * std::cos(q * n) + std::sin(q * n) * std::cos(q) / std::sin(q)) / (M + 1)
                         : 1.0;
    c[n] = (n == 0 ? 1.0 : 2.0) * g * mu[n];
  }
  for (int k = 0; k < K; ++k) {
    const double x = energies ? a * (energies[k] - b) : std::cos(pi * (k + 0.5) / K);
    E_out[k] = energies ? energies[k] : x / a + b;
    if (!(std::fabs(x) < 1.0)) {
      rho_out[k] = 0.0;  // outside the interval of orthogonality
      continue;
    }
    // Clenshaw: s = sum_n c_n T_n(x)
    double b1 = 0.0, b2 = 0.0;
    for (int n = M - 1; n >= 1; --n) {
      const double b0 = 2.0 * x * b1 - b2 + c[n];
      b2 = b1;
      b1 = b0;
    }
    const double s = x * b1 - b2 + c[0];
    rho_out[k] = a * s / (pi * std::sqrt(1.0 - x * x));
  }
  return KPM_OK;
}
