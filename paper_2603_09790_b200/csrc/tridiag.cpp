// tridiag.cpp -- eigenvalues of the Lanczos tridiagonal (<= 256 x 256).
//
// Replaces LAPACK dsterf (lapack.cpp:61-71), which the reference calls on the
// 40 Lanczos coefficients. This is bisection on Sturm sequence counts: each
// eigenvalue is bracketed inside the Gershgorin interval and halved until the
// bracket cannot shrink in floating point. It works on 40 numbers, after the
// device has done all n-sized work, so it is not a CPU fallback of the solve.
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "lanczos.cuh"

namespace csg {
namespace {

// number of eigenvalues strictly less than x
int sturm_count(int m, const double* d, const double* e2, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (std::fabs(q) < pivmin) q = -pivmin;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < m; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (std::fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

}  // namespace

void tridiag_eigenvalues(int m, const double* d, const double* e, double* out) {
  if (m <= 0) return;
  std::vector<double> e2(std::max(m - 1, 1), 0.0);
  double lo = d[0], hi = d[0], emax = 0.0;
  for (int i = 0; i < m; ++i) {
    const double left = (i > 0 ? std::fabs(e[i - 1]) : 0.0);
    const double right = (i + 1 < m ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - left - right);
    hi = std::max(hi, d[i] + left + right);
    if (i + 1 < m) {
      e2[i] = e[i] * e[i];
      emax = std::max(emax, e2[i]);
    }
  }
  const double span = std::max(std::fabs(lo), std::fabs(hi));
  const double pivmin = std::numeric_limits<double>::min() * std::max(1.0, emax);
  lo -= 2.0 * std::numeric_limits<double>::epsilon() * span + pivmin;
  hi += 2.0 * std::numeric_limits<double>::epsilon() * span + pivmin;
  for (int k = 0; k < m; ++k) {
    double a = lo, b = hi;  // invariant: count(a) <= k < count(b)
    for (int it = 0; it < 4096; ++it) {
      const double mid = 0.5 * (a + b);
      if (!(mid > a && mid < b)) break;
      if (sturm_count(m, d, e2.data(), mid, pivmin) > k) b = mid;
      else a = mid;
    }
    out[k] = 0.5 * (a + b);
  }
}

}  // namespace csg
