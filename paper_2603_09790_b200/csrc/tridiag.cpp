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

// Cyclic Jacobi rotations on a copy of the s x s (s <= 64) Gram matrix; used
// for kappa_2(W) of the collect_gram hook (the reference calls dsyevd there,
// solver.cpp:69-74). Converges quadratically; eigenvalues sorted ascending.
void sym_eigenvalues(int s, const double* w, double* out) {
  std::vector<double> a(w, w + static_cast<size_t>(s) * s);
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) + static_cast<size_t>(j) * s]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < s; ++i) {
        tot += A(i, j) * A(i, j);
        if (i != j) off += A(i, j) * A(i, j);
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int pp = 0; pp < s - 1; ++pp)
      for (int q = pp + 1; q < s; ++q) {
        const double apq = A(pp, q);
        if (apq == 0.0) continue;
        const double theta = (A(q, q) - A(pp, pp)) / (2.0 * apq);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(tt * tt + 1.0), sn = tt * c;
        for (int k = 0; k < s; ++k) {  // columns pp, q
          const double akp = A(k, pp), akq = A(k, q);
          A(k, pp) = c * akp - sn * akq;
          A(k, q) = sn * akp + c * akq;
        }
        for (int k = 0; k < s; ++k) {  // rows pp, q
          const double apk = A(pp, k), aqk = A(q, k);
          A(pp, k) = c * apk - sn * aqk;
          A(q, k) = sn * apk + c * aqk;
        }
      }
  }
  for (int i = 0; i < s; ++i) out[i] = A(i, i);
  std::sort(out, out + s);
}

}  // namespace csg
