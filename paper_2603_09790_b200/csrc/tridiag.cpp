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

// Largest singular value of a column-major s x s matrix: sqrt of the largest
// eigenvalue of M^T M (Jacobi). Used by fgs_rate where the reference calls
// dgesvd (gram.cpp:170, lapack.cpp:37-47) and takes the front (largest) value.
double max_singular_value(int s, const double* m) {
  if (s == 0) return 0.0;
  std::vector<double> g(static_cast<size_t>(s) * s), ev(s);
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < s; ++i) {
      double acc = 0.0;
      for (int k = 0; k < s; ++k) acc += m[k + static_cast<size_t>(i) * s] * m[k + static_cast<size_t>(j) * s];
      g[i + static_cast<size_t>(j) * s] = acc;
    }
  sym_eigenvalues(s, g.data(), ev.data());
  return std::sqrt(std::max(0.0, ev[s - 1]));
}

// Moduli of the eigenvalues of a general column-major n x n matrix (the
// reference calls dgeev, lapack.cpp:49-59): reduction to upper Hessenberg
// form by stabilised elimination, then Francis double-shift QR with
// deflation on the Hessenberg matrix (eigenvalues only).
void general_eig_moduli(int n, const double* m, double* out) {
  std::vector<double> h(static_cast<size_t>(n) * n);
  auto A = [&](int i, int j) -> double& { return h[static_cast<size_t>(i) * n + j]; };
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) A(i, j) = m[i + static_cast<size_t>(j) * n];
  // Hessenberg reduction
  for (int c = 1; c < n - 1; ++c) {
    int piv = c;
    double x = 0.0;
    for (int r = c; r < n; ++r)
      if (std::fabs(A(r, c - 1)) > std::fabs(x)) x = A(r, c - 1), piv = r;
    if (piv != c) {
      for (int j = c - 1; j < n; ++j) std::swap(A(piv, j), A(c, j));
      for (int i = 0; i < n; ++i) std::swap(A(i, piv), A(i, c));
    }
    if (x == 0.0) continue;
    for (int r = c + 1; r < n; ++r) {
      double y = A(r, c - 1);
      if (y == 0.0) continue;
      y /= x;
      A(r, c - 1) = 0.0;
      for (int j = c; j < n; ++j) A(r, j) -= y * A(c, j);
      for (int i = 0; i < n; ++i) A(i, c) += y * A(i, r);
    }
  }
  std::vector<double> wr(n, 0.0), wi(n, 0.0);
  double anorm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(i - 1, 0); j < n; ++j) anorm += std::fabs(A(i, j));
  auto sgn = [](double a, double b) { return b >= 0.0 ? std::fabs(a) : -std::fabs(a); };
  int nn = n - 1;
  double t = 0.0;
  bool failed = false;
  while (nn >= 0 && !failed) {
    int its = 0, l;
    do {
      for (l = nn; l >= 1; --l) {
        double sc = std::fabs(A(l - 1, l - 1)) + std::fabs(A(l, l));
        if (sc == 0.0) sc = anorm;
        if (std::fabs(A(l, l - 1)) + sc == sc) {
          A(l, l - 1) = 0.0;
          break;
        }
      }
      double x = A(nn, nn);
      if (l == nn) {  // one root
        wr[nn] = x + t;
        wi[nn] = 0.0;
        --nn;
      } else {
        double y = A(nn - 1, nn - 1), w = A(nn, nn - 1) * A(nn - 1, nn);
        if (l == nn - 1) {  // two roots
          const double p = 0.5 * (y - x), q = p * p + w;
          double z = std::sqrt(std::fabs(q));
          x += t;
          if (q >= 0.0) {
            z = p + sgn(z, p);
            wr[nn - 1] = wr[nn] = x + z;
            if (z != 0.0) wr[nn] = x - w / z;
            wi[nn - 1] = wi[nn] = 0.0;
          } else {
            wr[nn - 1] = wr[nn] = x + p;
            wi[nn - 1] = -z;
            wi[nn] = z;
          }
          nn -= 2;
        } else {
          if (its == 60) {
            failed = true;
            break;
          }
          if (its == 10 || its == 20 || its == 40) {  // exceptional shift
            t += x;
            for (int i = 0; i <= nn; ++i) A(i, i) -= x;
            const double sc = std::fabs(A(nn, nn - 1)) + std::fabs(A(nn - 1, nn - 2));
            y = x = 0.75 * sc;
            w = -0.4375 * sc * sc;
          }
          ++its;
          int mm;
          double p = 0.0, q = 0.0, r = 0.0, z;
          for (mm = nn - 2; mm >= l; --mm) {
            z = A(mm, mm);
            r = x - z;
            double sc = y - z;
            p = (r * sc - w) / A(mm + 1, mm) + A(mm, mm + 1);
            q = A(mm + 1, mm + 1) - z - r - sc;
            r = A(mm + 2, mm + 1);
            sc = std::fabs(p) + std::fabs(q) + std::fabs(r);
            p /= sc, q /= sc, r /= sc;
            if (mm == l) break;
            const double u = std::fabs(A(mm, mm - 1)) * (std::fabs(q) + std::fabs(r));
            const double v = std::fabs(p) * (std::fabs(A(mm - 1, mm - 1)) + std::fabs(z) +
                                             std::fabs(A(mm + 1, mm + 1)));
            if (u + v == v) break;
          }
          for (int i = mm + 2; i <= nn; ++i) {
            A(i, i - 2) = 0.0;
            if (i != mm + 2) A(i, i - 3) = 0.0;
          }
          for (int k = mm; k <= nn - 1; ++k) {
            if (k != mm) {
              p = A(k, k - 1);
              q = A(k + 1, k - 1);
              r = k != nn - 1 ? A(k + 2, k - 1) : 0.0;
              if ((x = std::fabs(p) + std::fabs(q) + std::fabs(r)) != 0.0) p /= x, q /= x, r /= x;
            }
            const double sc = sgn(std::sqrt(p * p + q * q + r * r), p);
            if (sc == 0.0) continue;
            if (k == mm) {
              if (l != mm) A(k, k - 1) = -A(k, k - 1);
            } else {
              A(k, k - 1) = -sc * x;
            }
            p += sc;
            x = p / sc;
            y = q / sc;
            z = r / sc;
            q /= p;
            r /= p;
            for (int j = k; j <= nn; ++j) {
              p = A(k, j) + q * A(k + 1, j);
              if (k != nn - 1) {
                p += r * A(k + 2, j);
                A(k + 2, j) -= p * z;
              }
              A(k + 1, j) -= p * y;
              A(k, j) -= p * x;
            }
            const int mmin = nn < k + 3 ? nn : k + 3;
            for (int i = l; i <= mmin; ++i) {
              p = x * A(i, k) + y * A(i, k + 1);
              if (k != nn - 1) {
                p += z * A(i, k + 2);
                A(i, k + 2) -= p * r;
              }
              A(i, k + 1) -= p * q;
              A(i, k) -= p;
            }
          }
        }
      }
    } while (!failed && l < nn - 1);
  }
  for (int i = 0; i < n; ++i)
    out[i] = failed ? std::numeric_limits<double>::quiet_NaN() : std::hypot(wr[i], wi[i]);
}

}  // namespace csg
