/* cs_oracle.c -- TEST INFRASTRUCTURE ONLY. CPU restatement ("port") of the
 * reference chebstep solve path, in plain C, used as the parity checker for
 * the CUDA product and as the "port" CPU baseline. It is never linked into,
 * called by, or shipped with the product (paper_2603_09790_b200).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Arithmetic follows the reference per-element
 * operation sequence exactly: separate multiply and add roundings (the
 * reference builds with -ffp-contract=off, CMakeLists.txt:11-15; this file is
 * compiled the same way), serial ascending-index reductions, the same loop
 * orders, true divisions. It is pinned against the compiled reference
 * (oracle/_ref) and the golden fixtures in tests/golden/ by
 * tests/test_oracle.py.
 *
 * The one intentional deviation: tridiagonal Ritz values come from an
 * implicit QL iteration (EISPACK tql1 style) instead of LAPACK dsterf
 * (lapack.cpp:61-71). Both are backward stable; results agree to ~1e-15
 * relative in lambda_max and ~1e-13 in lambda_min (tested).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_abi.h"

enum { OK = 0, E_DIM = 1, E_MATRIX = 2, E_NOTSPD = 3, E_BASIS = 4, E_SOLVER = 5,
       E_GUARD = 6, E_PARSE = 7, E_ARG = 8, E_GENERIC = 9, E_NOMEM = 9 };

static _Thread_local char g_msg[256];
static _Thread_local int g_payload;

static int fail(int code, int payload, const char* msg) {
  g_payload = payload;
  snprintf(g_msg, sizeof g_msg, "%s", msg);
  return code;
}

const char* orc_last_error(int* payload) {
  if (payload) *payload = g_payload;
  return g_msg;
}

#define TRY(expr)              \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != OK) return rc_; \
  } while (0)

/* ---------------------------------------------------------------- util */

/* util.hpp:25-40 SplitMix64; util.cpp:31-36 random_vector */
int orc_random_vector(int64_t n, uint64_t seed, double* out) {
  uint64_t state = seed;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    const double unit = (double)(z >> 11) * 0x1.0p-53;
    out[i] = 2.0 * unit - 1.0;
  }
  return OK;
}

/* dense_ops.cpp:10-17 */
static double dot(int64_t n, const double* x, const double* y) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc = acc + x[i] * y[i];
  return acc;
}
static double norm2(int64_t n, const double* x) { return sqrt(dot(n, x, x)); }

/* kernels_scalar.cpp:6-8 */
static void axpy(int64_t n, double a, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = y[i] + a * x[i];
}
/* kernels_scalar.cpp:10-12 */
static void xpby(int64_t n, const double* x, double b, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = x[i] + b * y[i];
}
/* kernels_scalar.cpp:14-20 */
static void lincomb3(int64_t n, double a, const double* x, double b, const double* y, double c,
                     const double* z, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double t = a * x[i] + b * y[i];
    out[i] = t + c * z[i];
  }
}
/* kernels_scalar.cpp:22-33 (the AVX2 variant, kernels_avx2.cpp:57-110, keeps
 * the same per-entry ascending chain, hence is bitwise equal) */
static void gram(int64_t n, int ucols, int vcols, const double* u, const double* v, double* g) {
  for (int j = 0; j < vcols; ++j)
    for (int i = 0; i < ucols; ++i) {
      const double* ui = u + (int64_t)i * n;
      const double* vj = v + (int64_t)j * n;
      double acc = 0.0;
      for (int64_t l = 0; l < n; ++l) acc = acc + ui[l] * vj[l];
      g[i + j * ucols] = acc;
    }
}

/* block.cpp:53-57 */
static double frobenius(int len, const double* m) {
  double acc = 0.0;
  for (int i = 0; i < len; ++i) acc += m[i] * m[i];
  return sqrt(acc);
}

static void* xcalloc(int64_t count, size_t size) {
  return calloc((size_t)(count > 0 ? count : 1), size);
}

/* ---------------------------------------------------------------- problems */

/* problems.cpp:13-53 -- HPCG 27-point, (dz,dy,dx) lexicographic loops give
 * ascending columns; diagonal 26, in-grid neighbours -1. Caller sizes the
 * arrays: rowptr n+1, col/val (3nx-2)(3ny-2)(3nz-2) (for n>1 dims). */
int orc_poisson27_fill(int64_t nx, int64_t ny, int64_t nz, int64_t* rowptr, int64_t* col,
                       double* val) {
  if (nx < 1 || ny < 1 || nz < 1) return fail(E_ARG, 0, "poisson27: grid dimensions must be >= 1");
  const int64_t kmax = (int64_t)1 << 31;
  if (nx > kmax / ny || nx * ny > kmax / nz) return fail(E_ARG, 0, "poisson27: grid size overflow");
  int64_t row = 0, k = 0;
  rowptr[0] = 0;
  for (int64_t iz = 0; iz < nz; ++iz)
    for (int64_t iy = 0; iy < ny; ++iy)
      for (int64_t ix = 0; ix < nx; ++ix, ++row) {
        for (int64_t dz = -1; dz <= 1; ++dz) {
          const int64_t jz = iz + dz;
          if (jz < 0 || jz >= nz) continue;
          for (int64_t dy = -1; dy <= 1; ++dy) {
            const int64_t jy = iy + dy;
            if (jy < 0 || jy >= ny) continue;
            for (int64_t dx = -1; dx <= 1; ++dx) {
              const int64_t jx = ix + dx;
              if (jx < 0 || jx >= nx) continue;
              const int64_t c = jx + nx * (jy + ny * jz);
              col[k] = c;
              val[k] = (c == row) ? 26.0 : -1.0;
              ++k;
            }
          }
        }
        rowptr[row + 1] = k;
      }
  return OK;
}

/* NEW (no reference function): 7-point operator with
 * per-direction coefficients, following poisson27's conventions
 * (problems.cpp:28-51): x-fastest rows, strictly ascending columns,
 * diagonal 2(cx+cy+cz) = sum of the full-grid off-diagonal magnitudes,
 * off-diagonals -c_dir for in-grid neighbours. (1,1,1) is poisson7;
 * (1,1,100) is the config-4 anisotropic operator. */
int orc_stencil7_fill(int64_t nx, int64_t ny, int64_t nz, double cx, double cy, double cz,
                      int64_t* rowptr, int64_t* col, double* val) {
  if (nx < 1 || ny < 1 || nz < 1) return fail(E_ARG, 0, "stencil7: grid dimensions must be >= 1");
  const double diag = 2.0 * (cx + cy + cz);
  const int64_t pxy = nx * ny;
  int64_t row = 0, k = 0;
  rowptr[0] = 0;
  for (int64_t iz = 0; iz < nz; ++iz)
    for (int64_t iy = 0; iy < ny; ++iy)
      for (int64_t ix = 0; ix < nx; ++ix, ++row) {
        if (iz > 0) { col[k] = row - pxy; val[k++] = -cz; }
        if (iy > 0) { col[k] = row - nx; val[k++] = -cy; }
        if (ix > 0) { col[k] = row - 1; val[k++] = -cx; }
        col[k] = row; val[k++] = diag;
        if (ix + 1 < nx) { col[k] = row + 1; val[k++] = -cx; }
        if (iy + 1 < ny) { col[k] = row + nx; val[k++] = -cy; }
        if (iz + 1 < nz) { col[k] = row + pxy; val[k++] = -cz; }
        rowptr[row + 1] = k;
      }
  return OK;
}

/* ---------------------------------------------------------------- csr / precond */

/* csr.cpp:111-124 -- row-serial, stored column order, acc = acc + v*x */
int orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x,
             double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc = acc + v[k] * x[ci[k]];
    y[i] = acc;
  }
  return OK;
}

/* csr.cpp:10-15 -- lower_bound over the row's sorted columns */
static double diagonal(const int64_t* rp, const int64_t* ci, const double* v, int64_t i) {
  int64_t lo = rp[i], hi = rp[i + 1];
  const int64_t end = hi;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (ci[mid] < i) lo = mid + 1;
    else hi = mid;
  }
  if (lo == end || ci[lo] != i) return 0.0;
  return v[lo];
}

/* precond.cpp:15-23 */
int orc_jacobi_invdiag(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                       double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double d = diagonal(rp, ci, v, i);
    if (!(d > 0.0)) return fail(E_NOTSPD, 0, "jacobi: diagonal must be strictly positive");
    out[i] = 1.0 / d;
  }
  return OK;
}

typedef struct {
  int kind;          /* 0 identity, 1 jacobi */
  double* inv_diag;  /* jacobi only */
} precond_t;

static int precond_make(precond_t* m, int kind, int64_t n, const int64_t* rp, const int64_t* ci,
                        const double* v) {
  m->kind = kind;
  m->inv_diag = NULL;
  if (kind == 0) return OK;
  if (kind != 1) return fail(E_ARG, 0, "unknown preconditioner kind");
  m->inv_diag = (double*)xcalloc(n, sizeof(double));
  if (!m->inv_diag) return fail(E_NOMEM, 0, "out of memory");
  const int rc = orc_jacobi_invdiag(n, rp, ci, v, m->inv_diag);
  if (rc != OK) {
    free(m->inv_diag);
    m->inv_diag = NULL;
  }
  return rc;
}
static void precond_free(precond_t* m) { free(m->inv_diag); }

/* precond.cpp:9-13 (identity: bitwise copy) and 25-30 (jacobi: inv_d*in) */
static void precond_apply(const precond_t* m, int64_t n, const double* in, double* out) {
  if (m->kind == 0) {
    memmove(out, in, sizeof(double) * (size_t)n);
    return;
  }
  for (int64_t i = 0; i < n; ++i) out[i] = m->inv_diag[i] * in[i];
}

/* ---------------------------------------------------------------- mpk */

static int all_finite(int64_t n, const double* x) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

/* mpk.cpp:11-16 ChebyshevParams::from_interval */
static int cheb_check(double lo, double hi) {
  if (!(hi > lo) || !(lo > 0.0) || !isfinite(hi))
    return fail(E_ARG, 0, "ChebyshevParams: need lambda_max > lambda_min > 0");
  return OK;
}

/* mpk.cpp:26-71 -- Alg. 2; z n x s, p n x (s+1), zp scratch n x s */
static int mpk_core(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    const precond_t* m, const double* r, int s, double lo, double hi, double* z,
                    double* p) {
  if (s < 1) return fail(E_ARG, 0, "mpk: s must be >= 1");
  const double alpha = 2.0 / (hi - lo);                /* mpk.hpp:22 */
  const double sigma = (hi + lo) / (hi - lo);          /* mpk.hpp:23-25 */
  const double gamma = 1.0;                            /* mpk.hpp:26 */
  double* zp = (double*)xcalloc(n * s, sizeof(double));
  if (!zp) return fail(E_NOMEM, 0, "out of memory");
  char msg[64];
#define COL(b, j) ((b) + (int64_t)(j) * n)
#define CHECK(vec, c)                                                  \
  do {                                                                 \
    if (!all_finite(n, (vec))) {                                       \
      free(zp);                                                        \
      snprintf(msg, sizeof msg, "mpk: non-finite basis column %d", (c) + 1); \
      return fail(E_BASIS, (c), msg);                                  \
    }                                                                  \
  } while (0)
  memcpy(COL(p, 0), r, sizeof(double) * (size_t)n);
  memcpy(COL(zp, 0), r, sizeof(double) * (size_t)n);
  precond_apply(m, n, COL(zp, 0), COL(z, 0));
  CHECK(COL(z, 0), 0);
  if (s > 1) {
    orc_spmv(n, rp, ci, v, COL(z, 0), COL(p, 1));
    lincomb3(n, alpha, COL(p, 1), -sigma, COL(zp, 0), 0.0, COL(zp, 0), COL(zp, 1));
    precond_apply(m, n, COL(zp, 1), COL(z, 1));
    CHECK(COL(z, 1), 1);
    for (int q = 2; q < s; ++q) {
      orc_spmv(n, rp, ci, v, COL(z, q - 1), COL(p, q));
      lincomb3(n, 2.0 * alpha, COL(p, q), -2.0 * sigma, COL(zp, q - 1), -gamma, COL(zp, q - 2),
               COL(zp, q));
      precond_apply(m, n, COL(zp, q), COL(z, q));
      CHECK(COL(z, q), q);
    }
  }
  orc_spmv(n, rp, ci, v, COL(z, s - 1), COL(p, s));
  CHECK(COL(p, s), s - 1);
#undef CHECK
  free(zp);
  return OK;
}

int orc_mpk(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int precond,
            const double* r, int s, double lo, double hi, double* z, double* p) {
  precond_t m;
  TRY(precond_make(&m, precond, n, rp, ci, v));
  int rc = cheb_check(lo, hi);
  if (rc == OK) {
    memset(z, 0, sizeof(double) * (size_t)(n * s));
    memset(p, 0, sizeof(double) * (size_t)(n * (s + 1)));
    rc = mpk_core(n, rp, ci, v, &m, r, s, lo, hi, z, p);
  }
  precond_free(&m);
  return rc;
}

/* ---------------------------------------------------------------- dense ops */

/* dense_ops.cpp:19-27 */
int orc_block_gram(int64_t n, int ku, int kv, const double* u, const double* w, double* g) {
  if (ku > 64 || kv > 64) return fail(E_DIM, 0, "SmallDense: dimensions must be in [0, 64]");
  gram(n, ku, kv, u, w, g);
  return OK;
}

/* dense_ops.cpp:29-42 -- out = y; out_j += c_qj x_q for q ascending */
int orc_block_update(int64_t n, int m, int k, const double* y, const double* x, const double* c,
                     double* out) {
  if (out != y) memcpy(out, y, sizeof(double) * (size_t)(n * k));
  for (int j = 0; j < k; ++j)
    for (int q = 0; q < m; ++q) axpy(n, c[q + j * m], x + (int64_t)q * n, out + (int64_t)j * n);
  return OK;
}

/* gram.cpp:22-35 finish_assembly: diagonal positive and finite */
static int finish_assembly(int s, const double* w) {
  for (int i = 0; i < s; ++i) {
    const double d = w[i + i * s];
    if (!(d > 0.0) || !isfinite(d))
      return fail(E_NOTSPD, 0, "gram: non-positive diagonal (basis degeneracy)");
  }
  return OK;
}

/* gram.cpp:38-49 -- W = q^T aq, symmetrised (W+W^T)/2 */
int orc_assemble_gram(int64_t n, int k, const double* q, const double* aq, double* w) {
  if (k > 64) return fail(E_DIM, 0, "SmallDense: dimensions must be in [0, 64]");
  gram(n, k, k, q, aq, w);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < j; ++i) {
      const double sym = 0.5 * (w[i + j * k] + w[j + i * k]);
      w[i + j * k] = sym;
      w[j + i * k] = sym;
    }
  return finish_assembly(k, w);
}

/* gram.cpp:78-119 -- nu forward GS sweeps per rhs column from x=0 */
static int fgs_core(int s, const double* w, int k, const double* rhs, int nu, double* x,
                    double* delta) {
  if (nu < 1) return fail(E_ARG, 0, "fgs: nu must be >= 1");
  for (int i = 0; i < s; ++i)
    if (!(w[i + i * s] > 0.0)) return fail(E_NOTSPD, 0, "fgs: zero diagonal");
  const double rn = frobenius(s * k, rhs);
  memset(x, 0, sizeof(double) * (size_t)(s * k));
  if (rn == 0.0) {
    *delta = 0.0;
    return OK;
  }
  for (int col = 0; col < k; ++col) {
    const double* b = rhs + col * s;
    double* xc = x + col * s;
    for (int sweep = 0; sweep < nu; ++sweep)
      for (int i = 0; i < s; ++i) {
        double acc = b[i];
        for (int j = 0; j < s; ++j)
          if (j != i) acc -= w[i + j * s] * xc[j];
        xc[i] = acc / w[i + i * s];
      }
  }
  double res_sq = 0.0;
  for (int col = 0; col < k; ++col)
    for (int i = 0; i < s; ++i) {
      double acc = rhs[i + col * s];
      for (int j = 0; j < s; ++j) acc -= w[i + j * s] * x[j + col * s];
      res_sq += acc * acc;
    }
  *delta = sqrt(res_sq) / rn;
  return OK;
}

/* gram.cpp:51-58 gram_from_matrix (exact symmetry + diagonal) then fgs_solve */
int orc_fgs_solve(int s, const double* w, int k, const double* rhs, int nu, double* x,
                  double* delta) {
  if (s > 64 || k > 64) return fail(E_DIM, 0, "SmallDense: dimensions must be in [0, 64]");
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < j; ++i)
      if (w[i + j * s] != w[j + i * s])
        return fail(E_MATRIX, 0, "gram_from_matrix: matrix not symmetric");
  TRY(finish_assembly(s, w));
  return fgs_core(s, w, k, rhs, nu, x, delta);
}

/* dense_ops.cpp:55-88 -- left-looking Cholesky, forward/back substitution */
int orc_cholesky_solve(int s, const double* w, int k, const double* rhs, double* x) {
  if (s > 64 || k > 64) return fail(E_DIM, 0, "SmallDense: dimensions must be in [0, 64]");
  double l[64 * 64];
  memset(l, 0, sizeof l);
  for (int j = 0; j < s; ++j) {
    double d = w[j + j * s];
    for (int q = 0; q < j; ++q) d -= l[j + q * s] * l[j + q * s];
    if (!(d > 0.0) || !isfinite(d))
      return fail(E_NOTSPD, 0, "cholesky: non-positive pivot (basis breakdown)");
    const double dg = sqrt(d);
    l[j + j * s] = dg;
    for (int i = j + 1; i < s; ++i) {
      double v = w[i + j * s];
      for (int q = 0; q < j; ++q) v -= l[i + q * s] * l[j + q * s];
      l[i + j * s] = v / dg;
    }
  }
  memcpy(x, rhs, sizeof(double) * (size_t)(s * k));
  for (int col = 0; col < k; ++col) {
    double* xc = x + col * s;
    for (int i = 0; i < s; ++i) {
      double v = xc[i];
      for (int q = 0; q < i; ++q) v -= l[i + q * s] * xc[q];
      xc[i] = v / l[i + i * s];
    }
    for (int i = s - 1; i >= 0; --i) {
      double v = xc[i];
      for (int q = i + 1; q < s; ++q) v -= l[q + i * s] * xc[q];
      xc[i] = v / l[i + i * s];
    }
  }
  return OK;
}

/* solver.cpp:33-44 gram_rel_residual */
static double gram_rel_residual(int s, const double* w, int k, const double* rhs,
                                const double* x) {
  double res_sq = 0.0;
  for (int col = 0; col < k; ++col)
    for (int i = 0; i < s; ++i) {
      double acc = rhs[i + col * s];
      for (int j = 0; j < s; ++j) acc -= w[i + j * s] * x[j + col * s];
      res_sq += acc * acc;
    }
  const double rn = frobenius(s * k, rhs);
  return rn == 0.0 ? 0.0 : sqrt(res_sq) / rn;
}

/* ---------------------------------------------------------------- spectral */

/* Replaces LAPACK dsterf (lapack.cpp:61-71): eigenvalues of the symmetric
 * tridiagonal (d, e), ascending, by the implicit QL iteration with Wilkinson
 * shifts. d[m], e[m-1]; out[m]. */
int orc_tridiag_eigvals(int m, const double* diag, const double* off, double* out) {
  if (m <= 0) return OK;
  double* d = out;
  double* e = (double*)xcalloc(m, sizeof(double));
  if (!e) return fail(E_NOMEM, 0, "out of memory");
  for (int i = 0; i < m; ++i) d[i] = diag[i];
  for (int i = 0; i + 1 < m; ++i) e[i] = off[i];
  e[m - 1] = 0.0;
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    for (;;) {
      int mm;
      for (mm = l; mm < m - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= 0x1.0p-53 * dd) break;
      }
      if (mm == l) break;
      if (++iter > 60) {
        free(e);
        return fail(E_GENERIC, 0, "tridiag_eigvals: no convergence");
      }
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? fabs(r) : -fabs(r)));
      double s = 1.0, c = 1.0, p = 0.0;
      int i;
      for (i = mm - 1; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        r = hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[mm] = 0.0;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
      }
      if (r == 0.0 && i >= l) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  free(e);
  for (int i = 1; i < m; ++i) { /* insertion sort, ascending */
    const double key = d[i];
    int j = i - 1;
    while (j >= 0 && d[j] > key) {
      d[j + 1] = d[j];
      --j;
    }
    d[j + 1] = key;
  }
  return OK;
}

/* spectral.cpp:60-132 -- Lanczos on M^{-1}A in the M inner product, full
 * (modified Gram-Schmidt) reorthogonalisation, Ritz extremes x0.9 / x1.1. */
static int lanczos_core(int64_t n, const int64_t* rp, const int64_t* ci, const double* v_,
                        const precond_t* m, int steps, uint64_t seed, double* lo, double* hi) {
  if (steps < 2) return fail(E_ARG, 0, "estimate_interval: steps >= 2");
  double* vs = (double*)xcalloc(n * steps, sizeof(double));
  double* gs = (double*)xcalloc(n * steps, sizeof(double));
  double* v = (double*)xcalloc(n, sizeof(double));
  double* g = (double*)xcalloc(n, sizeof(double));
  double* t = (double*)xcalloc(n, sizeof(double));
  double* r = (double*)xcalloc(n, sizeof(double));
  double* gr = (double*)xcalloc(n, sizeof(double));
  double* alpha = (double*)xcalloc(steps, sizeof(double));
  double* beta = (double*)xcalloc(steps, sizeof(double));
  double* ritz = (double*)xcalloc(steps, sizeof(double));
  int rc = OK, na = 0, nb = 0;
  if (!vs || !gs || !v || !g || !t || !r || !gr || !alpha || !beta || !ritz) {
    rc = fail(E_NOMEM, 0, "out of memory");
    goto done;
  }
  orc_random_vector(n, seed, v);
  memcpy(g, v, sizeof(double) * (size_t)n);
  precond_apply(m, n, g, v);
  {
    const double nrm = sqrt(dot(n, v, g));
    if (!(nrm > 0.0)) {
      rc = fail(E_GENERIC, 0, "estimate_interval: degenerate start vector");
      goto done;
    }
    for (int64_t i = 0; i < n; ++i) {
      v[i] /= nrm;
      g[i] /= nrm;
    }
  }
  for (int j = 0; j < steps; ++j) {
    orc_spmv(n, rp, ci, v_, v, t);
    const double aj = dot(n, v, t);
    if (!isfinite(aj)) {
      rc = fail(E_GENERIC, 0, "estimate_interval: non-finite value");
      goto done;
    }
    alpha[na++] = aj;
    double* vj = vs + (int64_t)j * n;
    double* gj = gs + (int64_t)j * n;
    memcpy(vj, v, sizeof(double) * (size_t)n);
    memcpy(gj, g, sizeof(double) * (size_t)n);
    precond_apply(m, n, t, r);
    memcpy(gr, t, sizeof(double) * (size_t)n);
    axpy(n, -aj, vj, r);
    axpy(n, -aj, gj, gr);
    if (j > 0) {
      axpy(n, -beta[nb - 1], vj - n, r);
      axpy(n, -beta[nb - 1], gj - n, gr);
    }
    for (int i = 0; i <= j; ++i) {
      const double proj = dot(n, gs + (int64_t)i * n, r);
      axpy(n, -proj, vs + (int64_t)i * n, r);
      axpy(n, -proj, gs + (int64_t)i * n, gr);
    }
    const double rg = dot(n, r, gr);
    const double bj = sqrt(0.0 < rg ? rg : 0.0); /* std::max(0.0, rg) */
    if (!isfinite(bj)) {
      rc = fail(E_GENERIC, 0, "estimate_interval: non-finite value");
      goto done;
    }
    if (bj == 0.0) break;
    if (j + 1 < steps) {
      beta[nb++] = bj;
      for (int64_t i = 0; i < n; ++i) {
        v[i] = r[i] / bj;
        g[i] = gr[i] / bj;
      }
    }
  }
  rc = orc_tridiag_eigvals(na, alpha, beta, ritz);
  if (rc != OK) goto done;
  *lo = 0.9 * ritz[0];
  *hi = 1.1 * ritz[na - 1];
  if (!(*lo > 0.0) || !isfinite(*hi))
    rc = fail(E_NOTSPD, 0, "estimate_interval: operator not positive definite");
done:
  free(vs); free(gs); free(v); free(g); free(t); free(r); free(gr);
  free(alpha); free(beta); free(ritz);
  return rc;
}

int orc_estimate_interval(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                          int precond, int steps, uint64_t seed, double* lo, double* hi) {
  precond_t m;
  TRY(precond_make(&m, precond, n, rp, ci, v));
  const int rc = lanczos_core(n, rp, ci, v, &m, steps, seed, lo, hi);
  precond_free(&m);
  return rc;
}

/* ---------------------------------------------------------------- solvers */

static void rep_reset(oc_report* rep) {
  rep->converged = 0;
  rep->outer_iters = 0;
  rep->spmv_count = rep->precond_count = rep->allreduce_count = 0;
  rep->local_update_flops = rep->gram_solve_flops = 0.0;
  rep->lambda_min = rep->lambda_max = 0.0;
  rep->n_rel = rep->n_da = rep->n_db = 0;
}
static void push(double* arr, int* len, int cap, double val) {
  if (arr && *len < cap) arr[*len] = val;
  ++*len;
}

/* solver.cpp:51-67 solve_gram: FGS or Cholesky + residual; NotSpd becomes
 * SolverBreakdownError(outer). */
static int solve_gram(int s, const double* w, int k, const double* rhs, const oc_cfg* cfg,
                      int outer, double* x, double* delta) {
  int rc;
  if (cfg->gram == 0) {
    rc = fgs_core(s, w, k, rhs, cfg->nu, x, delta);
  } else {
    rc = orc_cholesky_solve(s, w, k, rhs, x);
    if (rc == OK) *delta = gram_rel_residual(s, w, k, rhs, x);
  }
  if (rc == E_NOTSPD) {
    char msg[256];
    snprintf(msg, sizeof msg, "gram solve failed at outer iteration %d: %s", outer, g_msg);
    return fail(E_SOLVER, outer, msg);
  }
  return rc;
}

/* solver.cpp:78-190 -- PCG-S (Alg. 1) */
static int pcgs_core(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     const double* b, const precond_t* m, const oc_cfg* cfg, double* x,
                     oc_report* rep) {
  const int s = cfg->s;
  const double bnorm = norm2(n, b);
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    rep->converged = 1;
    push(rep->rel_residual, &rep->n_rel, rep->cap, 0.0);
    return OK;
  }
  double lo, hi;
  if (cfg->has_spectrum) {
    lo = cfg->lambda_min;
    hi = cfg->lambda_max;
  } else {
    TRY(lanczos_core(n, rp, ci, v, m, cfg->lanczos_steps, cfg->seed, &lo, &hi));
  }
  rep->lambda_min = lo;
  rep->lambda_max = hi;
  TRY(cheb_check(lo, hi));

  int rc = OK;
  double* r = (double*)xcalloc(n, sizeof(double));
  double* q = (double*)xcalloc(n * s, sizeof(double));
  double* aq = (double*)xcalloc(n * s, sizeof(double));
  double* z = (double*)xcalloc(n * s, sizeof(double));
  double* p = (double*)xcalloc(n * (s + 1), sizeof(double));
  double* tmp = (double*)xcalloc(n * s, sizeof(double));
  if (!r || !q || !aq || !z || !p || !tmp) {
    rc = fail(E_NOMEM, 0, "out of memory");
    goto done;
  }
  double w[64 * 64], b1[64], b2[64 * 64], alpha[64], beta[64 * 64], da, db;

  orc_spmv(n, rp, ci, v, x, r); /* r0 = b - A x0 */
  rep->spmv_count += 1;
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  push(rep->rel_residual, &rep->n_rel, rep->cap, norm2(n, r) / bnorm);

  rc = mpk_core(n, rp, ci, v, m, r, s, lo, hi, z, p);
  if (rc != OK) goto done;
  rep->spmv_count += s;
  rep->precond_count += s;
  memcpy(q, z, sizeof(double) * (size_t)(n * s));
  memcpy(aq, p + n, sizeof(double) * (size_t)(n * s));

  const double lflops = 3.5 * ((double)s * s + s) * (double)n;
  const double gflops = cfg->gram == 0 ? (double)cfg->nu * ((double)s * s + 2.0 * s)
                                       : (double)s * s * s / 3.0 + 2.0 * s * s * (s + 1.0);

  for (int k = 1; k <= cfg->max_outer; ++k) {
    gram(n, s, s, q, aq, w); /* assemble_gram, gram.cpp:38-49 */
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < j; ++i) {
        const double sym = 0.5 * (w[i + j * s] + w[j + i * s]);
        w[i + j * s] = sym;
        w[j + i * s] = sym;
      }
    if (finish_assembly(s, w) != OK) {
      char msg[256];
      snprintf(msg, sizeof msg, "Gram assembly degenerate at outer iteration %d: %s", k, g_msg);
      rc = fail(E_SOLVER, k, msg);
      goto done;
    }
    gram(n, s, 1, q, p, b1); /* b1 = Q^T p_0, solver.cpp:153-154 */
    rc = solve_gram(s, w, 1, b1, cfg, k, alpha, &da);
    if (rc != OK) goto done;
    push(rep->delta_alpha, &rep->n_da, rep->cap, da);
    rep->gram_solve_flops += gflops;
    for (int j = 0; j < s; ++j) { /* solver.cpp:159-162 */
      axpy(n, alpha[j], q + (int64_t)j * n, x);
      axpy(n, -alpha[j], aq + (int64_t)j * n, r);
    }
    rep->local_update_flops += lflops;
    rep->outer_iters = k;
    const double rel = norm2(n, r) / bnorm;
    push(rep->rel_residual, &rep->n_rel, rep->cap, rel);
    if (rel <= cfg->tol) {
      rep->converged = 1;
      break;
    }
    memset(z, 0, sizeof(double) * (size_t)(n * s));
    memset(p, 0, sizeof(double) * (size_t)(n * (s + 1)));
    rc = mpk_core(n, rp, ci, v, m, r, s, lo, hi, z, p);
    if (rc != OK) goto done;
    rep->spmv_count += s;
    rep->precond_count += s;
    const double* aq_new = p + n;
    gram(n, s, s, q, aq_new, b2); /* solver.cpp:178-179 */
    for (int i = 0; i < s * s; ++i) b2[i] = -b2[i];
    rc = solve_gram(s, w, s, b2, cfg, k, beta, &db);
    if (rc != OK) goto done;
    push(rep->delta_beta, &rep->n_db, rep->cap, db);
    rep->gram_solve_flops += gflops;
    /* q = block_update(z, q, beta); aq = block_update(aq_new, aq, beta) */
    orc_block_update(n, s, s, z, q, beta, tmp);
    memcpy(q, tmp, sizeof(double) * (size_t)(n * s));
    orc_block_update(n, s, s, aq_new, aq, beta, tmp);
    memcpy(aq, tmp, sizeof(double) * (size_t)(n * s));
  }
  rep->allreduce_count = 2 * (int64_t)rep->outer_iters;
done:
  free(r); free(q); free(aq); free(z); free(p); free(tmp);
  return rc;
}

int orc_pcg_s_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    const double* b, const double* x0, int precond, const oc_cfg* cfg, double* x,
                    oc_report* rep) {
  rep_reset(rep);
  /* solver.cpp:15-22 SolverConfig::validate */
  if (cfg->s < 1 || cfg->s > 64) return fail(E_ARG, 0, "SolverConfig: s must be in [1, 64]");
  if (!(cfg->tol > 0.0)) return fail(E_ARG, 0, "SolverConfig: tol must be > 0");
  if (cfg->max_outer < 1) return fail(E_ARG, 0, "SolverConfig: max_outer must be >= 1");
  if (cfg->nu < 1) return fail(E_ARG, 0, "SolverConfig: nu must be >= 1");
  precond_t m;
  TRY(precond_make(&m, precond, n, rp, ci, v));
  memcpy(x, x0, sizeof(double) * (size_t)n);
  const int rc = pcgs_core(n, rp, ci, v, b, &m, cfg, x, rep);
  precond_free(&m);
  return rc;
}

/* solver.cpp:192-264 -- classical PCG */
int orc_pcg_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  const double* b, const double* x0, int precond, double tol, int max_iter,
                  double* x, oc_report* rep) {
  rep_reset(rep);
  if (!(tol >= 0.0) || max_iter < 1) return fail(E_ARG, 0, "pcg_solve: bad tol/max_iter");
  precond_t m;
  TRY(precond_make(&m, precond, n, rp, ci, v));
  memcpy(x, x0, sizeof(double) * (size_t)n);
  int rc = OK;
  double *r = NULL, *z = NULL, *p = NULL, *q = NULL;
  const double bnorm = norm2(n, b);
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    rep->converged = 1;
    push(rep->rel_residual, &rep->n_rel, rep->cap, 0.0);
    goto done;
  }
  r = (double*)xcalloc(n, sizeof(double));
  z = (double*)xcalloc(n, sizeof(double));
  p = (double*)xcalloc(n, sizeof(double));
  q = (double*)xcalloc(n, sizeof(double));
  if (!r || !z || !p || !q) {
    rc = fail(E_NOMEM, 0, "out of memory");
    goto done;
  }
  orc_spmv(n, rp, ci, v, x, r);
  rep->spmv_count += 1;
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  push(rep->rel_residual, &rep->n_rel, rep->cap, norm2(n, r) / bnorm);
  precond_apply(&m, n, r, z);
  rep->precond_count += 1;
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rho = dot(n, r, z);
  for (int it = 1; it <= max_iter; ++it) {
    orc_spmv(n, rp, ci, v, p, q);
    rep->spmv_count += 1;
    const double pq = dot(n, p, q);
    if (!(pq > 0.0)) {
      char msg[96];
      snprintf(msg, sizeof msg, "pcg: non-positive curvature at iteration %d", it);
      rc = fail(E_SOLVER, it, msg);
      goto done;
    }
    const double step = rho / pq;
    axpy(n, step, p, x);
    axpy(n, -step, q, r);
    rep->local_update_flops += 8.0 * (double)n;
    rep->outer_iters = it;
    const double rel = norm2(n, r) / bnorm;
    push(rep->rel_residual, &rep->n_rel, rep->cap, rel);
    if (rel <= tol) {
      rep->converged = 1;
      break;
    }
    precond_apply(&m, n, r, z);
    rep->precond_count += 1;
    const double rho_new = dot(n, r, z);
    const double beta = rho_new / rho;
    rho = rho_new;
    xpby(n, z, beta, p);
  }
  rep->allreduce_count = 2 * (int64_t)rep->outer_iters;
done:
  free(r); free(z); free(p); free(q);
  precond_free(&m);
  return rc;
}
