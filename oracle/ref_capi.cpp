// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (see oracle_abi.h).
//
// extern "C" wrappers over the unmodified reference library. oracle/Makefile
// compiles /root/reference/proj/src/*.cpp in place with -Dchebstep=chebstep_ref
// and this file with the same flag, so every reference symbol lives in
// namespace chebstep_ref and cannot collide with the product's chebstep::
// drop-in API. Each wrapper converts plain arrays to the reference types,
// calls the reference function named in its comment, and maps the
// reference exception hierarchy (errors.hpp:9-56) to CS_* status codes.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "chebstep/block.hpp"
#include "chebstep/csr.hpp"
#include "chebstep/dense_ops.hpp"
#include "chebstep/errors.hpp"
#include "chebstep/gram.hpp"
#include "chebstep/lapack.hpp"
#include "chebstep/mpk.hpp"
#include <cmath>
#include <span>
#include <string_view>
#include "chebstep/precond.hpp"
#include "chebstep/problems.hpp"
#include "chebstep/solver.hpp"
#include "chebstep/spectral.hpp"
#include "chebstep/util.hpp"
#include "oracle_abi.h"

namespace cs = chebstep;  // == chebstep_ref under -Dchebstep=chebstep_ref

namespace {
thread_local std::string g_msg;
thread_local int g_payload = 0;

template <class F>
int guarded(F&& f) {
  g_msg.clear();
  g_payload = 0;
  try {
    f();
    return 0;
  } catch (const cs::DimensionError& e) {
    g_msg = e.what();
    return 1;
  } catch (const cs::InvalidMatrixError& e) {
    g_msg = e.what();
    return 2;
  } catch (const cs::NotSpdError& e) {
    g_msg = e.what();
    return 3;
  } catch (const cs::BasisBreakdownError& e) {
    g_msg = e.what();
    g_payload = e.column;
    return 4;
  } catch (const cs::SolverBreakdownError& e) {
    g_msg = e.what();
    g_payload = e.outer_iteration;
    return 5;
  } catch (const cs::GuardExceededError& e) {
    g_msg = e.what();
    return 6;
  } catch (const cs::ParseError& e) {
    g_msg = e.what();
    return 7;
  } catch (const cs::InvalidArgumentError& e) {
    g_msg = e.what();
    return 8;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 9;
  }
}

cs::CsrMatrix make_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
  cs::CsrMatrix a;
  a.n = n;
  a.row_offsets.assign(rp, rp + n + 1);
  const int64_t nnz = rp[n];
  a.col_indices.assign(ci, ci + nnz);
  a.values.assign(v, v + nnz);
  return a;
}

// Reference-side block-Jacobi subclass of the reference's own Preconditioner
// interface (precond.hpp:12-23) -- the parity partner of the device block
// Jacobi. Test infrastructure: dense diagonal blocks of bs rows
// (entries summed in stored order, a short last block padded with the
// identity), left-looking Cholesky in small_cholesky_solve's order
// (dense_ops.cpp:55-88), apply = forward then back substitution.
class BlockJacobiRef final : public cs::Preconditioner {
 public:
  BlockJacobiRef(const cs::CsrMatrix& a, int bs) : bs_(bs), n_(a.n) {
    if (bs < 1 || bs > 16) throw cs::InvalidArgumentError("block_jacobi: bs must be in [1, 16]");
    const int64_t nb = (a.n + bs - 1) / bs;
    const size_t q = static_cast<size_t>(bs) * bs;
    f_.assign(static_cast<size_t>(nb) * q, 0.0);
    for (int64_t r = 0; r < nb * bs; ++r) {
      double* blk = f_.data() + static_cast<size_t>(r / bs) * q;
      const int i = static_cast<int>(r % bs);
      if (r >= a.n) {
        blk[i + i * bs] = 1.0;
        continue;
      }
      const int64_t b0 = (r / bs) * bs;
      for (int64_t k = a.row_offsets[r]; k < a.row_offsets[r + 1]; ++k) {
        const int64_t c = a.col_indices[k];
        if (c >= b0 && c < b0 + bs) blk[i + (c - b0) * bs] += a.values[k];
      }
    }
    for (int64_t b = 0; b < nb; ++b) {
      double* L = f_.data() + static_cast<size_t>(b) * q;
      for (int j = 0; j < bs; ++j) {
        double d = L[j + j * bs];
        for (int t = 0; t < j; ++t) d -= L[j + t * bs] * L[j + t * bs];
        if (!(d > 0.0) || !std::isfinite(d))
          throw cs::NotSpdError("block_jacobi: diagonal block not positive definite");
        const double dg = std::sqrt(d);
        L[j + j * bs] = dg;
        for (int i = j + 1; i < bs; ++i) {
          double v = L[i + j * bs];
          for (int t = 0; t < j; ++t) v -= L[i + t * bs] * L[j + t * bs];
          L[i + j * bs] = v / dg;
        }
      }
    }
  }
  void apply(std::span<const double> in, std::span<double> out) const override {
    const int bs = bs_;
    double x[16];
    for (int64_t r0 = 0; r0 < n_; r0 += bs) {
      const double* L = f_.data() + static_cast<size_t>(r0 / bs) * bs * bs;
      for (int i = 0; i < bs; ++i) x[i] = r0 + i < n_ ? in[r0 + i] : 0.0;
      for (int i = 0; i < bs; ++i) {
        double v = x[i];
        for (int t = 0; t < i; ++t) v -= L[i + t * bs] * x[t];
        x[i] = v / L[i + i * bs];
      }
      for (int i = bs - 1; i >= 0; --i) {
        double v = x[i];
        for (int t = i + 1; t < bs; ++t) v -= L[t + i * bs] * x[t];
        x[i] = v / L[i + i * bs];
      }
      for (int i = 0; i < bs && r0 + i < n_; ++i) out[r0 + i] = x[i];
    }
  }
  std::string_view name() const override { return "block_jacobi"; }

 private:
  int bs_;
  int64_t n_;
  std::vector<double> f_;
};

struct Precond {
  cs::IdentityPreconditioner ident;
  std::unique_ptr<cs::JacobiPreconditioner> jac;
  std::unique_ptr<BlockJacobiRef> bj;
  const cs::Preconditioner& get() const {
    if (bj) return *bj;
    return jac ? static_cast<const cs::Preconditioner&>(*jac) : ident;
  }
};

// kind: 0 identity, 1 Jacobi, 100 + bs block Jacobi
void make_precond(Precond& p, const cs::CsrMatrix& a, int kind) {
  if (kind == 1) p.jac = std::make_unique<cs::JacobiPreconditioner>(a);
  else if (kind >= 101 && kind <= 116) p.bj = std::make_unique<BlockJacobiRef>(a, kind - 100);
  else if (kind != 0) throw cs::InvalidArgumentError("unknown preconditioner kind");
}

cs::VectorBlock block_of(int64_t n, int k, const double* d) {
  cs::VectorBlock b(n, k);
  std::memcpy(b.data.data(), d, sizeof(double) * static_cast<size_t>(n) * k);
  return b;
}

cs::SmallDense dense_of(int r, int c, const double* d) {
  cs::SmallDense m(r, c);
  std::memcpy(m.data.data(), d, sizeof(double) * static_cast<size_t>(r) * c);
  return m;
}

void fill_report(const cs::SolveReport& r, oc_report* o) {
  o->converged = r.converged ? 1 : 0;
  o->outer_iters = r.outer_iters;
  o->spmv_count = r.spmv_count;
  o->precond_count = r.precond_count;
  o->allreduce_count = r.allreduce_count;
  o->local_update_flops = r.local_update_flops;
  o->gram_solve_flops = r.gram_solve_flops;
  o->lambda_min = r.spectrum_used.lambda_min;
  o->lambda_max = r.spectrum_used.lambda_max;
  auto copy = [&](const std::vector<double>& src, double* dst, int* len) {
    const int m = static_cast<int>(src.size());
    *len = m;
    if (dst)
      for (int i = 0; i < m && i < o->cap; ++i) dst[i] = src[i];
  };
  copy(r.rel_residual, o->rel_residual, &o->n_rel);
  copy(r.delta_alpha, o->delta_alpha, &o->n_da);
  copy(r.delta_beta, o->delta_beta, &o->n_db);
}
}  // namespace

extern "C" {

// problems.cpp:13-53
int ref_poisson27_fill(int64_t nx, int64_t ny, int64_t nz, int64_t* rowptr, int64_t* col,
                       double* val) {
  return guarded([&] {
    cs::PoissonSystem sys = cs::poisson27({nx, ny, nz});
    std::memcpy(rowptr, sys.a.row_offsets.data(), sizeof(int64_t) * (sys.a.n + 1));
    std::memcpy(col, sys.a.col_indices.data(), sizeof(int64_t) * sys.a.nnz());
    std::memcpy(val, sys.a.values.data(), sizeof(double) * sys.a.nnz());
  });
}

// csr.cpp:111-124
int ref_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x,
             double* y) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    cs::spmv_into(a, {x, static_cast<size_t>(n)}, {y, static_cast<size_t>(n)});
  });
}

// precond.cpp:15-30 (the inverse diagonal is private; apply to ones)
int ref_jacobi_invdiag(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                       double* out) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    cs::JacobiPreconditioner m(a);
    std::vector<double> ones(static_cast<size_t>(n), 1.0);
    m.apply(ones, {out, static_cast<size_t>(n)});
  });
}

// mpk.cpp:26-71
int ref_mpk(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int precond,
            const double* r, int s, double lo, double hi, double* z, double* p) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    Precond m;
    make_precond(m, a, precond);
    const auto params = cs::ChebyshevParams::from_interval(lo, hi);
    cs::MpkResult res = cs::mpk_chebyshev(a, {r, static_cast<size_t>(n)}, s, m.get(), params);
    std::memcpy(z, res.z.data.data(), sizeof(double) * res.z.data.size());
    std::memcpy(p, res.p.data.data(), sizeof(double) * res.p.data.size());
  });
}

// dense_ops.cpp:19-27
int ref_block_gram(int64_t n, int ku, int kv, const double* u, const double* w, double* g) {
  return guarded([&] {
    const cs::SmallDense out = cs::block_gram(block_of(n, ku, u), block_of(n, kv, w));
    std::memcpy(g, out.data.data(), sizeof(double) * out.data.size());
  });
}

// dense_ops.cpp:29-42
int ref_block_update(int64_t n, int m, int k, const double* y, const double* x, const double* c,
                     double* out) {
  return guarded([&] {
    const cs::VectorBlock r =
        cs::block_update(block_of(n, k, y), block_of(n, m, x), dense_of(m, k, c));
    std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
  });
}

// gram.cpp:38-49
int ref_assemble_gram(int64_t n, int k, const double* q, const double* aq, double* w) {
  return guarded([&] {
    const cs::GramSystem g = cs::assemble_gram(block_of(n, k, q), block_of(n, k, aq));
    std::memcpy(w, g.w.data.data(), sizeof(double) * g.w.data.size());
  });
}

// gram.cpp:51-58 + 78-119
int ref_fgs_solve(int s, const double* w, int k, const double* rhs, int nu, double* x,
                  double* delta) {
  return guarded([&] {
    const cs::GramSystem g = cs::gram_from_matrix(dense_of(s, s, w));
    cs::FgsConfig cfg;
    cfg.nu = nu;
    const cs::FgsResult r = cs::fgs_solve(g, dense_of(s, k, rhs), cfg);
    std::memcpy(x, r.x.data.data(), sizeof(double) * r.x.data.size());
    *delta = r.rel_residual;
  });
}

// dense_ops.cpp:55-88
int ref_cholesky_solve(int s, const double* w, int k, const double* rhs, double* x) {
  return guarded([&] {
    const cs::SmallDense r = cs::small_cholesky_solve(dense_of(s, s, w), dense_of(s, k, rhs));
    std::memcpy(x, r.data.data(), sizeof(double) * r.data.size());
  });
}

// util.cpp:31-36
int ref_random_vector(int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const std::vector<double> r = cs::random_vector(n, seed);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

// lapack.cpp:61-71 (LAPACKE_dsterf)
int ref_tridiag_eigvals(int m, const double* diag, const double* off, double* out) {
  return guarded([&] {
    std::vector<double> d(diag, diag + m);
    std::vector<double> e(off, off + (m > 0 ? m - 1 : 0));
    const std::vector<double> r = cs::lapack::tridiag_eigvals(d, e);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

// spectral.cpp:60-132
int ref_estimate_interval(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                          int precond, int steps, uint64_t seed, double* lo, double* hi) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    Precond m;
    make_precond(m, a, precond);
    const cs::SpectrumEstimate e = cs::estimate_interval(a, m.get(), steps, seed);
    *lo = e.lambda_min;
    *hi = e.lambda_max;
  });
}

// solver.cpp:78-190
int ref_pcg_s_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    const double* b, const double* x0, int precond, const oc_cfg* c, double* x,
                    oc_report* rep) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    Precond m;
    make_precond(m, a, precond);
    cs::SolverConfig cfg;
    cfg.s = c->s;
    cfg.tol = c->tol;
    cfg.max_outer = c->max_outer;
    cfg.fgs.nu = c->nu;
    cfg.gram_solver = c->gram == 1 ? cs::GramSolverKind::cholesky : cs::GramSolverKind::fgs;
    if (c->has_spectrum) {
      cs::SpectrumEstimate e;
      e.lambda_min = c->lambda_min;
      e.lambda_max = c->lambda_max;
      cfg.spectrum = e;
    }
    cfg.lanczos_steps = c->lanczos_steps;
    cfg.seed = c->seed;
    const cs::SolveResult res = cs::pcg_s_solve(a, {b, static_cast<size_t>(n)},
                                                {x0, static_cast<size_t>(n)}, m.get(), cfg);
    std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
    fill_report(res.report, rep);
  });
}

// solver.cpp:192-264
int ref_pcg_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  const double* b, const double* x0, int precond, double tol, int max_iter,
                  double* x, oc_report* rep) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    Precond m;
    make_precond(m, a, precond);
    const cs::SolveResult res = cs::pcg_solve(a, {b, static_cast<size_t>(n)},
                                              {x0, static_cast<size_t>(n)}, m.get(), tol, max_iter);
    std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
    fill_report(res.report, rep);
  });
}

// solver.cpp:78-190 with the analysis hooks of SolverConfig (solver.hpp:30-34)
static void copy_hooks(const cs::SolveReport& r, oc_hooks* hk, int s, int64_t n) {
  auto put = [&](const std::vector<double>& src, double* dst, int* len) {
    *len = static_cast<int>(src.size());
    if (dst)
      for (int i = 0; i < *len && i < hk->cap; ++i) dst[i] = src[i];
  };
  put(r.kappa_w, hk->kappa_w, &hk->n_kappa);
  put(r.true_rel_residual, hk->true_rel_residual, &hk->n_true);
  put(r.a_norm_error, hk->a_norm_error, &hk->n_aerr);
  if (hk->gram_history)
    for (size_t i = 0; i < r.gram_history.size() && static_cast<int>(i) < hk->cap; ++i)
      std::memcpy(hk->gram_history + i * s * s, r.gram_history[i].data.data(),
                  sizeof(double) * s * s);
  hk->n_iter = static_cast<int>(r.iterates.size());
  if (hk->iterates)
    for (size_t i = 0; i < r.iterates.size() && static_cast<int>(i) < hk->cap; ++i)
      std::memcpy(hk->iterates + i * n, r.iterates[i].data(), sizeof(double) * n);
}

int ref_pcg_s_solve_hooks(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                          const double* b, const double* x0, int precond, const oc_cfg* c,
                          oc_hooks* hk, double* x, oc_report* rep) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    Precond m;
    make_precond(m, a, precond);
    cs::SolverConfig cfg;
    cfg.s = c->s;
    cfg.tol = c->tol;
    cfg.max_outer = c->max_outer;
    cfg.fgs.nu = c->nu;
    cfg.gram_solver = c->gram == 1 ? cs::GramSolverKind::cholesky : cs::GramSolverKind::fgs;
    if (c->has_spectrum) {
      cs::SpectrumEstimate e;
      e.lambda_min = c->lambda_min;
      e.lambda_max = c->lambda_max;
      cfg.spectrum = e;
    }
    cfg.lanczos_steps = c->lanczos_steps;
    cfg.seed = c->seed;
    cfg.collect_gram = hk->collect_gram != 0;
    cfg.track_true_residual = hk->track_true_residual != 0;
    cfg.collect_iterates = hk->collect_iterates != 0;
    if (hk->error_reference) cfg.error_reference = std::vector<double>(hk->error_reference, hk->error_reference + n);
    const cs::SolveResult res = cs::pcg_s_solve(a, {b, static_cast<size_t>(n)},
                                                {x0, static_cast<size_t>(n)}, m.get(), cfg);
    std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
    fill_report(res.report, rep);
    copy_hooks(res.report, hk, c->s, n);
  });
}

int ref_pcg_solve_hooks(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        const double* b, const double* x0, int precond, double tol, int max_iter,
                        oc_hooks* hk, double* x, oc_report* rep) {
  return guarded([&] {
    const cs::CsrMatrix a = make_csr(n, rp, ci, v);
    Precond m;
    make_precond(m, a, precond);
    cs::PcgConfig cfg;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    cfg.collect_iterates = hk->collect_iterates != 0;
    if (hk->error_reference) cfg.error_reference = std::vector<double>(hk->error_reference, hk->error_reference + n);
    const cs::SolveResult res = cs::pcg_solve(a, {b, static_cast<size_t>(n)},
                                              {x0, static_cast<size_t>(n)}, m.get(), cfg);
    std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
    fill_report(res.report, rep);
    copy_hooks(res.report, hk, 1, n);
  });
}

int ref_mm_read(const char* path, int require_spd, int64_t* n, int64_t* nnz, int64_t* rp,
                int64_t* ci, double* v) {
  return guarded([&] {
    const cs::CsrMatrix a = cs::read_matrix_market(path, require_spd != 0);
    *n = a.n;
    *nnz = a.nnz();
    if (rp == nullptr) return;
    std::memcpy(rp, a.row_offsets.data(), sizeof(int64_t) * (a.n + 1));
    std::memcpy(ci, a.col_indices.data(), sizeof(int64_t) * a.nnz());
    std::memcpy(v, a.values.data(), sizeof(double) * a.nnz());
  });
}

int ref_mm_write(const char* path, int64_t n, const int64_t* rp, const int64_t* ci,
                 const double* v) {
  return guarded([&] { cs::write_matrix_market(path, make_csr(n, rp, ci, v)); });
}

// check: 0 validate_structure, 1 validate_symmetric, 2 validate_spd_diagonal
int ref_csr_validate(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     int64_t nnz, int check) {
  return guarded([&] {
    cs::CsrMatrix a;
    a.n = n;
    a.row_offsets.assign(rp, rp + n + 1);
    a.col_indices.assign(ci, ci + nnz);
    a.values.assign(v, v + nnz);
    if (check == 0) cs::validate_structure(a);
    else if (check == 1) cs::validate_symmetric(a);
    else cs::validate_spd_diagonal(a);
  });
}

int ref_fgs_rate_normalized(int s, const double* w, double* norm, double* radius) {
  return guarded([&] {
    cs::SmallDense m(s, s);
    std::memcpy(m.data.data(), w, sizeof(double) * s * s);
    const cs::FgsRate r = cs::fgs_rate(cs::normalize_gram(cs::gram_from_matrix(m)));
    *norm = r.spectral_norm;
    *radius = r.spectral_radius;
  });
}

int ref_sym_eigvals(int s, const double* w, double* out) {
  return guarded([&] {
    const auto e = cs::lapack::sym_eigvals(s, std::vector<double>(w, w + s * s));
    std::memcpy(out, e.data(), sizeof(double) * s);
  });
}

// solver.cpp:275-282 over a report carrying only what the verdict reads
int ref_monitor_inexact(int outer_iters, int n_da, const double* delta_alpha, double delta_cap,
                        double* max_delta, double* budget, int* pass) {
  return guarded([&] {
    cs::SolveReport r;
    r.outer_iters = outer_iters;
    r.delta_alpha.assign(delta_alpha, delta_alpha + n_da);
    const cs::InexactVerdict v = cs::monitor_inexact(r, delta_cap);
    *max_delta = v.max_delta;
    *budget = v.budget;
    *pass = v.pass ? 1 : 0;
  });
}

const char* ref_last_error(int* payload) {
  if (payload) *payload = g_payload;
  return g_msg.c_str();
}

}  // extern "C"
