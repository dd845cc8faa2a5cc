// ref_probe.cpp -- TEST INFRASTRUCTURE ONLY: command-line driver over the
// unmodified reference library (namespace chebstep_ref) used to produce the
// golden outer-iteration counts / spectra in tests/golden/ for sizes that take
// minutes to hours on one CPU core. Prints one JSON line.
//   ref_probe <7|27> <N> <s> <nu> <tol> <jacobi|identity> [pcg|cholesky] [maxouter=M]
//             [lo=.. hi=..]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "chebstep/precond.hpp"
#include "chebstep/problems.hpp"
#include "chebstep/solver.hpp"
#include "chebstep/spectral.hpp"

namespace cs = chebstep;

static cs::CsrMatrix stencil7(int64_t N) {
  // 7-point restatement: x-fastest rows, ascending columns,
  // diagonal 6, -1 on in-grid faces, same conventions as problems.cpp:28-51.
  cs::CsrMatrix a;
  const int64_t n = N * N * N;
  a.n = n;
  a.row_offsets.assign(n + 1, 0);
  a.col_indices.reserve(n * 7);
  a.values.reserve(n * 7);
  int64_t row = 0;
  for (int64_t z = 0; z < N; ++z)
    for (int64_t y = 0; y < N; ++y)
      for (int64_t x = 0; x < N; ++x, ++row) {
        auto push = [&](int64_t c, double v) {
          a.col_indices.push_back(c);
          a.values.push_back(v);
        };
        if (z > 0) push(row - N * N, -1.0);
        if (y > 0) push(row - N, -1.0);
        if (x > 0) push(row - 1, -1.0);
        push(row, 6.0);
        if (x + 1 < N) push(row + 1, -1.0);
        if (y + 1 < N) push(row + N, -1.0);
        if (z + 1 < N) push(row + N * N, -1.0);
        a.row_offsets[row + 1] = static_cast<int64_t>(a.col_indices.size());
      }
  return a;
}

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: ref_probe <7|27> N s nu tol jacobi|identity [pcg|cholesky] "
                         "[maxouter=M] [lo=.. hi=..]\n");
    return 64;
  }
  const int stencil = std::atoi(argv[1]);
  const int64_t N = std::atoll(argv[2]);
  const int s = std::atoi(argv[3]);
  const int nu = std::atoi(argv[4]);
  const double tol = std::atof(argv[5]);
  const bool jacobi = std::strcmp(argv[6], "jacobi") == 0;
  bool pcg = false, chol = false;
  int max_outer = 100000;
  double lo = 0, hi = 0;
  for (int i = 7; i < argc; ++i) {
    if (!std::strcmp(argv[i], "pcg")) pcg = true;
    else if (!std::strcmp(argv[i], "cholesky")) chol = true;
    else if (!std::strncmp(argv[i], "maxouter=", 9)) max_outer = std::atoi(argv[i] + 9);
    else if (!std::strncmp(argv[i], "lo=", 3)) lo = std::atof(argv[i] + 3);
    else if (!std::strncmp(argv[i], "hi=", 3)) hi = std::atof(argv[i] + 3);
  }
  using clk = std::chrono::steady_clock;
  auto t0 = clk::now();
  cs::CsrMatrix a = stencil == 27 ? cs::poisson27({N, N, N}).a : stencil7(N);
  std::vector<double> b(a.n, 1.0), x0(a.n, 0.0);
  auto t1 = clk::now();
  cs::IdentityPreconditioner ident;
  std::unique_ptr<cs::JacobiPreconditioner> jac;
  if (jacobi) jac = std::make_unique<cs::JacobiPreconditioner>(a);
  const cs::Preconditioner& m = jacobi ? static_cast<const cs::Preconditioner&>(*jac) : ident;
  double t_lanczos = 0;
  cs::SolveResult res;
  int code = 0;
  std::string err;
  try {
    if (pcg) {
      res = cs::pcg_solve(a, b, x0, m, tol, max_outer);
    } else {
      cs::SolverConfig cfg;
      cfg.s = s;
      cfg.tol = tol;
      cfg.max_outer = max_outer;
      cfg.fgs.nu = nu;
      if (chol) cfg.gram_solver = cs::GramSolverKind::cholesky;
      if (lo > 0 && hi > lo) {
        cfg.spectrum = cs::SpectrumEstimate{lo, hi};
      } else {
        auto tl = clk::now();
        cfg.spectrum = cs::estimate_interval(a, m, cfg.lanczos_steps, cfg.seed);
        t_lanczos = std::chrono::duration<double>(clk::now() - tl).count();
      }
      res = cs::pcg_s_solve(a, b, x0, m, cfg);
    }
  } catch (const std::exception& e) {
    code = 1;
    err = e.what();
  }
  auto t2 = clk::now();
  const double t_solve = std::chrono::duration<double>(t2 - t1).count() - t_lanczos;
  double xs = 0, xn = 0;
  for (double v : res.x) {
    xs += v;
    xn += v * v;
  }
  double maxda = 0;
  for (double d : res.report.delta_alpha) maxda = std::max(maxda, d);
  std::printf("{\"stencil\": %d, \"N\": %lld, \"s\": %d, \"nu\": %d, \"tol\": %.17g, "
              "\"precond\": \"%s\", \"method\": \"%s\", \"error\": \"%s\", "
              "\"converged\": %d, \"outer_iters\": %d, \"spmv_count\": %lld, "
              "\"lambda_min\": %.17g, \"lambda_max\": %.17g, \"final_rel_residual\": %.17g, "
              "\"max_delta_alpha\": %.17g, \"x_sum\": %.17g, \"x_norm\": %.17g, "
              "\"t_assembly_s\": %.3f, \"t_lanczos_s\": %.3f, \"t_solve_s\": %.3f}\n",
              stencil, (long long)N, s, nu, tol, jacobi ? "jacobi" : "identity",
              pcg ? "pcg" : (chol ? "pcgs-cholesky" : "pcgs-fgs"), err.c_str(),
              res.report.converged ? 1 : 0, res.report.outer_iters,
              (long long)res.report.spmv_count, res.report.spectrum_used.lambda_min,
              res.report.spectrum_used.lambda_max,
              res.report.rel_residual.empty() ? 0.0 : res.report.rel_residual.back(), maxda, xs,
              std::sqrt(xn), std::chrono::duration<double>(t1 - t0).count(), t_lanczos, t_solve);
  return code;
}
