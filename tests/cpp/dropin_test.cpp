// dropin_test.cpp -- a reference-style C++ caller of the chebstep:: API,
// linked against libchebstep_gpu.so (the B200 drop-in) and checked against the
// unmodified reference library through the oracle's C ABI (test infrastructure,
// oracle/oracle_abi.h). Built and run by tests/test_gpu_cpp.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "chebstep/solver.hpp"
#include "chebstep/problems.hpp"
#include "chebstep/mpk.hpp"
#include "chebstep/gram.hpp"
#include "oracle_abi.h"

namespace cs = chebstep;
static int failures = 0;
#define EXPECT(cond)                                                  \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <class A, class B>
static bool same_bits(const A& a, const B& b, size_t n) {
  return std::memcmp(a, b, n * sizeof(*a)) == 0;
}

int main() {
  // --- assembly: device poisson27 == reference poisson27, bit for bit
  const cs::PoissonSystem sys = cs::poisson27({20, 18, 22});
  const int64_t n = sys.a.n, nnz = sys.a.nnz();
  std::vector<int64_t> rp(n + 1), ci(nnz);
  std::vector<double> v(nnz);
  EXPECT(ref_poisson27_fill(20, 18, 22, rp.data(), ci.data(), v.data()) == 0);
  EXPECT(same_bits(rp.data(), sys.a.row_offsets.data(), n + 1));
  EXPECT(same_bits(ci.data(), sys.a.col_indices.data(), nnz));
  EXPECT(same_bits(v.data(), sys.a.values.data(), nnz));

  // --- spmv_into
  std::vector<double> x = cs::random_vector(n, 77), y(n), yr(n), xr(n);
  EXPECT(ref_random_vector(n, 77, xr.data()) == 0 && same_bits(x.data(), xr.data(), n));
  cs::spmv_into(sys.a, x, y);
  ref_spmv(n, rp.data(), ci.data(), v.data(), x.data(), yr.data());
  EXPECT(same_bits(y.data(), yr.data(), n));

  // --- mpk_chebyshev (Jacobi)
  cs::JacobiPreconditioner jac(sys.a);
  const auto params = cs::ChebyshevParams::from_interval(0.01, 1.6);
  const cs::MpkResult mk = cs::mpk_chebyshev(sys.a, x, 6, jac, params);
  std::vector<double> z(n * 6), p(n * 7);
  ref_mpk(n, rp.data(), ci.data(), v.data(), 1, x.data(), 6, 0.01, 1.6, z.data(), p.data());
  EXPECT(same_bits(mk.z.data.data(), z.data(), n * 6));
  EXPECT(same_bits(mk.p.data.data(), p.data(), n * 7));

  // --- fgs_solve KAT
  cs::SmallDense w(2, 2);
  w.at(0, 0) = 1.0, w.at(0, 1) = 0.5, w.at(1, 0) = 0.5, w.at(1, 1) = 1.0;
  cs::SmallDense rhs(2, 1);
  rhs.at(0, 0) = 1.0;
  const auto fr = cs::fgs_solve(cs::gram_from_matrix(w), rhs, cs::FgsConfig{1, true});
  EXPECT(fr.x.at(0, 0) == 1.0 && fr.x.at(1, 0) == -0.5 && fr.rel_residual == 0.25);

  // --- pcg_s_solve, reference algebra, reference spectrum: bitwise the reference
  double lo = 0, hi = 0;
  EXPECT(ref_estimate_interval(n, rp.data(), ci.data(), v.data(), 1, 40, 1234, &lo, &hi) == 0);
  cs::SolverConfig cfg;
  cfg.s = 5;
  cfg.tol = 1e-9;
  cfg.spectrum = cs::SpectrumEstimate{lo, hi};
  cs::gpu::set_mode(cs::gpu::Mode::reference);
  const std::vector<double> b(n, 1.0), x0(n, 0.0);
  const cs::SolveResult res = cs::pcg_s_solve(sys.a, b, x0, jac, cfg);
  oc_cfg oc{5, 1e-9, 500, 30, 0, 1, lo, hi, 40, 1234};
  std::vector<double> xo(n), rel(600), da(600), db(600);
  oc_report orep{};
  orep.cap = 600;
  orep.rel_residual = rel.data();
  orep.delta_alpha = da.data();
  orep.delta_beta = db.data();
  EXPECT(ref_pcg_s_solve(n, rp.data(), ci.data(), v.data(), b.data(), x0.data(), 1, &oc, xo.data(),
                         &orep) == 0);
  EXPECT(res.report.outer_iters == orep.outer_iters);
  EXPECT(same_bits(res.x.data(), xo.data(), n));
  EXPECT(static_cast<int>(res.report.rel_residual.size()) == orep.n_rel &&
         same_bits(res.report.rel_residual.data(), rel.data(), orep.n_rel));
  EXPECT(res.report.spmv_count == orep.spmv_count);
  EXPECT(res.report.gram_solve_flops == orep.gram_solve_flops);

  // --- fast algebra with device Lanczos: same count +-1, x within 1e-8
  cs::gpu::set_mode(cs::gpu::Mode::fast);
  cfg.spectrum.reset();
  const cs::SolveResult fast = cs::pcg_s_solve(sys.a, b, x0, jac, cfg);
  double num = 0, den = 0;
  for (int64_t i = 0; i < n; ++i) {
    num += (fast.x[i] - xo[i]) * (fast.x[i] - xo[i]);
    den += xo[i] * xo[i];
  }
  EXPECT(std::abs(fast.report.outer_iters - orep.outer_iters) <= 1);
  EXPECT(std::sqrt(num / den) <= 1e-8);
  EXPECT(cs::monitor_inexact(fast.report).max_delta >= 0.0);

  // --- monitor_inexact verdict parity (solver.cpp:275-282): a nu = 2 run whose
  // alpha-system residual budget fails, the verdict of both libraries on it
  {
    cs::SolverConfig c2;
    c2.s = 6;
    c2.tol = 1e-9;
    c2.fgs.nu = 2;
    c2.spectrum = cs::SpectrumEstimate{lo, hi};
    cs::gpu::set_mode(cs::gpu::Mode::reference);
    const cs::SolveResult r2 = cs::pcg_s_solve(sys.a, b, x0, jac, c2);
    const cs::InexactVerdict vd = cs::monitor_inexact(r2.report);
    double md = 0, bud = 0;
    int pass = -1;
    EXPECT(ref_monitor_inexact(r2.report.outer_iters, static_cast<int>(r2.report.delta_alpha.size()),
                               r2.report.delta_alpha.data(), 1.0, &md, &bud, &pass) == 0);
    EXPECT(vd.max_delta == md && vd.budget == bud && (vd.pass ? 1 : 0) == pass);
    EXPECT(!vd.pass);  // nu = 2: the budget exceeds the default cap
    const cs::InexactVerdict v5 = cs::monitor_inexact(r2.report, 1e9);
    EXPECT(ref_monitor_inexact(r2.report.outer_iters, static_cast<int>(r2.report.delta_alpha.size()),
                               r2.report.delta_alpha.data(), 1e9, &md, &bud, &pass) == 0);
    EXPECT(v5.pass && pass == 1);
    cs::gpu::set_mode(cs::gpu::Mode::fast);
  }

  // --- block-Jacobi preconditioner through the same Preconditioner
  // interface: reference algebra bitwise the reference library driving its own
  // block-Jacobi Preconditioner subclass (oracle ref_capi.cpp, kind 100 + bs)
  {
    const cs::BlockJacobiPreconditioner bj(sys.a, 4);
    double blo = 0, bhi = 0;
    EXPECT(ref_estimate_interval(n, rp.data(), ci.data(), v.data(), 104, 40, 1234, &blo, &bhi) == 0);
    cs::SolverConfig cb;
    cb.s = 4;
    cb.tol = 1e-9;
    cb.spectrum = cs::SpectrumEstimate{blo, bhi};
    cs::gpu::set_mode(cs::gpu::Mode::reference);
    const cs::SolveResult rb = cs::pcg_s_solve(sys.a, b, x0, bj, cb);
    oc_cfg ob{4, 1e-9, 500, 30, 0, 1, blo, bhi, 40, 1234};
    std::vector<double> xb(n);
    oc_report brep{};
    brep.cap = 600;
    brep.rel_residual = rel.data();
    brep.delta_alpha = da.data();
    brep.delta_beta = db.data();
    EXPECT(ref_pcg_s_solve(n, rp.data(), ci.data(), v.data(), b.data(), x0.data(), 104, &ob,
                           xb.data(), &brep) == 0);
    EXPECT(rb.report.outer_iters == brep.outer_iters);
    EXPECT(same_bits(rb.x.data(), xb.data(), n));
    // host apply() of the drop-in class == the device apply (through mpk z_0 = M^-1 r)
    std::vector<double> hz(n);
    bj.apply(x, hz);
    const cs::MpkResult mb = cs::mpk_chebyshev(sys.a, x, 2, bj, params);
    EXPECT(same_bits(hz.data(), mb.z.data.data(), n));
    cs::gpu::set_mode(cs::gpu::Mode::fast);
  }

  // --- classical PCG comparator
  const cs::SolveResult pcg = cs::pcg_solve(sys.a, b, x0, jac, 1e-9, 1000);
  EXPECT(pcg.report.converged);

  // --- error convention: A = I, M = I, s = 4, interval [0.9, 1.1] (the auto
  // estimate's widening of lambda = 1): z_1 = (alpha - sigma) r = 0 exactly, so the
  // Gram diagonal vanishes -> SolverBreakdownError at outer 1
  const cs::CsrMatrix eye = cs::CsrMatrix::identity(40);
  const std::vector<double> b40(40, 1.0), z40(40, 0.0);
  cs::SolverConfig c4;
  c4.s = 4;
  c4.spectrum = cs::SpectrumEstimate{0.9, 1.1};
  cs::gpu::set_mode(cs::gpu::Mode::reference);
  bool thrown = false;
  try {
    cs::pcg_s_solve(eye, b40, z40, cs::IdentityPreconditioner{}, c4);
  } catch (const cs::SolverBreakdownError& e) {
    thrown = e.outer_iteration == 1;
  }
  EXPECT(thrown);
  bool dim = false;
  try {
    cs::pcg_s_solve(eye, std::vector<double>(39, 1.0), z40, cs::IdentityPreconditioner{}, c4);
  } catch (const cs::DimensionError&) {
    dim = true;
  }
  EXPECT(dim);
  // --- Matrix Market round trip: drop-in writer/reader == reference reader
  {
    const char* path = "/tmp/dropin_mm_test.mtx";
    cs::write_matrix_market(path, sys.a);
    const cs::CsrMatrix back = cs::read_matrix_market(path, true);
    int64_t rn = 0, rnnz = 0;
    EXPECT(ref_mm_read(path, 1, &rn, &rnnz, nullptr, nullptr, nullptr) == 0);
    std::vector<int64_t> rrp(rn + 1), rci(rnnz);
    std::vector<double> rv(rnnz);
    EXPECT(ref_mm_read(path, 1, &rn, &rnnz, rrp.data(), rci.data(), rv.data()) == 0);
    EXPECT(back.n == rn && back.nnz() == rnnz);
    EXPECT(same_bits(back.row_offsets.data(), rrp.data(), rn + 1));
    EXPECT(same_bits(back.col_indices.data(), rci.data(), rnnz));
    EXPECT(same_bits(back.values.data(), rv.data(), rnnz));
    EXPECT(same_bits(back.values.data(), sys.a.values.data(), nnz));
    bool parse = false;
    try {
      cs::read_matrix_market("/nonexistent/x.mtx");
    } catch (const cs::ParseError&) {
      parse = true;
    }
    EXPECT(parse);
    std::remove(path);
  }
  std::printf("%s (%d failures)\n", failures ? "DROPIN FAIL" : "DROPIN OK", failures);
  return failures ? 1 : 0;
}
