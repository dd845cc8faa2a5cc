// api.cpp -- the C++ drop-in (include/chebstep/api.hpp) on top of the C ABI.
//
// Every n-sized computation goes through libchebstep_gpu's CUDA kernels via
// chebstep_gpu.h; what stays on the host is what the reference's interface
// itself defines as host data handling (CSR/block containers, validators,
// the O(s^2) report bookkeeping). Reductions exposed here (dot, norm2,
// block_gram, assemble_gram) run in the reference's serial order on the
// device, so they are bitwise the reference's.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "chebstep/api.hpp"
#include "chebstep_gpu.h"

namespace chebstep {
namespace {

int g_device = 0;
gpu::Mode g_mode = gpu::Mode::fast;

[[noreturn]] void rethrow(int rc) {
  int payload = 0;
  const std::string msg = cs_last_error(&payload);
  switch (rc) {
    case CS_ERR_DIMENSION: throw DimensionError(msg);
    case CS_ERR_INVALID_MATRIX: throw InvalidMatrixError(msg);
    case CS_ERR_NOT_SPD: throw NotSpdError(msg);
    case CS_ERR_BASIS_BREAKDOWN: throw BasisBreakdownError(msg, payload);
    case CS_ERR_SOLVER_BREAKDOWN: throw SolverBreakdownError(msg, payload);
    case CS_ERR_GUARD_EXCEEDED: throw GuardExceededError(msg);
    case CS_ERR_PARSE: throw ParseError(msg);
    case CS_ERR_INVALID_ARGUMENT: throw InvalidArgumentError(msg);
    case CS_ERR_CUDA:
    case CS_ERR_NCCL: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

inline void check(int rc) {
  if (rc != CS_OK) rethrow(rc);
}

cs_ctx* ctx() {
  static std::mutex mu;
  static cs_ctx* c = nullptr;
  static int dev = -1;
  std::lock_guard<std::mutex> lk(mu);
  if (c == nullptr || dev != g_device) {
    if (c) cs_ctx_destroy(c);
    c = nullptr;
    check(cs_ctx_create(g_device, &c));
    dev = g_device;
  }
  return c;
}

}  // namespace
void attach_precond(cs_problem* p, const Preconditioner& m);
namespace {

// device-resident copy of a reference CsrMatrix for one call
struct Problem {
  cs_problem* p = nullptr;
  Problem(const CsrMatrix& a, const Preconditioner* m) {
    check(cs_problem_upload_csr(ctx(), a.n, a.row_offsets.data(), a.col_indices.data(),
                                a.values.data(), &p));
    if (m) attach_precond(p, *m);
  }
  ~Problem() { cs_problem_destroy(p); }
  Problem(const Problem&) = delete;
  Problem& operator=(const Problem&) = delete;
};

int mode_code() { return g_mode == gpu::Mode::reference ? CS_MODE_REFERENCE : CS_MODE_FAST; }

}  // namespace

namespace gpu {
void set_mode(Mode m) { g_mode = m; }
Mode mode() { return g_mode; }
void set_device(int device) { g_device = device; }
}  // namespace gpu

// ------------------------------------------------------------------ util (util.cpp:8-36)
int log_level() {
  static const int level = [] {
    const char* env = std::getenv("CHEBSTEP_LOG");
    return (env == nullptr || *env == '\0') ? 0 : std::atoi(env);
  }();
  return level;
}
void log_info(const std::string& msg) {
  if (log_level() >= 1) std::fprintf(stderr, "[chebstep] %s\n", msg.c_str());
}
void log_debug(const std::string& msg) {
  if (log_level() >= 2) std::fprintf(stderr, "[chebstep:debug] %s\n", msg.c_str());
}
std::string fmt_double(double x) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}
std::vector<double> random_vector(index_t n, std::uint64_t seed) {
  std::vector<double> v(static_cast<std::size_t>(n));
  if (n > 0) check(cs_random_vector(ctx(), n, seed, v.data()));
  return v;
}

// ------------------------------------------------------------------ csr
double CsrMatrix::diagonal(index_t i) const {
  const auto c = row_cols(i);
  const auto it = std::lower_bound(c.begin(), c.end(), i);
  if (it == c.end() || *it != i) return 0.0;
  return values[row_offsets[i] + (it - c.begin())];
}

CsrMatrix CsrMatrix::identity(index_t n) {
  CsrMatrix a;
  a.n = n;
  a.row_offsets.resize(n + 1);
  a.col_indices.resize(n);
  a.values.assign(n, 1.0);
  for (index_t i = 0; i <= n; ++i) a.row_offsets[i] = i;
  for (index_t i = 0; i < n; ++i) a.col_indices[i] = i;
  return a;
}

CsrMatrix CsrMatrix::diagonal_matrix(std::span<const double> d) {
  CsrMatrix a = identity(static_cast<index_t>(d.size()));
  std::copy(d.begin(), d.end(), a.values.begin());
  return a;
}

CsrMatrix CsrMatrix::from_triplets(index_t n,
                                   std::vector<std::pair<std::pair<index_t, index_t>, double>> t) {
  std::sort(t.begin(), t.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  for (std::size_t k = 1; k < t.size(); ++k)
    if (t[k].first == t[k - 1].first) throw InvalidMatrixError("duplicate entry in triplet list");
  CsrMatrix a;
  a.n = n;
  a.row_offsets.assign(n + 1, 0);
  for (const auto& e : t) {
    const auto [i, j] = e.first;
    if (i < 0 || i >= n || j < 0 || j >= n) throw InvalidMatrixError("triplet index out of range");
    ++a.row_offsets[i + 1];
    a.col_indices.push_back(j);
    a.values.push_back(e.second);
  }
  for (index_t i = 0; i < n; ++i) a.row_offsets[i + 1] += a.row_offsets[i];
  return a;
}

void validate_structure(const CsrMatrix& a) {
  if (a.n < 0 || static_cast<index_t>(a.row_offsets.size()) != a.n + 1)
    throw InvalidMatrixError("row_offsets length must be n+1");
  if (a.row_offsets.front() != 0) throw InvalidMatrixError("row_offsets[0] must be 0");
  if (a.row_offsets.back() != a.nnz() || a.values.size() != a.col_indices.size())
    throw InvalidMatrixError("row_offsets[n] must equal nnz");
  for (index_t i = 0; i < a.n; ++i) {
    if (a.row_offsets[i] > a.row_offsets[i + 1])
      throw InvalidMatrixError("row_offsets must be nondecreasing");
    const auto c = a.row_cols(i);
    for (std::size_t k = 0; k < c.size(); ++k) {
      if (c[k] < 0 || c[k] >= a.n) throw InvalidMatrixError("column index out of range");
      if (k > 0 && c[k] <= c[k - 1])
        throw InvalidMatrixError("column indices must be strictly increasing");
    }
  }
  for (double v : a.values)
    if (!std::isfinite(v)) throw InvalidMatrixError("non-finite matrix value");
}

void validate_symmetric(const CsrMatrix& a) {
  validate_structure(a);
  for (index_t i = 0; i < a.n; ++i) {
    const auto c = a.row_cols(i);
    const auto v = a.row_vals(i);
    for (std::size_t k = 0; k < c.size(); ++k) {
      const auto jc = a.row_cols(c[k]);
      const auto it = std::lower_bound(jc.begin(), jc.end(), i);
      if (it == jc.end() || *it != i) throw InvalidMatrixError("missing symmetric counterpart entry");
      if (a.values[a.row_offsets[c[k]] + (it - jc.begin())] != v[k])
        throw InvalidMatrixError("symmetric counterpart value differs");
    }
  }
}

void validate_spd_diagonal(const CsrMatrix& a) {
  for (index_t i = 0; i < a.n; ++i) {
    const auto c = a.row_cols(i);
    const auto it = std::lower_bound(c.begin(), c.end(), i);
    if (it == c.end() || *it != i) throw NotSpdError("missing diagonal entry in SPD matrix");
    if (a.values[a.row_offsets[i] + (it - c.begin())] <= 0.0)
      throw NotSpdError("non-positive diagonal entry in SPD matrix");
  }
}

void spmv_into(const CsrMatrix& a, std::span<const double> x, std::span<double> y) {
  if (static_cast<index_t>(x.size()) != a.n || static_cast<index_t>(y.size()) != a.n)
    throw DimensionError("spmv: vector length must equal matrix dimension");
  if (a.n == 0) return;
  Problem p(a, nullptr);
  check(cs_spmv(p.p, x.data(), y.data()));
}

std::vector<double> spmv(const CsrMatrix& a, std::span<const double> x) {
  std::vector<double> y(static_cast<std::size_t>(a.n));
  spmv_into(a, x, y);
  return y;
}

// ------------------------------------------------------------------ blocks
VectorBlock::VectorBlock(index_t n_, index_t k_) : n(n_), k(k_) {
  if (n_ < 0 || k_ < 0) throw DimensionError("VectorBlock: negative shape");
  data.assign(static_cast<std::size_t>(n_ * k_), 0.0);
}
void VectorBlock::set_col(index_t j, std::span<const double> v) {
  if (static_cast<index_t>(v.size()) != n) throw DimensionError("set_col: length mismatch");
  std::copy(v.begin(), v.end(), col(j));
}
VectorBlock VectorBlock::columns(index_t first, index_t count) const {
  if (first < 0 || count < 0 || first + count > k)
    throw DimensionError("columns: range out of bounds");
  VectorBlock out(n, count);
  std::copy(col(first), col(first) + n * count, out.data.begin());
  return out;
}
VectorBlock VectorBlock::from_column(std::span<const double> v) {
  VectorBlock out(static_cast<index_t>(v.size()), 1);
  out.set_col(0, v);
  return out;
}
SmallDense::SmallDense(int r, int c) : rows(r), cols(c) {
  if (r < 0 || c < 0 || r > kSmallDenseMax || c > kSmallDenseMax)
    throw DimensionError("SmallDense: dimensions must be in [0, 64]");
  data.assign(static_cast<std::size_t>(r) * c, 0.0);
}
SmallDense SmallDense::identity(int m) {
  SmallDense o(m, m);
  for (int i = 0; i < m; ++i) o.at(i, i) = 1.0;
  return o;
}
SmallDense SmallDense::from_column(std::span<const double> v) {
  SmallDense o(static_cast<int>(v.size()), 1);
  std::copy(v.begin(), v.end(), o.data.begin());
  return o;
}
double frobenius_norm(const SmallDense& m) {
  double acc = 0.0;
  for (double x : m.data) acc += x * x;
  return std::sqrt(acc);
}
double max_abs(const SmallDense& m) {
  double best = 0.0;
  for (double x : m.data) best = std::max(best, std::abs(x));
  return best;
}

// ------------------------------------------------------------------ dense ops
double dot(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size()) throw DimensionError("dot: length mismatch");
  if (x.empty()) return 0.0;
  double g = 0.0;
  check(cs_block_gram(ctx(), static_cast<int64_t>(x.size()), 1, 1, x.data(), y.data(), &g,
                      CS_MODE_REFERENCE));
  return g;
}
double norm2(std::span<const double> x) { return std::sqrt(dot(x, x)); }

SmallDense block_gram(const VectorBlock& u, const VectorBlock& v) {
  if (u.n != v.n) throw DimensionError("block_gram: row counts differ");
  SmallDense g(static_cast<int>(u.k), static_cast<int>(v.k));
  if (u.k && v.k && u.n)
    check(cs_block_gram(ctx(), u.n, static_cast<int>(u.k), static_cast<int>(v.k), u.data.data(),
                        v.data.data(), g.data.data(), CS_MODE_REFERENCE));
  return g;
}

VectorBlock block_update(const VectorBlock& y, const VectorBlock& x, const SmallDense& c) {
  if (x.n != y.n || x.k != c.rows || y.k != c.cols)
    throw DimensionError("block_update: shape mismatch");
  VectorBlock out(y.n, y.k);
  if (y.n && y.k)
    check(cs_block_update(ctx(), y.n, static_cast<int>(x.k), static_cast<int>(y.k), y.data.data(),
                          x.data.data(), c.data.data(), out.data.data()));
  return out;
}

SmallDense small_cholesky_solve(const SmallDense& w, const SmallDense& rhs) {
  if (w.rows != w.cols) throw DimensionError("cholesky: matrix not square");
  if (rhs.rows != w.rows) throw DimensionError("cholesky: rhs rows mismatch");
  SmallDense x(rhs.rows, rhs.cols);
  check(cs_cholesky_solve(ctx(), w.rows, w.data.data(), rhs.cols, rhs.data.data(), x.data.data()));
  return x;
}

// ------------------------------------------------------------------ precond (precond.cpp:9-30)
void IdentityPreconditioner::apply(std::span<const double> in, std::span<double> out) const {
  if (in.size() != out.size()) throw DimensionError("identity: size mismatch");
  std::copy(in.begin(), in.end(), out.begin());
}
JacobiPreconditioner::JacobiPreconditioner(const CsrMatrix& a) {
  inv_diag_.resize(static_cast<std::size_t>(a.n));
  for (index_t i = 0; i < a.n; ++i) {
    const double d = a.diagonal(i);
    if (!(d > 0.0)) throw NotSpdError("jacobi: diagonal must be strictly positive");
    inv_diag_[static_cast<std::size_t>(i)] = 1.0 / d;
  }
}
void JacobiPreconditioner::apply(std::span<const double> in, std::span<double> out) const {
  if (in.size() != out.size() || in.size() != inv_diag_.size())
    throw DimensionError("jacobi: size mismatch");
  for (std::size_t i = 0; i < in.size(); ++i) out[i] = inv_diag_[i] * in[i];
}

// block Jacobi: host extraction + factorisation; the device factorises the same
// blocks with the same operation order (vec.cu bj_factor_kernel)
BlockJacobiPreconditioner::BlockJacobiPreconditioner(const CsrMatrix& a, int bs)
    : bs_(bs), n_(a.n) {
  if (bs < 1 || bs > 16) throw InvalidArgumentError("block_jacobi: bs must be in [1, 16]");
  const index_t nb = (a.n + bs - 1) / bs;
  const std::size_t q = static_cast<std::size_t>(bs) * bs;
  blocks_.assign(static_cast<std::size_t>(nb) * q, 0.0);
  for (index_t r = 0; r < nb * bs; ++r) {
    double* blk = blocks_.data() + static_cast<std::size_t>(r / bs) * q;
    const int i = static_cast<int>(r % bs);
    if (r >= a.n) {
      blk[i + i * bs] = 1.0;
      continue;
    }
    const index_t b0 = (r / bs) * bs;
    for (index_t k = a.row_offsets[r]; k < a.row_offsets[r + 1]; ++k) {
      const index_t c = a.col_indices[k];
      if (c >= b0 && c < b0 + bs) blk[i + (c - b0) * bs] += a.values[k];
    }
  }
  factor_ = blocks_;
  for (index_t b = 0; b < nb; ++b) {
    double* L = factor_.data() + static_cast<std::size_t>(b) * q;
    for (int j = 0; j < bs; ++j) {
      double d = L[j + j * bs];
      for (int t = 0; t < j; ++t) d -= L[j + t * bs] * L[j + t * bs];
      if (!(d > 0.0) || !std::isfinite(d))
        throw NotSpdError("block_jacobi: diagonal block " + std::to_string(b) +
                          " is not positive definite");
      const double dg = std::sqrt(d);
      L[j + j * bs] = dg;
      for (int i = j + 1; i < bs; ++i) {
        double v = L[i + j * bs];
        for (int t = 0; t < j; ++t) v -= L[i + t * bs] * L[j + t * bs];
        L[i + j * bs] = v / dg;
      }
      for (int i = 0; i < j; ++i) L[i + j * bs] = 0.0;
    }
  }
}

void BlockJacobiPreconditioner::apply(std::span<const double> in, std::span<double> out) const {
  if (in.size() != out.size() || static_cast<index_t>(in.size()) != n_)
    throw DimensionError("block_jacobi: size mismatch");
  const int bs = bs_;
  std::vector<double> x(static_cast<std::size_t>(bs));
  for (index_t r0 = 0; r0 < n_; r0 += bs) {
    const double* L = factor_.data() + static_cast<std::size_t>(r0 / bs) * bs * bs;
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

// ------------------------------------------------------------------ problems
namespace {
PoissonSystem generated(int kind, const PoissonSpec& spec, const double* coef) {
  cs_problem* p = nullptr;
  check(cs_problem_generate(ctx(), kind, spec.nx, spec.ny, spec.nz, coef, &p));
  int64_t info[12];
  cs_problem_info(p, info);
  PoissonSystem sys;
  sys.a.n = info[1];
  sys.a.row_offsets.resize(info[1] + 1);
  sys.a.col_indices.resize(info[2]);
  sys.a.values.resize(info[2]);
  const int rc = cs_problem_download_csr(p, sys.a.row_offsets.data(), sys.a.col_indices.data(),
                                         sys.a.values.data());
  cs_problem_destroy(p);
  check(rc);
  sys.rhs.assign(static_cast<std::size_t>(sys.a.n), 1.0);
  return sys;
}
}  // namespace

CsrMatrix read_matrix_market(const std::string& path, bool require_spd) {
  cs_csr_host* h = nullptr;
  int64_t n = 0, nnz = 0;
  check(cs_mm_read(path.c_str(), require_spd ? 1 : 0, &h, &n, &nnz));
  CsrMatrix a;
  a.n = n;
  a.row_offsets.resize(static_cast<size_t>(n) + 1);
  a.col_indices.resize(static_cast<size_t>(nnz));
  a.values.resize(static_cast<size_t>(nnz));
  const int rc = cs_csr_host_rows(h, 0, n, a.row_offsets.data(), a.col_indices.data(),
                                  a.values.data());
  cs_csr_host_free(h);
  check(rc);
  return a;
}

void write_matrix_market(const std::string& path, const CsrMatrix& a) {
  check(cs_mm_write(path.c_str(), a.n, a.row_offsets.data(), a.col_indices.data(),
                    a.values.data()));
}

PoissonSystem poisson27(const PoissonSpec& spec) { return generated(CS_GEN_POISSON27, spec, nullptr); }

PoissonSystem stencil7(const PoissonSpec& spec, double cx, double cy, double cz) {
  const double coef[3] = {cx, cy, cz};
  return generated(CS_GEN_STENCIL7, spec, coef);
}

// ------------------------------------------------------------------ spectral
SpectrumEstimate estimate_interval(const CsrMatrix& a, const Preconditioner& m, int steps,
                                   std::uint64_t seed) {
  Problem p(a, &m);
  SpectrumEstimate e;
  check(cs_estimate_interval(p.p, steps, seed, mode_code(), &e.lambda_min, &e.lambda_max));
  e.method = SpectrumMethod::lanczos;
  e.low_factor = 0.9;
  e.high_factor = 1.1;
  return e;
}

std::pair<double, double> gershgorin_bounds(const CsrMatrix& a) {
  double lo = INFINITY, hi = -INFINITY;
  for (index_t i = 0; i < a.n; ++i) {
    const auto c = a.row_cols(i);
    const auto v = a.row_vals(i);
    double d = 0.0, r = 0.0;
    for (std::size_t k = 0; k < c.size(); ++k) {
      if (c[k] == i) d = v[k];
      else r += std::abs(v[k]);
    }
    lo = std::min(lo, d - r);
    hi = std::max(hi, d + r);
  }
  return {lo, hi};
}

// ------------------------------------------------------------------ mpk
ChebyshevParams ChebyshevParams::from_interval(double lo, double hi) {
  if (!(hi > lo) || !(lo > 0.0) || !std::isfinite(hi))
    throw InvalidArgumentError("ChebyshevParams: need lambda_max > lambda_min > 0");
  return {lo, hi};
}

MpkResult mpk_chebyshev(const CsrMatrix& a, std::span<const double> r, int s,
                        const Preconditioner& m, const ChebyshevParams& params) {
  if (s < 1) throw InvalidArgumentError("mpk: s must be >= 1");
  if (static_cast<index_t>(r.size()) != a.n) throw DimensionError("mpk: residual length mismatch");
  Problem p(a, &m);
  MpkResult out;
  out.z = VectorBlock(a.n, s);
  out.p = VectorBlock(a.n, s + 1);
  check(cs_mpk(p.p, r.data(), s, params.lambda_min, params.lambda_max, out.z.data.data(),
               out.p.data.data()));
  return out;
}

// ------------------------------------------------------------------ gram
SmallDense GramSystem::strict_lower() const {
  const int s = order();
  SmallDense l(s, s);
  for (int j = 0; j < s; ++j)
    for (int i = j + 1; i < s; ++i) l.at(i, j) = w.at(i, j);
  return l;
}

namespace {
GramSystem finish(SmallDense w) {
  GramSystem g;
  for (int i = 0; i < w.rows; ++i) {
    const double d = w.at(i, i);
    if (!(d > 0.0) || !std::isfinite(d))
      throw NotSpdError("gram: non-positive diagonal (basis degeneracy)");
    g.diag.push_back(d);
  }
  g.w = std::move(w);
  return g;
}
}  // namespace

GramSystem assemble_gram(const VectorBlock& q, const VectorBlock& aq) {
  if (q.n != aq.n || q.k != aq.k) throw DimensionError("assemble_gram: block shapes differ");
  SmallDense w(static_cast<int>(q.k), static_cast<int>(q.k));
  check(cs_assemble_gram(ctx(), q.n, static_cast<int>(q.k), q.data.data(), aq.data.data(),
                         w.data.data(), CS_MODE_REFERENCE));
  return finish(std::move(w));
}

GramSystem gram_from_matrix(const SmallDense& w) {
  if (w.rows != w.cols) throw DimensionError("gram_from_matrix: not square");
  for (int j = 0; j < w.cols; ++j)
    for (int i = 0; i < j; ++i)
      if (w.at(i, j) != w.at(j, i)) throw InvalidMatrixError("gram_from_matrix: matrix not symmetric");
  return finish(w);
}

GramSystem normalize_gram(const GramSystem& g) {  // gram.cpp:60-76
  const int s = g.order();
  SmallDense wc(s, s);
  std::vector<double> inv_sqrt(static_cast<size_t>(s));
  for (int i = 0; i < s; ++i) inv_sqrt[i] = 1.0 / std::sqrt(g.diag[i]);
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < s; ++i)
      wc.at(i, j) = (i == j) ? 1.0 : g.w.at(i, j) * inv_sqrt[i] * inv_sqrt[j];
  GramSystem out;
  out.w = std::move(wc);
  out.diag.assign(static_cast<size_t>(s), 1.0);
  out.normalized = true;
  return out;
}

FgsRate fgs_rate(const GramSystem& g) {
  if (!g.normalized) throw InvalidArgumentError("fgs_rate: system must be normalized");
  FgsRate r{0.0, 0.0};
  check(cs_fgs_rate(g.order(), g.w.data.data(), &r.spectral_norm, &r.spectral_radius));
  return r;
}

FgsResult fgs_solve(const GramSystem& g, const SmallDense& rhs, const FgsConfig& cfg) {
  if (cfg.nu < 1) throw InvalidArgumentError("fgs: nu must be >= 1");
  if (rhs.rows != g.order()) throw DimensionError("fgs: rhs rows mismatch");
  if (!cfg.multi_rhs && rhs.cols > 1)
    throw InvalidArgumentError("fgs: multiple right-hand sides disabled");
  FgsResult r{SmallDense(rhs.rows, rhs.cols), 0.0};
  check(cs_fgs_solve(ctx(), g.order(), g.w.data.data(), rhs.cols, rhs.data.data(), cfg.nu,
                     r.x.data.data(), &r.rel_residual));
  return r;
}

// ------------------------------------------------------------------ solver
void SolverConfig::validate() const {
  if (s < 1 || s > kSmallDenseMax) throw InvalidArgumentError("SolverConfig: s must be in [1, 64]");
  if (!(tol > 0.0)) throw InvalidArgumentError("SolverConfig: tol must be > 0");
  if (max_outer < 1) throw InvalidArgumentError("SolverConfig: max_outer must be >= 1");
  if (fgs.nu < 1) throw InvalidArgumentError("SolverConfig: nu must be >= 1");
}

namespace {
void fill(SolveReport& r, const cs_report& c, const std::vector<double>& rel,
          const std::vector<double>& da, const std::vector<double>& db) {
  r.converged = c.converged != 0;
  r.outer_iters = c.outer_iters;
  r.rel_residual.assign(rel.begin(), rel.begin() + std::min<std::size_t>(c.n_rel, rel.size()));
  r.delta_alpha.assign(da.begin(), da.begin() + std::min<std::size_t>(c.n_da, da.size()));
  r.delta_beta.assign(db.begin(), db.begin() + std::min<std::size_t>(c.n_db, db.size()));
  r.spmv_count = c.spmv_count;
  r.precond_count = c.precond_count;
  r.allreduce_count = c.allreduce_count;
  r.local_update_flops = c.local_update_flops;
  r.gram_solve_flops = c.gram_solve_flops;
  r.spectrum_used.lambda_min = c.lambda_min;
  r.spectrum_used.lambda_max = c.lambda_max;
}
}  // namespace

namespace {
// caller-side buffers for the analysis-hook histories
struct HookBufs {
  std::vector<double> kappa, gram, truer, aerr, iter;
  void attach(cs_report& r, int cap, int s, index_t n, bool g, bool t, bool e, bool it) {
    if (g) {
      kappa.assign(cap, 0.0);
      gram.assign(static_cast<size_t>(cap) * s * s, 0.0);
      r.kappa_w = kappa.data();
      r.gram_history = gram.data();
    }
    if (t) {
      truer.assign(cap, 0.0);
      r.true_rel_residual = truer.data();
    }
    if (e) {
      aerr.assign(cap, 0.0);
      r.a_norm_error = aerr.data();
    }
    if (it) {
      iter.assign(static_cast<size_t>(cap) * n, 0.0);
      r.iterates = iter.data();
    }
  }
  void fill(SolveReport& rep, const cs_report& r, int s, index_t n) const {
    for (int i = 0; i < r.n_kappa && i < static_cast<int>(kappa.size()); ++i) {
      rep.kappa_w.push_back(kappa[i]);
      SmallDense w(s, s);
      std::copy(gram.begin() + static_cast<size_t>(i) * s * s,
                gram.begin() + static_cast<size_t>(i + 1) * s * s, w.data.begin());
      rep.gram_history.push_back(std::move(w));
    }
    rep.true_rel_residual.assign(truer.begin(),
                                 truer.begin() + std::min<size_t>(r.n_true, truer.size()));
    rep.a_norm_error.assign(aerr.begin(), aerr.begin() + std::min<size_t>(r.n_aerr, aerr.size()));
    for (int i = 0; i < r.n_iter && static_cast<size_t>(i + 1) * n <= iter.size(); ++i)
      rep.iterates.emplace_back(iter.begin() + static_cast<size_t>(i) * n,
                                iter.begin() + static_cast<size_t>(i + 1) * n);
  }
};
}  // namespace

namespace {
cs_config to_cs(const SolverConfig& cfg, index_t n) {
  cfg.validate();
  cs_config c;
  cs_config_default(&c);
  c.s = cfg.s;
  c.tol = cfg.tol;
  c.max_outer = cfg.max_outer;
  c.nu = cfg.fgs.nu;
  c.gram = cfg.gram_solver == GramSolverKind::cholesky ? CS_GRAM_CHOLESKY : CS_GRAM_FGS;
  if (cfg.spectrum) {
    c.has_spectrum = 1;
    c.lambda_min = cfg.spectrum->lambda_min;
    c.lambda_max = cfg.spectrum->lambda_max;
  }
  c.lanczos_steps = cfg.lanczos_steps;
  c.seed = cfg.seed;
  c.mode = mode_code();
  c.collect_gram = cfg.collect_gram;
  c.track_true_residual = cfg.track_true_residual;
  c.collect_iterates = cfg.collect_iterates;
  if (cfg.error_reference) {
    if (static_cast<index_t>(cfg.error_reference->size()) != n)
      throw DimensionError("pcg_s_solve: error_reference length mismatch");
    c.error_reference = cfg.error_reference->data();
  }
  return c;
}

// one s-step solve through `call` (fills cs_report), histories + hooks unpacked
template <class Call>
SolveResult run_pcgs(const SolverConfig& cfg, index_t n, Call&& call) {
  cs_config c = to_cs(cfg, n);
  SolveResult out;
  out.x.resize(static_cast<std::size_t>(n));
  const int cap = cfg.max_outer + 2;
  std::vector<double> rel(cap), da(cap), db(cap);
  cs_report r{};
  r.cap = cap;
  r.rel_residual = rel.data();
  r.delta_alpha = da.data();
  r.delta_beta = db.data();
  HookBufs hb;
  hb.attach(r, cap, cfg.s, n, cfg.collect_gram, cfg.track_true_residual,
            cfg.error_reference.has_value(), cfg.collect_iterates);
  check(call(&c, out.x.data(), &r));
  fill(out.report, r, rel, da, db);
  hb.fill(out.report, r, cfg.s, n);
  if (cfg.spectrum) out.report.spectrum_used = *cfg.spectrum;
  else if (r.lambda_max > 0.0) {
    out.report.spectrum_used.low_factor = 0.9;
    out.report.spectrum_used.high_factor = 1.1;
  }
  return out;
}

template <class Call>
SolveResult run_pcg(const PcgConfig& cfg, index_t n, Call&& call) {
  if (!(cfg.tol >= 0.0) || cfg.max_iter < 1) throw InvalidArgumentError("pcg_solve: bad tol/max_iter");
  cs_config c;
  cs_config_default(&c);
  c.tol = cfg.tol;
  c.max_outer = cfg.max_iter;
  c.mode = mode_code();
  c.collect_iterates = cfg.collect_iterates;
  if (cfg.error_reference) {
    if (static_cast<index_t>(cfg.error_reference->size()) != n)
      throw DimensionError("pcg_solve: error_reference length mismatch");
    c.error_reference = cfg.error_reference->data();
  }
  SolveResult out;
  out.x.resize(static_cast<std::size_t>(n));
  const int cap = cfg.max_iter + 2;
  std::vector<double> rel(cap);
  cs_report r{};
  r.cap = cap;
  r.rel_residual = rel.data();
  HookBufs hb;
  hb.attach(r, cap, 1, n, false, false, cfg.error_reference.has_value(), cfg.collect_iterates);
  check(call(&c, out.x.data(), &r));
  fill(out.report, r, rel, {}, {});
  hb.fill(out.report, r, 1, n);
  out.report.spectrum_used = SpectrumEstimate{};
  return out;
}

int precond_kind(const Preconditioner& m) {
  const std::string_view nm = m.name();
  const int kind = nm == "jacobi" ? CS_PRECOND_JACOBI : nm == "identity" ? CS_PRECOND_IDENTITY : -1;
  if (kind < 0) throw InvalidArgumentError("preconditioner has no device implementation");
  return kind;
}

bool general_precond(const Preconditioner& m) {
  return dynamic_cast<const BlockJacobiPreconditioner*>(&m) != nullptr ||
         dynamic_cast<const gpu::DevicePreconditioner*>(&m) != nullptr;
}

int device_precond_trampoline(void* user, const double* in, double* out, int64_t n, void* stream) {
  try {
    static_cast<const gpu::DevicePreconditioner*>(user)->device_apply(in, out, n, stream);
    return 0;
  } catch (...) {
    return 1;
  }
}
}  // namespace

// every preconditioner kind onto a problem: identity/jacobi (fused), block
// Jacobi (device-factored blocks), device plugin
void attach_precond(cs_problem* p, const Preconditioner& m) {
  if (const auto* bj = dynamic_cast<const BlockJacobiPreconditioner*>(&m)) {
    check(cs_problem_set_precond_block_jacobi(p, bj->block_size(), bj->blocks().data()));
    return;
  }
  if (const auto* dp = dynamic_cast<const gpu::DevicePreconditioner*>(&m)) {
    check(cs_problem_set_precond_fn(p, device_precond_trampoline,
                                    const_cast<gpu::DevicePreconditioner*>(dp)));
    return;
  }
  const std::string_view nm = m.name();
  if (nm != "identity" && nm != "jacobi")
    throw InvalidArgumentError("preconditioner '" + std::string(nm) +
                               "' has no device implementation (identity, jacobi, "
                               "BlockJacobiPreconditioner, gpu::DevicePreconditioner)");
  check(cs_problem_set_precond(p, precond_kind(m)));
}

SolveResult pcg_s_solve(const CsrMatrix& a, std::span<const double> b, std::span<const double> x0,
                        const Preconditioner& m, const SolverConfig& cfg) {
  cfg.validate();
  if (static_cast<index_t>(b.size()) != a.n || static_cast<index_t>(x0.size()) != a.n)
    throw DimensionError("pcg_s_solve: vector length mismatch");
  if (general_precond(m)) {  // upload, attach the device preconditioner, solve
    Problem p(a, &m);
    return run_pcgs(cfg, a.n, [&](const cs_config* c, double* x, cs_report* r) {
      return cs_pcg_s_solve(p.p, b.data(), x0.data(), c, x, r);
    });
  }
  const int kind = precond_kind(m);
  return run_pcgs(cfg, a.n, [&](const cs_config* c, double* x, cs_report* r) {
    return cs_pcg_s_solve_csr(ctx(), a.n, a.row_offsets.data(), a.col_indices.data(),
                              a.values.data(), kind, b.data(), x0.data(), c, x, r);
  });
}

SolveResult pcg_solve(const CsrMatrix& a, std::span<const double> b, std::span<const double> x0,
                      const Preconditioner& m, const PcgConfig& cfg) {
  if (!(cfg.tol >= 0.0) || cfg.max_iter < 1) throw InvalidArgumentError("pcg_solve: bad tol/max_iter");
  if (static_cast<index_t>(b.size()) != a.n || static_cast<index_t>(x0.size()) != a.n)
    throw DimensionError("pcg_solve: vector length mismatch");
  Problem p(a, &m);
  return run_pcg(cfg, a.n, [&](const cs_config* c, double* x, cs_report* r) {
    return cs_pcg_solve_cfg(p.p, b.data(), x0.data(), c, x, r);
  });
}

// ------------------------------------------------------------------ device-resident problems
namespace gpu {

DeviceProblem::DeviceProblem(cs_problem* p) : p_(p) {
  int64_t info[12];
  check(cs_problem_info(p_, info));
  n_global_ = info[0], n_local_ = info[1], nnz_local_ = info[2], row_begin_ = info[3];
}
DeviceProblem::~DeviceProblem() {
  if (p_) cs_problem_destroy(p_);
}
DeviceProblem::DeviceProblem(DeviceProblem&& o) noexcept { *this = std::move(o); }
DeviceProblem& DeviceProblem::operator=(DeviceProblem&& o) noexcept {
  if (this != &o) {
    if (p_) cs_problem_destroy(p_);
    p_ = o.p_;
    n_global_ = o.n_global_, n_local_ = o.n_local_, nnz_local_ = o.nnz_local_;
    row_begin_ = o.row_begin_;
    o.p_ = nullptr;
  }
  return *this;
}

DeviceProblem DeviceProblem::poisson27(const PoissonSpec& spec) {
  cs_problem* p = nullptr;
  check(cs_problem_generate(ctx(), CS_GEN_POISSON27, spec.nx, spec.ny, spec.nz, nullptr, &p));
  return DeviceProblem(p);
}
DeviceProblem DeviceProblem::stencil7(const PoissonSpec& spec, double cx, double cy, double cz) {
  const double coef[3] = {cx, cy, cz};
  cs_problem* p = nullptr;
  check(cs_problem_generate(ctx(), CS_GEN_STENCIL7, spec.nx, spec.ny, spec.nz, coef, &p));
  return DeviceProblem(p);
}
DeviceProblem DeviceProblem::from_csr(const CsrMatrix& a) {
  cs_problem* p = nullptr;
  check(cs_problem_upload_csr(ctx(), a.n, a.row_offsets.data(), a.col_indices.data(),
                              a.values.data(), &p));
  return DeviceProblem(p);
}
DeviceProblem DeviceProblem::read_matrix_market(const std::string& path, bool require_spd) {
  cs_problem* p = nullptr;
  check(cs_problem_read_mm(ctx(), path.c_str(), require_spd ? 1 : 0, &p));
  return DeviceProblem(p);
}
void DeviceProblem::set_precond(const Preconditioner& m) {
  attach_precond(p_, m);
}

SolveResult pcg_s_solve(const DeviceProblem& p, std::span<const double> b,
                        std::span<const double> x0, const SolverConfig& cfg) {
  cfg.validate();
  if (static_cast<index_t>(b.size()) != p.n_local() || static_cast<index_t>(x0.size()) != p.n_local())
    throw DimensionError("pcg_s_solve: vector length mismatch");
  return run_pcgs(cfg, p.n_local(), [&](const cs_config* c, double* x, cs_report* r) {
    return cs_pcg_s_solve(p.handle(), b.data(), x0.data(), c, x, r);
  });
}

SolveResult pcg_solve(const DeviceProblem& p, std::span<const double> b,
                      std::span<const double> x0, const PcgConfig& cfg) {
  if (static_cast<index_t>(b.size()) != p.n_local() || static_cast<index_t>(x0.size()) != p.n_local())
    throw DimensionError("pcg_solve: vector length mismatch");
  return run_pcg(cfg, p.n_local(), [&](const cs_config* c, double* x, cs_report* r) {
    return cs_pcg_solve_cfg(p.handle(), b.data(), x0.data(), c, x, r);
  });
}

}  // namespace gpu

SolveResult pcg_solve(const CsrMatrix& a, std::span<const double> b, std::span<const double> x0,
                      const Preconditioner& m, double tol, int max_iter) {
  PcgConfig cfg;
  cfg.tol = tol;
  cfg.max_iter = max_iter;
  return pcg_solve(a, b, x0, m, cfg);
}

InexactVerdict monitor_inexact(const SolveReport& report, double delta_cap) {
  double max_delta = 0.0;
  for (double d : report.delta_alpha) max_delta = std::max(max_delta, d);
  const double budget = static_cast<double>(report.outer_iters) * max_delta;
  return {max_delta, budget, budget <= delta_cap};
}

double a_norm_error(const CsrMatrix& a, std::span<const double> x, std::span<const double> ref) {
  std::vector<double> e(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) e[i] = x[i] - ref[i];
  return std::sqrt(std::max(0.0, dot(e, spmv(a, e))));
}

}  // namespace chebstep
