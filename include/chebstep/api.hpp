// chebstep/api.hpp -- C++ drop-in for the reference chebstep solve path,
// executed on B200 by libchebstep_gpu.so.
//
// Source- and link-compatible subset of the reference public headers
// (/root/reference/proj/include/chebstep/*.hpp): same namespace, type names,
// member order and function signatures for everything on the solve path, so
// solve-path callers compile and link against this library unchanged. Callers
// that also use the reference's analysis modules do not: e.g. the reference
// cli.cpp includes moments.hpp / perf_model.hpp (cli.cpp:13-14), and
// dense_ops.hpp:24-53 (block_combine, ldlt_pivots, InnerProduct,
// mgs_orthogonalize_first), gram.hpp:55-78 (fgs_residual_oracle,
// ruhe_equivalence_check, gram_kappa_check) and the dense paths of
// spectral.hpp:35-53 are not declared here (out of scope). The repo's
// own CLI (csrc/cli.cpp) covers solve / compare / gram-analysis. The per-module headers next to this file (csr.hpp,
// solver.hpp, ...) all forward here. Compute entries go through the C ABI in
// chebstep_gpu.h (CUDA kernels for sm_100a, no CPU fallback); the analysis-only
// modules of the reference (moments, perf_model, cli, dense LAPACK paths,
// Matrix Market I/O) are not part of this library -- see DESIGN.md.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

typedef struct cs_problem cs_problem;

namespace chebstep {

using index_t = std::int64_t;  // util.hpp:10

// ------------------------------------------------------------------ errors (errors.hpp:9-56)
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct InvalidMatrixError : Error {
  using Error::Error;
};
struct NotSpdError : Error {
  using Error::Error;
};
struct BasisBreakdownError : Error {
  BasisBreakdownError(const std::string& what, int col) : Error(what), column(col) {}
  int column;
};
struct SolverBreakdownError : Error {
  SolverBreakdownError(const std::string& what, int outer) : Error(what), outer_iteration(outer) {}
  int outer_iteration;
};
struct GuardExceededError : Error {
  using Error::Error;
};
struct ParseError : Error {
  using Error::Error;
};
struct InvalidArgumentError : Error {
  using Error::Error;
};
/// Device or collective failure (no counterpart in the CPU reference).
struct DeviceError : Error {
  using Error::Error;
};

// ------------------------------------------------------------------ util (util.hpp:10-42)
int log_level();
void log_info(const std::string& msg);
void log_debug(const std::string& msg);
std::string fmt_double(double x);

struct SplitMix64 {
  std::uint64_t state;
  explicit SplitMix64(std::uint64_t seed) : state(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double next_symmetric() { return 2.0 * next_unit() - 1.0; }
};

/// Generated on the device (counter-based SplitMix64, bitwise the sequential stream).
std::vector<double> random_vector(index_t n, std::uint64_t seed);

// ------------------------------------------------------------------ csr (csr.hpp:12-53)
struct CsrMatrix {
  index_t n = 0;
  std::vector<index_t> row_offsets;
  std::vector<index_t> col_indices;
  std::vector<double> values;

  index_t nnz() const { return static_cast<index_t>(col_indices.size()); }
  std::span<const index_t> row_cols(index_t i) const {
    return {col_indices.data() + row_offsets[i],
            static_cast<std::size_t>(row_offsets[i + 1] - row_offsets[i])};
  }
  std::span<const double> row_vals(index_t i) const {
    return {values.data() + row_offsets[i],
            static_cast<std::size_t>(row_offsets[i + 1] - row_offsets[i])};
  }
  double diagonal(index_t i) const;
  static CsrMatrix identity(index_t n);
  static CsrMatrix diagonal_matrix(std::span<const double> d);
  static CsrMatrix from_triplets(index_t n,
                                 std::vector<std::pair<std::pair<index_t, index_t>, double>> t);
};

void validate_structure(const CsrMatrix& a);
void validate_symmetric(const CsrMatrix& a);
void validate_spd_diagonal(const CsrMatrix& a);

std::vector<double> spmv(const CsrMatrix& a, std::span<const double> x);
void spmv_into(const CsrMatrix& a, std::span<const double> x, std::span<double> y);

// ------------------------------------------------------------------ blocks (block.hpp:13-60)
struct VectorBlock {
  index_t n = 0;
  index_t k = 0;
  std::vector<double> data;

  VectorBlock() = default;
  VectorBlock(index_t n_, index_t k_);
  double* col(index_t j) { return data.data() + j * n; }
  const double* col(index_t j) const { return data.data() + j * n; }
  std::span<double> col_span(index_t j) { return {col(j), static_cast<std::size_t>(n)}; }
  std::span<const double> col_span(index_t j) const {
    return {col(j), static_cast<std::size_t>(n)};
  }
  void set_col(index_t j, std::span<const double> v);
  VectorBlock columns(index_t first, index_t count) const;
  static VectorBlock from_column(std::span<const double> v);
};

inline constexpr int kSmallDenseMax = 64;

struct SmallDense {
  int rows = 0, cols = 0;
  std::vector<double> data;

  SmallDense() = default;
  SmallDense(int r, int c);
  double& at(int i, int j) {
    return data[static_cast<std::size_t>(i) + static_cast<std::size_t>(j) * rows];
  }
  double at(int i, int j) const {
    return data[static_cast<std::size_t>(i) + static_cast<std::size_t>(j) * rows];
  }
  std::span<double> col_span(int j) {
    return {data.data() + static_cast<std::size_t>(j) * rows, static_cast<std::size_t>(rows)};
  }
  std::span<const double> col_span(int j) const {
    return {data.data() + static_cast<std::size_t>(j) * rows, static_cast<std::size_t>(rows)};
  }
  static SmallDense identity(int m);
  static SmallDense from_column(std::span<const double> v);
};

double frobenius_norm(const SmallDense& m);
double max_abs(const SmallDense& m);

// ------------------------------------------------------------------ dense ops (dense_ops.hpp:13-28)
/// Serial ascending-order reductions, evaluated on the device (bitwise the reference).
double dot(std::span<const double> x, std::span<const double> y);
double norm2(std::span<const double> x);
SmallDense block_gram(const VectorBlock& u, const VectorBlock& v);
VectorBlock block_update(const VectorBlock& y, const VectorBlock& x, const SmallDense& c);
SmallDense small_cholesky_solve(const SmallDense& w, const SmallDense& rhs);

// ------------------------------------------------------------------ precond (precond.hpp:12-41)
class Preconditioner {
 public:
  virtual ~Preconditioner() = default;
  virtual void apply(std::span<const double> in, std::span<double> out) const = 0;
  virtual std::string_view name() const = 0;
  std::vector<double> apply_copy(std::span<const double> in) const {
    std::vector<double> out(in.size());
    apply(in, out);
    return out;
  }
};

class IdentityPreconditioner final : public Preconditioner {
 public:
  void apply(std::span<const double> in, std::span<double> out) const override;
  std::string_view name() const override { return "identity"; }
};

/// The solver recomputes 1/a_ii on the device (bitwise the ctor's values);
/// apply() is the reference's host utility method for callers.
class JacobiPreconditioner final : public Preconditioner {
 public:
  explicit JacobiPreconditioner(const CsrMatrix& a);
  void apply(std::span<const double> in, std::span<double> out) const override;
  std::string_view name() const override { return "jacobi"; }

 private:
  std::vector<double> inv_diag_;
};

/// Block Jacobi, M = blockdiag(A_11, A_22, ...) over blocks of `bs` consecutive
/// rows (a preconditioner beyond the reference's two, through the
/// same `Preconditioner` interface, precond.hpp:12-23). The ctor extracts the
/// dense diagonal blocks (a short last block padded with the identity) and
/// Cholesky-factors them (small_cholesky_solve's order, dense_ops.cpp:55-88);
/// NotSpdError if a block is not SPD. apply() is the host method (forward then
/// back substitution); the solver factors the same blocks on the device and
/// applies them there, bitwise equal.
class BlockJacobiPreconditioner final : public Preconditioner {
 public:
  BlockJacobiPreconditioner(const CsrMatrix& a, int bs);
  void apply(std::span<const double> in, std::span<double> out) const override;
  std::string_view name() const override { return "block_jacobi"; }
  int block_size() const { return bs_; }
  /// ceil(n/bs) dense bs x bs column-major diagonal blocks of A (unfactored)
  const std::vector<double>& blocks() const { return blocks_; }

 private:
  int bs_;
  index_t n_;
  std::vector<double> blocks_, factor_;
};

// ------------------------------------------------------------------ problems (problems.hpp:13-34)
struct PoissonSpec {
  index_t nx = 1, ny = 1, nz = 1;
  index_t size() const { return nx * ny * nz; }
};
struct PoissonSystem {
  CsrMatrix a;
  std::vector<double> rhs;
};
/// Assembled on the device (SELL-32) and downloaded; bitwise problems.cpp:13-53.
PoissonSystem poisson27(const PoissonSpec& spec);

/// Matrix Market coordinate real symmetric, 1-based, expanded to the full
/// pattern (problems.hpp:28-31); parsed on all host cores.
CsrMatrix read_matrix_market(const std::string& path, bool require_spd = false);
/// Lower triangle with round-trip-exact decimal values (problems.hpp:33-34).
void write_matrix_market(const std::string& path, const CsrMatrix& a);
/// New 7-point generator with the same conventions (poisson7 = (1,1,1), aniso (1,1,100)).
PoissonSystem stencil7(const PoissonSpec& spec, double cx = 1.0, double cy = 1.0,
                       double cz = 1.0);

// ------------------------------------------------------------------ spectral (spectral.hpp:13-57)
inline constexpr index_t kDenseAnalysisGuard = 2048;
enum class SpectrumMethod { lanczos, gershgorin, exact_dense };
struct SpectrumEstimate {
  double lambda_min = 0.0;
  double lambda_max = 0.0;
  SpectrumMethod method = SpectrumMethod::lanczos;
  double low_factor = 1.0;
  double high_factor = 1.0;
};
/// Device Lanczos (spectral.cpp:60-132).
SpectrumEstimate estimate_interval(const CsrMatrix& a, const Preconditioner& m, int steps,
                                   std::uint64_t seed);
std::pair<double, double> gershgorin_bounds(const CsrMatrix& a);

// ------------------------------------------------------------------ mpk (mpk.hpp:14-44)
struct ChebyshevParams {
  double lambda_min = 0.0;
  double lambda_max = 0.0;
  static ChebyshevParams from_interval(double lo, double hi);
  static ChebyshevParams from_estimate(const SpectrumEstimate& e) {
    return from_interval(e.lambda_min, e.lambda_max);
  }
  double alpha() const { return 2.0 / (lambda_max - lambda_min); }
  double sigma() const { return (lambda_max + lambda_min) / (lambda_max - lambda_min); }
  double gamma() const { return 1.0; }
};
struct MpkResult {
  VectorBlock z;
  VectorBlock p;
};
MpkResult mpk_chebyshev(const CsrMatrix& a, std::span<const double> r, int s,
                        const Preconditioner& m, const ChebyshevParams& params);

// ------------------------------------------------------------------ gram (gram.hpp:14-50)
struct GramSystem {
  SmallDense w;
  std::vector<double> diag;
  bool normalized = false;
  int order() const { return w.rows; }
  SmallDense strict_lower() const;
};
GramSystem assemble_gram(const VectorBlock& q, const VectorBlock& aq);
GramSystem gram_from_matrix(const SmallDense& w);
/// W_c = D^-1/2 W D^-1/2 with an exact unit diagonal (gram.hpp:52-56).
GramSystem normalize_gram(const GramSystem& g);
struct FgsRate {
  double spectral_norm;    // ||L^T (I+L)^{-1}||_2
  double spectral_radius;  // rho(L^T (I+L)^{-1})
};
/// Norm and radius of the FGS residual iteration matrix of a normalized
/// system (gram.hpp:58-66); host eigensolvers instead of dgesvd/dgeev.
FgsRate fgs_rate(const GramSystem& g);
struct FgsConfig {
  int nu = 30;
  bool multi_rhs = true;
};
struct FgsResult {
  SmallDense x;
  double rel_residual;
};
FgsResult fgs_solve(const GramSystem& g, const SmallDense& rhs, const FgsConfig& cfg);

// ------------------------------------------------------------------ solver (solver.hpp:14-116)
enum class GramSolverKind { fgs, cholesky };

struct SolverConfig {
  int s = 4;
  double tol = 1e-6;
  int max_outer = 500;
  FgsConfig fgs{};
  GramSolverKind gram_solver = GramSolverKind::fgs;
  std::optional<SpectrumEstimate> spectrum{};
  int lanczos_steps = 40;
  std::uint64_t seed = 1234;
  bool collect_gram = false;
  bool track_true_residual = false;
  std::optional<std::vector<double>> error_reference{};
  bool collect_iterates = false;
  void validate() const;
};

struct SolveReport {
  bool converged = false;
  int outer_iters = 0;
  std::vector<double> rel_residual;
  std::vector<double> delta_alpha;
  std::vector<double> delta_beta;
  std::vector<double> kappa_w;
  std::vector<SmallDense> gram_history;
  std::vector<double> true_rel_residual;
  std::vector<double> a_norm_error;
  std::vector<std::vector<double>> iterates;
  std::int64_t spmv_count = 0;
  std::int64_t precond_count = 0;
  std::int64_t allreduce_count = 0;
  double local_update_flops = 0.0;
  double gram_solve_flops = 0.0;
  SpectrumEstimate spectrum_used{};
};

struct SolveResult {
  std::vector<double> x;
  SolveReport report;
};

SolveResult pcg_s_solve(const CsrMatrix& a, std::span<const double> b,
                        std::span<const double> x0, const Preconditioner& m,
                        const SolverConfig& cfg);

struct PcgConfig {
  double tol = 1e-6;
  int max_iter = 1000;
  std::optional<std::vector<double>> error_reference{};
  bool collect_iterates = false;
};

SolveResult pcg_solve(const CsrMatrix& a, std::span<const double> b,
                      std::span<const double> x0, const Preconditioner& m,
                      const PcgConfig& cfg);
SolveResult pcg_solve(const CsrMatrix& a, std::span<const double> b,
                      std::span<const double> x0, const Preconditioner& m, double tol,
                      int max_iter);

struct InexactVerdict {
  double max_delta;
  double budget;
  bool pass;
};
InexactVerdict monitor_inexact(const SolveReport& report, double delta_cap = 1.0);
double a_norm_error(const CsrMatrix& a, std::span<const double> x, std::span<const double> ref);

// ------------------------------------------------------------------ B200 extensions
namespace gpu {
/// Arithmetic of pcg_s_solve: fast (one packed reduction per outer iteration,
/// default) or reference (bitwise the CPU reference given the same spectrum).
enum class Mode { fast = 0, reference = 1 };
void set_mode(Mode m);
Mode mode();
/// CUDA device used by the drop-in entry points (default 0).
void set_device(int device);

/// Plugin for a preconditioner whose apply runs on the device:
/// device_apply enqueues out = M^-1 in (n doubles, device pointers) on
/// `stream` (a cudaStream_t). The solver calls it wherever the reference calls
/// Preconditioner::apply (mpk.cpp:51-67, spectral.cpp:81,94, solver.cpp:228,254);
/// the host apply() stays the reference's utility method.
class DevicePreconditioner : public Preconditioner {
 public:
  virtual void device_apply(const double* in, double* out, index_t n, void* stream) const = 0;
};

/// Device-resident operator (SELL-32P in HBM + preconditioner), the
/// boundary's addition for sizes whose host CSR would not fit.
/// Generated problems are assembled on the device; Matrix Market files are
/// parsed on the host and uploaded once.
class DeviceProblem {
 public:
  static DeviceProblem poisson27(const PoissonSpec& spec);
  static DeviceProblem stencil7(const PoissonSpec& spec, double cx = 1.0, double cy = 1.0,
                                double cz = 1.0);
  static DeviceProblem from_csr(const CsrMatrix& a);
  static DeviceProblem read_matrix_market(const std::string& path, bool require_spd = true);
  void set_precond(const Preconditioner& m);
  index_t n_global() const { return n_global_; }
  index_t n_local() const { return n_local_; }
  index_t nnz_local() const { return nnz_local_; }
  index_t row_begin() const { return row_begin_; }
  cs_problem* handle() const { return p_; }
  ~DeviceProblem();
  DeviceProblem(DeviceProblem&& o) noexcept;
  DeviceProblem& operator=(DeviceProblem&& o) noexcept;
  DeviceProblem(const DeviceProblem&) = delete;
  DeviceProblem& operator=(const DeviceProblem&) = delete;

 private:
  explicit DeviceProblem(cs_problem* p);
  cs_problem* p_ = nullptr;
  index_t n_global_ = 0, n_local_ = 0, nnz_local_ = 0, row_begin_ = 0;
};

/// pcg_s_solve / pcg_solve on a device-resident problem (b, x0, x host vectors).
SolveResult pcg_s_solve(const DeviceProblem& p, std::span<const double> b,
                        std::span<const double> x0, const SolverConfig& cfg);
SolveResult pcg_solve(const DeviceProblem& p, std::span<const double> b,
                      std::span<const double> x0, const PcgConfig& cfg);
}  // namespace gpu

}  // namespace chebstep
