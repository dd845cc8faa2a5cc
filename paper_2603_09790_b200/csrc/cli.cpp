// cli.cpp -- the `chebstep` command line over the B200 solve path: the
// reference CLI's solve / compare / gram-analysis subcommands (reference
// src/cli.cpp:30-305) with the same flags, defaults, output files, CSV
// schema lines ("# chebstep-csv v1 <schema>"), JSON summary schemas and exit
// codes. The reference parses with CLI11 and writes JSON with nlohmann::json
// (neither is vendored here), so this file carries a small argument parser
// and a JSON writer that reproduces nlohmann's dump(2) layout (sorted keys,
// shortest round-trip numbers, NaN/inf as null).
//
// Problems are device-resident: --poisson assembles the 27-point operator on
// the GPU, --matrix parses the Matrix Market file on the host and uploads it
// once; b = 1, x0 = 0 as in the reference (cli.cpp:40-50).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "chebstep/api.hpp"
#include "chebstep/cli.hpp"

namespace chebstep::cli {
namespace {

namespace fs = std::filesystem;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ JSON (nlohmann dump(2) layout)
struct Json {
  enum Kind { Null, Bool, Int, Uint, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;  // std::map: nlohmann's default object orders keys

  Json() = default;
  Json(bool v) : kind(Bool), b(v) {}
  Json(int v) : kind(Int), i(v) {}
  Json(int64_t v) : kind(Int), i(v) {}
  Json(uint64_t v) : kind(Uint), u(v) {}
  Json(double v) : kind(Num), d(v) {}
  Json(const char* v) : kind(Str), s(v) {}
  Json(std::string v) : kind(Str), s(std::move(v)) {}
  Json(const std::vector<double>& v) : kind(Arr) {
    for (double x : v) arr.emplace_back(x);
  }
  static Json object() {
    Json j;
    j.kind = Obj;
    return j;
  }
  static Json array() {
    Json j;
    j.kind = Arr;
    return j;
  }
  Json& operator[](const std::string& k) {
    kind = Obj;
    return obj[k];
  }
  void push_back(Json v) {
    kind = Arr;
    arr.push_back(std::move(v));
  }
};

// nlohmann::detail::to_chars: shortest round-trip digits, fixed notation for
// decimal exponents in (-4, 15], otherwise d.ddde[+-]XX; always a '.0' or an
// exponent so the value reads back as a float.
std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  std::string out = v < 0 ? "-" : "";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof buf, std::fabs(v), std::chars_format::scientific);
  std::string sci(buf, res.ptr);
  const size_t epos = sci.find('e');
  std::string digits;
  for (size_t k = 0; k < epos; ++k)
    if (sci[k] != '.') digits += sci[k];
  const int exp10 = std::atoi(sci.c_str() + epos + 1);
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // decimal point position relative to the digits
  if (k <= n && n <= 15) {
    out += digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[8];
    std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', std::abs(e));
    out += eb;
  }
  return out;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += static_cast<char>(c);
        }
    }
  }
  return o + "\"";
}

void dump(const Json& j, std::string& o, int level) {
  const std::string pad(static_cast<size_t>(2 * (level + 1)), ' ');
  const std::string end_pad(static_cast<size_t>(2 * level), ' ');
  switch (j.kind) {
    case Json::Null: o += "null"; break;
    case Json::Bool: o += j.b ? "true" : "false"; break;
    case Json::Int: o += std::to_string(j.i); break;
    case Json::Uint: o += std::to_string(j.u); break;
    case Json::Num: o += json_number(j.d); break;
    case Json::Str: o += json_string(j.s); break;
    case Json::Arr:
      if (j.arr.empty()) {
        o += "[]";
        break;
      }
      o += "[\n";
      for (size_t k = 0; k < j.arr.size(); ++k) {
        o += pad;
        dump(j.arr[k], o, level + 1);
        o += k + 1 < j.arr.size() ? ",\n" : "\n";
      }
      o += end_pad + "]";
      break;
    case Json::Obj:
      if (j.obj.empty()) {
        o += "{}";
        break;
      }
      o += "{\n";
      {
        size_t k = 0;
        for (const auto& [key, val] : j.obj) {
          o += pad + json_string(key) + ": ";
          dump(val, o, level + 1);
          o += ++k < j.obj.size() ? ",\n" : "\n";
        }
      }
      o += end_pad + "}";
      break;
  }
}

void write_json(const fs::path& path, const Json& j) {
  std::ofstream out(path);
  if (!out) throw Error("cannot open for writing: " + path.string());
  std::string s;
  dump(j, s, 0);
  out << s << "\n";
}

// ------------------------------------------------------------------ CSV (cli.cpp:122-142)
class CsvWriter {
 public:
  CsvWriter(const fs::path& path, const std::string& schema, const std::string& header)
      : out_(path) {
    if (!out_) throw Error("cannot open for writing: " + path.string());
    out_ << "# chebstep-csv v1 " << schema << "\n" << header << "\n";
  }
  void row(const std::vector<std::string>& cells) {
    for (size_t i = 0; i < cells.size(); ++i) out_ << (i ? "," : "") << cells[i];
    out_ << "\n";
  }

 private:
  std::ofstream out_;
};

std::string cell(double v) { return fmt_double(v); }
std::string cell(int v) { return std::to_string(v); }
std::string cell(int64_t v) { return std::to_string(v); }

std::string delta_cell(const std::vector<double>& deltas, int k) {
  if (k < 1 || k > static_cast<int>(deltas.size())) return "";
  return fmt_double(deltas[static_cast<size_t>(k - 1)]);
}

// ------------------------------------------------------------------ argument parsing
struct Parser {
  struct Opt {
    std::string help;
    int nargs = 1;  // -1: one or more
    std::function<void(const std::vector<std::string>&)> set;
  };
  std::string name, about;
  std::map<std::string, Opt> opts;

  template <class T>
  static T number(const std::string& flag, const std::string& v) {
    T out{};
    const char* b = v.data();
    const char* e = b + v.size();
    std::from_chars_result r;
    if constexpr (std::is_floating_point_v<T>) {
      char* end = nullptr;
      out = std::strtod(v.c_str(), &end);
      r.ptr = end;
      r.ec = (end == b) ? std::errc::invalid_argument : std::errc{};
    } else {
      r = std::from_chars(b, e, out);
    }
    if (r.ec != std::errc{} || r.ptr != e)
      throw UsageError("--" + flag + ": Value " + v + " could not be converted");
    return out;
  }
  template <class T>
  void add(const std::string& flag, T* dst, const std::string& help) {
    opts[flag] = {help, 1, [=](const std::vector<std::string>& v) {
                    if constexpr (std::is_same_v<T, std::string>) *dst = v[0];
                    else *dst = number<T>(flag, v[0]);
                  }};
  }
  template <class T>
  void add_list(const std::string& flag, std::vector<T>* dst, int nargs, const std::string& help) {
    opts[flag] = {help, nargs, [=](const std::vector<std::string>& v) {
                    dst->clear();
                    for (const auto& x : v) dst->push_back(number<T>(flag, x));
                  }};
  }
  void add_choice(const std::string& flag, std::string* dst, std::vector<std::string> allowed,
                  const std::string& help) {
    opts[flag] = {help, 1, [=](const std::vector<std::string>& v) {
                    if (std::find(allowed.begin(), allowed.end(), v[0]) == allowed.end())
                      throw UsageError("--" + flag + ": " + v[0] + " not in {" +
                                       [&] {
                                         std::string s;
                                         for (size_t i = 0; i < allowed.size(); ++i)
                                           s += (i ? "," : "") + allowed[i];
                                         return s;
                                       }() + "}");
                    *dst = v[0];
                  }};
  }
  std::string help_text() const {
    std::string h = name + ": " + about + "\nOptions:\n  -h,--help  print this help\n";
    for (const auto& [k, o] : opts) h += "  --" + k + "  " + o.help + "\n";
    return h;
  }
  // returns false when help was requested
  bool parse(const std::vector<std::string>& args) {
    for (size_t a = 0; a < args.size(); ++a) {
      std::string tok = args[a];
      if (tok == "-h" || tok == "--help") return false;
      if (tok.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + tok);
      std::string key = tok.substr(2), inline_val;
      const bool has_inline = key.find('=') != std::string::npos;
      if (has_inline) {
        inline_val = key.substr(key.find('=') + 1);
        key = key.substr(0, key.find('='));
      }
      auto it = opts.find(key);
      if (it == opts.end()) throw UsageError("The following argument was not expected: " + tok);
      std::vector<std::string> vals;
      if (has_inline) vals.push_back(inline_val);
      const int want = it->second.nargs;
      while (a + 1 < args.size() && (want < 0 || static_cast<int>(vals.size()) < want) &&
             !(args[a + 1].rfind("--", 0) == 0 && args[a + 1].size() > 2 &&
               !std::isdigit(static_cast<unsigned char>(args[a + 1][2])) && args[a + 1][2] != '.'))
        vals.push_back(args[++a]);
      if (vals.empty() || (want > 0 && static_cast<int>(vals.size()) != want))
        throw UsageError("--" + key + ": " + std::to_string(want < 0 ? 1 : want) +
                         " required argument(s) missing");
      it->second.set(vals);
    }
    return true;
  }
};

// ------------------------------------------------------------------ options (cli.cpp:30-120)
struct ProblemOptions {
  std::vector<int64_t> poisson;
  std::string matrix_path;
  void add_flags(Parser& p) {
    p.add_list("poisson", &poisson, 3, "Poisson grid dimensions NX NY NZ");
    p.add("matrix", &matrix_path, "Matrix Market file (symmetric)");
  }
  gpu::DeviceProblem load() const {
    const bool have_poisson = !poisson.empty(), have_matrix = !matrix_path.empty();
    if (have_poisson == have_matrix)
      throw UsageError("exactly one of --poisson or --matrix is required");
    if (have_poisson) return gpu::DeviceProblem::poisson27({poisson[0], poisson[1], poisson[2]});
    return gpu::DeviceProblem::read_matrix_market(matrix_path, /*require_spd=*/true);
  }
  std::string label() const {
    if (!poisson.empty()) {
      std::ostringstream os;
      os << "poisson-" << poisson[0] << "x" << poisson[1] << "x" << poisson[2];
      return os.str();
    }
    return fs::path(matrix_path).filename().string();
  }
};

struct SolverOptions {
  int s = 4;
  std::string gram = "fgs";
  int nu = 30;
  double tol = 1e-6;
  int max_outer = 500;
  std::string precond = "identity";
  uint64_t seed = 1234;
  std::string mode = "fast";  // device extension
  int device = 0;             // device extension
  void add_flags(Parser& p, bool with_s = true) {
    if (with_s) p.add("s", &s, "step size");
    p.add_choice("gram", &gram, {"fgs", "cholesky"}, "Gram solver: fgs | cholesky");
    p.add("nu", &nu, "FGS sweep count");
    p.add("tol", &tol, "relative residual tolerance");
    p.add("max-outer", &max_outer, "maximum outer iterations");
    p.add_choice("precond", &precond, {"identity", "jacobi"}, "preconditioner: identity | jacobi");
    p.add("seed", &seed, "seed for the spectrum estimate");
    p.add_choice("mode", &mode, {"fast", "reference"},
                 "device algebra: fast (one reduction per outer) | reference (bitwise)");
    p.add("device", &device, "CUDA device");
  }
  SolverConfig to_config() const {
    SolverConfig cfg;
    cfg.s = s;
    cfg.tol = tol;
    cfg.max_outer = max_outer;
    cfg.fgs.nu = nu;
    cfg.gram_solver = gram == "cholesky" ? GramSolverKind::cholesky : GramSolverKind::fgs;
    cfg.seed = seed;
    return cfg;
  }
  void apply_device() const {
    gpu::set_device(device);
    gpu::set_mode(mode == "reference" ? gpu::Mode::reference : gpu::Mode::fast);
  }
  void set_precond(gpu::DeviceProblem& p) const {
    if (precond == "jacobi") {
      // the device recomputes 1/a_ii (precond.cpp:17-22); no host matrix needed
      struct J : Preconditioner {
        std::string_view name() const override { return "jacobi"; }
        void apply(std::span<const double>, std::span<double>) const override {}
      } j;
      p.set_precond(j);
    } else {
      p.set_precond(IdentityPreconditioner{});
    }
  }
};

struct OutputOptions {
  std::string out_dir = ".";
  std::string format = "csv";
  void add_flags(Parser& p) {
    p.add("out", &out_dir, "output directory");
    p.add_choice("format", &format, {"csv", "json"}, "history format: csv | json");
  }
  fs::path prepare() const {
    fs::path dir(out_dir);
    std::error_code ec;
    fs::create_directories(dir, ec);
    if (ec || !fs::is_directory(dir)) throw Error("cannot create output directory: " + out_dir);
    return dir;
  }
};

Json summary_json(const SolveReport& rep, const std::string& method, const ProblemOptions& prob,
                  const SolverOptions& sopt) {
  const InexactVerdict verdict = monitor_inexact(rep);
  Json j = Json::object();
  j["schema"] = "chebstep-solve-summary/1";
  j["problem"] = prob.label();
  j["method"] = method;
  j["converged"] = rep.converged;
  j["outer_iters"] = rep.outer_iters;
  j["final_rel_residual"] = rep.rel_residual.back();
  j["counts"]["spmv"] = static_cast<int64_t>(rep.spmv_count);
  j["counts"]["precond"] = static_cast<int64_t>(rep.precond_count);
  j["counts"]["allreduce"] = static_cast<int64_t>(rep.allreduce_count);
  j["model_flops"]["local_updates"] = rep.local_update_flops;
  j["model_flops"]["gram_solves"] = rep.gram_solve_flops;
  j["inexact"]["max_delta"] = verdict.max_delta;
  j["inexact"]["budget"] = verdict.budget;
  j["inexact"]["pass"] = verdict.pass;
  Json& c = j["config"];
  c["s"] = sopt.s;
  c["gram"] = sopt.gram;
  c["nu"] = sopt.nu;
  c["tol"] = sopt.tol;
  c["max_outer"] = sopt.max_outer;
  c["precond"] = sopt.precond;
  c["seed"] = sopt.seed;
  j["spectrum"]["lambda_min"] = rep.spectrum_used.lambda_min;
  j["spectrum"]["lambda_max"] = rep.spectrum_used.lambda_max;
  return j;
}

struct Rhs {
  std::vector<double> b, x0;
  explicit Rhs(const gpu::DeviceProblem& p)
      : b(static_cast<size_t>(p.n_local()), 1.0), x0(static_cast<size_t>(p.n_local()), 0.0) {}
};

// cli.cpp:184-212
int cmd_solve(const ProblemOptions& prob, const SolverOptions& sopt, const OutputOptions& oopt) {
  sopt.apply_device();
  gpu::DeviceProblem p = prob.load();
  sopt.set_precond(p);
  const Rhs v(p);
  const SolveResult res = gpu::pcg_s_solve(p, v.b, v.x0, sopt.to_config());
  const SolveReport& rep = res.report;
  const fs::path dir = oopt.prepare();
  Json summary = summary_json(rep, "pcgs-" + sopt.gram, prob, sopt);
  if (oopt.format == "csv") {
    CsvWriter csv(dir / "solve_history.csv", "solve-history", "k,rel_res,delta_alpha,delta_beta");
    for (size_t k = 0; k < rep.rel_residual.size(); ++k)
      csv.row({cell(static_cast<int>(k)), cell(rep.rel_residual[k]),
               delta_cell(rep.delta_alpha, static_cast<int>(k)),
               delta_cell(rep.delta_beta, static_cast<int>(k))});
  } else {
    summary["history"]["rel_residual"] = Json(rep.rel_residual);
    summary["history"]["delta_alpha"] = Json(rep.delta_alpha);
    summary["history"]["delta_beta"] = Json(rep.delta_beta);
  }
  write_json(dir / "solve_summary.json", summary);
  log_info("solve: " + std::string(rep.converged ? "converged" : "not converged") + " in " +
           std::to_string(rep.outer_iters) + " outer iterations");
  return rep.converged ? kExitOk : kExitNotConverged;
}

// cli.cpp:214-258
int cmd_compare(const ProblemOptions& prob, const SolverOptions& sopt, const OutputOptions& oopt,
                const std::vector<int>& s_list) {
  if (s_list.empty()) throw UsageError("compare: --s list must not be empty");
  sopt.apply_device();
  gpu::DeviceProblem p = prob.load();
  sopt.set_precond(p);
  const Rhs v(p);
  const fs::path dir = oopt.prepare();
  CsvWriter csv(dir / "compare.csv", "compare-history", "method,s,k,rel_res");
  Json summary = Json::object();
  summary["schema"] = "chebstep-compare-summary/1";
  summary["problem"] = prob.label();
  summary["runs"] = Json::array();
  const auto emit = [&](const std::string& method, int s, const SolveReport& rep) {
    for (size_t k = 0; k < rep.rel_residual.size(); ++k)
      csv.row({method, cell(s), cell(static_cast<int>(k)), cell(rep.rel_residual[k])});
    Json run = Json::object();
    run["method"] = method;
    run["s"] = s;
    run["converged"] = rep.converged;
    run["iters"] = rep.outer_iters;
    run["final_rel_residual"] = rep.rel_residual.back();
    summary["runs"].push_back(run);
  };
  bool all_converged = true;
  {
    PcgConfig pc;
    pc.tol = sopt.tol;
    pc.max_iter = sopt.max_outer * std::max(1, sopt.s);
    const SolveResult res = gpu::pcg_solve(p, v.b, v.x0, pc);
    emit("pcg", 1, res.report);
    all_converged &= res.report.converged;
  }
  for (const GramSolverKind kind : {GramSolverKind::cholesky, GramSolverKind::fgs}) {
    for (int s : s_list) {
      SolverConfig cfg = sopt.to_config();
      cfg.s = s;
      cfg.gram_solver = kind;
      const SolveResult res = gpu::pcg_s_solve(p, v.b, v.x0, cfg);
      emit(kind == GramSolverKind::cholesky ? "pcgs-cholesky" : "pcgs-fgs", s, res.report);
      all_converged &= res.report.converged;
    }
  }
  write_json(dir / "compare_summary.json", summary);
  return all_converged ? kExitOk : kExitNotConverged;
}

// cli.cpp:262-305; the structure_dev column (dense moment analysis,
// moments.cpp, n <= 2048) is left empty: the moments module is not part of
// the device path.
int cmd_gram_analysis(const ProblemOptions& prob, const SolverOptions& sopt,
                      const OutputOptions& oopt) {
  sopt.apply_device();
  gpu::DeviceProblem p = prob.load();
  sopt.set_precond(p);
  const Rhs v(p);
  SolverConfig cfg = sopt.to_config();
  cfg.collect_gram = true;
  const SolveResult res = gpu::pcg_s_solve(p, v.b, v.x0, cfg);
  const SolveReport& rep = res.report;
  const fs::path dir = oopt.prepare();
  {
    CsvWriter csv(dir / "gram_analysis.csv", "gram-analysis",
                  "k,rel_res,delta_alpha,delta_beta,kappa_w,fgs_spectral_norm,"
                  "fgs_spectral_radius,structure_dev");
    for (int k = 1; k <= rep.outer_iters && k <= static_cast<int>(rep.gram_history.size()); ++k) {
      const GramSystem g = gram_from_matrix(rep.gram_history[static_cast<size_t>(k - 1)]);
      const FgsRate rate = fgs_rate(normalize_gram(g));
      csv.row({cell(k), cell(rep.rel_residual[static_cast<size_t>(k)]),
               delta_cell(rep.delta_alpha, k), delta_cell(rep.delta_beta, k),
               cell(rep.kappa_w[static_cast<size_t>(k - 1)]), cell(rate.spectral_norm),
               cell(rate.spectral_radius), ""});
    }
  }
  {
    CsvWriter csv(dir / "gram_matrices.csv", "gram-entries", "k,i,j,w_ij");
    for (int k = 1; k <= rep.outer_iters && k <= static_cast<int>(rep.gram_history.size()); ++k) {
      const SmallDense& w = rep.gram_history[static_cast<size_t>(k - 1)];
      for (int i = 0; i < w.rows; ++i)
        for (int j = 0; j < w.cols; ++j)
          csv.row({cell(k), cell(i + 1), cell(j + 1), cell(w.at(i, j))});
    }
  }
  return rep.converged ? kExitOk : kExitNotConverged;
}

const char* kTopHelp =
    "Chebyshev-basis s-step PCG solver (B200 device path)\n"
    "Usage: chebstep SUBCOMMAND [OPTIONS]\n"
    "Subcommands:\n"
    "  solve          run the s-step solver\n"
    "  compare        classical PCG vs s-step with Cholesky and FGS Gram solves\n"
    "  gram-analysis  per-iteration Gram matrices, conditioning and deltas\n"
    "  perf-model     (not provided by the device build)\n"
    "  moments        (not provided by the device build)\n";

}  // namespace

int run(int argc, const char* const* argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  if (args.empty()) {
    std::fprintf(stderr, "A subcommand is required\n%s", kTopHelp);
    return kExitUsage;
  }
  if (args[0] == "-h" || args[0] == "--help") {
    std::printf("%s", kTopHelp);
    return kExitOk;
  }
  const std::string sub = args[0];
  args.erase(args.begin());
  ProblemOptions prob;
  SolverOptions sopt;
  OutputOptions oopt;
  std::vector<int> compare_s{2, 4, 6};
  Parser p;
  p.name = "chebstep " + sub;
  if (sub == "solve" || sub == "gram-analysis") {
    p.about = sub == "solve" ? "run the s-step solver"
                             : "per-iteration Gram matrices, conditioning and deltas";
    prob.add_flags(p);
    sopt.add_flags(p);
    oopt.add_flags(p);
  } else if (sub == "compare") {
    p.about = "classical PCG vs s-step with Cholesky and FGS Gram solves";
    prob.add_flags(p);
    sopt.add_flags(p, /*with_s=*/false);
    p.add_list("s", &compare_s, -1, "step sizes to sweep");
    oopt.add_flags(p);
  } else if (sub == "perf-model" || sub == "moments") {
    std::fprintf(stderr,
                 "error: %s is an analysis subcommand of the reference CPU tool and is not "
                 "part of the B200 solve path\n",
                 sub.c_str());
    return kExitUsage;
  } else {
    std::fprintf(stderr, "The following argument was not expected: %s\n%s", sub.c_str(), kTopHelp);
    return kExitUsage;
  }
  try {
    if (!p.parse(args)) {
      std::printf("%s", p.help_text().c_str());
      return kExitOk;
    }
  } catch (const UsageError& e) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
    return kExitUsage;
  }
  try {
    if (sub == "solve") return cmd_solve(prob, sopt, oopt);
    if (sub == "compare") return cmd_compare(prob, sopt, oopt, compare_s);
    return cmd_gram_analysis(prob, sopt, oopt);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    std::fprintf(stderr, "%s\n", p.help_text().c_str());
    return kExitUsage;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitError;
  }
}

int run(const std::vector<std::string>& args) {
  std::vector<const char*> argv;
  argv.push_back("chebstep");
  for (const auto& a : args) argv.push_back(a.c_str());
  return run(static_cast<int>(argv.size()), argv.data());
}

}  // namespace chebstep::cli
