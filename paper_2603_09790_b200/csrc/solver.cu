// solver.cu -- host orchestration of the device solve path:
//   pcg_s_solve   (solver.cpp:78-190)  Chebyshev s-step PCG, fast or reference algebra
//   pcg_solve     (solver.cpp:192-264) classical PCG comparator
//   estimate_interval (spectral.cpp:60-132) device Lanczos
// All n-sized work is device kernels; the host only enqueues work and polls
// an 4-byte convergence flag every `check_every` outer iterations while the
// next batch is already queued (stop decisions are taken on the device).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "runtime.cuh"

namespace csg {
namespace {

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    CS_CUDA(cudaEventCreate(&a));
    CS_CUDA(cudaEventCreate(&b));
    CS_CUDA(cudaEventRecord(a, s));
  }
  double stop() {
    CS_CUDA(cudaEventRecord(b, s));
    CS_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    CS_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

DevState read_state(cs_ctx* c) {
  DevState h;
  CS_CUDA(cudaMemcpyAsync(&h, c->state.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  return h;
}

void init_state(cs_ctx* c, double bnorm, int k) {
  DevState h;
  std::memset(&h, 0, sizeof h);
  h.bnorm = bnorm;
  h.k = k;
  CS_CUDA(cudaMemcpyAsync(c->state.p, &h, sizeof h, cudaMemcpyHostToDevice, c->stream));
}

void raise_device_error(const DevState& h, int s) {
  if (h.err == 0ull) return;
  const int code = static_cast<int>((h.err >> 32) & 0xff);
  const int payload = static_cast<int>(h.err & 0xffffffffu);
  fail(code, payload, format_device_error(h.err, s));
}

// bump allocator over one device buffer
struct Arena {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += sizeof(T) * std::max<size_t>(count, 1);
    return p;
  }
};

// global dot product (tree or serial order) into dev[0], then allreduce
void dot_into(cs_problem* p, const double* u, const double* v, double* dev, int mode,
              double* partial, unsigned* ticket, DevState* st) {
  cs_ctx* c = p->ctx;
  {
    Launch L(c, CS_PHASE_REDUCE);
    if (mode == CS_MODE_REFERENCE)
      launch_serial_gram(p->n_local, 1, 1, u, p->ld, v, p->ld, dev, st, c->stream);
    else
      launch_tree_gram(p->n_local, 1, 1, u, p->ld, v, p->ld, dev, partial, ticket, st, c->stream);
  }
  allreduce_sum(c, dev, 1);
}

double host_norm(cs_problem* p, const double* v, int mode) {
  cs_ctx* c = p->ctx;
  const size_t need = sizeof(double) * (tree_gram_partial_doubles(p->n_local, 1, 1) + 64) + 1024;
  if (c->normbuf.bytes < need) c->normbuf.alloc(need);
  Arena ar{c->normbuf.as<char>()};
  double* d = ar.take<double>(1);
  unsigned* ticket = ar.take<unsigned>(1);
  double* partial = ar.take<double>(tree_gram_partial_doubles(p->n_local, 1, 1));
  CS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), c->stream));
  dot_into(p, v, v, d, mode, partial, ticket, nullptr);
  double h = 0;
  CS_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  return std::sqrt(h);
}

}  // namespace

// ====================================================================== Lanczos

void estimate_interval_dev(cs_problem* p, int steps, uint64_t seed, int mode, double* lo,
                           double* hi, double* t_ms) {
  cs_ctx* c = p->ctx;
  NvtxRange nvtx_("cs:estimate_interval (Lanczos)");
  if (steps < 2) fail(CS_ERR_INVALID_ARGUMENT, 0, "estimate_interval: steps >= 2");
  if (steps > kLanczosMax) fail(CS_ERR_INVALID_ARGUMENT, 0, "estimate_interval: steps > 256");
  if (mode == CS_MODE_REFERENCE && c->nranks > 1)
    fail(CS_ERR_INVALID_ARGUMENT, 0, "reference mode is single-GPU");
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  const int64_t n = p->n_local, ld = p->ld;
  // The 2*steps basis vectors are cached on the context (every problem of it
  // reuses them); when HBM is short (512^3: 86 GB of basis next to the solve
  // workspace) this problem's workspace is released first and rebuilt after.
  // fast mode with a diagonal M: the G-only variant (v = D^-1 g, r = D^-1 gr
  // formed per row, never stored: half the basis, ~40 % fewer bytes per step)
  static const bool gonly_env = [] {
    const char* e = std::getenv("CS_LZ_GONLY");
    return e == nullptr || std::atoi(e) != 0;
  }();
  const bool gonly = gonly_env && mode == CS_MODE_FAST && !p->precond_general() && steps <= 40;
  const size_t lz_bytes =
      sizeof(double) * (static_cast<size_t>(gonly ? steps + 3 : 2 * steps + 3) * ld);
  if (c->lz.bytes < lz_bytes) {
    CS_CUDA(cudaStreamSynchronize(c->stream));
    c->lz.release();
    size_t free_b = 0, total_b = 0;
    CS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (free_b < lz_bytes + (size_t{1} << 30)) {
      p->ws.release();
      p->ws_s = -1;
    }
    c->lz.alloc(lz_bytes);
  }
  double* V = c->lz.as<double>();
  double* G = V + steps * ld;
  double* t = G + steps * ld;
  double* r = t + ld;
  double* gr = r + ld;
  const size_t tree_part = std::max(tree_gram_partial_doubles(n, steps, 1),
                                    lz_proj_partial_doubles(std::min(steps, 40)));
  const size_t part = std::max<size_t>(tree_part, static_cast<size_t>(lz_cgs_blocks(n)) + 16);
  char* scr = static_cast<char*>(ctx_scratch(
      c, sizeof(LanczosScalars) + sizeof(double) * (part + spmv_dot_blocks(p->nslices)) + 4096));
  Arena ar{scr};
  LanczosScalars* sc = ar.take<LanczosScalars>(1);
  double* partial = ar.take<double>(part + spmv_dot_blocks(p->nslices));
  unsigned* ticket = ar.take<unsigned>(4);
  CS_CUDA(cudaMemsetAsync(sc, 0, sizeof(LanczosScalars), c->stream));
  CS_CUDA(cudaMemsetAsync(ticket, 0, 4 * sizeof(unsigned), c->stream));
  init_state(c, 0.0, 0);
  DevState* st = c->state.as<DevState>();
  const double* inv = p->view().inv_diag;
  Timer timer(c->stream);
  auto L = [&]() { return Launch(c, CS_PHASE_LANCZOS); };

  const bool general = p->precond_general();
  auto reduce_dot = [&](const double* u, const double* v) {
    auto l = L();
    if (mode == CS_MODE_REFERENCE)
      launch_serial_gram(n, 1, 1, u, ld, v, ld, &sc->dot, st, c->stream);
    else
      launch_tree_gram(n, 1, 1, u, ld, v, ld, &sc->dot, partial, ticket, st, c->stream);
  };
  if (!gonly) {
    // start: g = random_vector(n, seed); v = M^-1 g; normalise by sqrt(v.g)  (spectral.cpp:72-83)
    {
      auto l = L();
      launch_random_vector(n, p->row_begin, seed, G, c->stream);
    }
    {
      auto l = L();
      precond_apply(p, G, V, nullptr, -1, 0);
    }
    reduce_dot(V, G);
  }
  int loop_steps = steps;  // the general loop's step count (0 after the G-only variant ran)
  if (gonly) {
    // layout [G: steps | v | t | gr]; the start pair is (v, g_0) as above
    G = V;
    double* v = G + steps * ld;
    double* tt = v + ld;
    double* grr = tt + ld;
    double dconst = 1.0;  // identity
    const double* dinv = nullptr;
    if (inv != nullptr) {  // Jacobi: the uniform 1/a_ii of the CDIA classes, else the vector
      const SellView A = p->view();
      double d0 = A.ncdia > 0 ? A.cdia[0].t.diag : 0.0;
      for (int k = 1; k < A.ncdia; ++k)
        if (std::memcmp(&A.cdia[k].t.diag, &d0, sizeof d0) != 0) d0 = 0.0;
      if (d0 != 0.0) dconst = 1.0 / d0;  // = inv_diag_kernel's value for every row
      else dinv = inv;
    }
    {
      auto l = L();
      launch_random_vector(n, p->row_begin, seed, G, c->stream);
    }
    {
      auto l = L();
      launch_precond_apply(n, inv, G, v, nullptr, -1, 0, c->stream);
    }
    reduce_dot(v, G);
    allreduce_sum(c, &sc->dot, 1);
    {
      auto l = L();
      lz_scalar(0, 0, steps, sc, st, c->stream);
    }
    {
      auto l = L();
      launch_scale2(n, v, G, v, G, &sc->denom, st, c->stream);
    }
    for (int j = 0; j < steps; ++j) {
      SpmvArgs g;
      g.x = v;
      g.y = tt;
      g.st = st;
      g.partial = partial;
      g.ticket = ticket + 1;
      g.result = &sc->dot;
      spmv_halo(p, kDot, g, v);  // t = A v_j, alpha_j = v_j . t
      allreduce_sum(c, &sc->dot, 1);
      {
        auto l = L();
        lz_scalar(1, j, steps, sc, st, c->stream);
      }
      {
        auto l = L();
        lz2_resid_proj(n, ld, j + 1, tt, G, dinv, dconst, grr, sc, j, sc->proj, partial, ticket + 2,
                       st, c->stream);
      }
      allreduce_sum(c, sc->proj, j + 1);
      {
        auto l = L();
        lz2_cgs(n, ld, j + 1, G, dinv, dconst, grr, sc->proj, partial, ticket + 3, &sc->dot, st,
                c->stream);
      }
      allreduce_sum(c, &sc->dot, 1);
      {
        auto l = L();
        lz_scalar(2, j, steps, sc, st, c->stream);
      }
      if (j + 1 < steps) {
        auto l = L();
        lz2_scale(n, grr, dinv, dconst, G + (j + 1) * ld, v, sc, st, c->stream);
      }
    }
    loop_steps = 0;  // the general loop below is skipped
  } else {
    allreduce_sum(c, &sc->dot, 1);
    {
      auto l = L();
      lz_scalar(0, 0, steps, sc, st, c->stream);
    }
    {
      auto l = L();
      launch_scale2(n, V, G, V, G, &sc->denom, st, c->stream);
    }
  }
  for (int j = 0; j < loop_steps; ++j) {
    double* vj = V + j * ld;
    double* gj = G + j * ld;
    SpmvArgs g;
    g.x = vj;
    g.y = t;
    g.st = st;
    if (mode == CS_MODE_REFERENCE) {
      spmv_halo(p, kPlain, g, vj);
      reduce_dot(vj, t);
    } else {
      g.partial = partial;
      g.ticket = ticket + 1;
      g.result = &sc->dot;
      spmv_halo(p, kDot, g, vj);
    }
    allreduce_sum(c, &sc->dot, 1);
    {
      auto l = L();
      lz_scalar(1, j, steps, sc, st, c->stream);
    }
    if (general) {  // r = M^-1 t first (spectral.cpp:94)
      auto l = L();
      precond_apply(p, t, r, st, -1, 0);
    }
    {
      auto l = L();
      lz_resid(n, t, inv, general ? r : nullptr, vj, gj, j > 0 ? vj - ld : nullptr,
               j > 0 ? gj - ld : nullptr, r, gr, sc, j, st, c->stream);
    }
    if (mode == CS_MODE_REFERENCE) {
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt, spectral.cpp:104-108
        {
          auto l = L();
          launch_serial_gram(n, 1, 1, G + i * ld, ld, r, ld, &sc->proj[0], st, c->stream);
        }
        auto l = L();
        lz_axpy2(n, V + i * ld, G + i * ld, r, gr, &sc->proj[0], st, c->stream);
      }
      reduce_dot(r, gr);
    } else {
      {  // classical Gram-Schmidt: all projections in one pass over r and G
        auto l = L();
        if (lz_proj_supported(j + 1))
          lz_proj(n, ld, j + 1, G, r, sc->proj, partial, ticket + 2, st, c->stream);
        else
          launch_tree_gram(n, j + 1, 1, G, ld, r, ld, sc->proj, partial, ticket + 2, st, c->stream);
      }
      allreduce_sum(c, sc->proj, j + 1);
      auto l = L();
      lz_cgs(n, ld, j + 1, V, G, r, gr, sc->proj, partial, ticket + 3, &sc->dot, st, c->stream);
    }
    allreduce_sum(c, &sc->dot, 1);
    {
      auto l = L();
      lz_scalar(2, j, steps, sc, st, c->stream);
    }
    if (j + 1 < steps) {
      auto l = L();
      launch_scale2(n, vj + ld, gj + ld, r, gr, &sc->denom, st, c->stream);
    }
  }
  const double ms = timer.stop();
  if (t_ms) *t_ms = ms;
  collect_timing(c);
  const DevState h = read_state(c);
  raise_device_error(h, 0);
  LanczosScalars hs;
  CS_CUDA(cudaMemcpy(&hs, sc, sizeof hs, cudaMemcpyDeviceToHost));
  const int m = hs.count;
  if (m < 1) fail(CS_ERR_GENERIC, 0, "estimate_interval: no Lanczos step completed");
  std::vector<double> ritz(m);
  tridiag_eigenvalues(m, hs.alpha, hs.beta, ritz.data());
  *lo = 0.9 * ritz.front();  // spectral.cpp:123-128
  *hi = 1.1 * ritz.back();
  if (!(*lo > 0.0) || !std::isfinite(*hi))
    fail(CS_ERR_NOT_SPD, 0, "estimate_interval: operator not positive definite");
}

// ====================================================================== PCG-S

namespace {

struct Blocks {
  double *Q, *AQ, *Z, *P, *x, *r, *b, *zpA, *zpB;
};

Blocks workspace(cs_problem* p, int s) {
  const int64_t ld = p->ld;
  const size_t vecs = static_cast<size_t>(4 * s + 5);
  if (p->ws_s != s) {
    p->ws.release();
    {
      // multi-GPU: a plain cudaMalloc allocation, exportable to the neighbours
      // for the peer-memory halo (pool allocations cannot be IPC-mapped)
      StreamBind plain(p->ctx->nranks > 1 ? nullptr : g_alloc_stream);
      p->ws.alloc(sizeof(double) * vecs * ld);
    }
    ++p->ws_gen;
    CS_CUDA(cudaMemsetAsync(p->ws.p, 0, sizeof(double) * vecs * ld, p->ctx->stream));
    p->ws_s = s;
  }
  double* base = p->ws.as<double>();
  Blocks bk;
  bk.Q = base;
  bk.AQ = bk.Q + s * ld;
  bk.Z = bk.AQ + s * ld;
  bk.P = bk.Z + s * ld;
  bk.x = bk.P + s * ld;
  bk.r = bk.x + ld;
  bk.b = bk.r + ld;
  bk.zpA = bk.b + ld;
  bk.zpB = bk.zpA + ld;
  return bk;
}

// MPK steps 1..s on a basis whose z_0 is already in Z column 0 (mpk.cpp:53-69).
// zs != nullptr (fast, diagonal M): PZ schedule -- no P column is written; the
// last step writes the virtual z_s instead of p_s (see PzArgs).
void mpk_steps(cs_problem* p, const Blocks& bk, int s, double lo, double hi, int pending,
               DevState* st, bool fast = false, bool p2p = false, double* zs = nullptr) {
  const int64_t ld = p->ld;
  const double alpha = 2.0 / (hi - lo);           // mpk.hpp:22
  const double sigma = (hi + lo) / (hi - lo);     // mpk.hpp:23-25
  const double gamma = 1.0;
  const bool jac = p->precond == CS_PRECOND_JACOBI;
  // general preconditioner (block Jacobi, device plugin): the reference
  // recurrence on zp with an identity epilogue writing zp_q, then z_q = M^-1 zp_q
  const bool gen = p->precond_general();
  if (gen) fast = false;
  auto zcol = [&](int q) { return bk.Z + q * ld; };
  auto zp = [&](int q) -> double* {  // zp_q storage
    if (q == 0) return bk.r;
    if (!jac && !gen) return zcol(q);
    return (q & 1) ? bk.zpA : bk.zpB;
  };
  const bool pz = zs != nullptr && fast && !gen;
  for (int q = 1; q < (pz ? s + 1 : s); ++q) {
    SpmvArgs g;
    g.x = zcol(q - 1);
    g.y = pz ? nullptr : bk.P + (q - 1) * ld;
    g.zp1 = zp(q - 1);
    g.zp2 = q >= 2 ? (fast ? zcol(q - 2) : zp(q - 2)) : nullptr;
    g.zpout = jac && !fast ? zp(q) : nullptr;
    g.zout = gen ? zp(q) : (pz && q == s) ? zs : zcol(q);
    if (q == 1) {
      g.ca = alpha;
      g.cb = -sigma;
      g.cc = 0.0;
    } else {
      g.ca = 2.0 * alpha;
      g.cb = -2.0 * sigma;
      g.cc = -gamma;
    }
    g.col = q;
    g.pending = pending;
    g.st = st;
    const int kind = fast ? (q == 1 ? kMpkFirstF : kMpkMidF) : (q == 1 ? kMpkFirst : kMpkMid);
    if (gen) g.col = -1;  // the breakdown check follows the apply
    if (pz && q == s) g.col = s - 1;  // z_s stands for p_s (mpk.cpp:69 checks p_s)
    // z_q's boundary rows go straight to the neighbours (z_s feeds no SpMV)
    if (p2p) spmv_p2p(p, kind, g, pz && q == s ? -1 : q);
    else spmv_halo(p, kind, g, zcol(q - 1));
    if (gen) {
      Launch L(p->ctx, CS_PHASE_UPDATE);
      precond_apply(p, zp(q), zcol(q), st, q, pending);  // mpk.cpp:58-59
    }
  }
  if (pz) return;
  SpmvArgs g;
  g.x = zcol(s - 1);
  g.y = bk.P + (s - 1) * ld;
  g.col = s - 1;
  g.pending = pending;
  g.st = st;
  if (p2p) spmv_p2p(p, kMpkLast, g, -1);
  else spmv_halo(p, kMpkLast, g, zcol(s - 1));
}

}  // namespace

void mpk_unit(cs_problem* p, double* Z, double* P, double* r, double* zpA, double* zpB, int s,
              double lo, double hi, DevState* st) {
  Blocks bk{};
  bk.Z = Z;
  bk.P = P;
  bk.r = r;
  bk.zpA = zpA;
  bk.zpB = zpB;
  mpk_steps(p, bk, s, lo, hi, /*pending=*/0, st);
}

namespace {

// Analysis hooks (solver.hpp:30-34, recorded as in solver.cpp:107-116 and
// 148-151): after r0 and after every outer update, on the host, without
// touching the iterates. Reductions follow the solve's mode (serial order in
// reference mode, so the histories are bitwise the reference's there).
struct Hooks {
  cs_problem* p;
  cs_report* rep;
  int mode, s;
  double bnorm;
  bool gram, truer, aerr, iter;
  const double* b_dev;
  DBuf buf;
  double *t = nullptr, *e = nullptr, *y = nullptr, *ref = nullptr, *dot = nullptr,
         *partial = nullptr;
  unsigned* ticket = nullptr;

  Hooks(cs_problem* p_, cs_report* r, const cs_config& cfg, int s_, const double* b)
      : p(p_), rep(r), mode(cfg.mode), s(s_), bnorm(0.0), b_dev(b) {
    gram = cfg.collect_gram != 0;
    truer = cfg.track_true_residual != 0;
    aerr = cfg.error_reference != nullptr;
    iter = cfg.collect_iterates != 0;
    rep->n_kappa = rep->n_true = rep->n_aerr = rep->n_iter = 0;
    if (!truer && !aerr) return;
    const int64_t ld = p->ld, n = p->n_local;
    const size_t part = tree_gram_partial_doubles(n, 1, 1);
    buf.alloc(sizeof(double) * (3 * ld + n + part + 64));
    t = buf.as<double>();
    e = t + ld;
    y = e + ld;
    ref = y + ld;
    dot = ref + n;
    partial = dot + 8;
    ticket = reinterpret_cast<unsigned*>(partial + part);
    CS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), p->ctx->stream));
    if (aerr)
      CS_CUDA(cudaMemcpyAsync(ref, cfg.error_reference, sizeof(double) * n,
                              cudaMemcpyHostToDevice, p->ctx->stream));
  }
  bool any() const { return gram || truer || aerr || iter; }

  double global_dot(const double* u, const double* v) {
    cs_ctx* c = p->ctx;
    {
      Launch L(c, CS_PHASE_OTHER);
      if (mode == CS_MODE_REFERENCE)
        launch_serial_gram(p->n_local, 1, 1, u, p->ld, v, p->ld, dot, nullptr, c->stream);
      else
        launch_tree_gram(p->n_local, 1, 1, u, p->ld, v, p->ld, dot, partial, ticket, nullptr,
                         c->stream);
    }
    allreduce_sum(c, dot, 1);
    double h = 0.0;
    CS_CUDA(cudaMemcpyAsync(&h, dot, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CS_CUDA(cudaStreamSynchronize(c->stream));
    return h;
  }

  static void push(double* arr, int* len, int cap, double v) {
    if (arr && *len < cap) arr[*len] = v;
    ++*len;
  }

  void record_x(double* x) {
    cs_ctx* c = p->ctx;
    const int64_t n = p->n_local;
    if (iter) {
      if (rep->iterates && rep->n_iter < rep->cap)
        CS_CUDA(cudaMemcpyAsync(rep->iterates + static_cast<int64_t>(rep->n_iter) * n, x,
                                sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
      ++rep->n_iter;
    }
    if (truer) {  // ||b - A x|| / ||b||   (solver.cpp:111-115)
      SpmvArgs g;
      g.x = x;
      g.y = t;
      g.b = b_dev;
      spmv_halo(p, kResid, g, x);
      push(rep->true_rel_residual, &rep->n_true, rep->cap, std::sqrt(global_dot(t, t)) / bnorm);
    }
    if (aerr) {  // sqrt(max(0, e^T A e)), e = x - x*   (solver.cpp:24-29)
      {
        Launch L(c, CS_PHASE_OTHER);
        static const double minus_one = -1.0;
        DBuf cm(sizeof(double));
        CS_CUDA(cudaMemcpyAsync(cm.p, &minus_one, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        launch_block_update(n, 1, 1, x, ref, cm.as<double>(), e, c->stream);  // e = x + (-1) x*
        CS_CUDA(cudaStreamSynchronize(c->stream));
      }
      SpmvArgs g;
      g.x = e;
      g.y = y;
      spmv_halo(p, kPlain, g, e);
      const double d = global_dot(e, y);
      push(rep->a_norm_error, &rep->n_aerr, rep->cap, std::sqrt(0.0 < d ? d : 0.0));
    }
    CS_CUDA(cudaStreamSynchronize(c->stream));
  }

  void record_gram(const double* W) {  // W_k and kappa_2(W_k)  (solver.cpp:148-151)
    if (!gram) return;
    std::vector<double> w(static_cast<size_t>(s) * s);
    CS_CUDA(cudaMemcpyAsync(w.data(), W, sizeof(double) * w.size(), cudaMemcpyDeviceToHost,
                            p->ctx->stream));
    CS_CUDA(cudaStreamSynchronize(p->ctx->stream));
    if (rep->gram_history && rep->n_kappa < rep->cap)
      std::copy(w.begin(), w.end(), rep->gram_history + static_cast<int64_t>(rep->n_kappa) * s * s);
    std::vector<double> ev(s);
    sym_eigenvalues(s, w.data(), ev.data());
    const double kappa =
        ev.front() > 0.0 ? ev.back() / ev.front() : std::numeric_limits<double>::infinity();
    push(rep->kappa_w, &rep->n_kappa, rep->cap, kappa);
  }
};

}  // namespace

namespace {
// CS_TRACE=1: host-side phase times of a solve (synchronising; diagnostics only)
struct SolveTrace {
  cudaStream_t st;
  bool on = std::getenv("CS_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit SolveTrace(cudaStream_t s) : st(s) {}
  void mark(const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cs-trace]   solve %s %.1f ms\n", phase,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};
}  // namespace

void pcgs_solve_dev(cs_problem* p, const double* b_dev, const double* x0_dev,
                    const cs_config& cfg, double* x_dev, cs_report* rep) {
  cs_ctx* c = p->ctx;
  NvtxRange nvtx_("cs:pcg_s_solve");
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  // SolverConfig::validate, solver.cpp:15-22
  if (cfg.s < 1 || cfg.s > kMaxS) fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: s must be in [1, 64]");
  if (!(cfg.tol > 0.0)) fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: tol must be > 0");
  if (cfg.max_outer < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: max_outer must be >= 1");
  if (cfg.nu < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: nu must be >= 1");
  const int mode = cfg.mode;
  if (mode == CS_MODE_REFERENCE && c->nranks > 1)
    fail(CS_ERR_INVALID_ARGUMENT, 0, "reference mode is single-GPU");
  const int var = cfg.variant;
  const bool explicit_w = mode == CS_MODE_FAST && (var & CS_VAR_EXPLICIT_W) != 0;
  const bool fast_mpk = (var & CS_VAR_REF_MPK) == 0;
  const bool tree_ref = mode == CS_MODE_REFERENCE && (var & CS_VAR_TREE) != 0;
  const int s = cfg.s;
  const int64_t n = p->n_local, ld = p->ld;
  const int64_t launches0 = c->launches, allred0 = c->allreduces;
  const double nglob = static_cast<double>(p->n_global);

  SolveTrace trace(c->stream);
  Blocks bk = workspace(p, s);
  DevState* st = c->state.as<DevState>();
  trace.mark("workspace");

  // vectors in: x (ghost slots filled by the halo), b
  CS_CUDA(cudaMemcpyAsync(bk.x, x0_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  CS_CUDA(cudaMemcpyAsync(bk.b, b_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));

  std::memset(rep, 0, offsetof(cs_report, cap));
  rep->schedule = 0;
  rep->n_rel = rep->n_da = rep->n_db = 0;
  const double bnorm = host_norm(p, bk.b, mode);  // solver.cpp:93
  if (bnorm == 0.0) {
    CS_CUDA(cudaMemsetAsync(x_dev, 0, sizeof(double) * n, c->stream));
    CS_CUDA(cudaStreamSynchronize(c->stream));
    rep->converged = 1;
    rep->n_rel = 1;
    if (rep->rel_residual && rep->cap > 0) rep->rel_residual[0] = 0.0;
    return;
  }
  trace.mark("vectors+bnorm");
  double lo = cfg.lambda_min, hi = cfg.lambda_max, t_lz = 0.0;
  if (!cfg.has_spectrum) {
    estimate_interval_dev(p, cfg.lanczos_steps, cfg.seed, mode, &lo, &hi, &t_lz);
    if (p->ws_s != s) {  // the estimate released the workspace for memory: rebuild, re-stage b/x0
      bk = workspace(p, s);
      CS_CUDA(cudaMemcpyAsync(bk.x, x0_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
      CS_CUDA(cudaMemcpyAsync(bk.b, b_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  trace.mark("lanczos");
  rep->lambda_min = lo;
  rep->lambda_max = hi;
  if (!(hi > lo) || !(lo > 0.0) || !std::isfinite(hi))  // mpk.cpp:11-16
    fail(CS_ERR_INVALID_ARGUMENT, 0, "ChebyshevParams: need lambda_max > lambda_min > 0");
  const int hist = cfg.max_outer + 2;
  const int q = s * s;
  const bool use_pack = mode == CS_MODE_FAST && pack_supported(s);
  const size_t partial_n = std::max({use_pack ? pack_partial_doubles(s, n) : size_t{0},
                                     tree_gram_partial_doubles(n, s, s),
                                     explicit_w ? update_gram_partial_doubles(s) : size_t{0}}) +
                           spmv_dot_blocks(p->nslices) + 64;
  char* scr = static_cast<char*>(ctx_scratch(
      c, sizeof(double) * (3 * static_cast<size_t>(hist) + 4 * q + 8 * s + 64 + partial_n) +
             64 * 256));
  Arena ar{scr};
  // packed block [G1 | G2 | c1 | c2 | rr | W_k raw (explicit W only) | breakdown
  // column flags (multi-rank only)]
  const int off_w = 2 * q + 2 * s + 1;
  const int off_flags = off_w + (explicit_w ? q : 0);
  const bool rank_flags = mode == CS_MODE_FAST && c->nranks > 1;
  const int npack = off_flags + (rank_flags ? s : 0);
  double* raw = ar.take<double>(npack);
  double* W = ar.take<double>(q);
  double* alpha_d = ar.take<double>(s);
  double* beta_d = ar.take<double>(q);
  double* rel = ar.take<double>(hist);
  double* da = ar.take<double>(hist);
  double* db = ar.take<double>(hist);
  double* partial = ar.take<double>(partial_n);
  unsigned* ticket = ar.take<unsigned>(8);
  CS_CUDA(cudaMemsetAsync(ticket, 0, 8 * sizeof(unsigned), c->stream));

  Hooks hooks(p, rep, cfg, s, bk.b);
  hooks.bnorm = bnorm;
  init_state(c, bnorm, 0);
  SmallArgs sa;
  sa.s = s;
  sa.nu = cfg.nu;
  sa.gram = cfg.gram;
  sa.max_outer = cfg.max_outer;
  sa.tol = cfg.tol;
  sa.st = st;
  sa.W = W;
  sa.alpha = alpha_d;
  sa.beta = beta_d;
  sa.raw = raw;
  sa.rel = rel;
  sa.da = da;
  sa.db = db;
  sa.Wexp = explicit_w ? raw + off_w : nullptr;
  sa.flags = rank_flags ? raw + off_flags : nullptr;
  double* flags = rank_flags ? raw + off_flags : nullptr;
  sa.fast_fgs = (var & CS_VAR_REF_FGS) ? 0 : 1;
  const SellView A = p->view();
  UpdateArgs ua;
  ua.s = s;
  ua.n = n;
  ua.ld = ld;
  ua.x = bk.x;
  ua.r = bk.r;
  ua.inv_diag = A.inv_diag;
  double diag_const = 0.0;  // the uniform a_ii when every row shares it (CDIA), else 0
  {  // one diagonal value for every row (constant-coefficient stencils): 1/a_ii as a constant
    double d0 = A.ncdia > 0 ? A.cdia[0].t.diag : 0.0;
    for (int k = 1; k < A.ncdia; ++k)
      if (std::memcmp(&A.cdia[k].t.diag, &d0, sizeof d0) != 0) d0 = 0.0;
    ua.inv_const = A.inv_diag != nullptr && d0 != 0.0 ? 1.0 / d0 : 0.0;  // = inv_diag_kernel
    diag_const = A.inv_diag != nullptr ? d0 : 0.0;
  }
  ua.alpha = alpha_d;
  ua.st = st;
  const bool general_pc = p->precond_general();
  if (general_pc) {  // the update pass writes z_0 = r into a scratch, the apply follows
    ua.inv_diag = nullptr;
    ua.inv_const = 0.0;
  }
  // PZ schedule (diagonal M, specialised order): P derived from Z in the pack
  // and update passes, z_s in the (otherwise unused) P block's first column
  const bool pz_on = mode == CS_MODE_FAST && fast_mpk && !general_pc && use_pack &&
                     update_gram_supported(s) && (var & CS_VAR_P_STORED) == 0;
  // true-residual schedule: r_{k+1} = b - A x_{k+1} (+ z_0) in one residual SpMV,
  // the update pass keeps only Q and x (no AQ block, no recursive r)
  // (the default of the fast PZ schedule; CS_VAR_RECUR_R keeps the recursive r)
  const bool tr_on = pz_on && !explicit_w && (var & CS_VAR_RECUR_R) == 0;
  PzArgs pz;
  if (pz_on) {
    const double alpha = 2.0 / (hi - lo), sigma = (hi + lo) / (hi - lo);  // mpk.hpp:22-25
    const bool jac = p->precond == CS_PRECOND_JACOBI;
    pz.sig1 = sigma;
    pz.sig2 = 2.0 * sigma;
    pz.k1 = 1.0 / alpha;
    pz.k2 = 1.0 / (2.0 * alpha);
    pz.dconst = jac && diag_const != 0.0 ? diag_const : 1.0;
    pz.diag = jac && diag_const == 0.0 ? p->diag.as<double>() : nullptr;
  }

  auto gram = [&](const double* u, int ku, const double* v, int kv, double* out) {
    Launch L(c, CS_PHASE_REDUCE);
    if (mode == CS_MODE_REFERENCE && !tree_ref)
      launch_serial_gram(n, ku, kv, u, ld, v, ld, out, st, c->stream);
    else
      launch_tree_gram(n, ku, kv, u, ld, v, ld, out, partial, ticket, st, c->stream);
  };
  // packed one-allreduce block {Q^T P, Z^T P, Z^T r, Q^T r, r^T r}
  auto packed_reduce = [&](const double* Qm, const double* Zm, const PzArgs& pza = PzArgs{}) {
    if (use_pack && p->xred_ok && pza.zs != nullptr && npack <= kXredSlot) {
      // the allreduce fused into the pack over NVLink peer memory (no NCCL call)
      ++c->allreduces;
      Launch L(c, CS_PHASE_REDUCE);
      launch_pack(s, n, ld, Qm, Zm, bk.P, bk.r, raw, partial, ticket + 1, st, flags, c->stream,
                  pza, xred_next(p, npack));
      return;
    }
    if (use_pack) {
      Launch L(c, CS_PHASE_REDUCE);
      launch_pack(s, n, ld, Qm, Zm, bk.P, bk.r, raw, partial, ticket + 1, st, flags, c->stream,
                  pza);
    } else {
      gram(Qm, s, bk.P, s, raw);
      gram(Zm, s, bk.P, s, raw + q);
      gram(Zm, s, bk.r, 1, raw + 2 * q);
      gram(Qm, s, bk.r, 1, raw + 2 * q + s);
      gram(bk.r, 1, bk.r, 1, raw + 2 * q + 2 * s);
      if (flags) launch_pending_flags(s, st, flags, c->stream);
    }
    allreduce_sum(c, raw, npack);
  };
  // The update pass of outer k forms Q_k, AQ_k, x_k, r_k, z_0. With the explicit
  // W it also reduces W_k = Q_k^T AQ_k from the rows it writes (fused, no extra
  // HBM traffic; a separate tree Gram for orders the fused kernel lacks). The
  // rank partial W_k travels in the packed block's single allreduce.
  auto update_pass = [&](bool first) {
    ua.beta = first ? nullptr : beta_d;
    sa.Wexp = explicit_w && !first ? raw + off_w : nullptr;  // outer 1: W_1 is explicit already
    if (tr_on) {
      Launch L(c, CS_PHASE_UPDATE);
      if (!launch_fast_update_tr(ua, c->stream))
        fail(CS_ERR_INVALID_ARGUMENT, 0, "true-residual schedule: unsupported s");
      return;
    }
    {
      Launch L(c, CS_PHASE_UPDATE);
      if (!(sa.Wexp && launch_fast_update_gram(ua, partial, ticket + 4, raw + off_w, c->stream))) {
        launch_fast_update(ua, c->stream);
        if (sa.Wexp) gram(bk.Q, s, bk.AQ, s, raw + off_w);
      }
    }
    if (general_pc) {  // z_0 = M^-1 r_k (the pass wrote r_k into the zp scratch)
      Launch L(c, CS_PHASE_UPDATE);
      precond_apply(p, bk.r, bk.Z, st, 0, /*pending=*/1);
    }
  };
  auto small = [&](void (*fn)(const SmallArgs&, cudaStream_t)) {
    Launch L(c, CS_PHASE_SMALL);
    fn(sa, c->stream);
  };

  Timer timer(c->stream);
  // ---- setup: r0 = b - A x0 (solver.cpp:118-122), MPK(r0) (:125-129)
  {
    SpmvArgs g;
    g.x = bk.x;
    g.y = bk.r;
    g.b = bk.b;
    g.st = st;
    spmv_halo(p, kResid, g, bk.x);
  }
  if (hooks.any()) hooks.record_x(bk.x);  // record_extras() after r0, solver.cpp:122-123
  if (mode == CS_MODE_REFERENCE) {
    gram(bk.r, 1, bk.r, 1, raw + q + s);
    {
      Launch L(c, CS_PHASE_SMALL);
      launch_ref_test(sa, c->stream);  // rel[0], k = 1
    }
  }
  {
    Launch L(c, CS_PHASE_UPDATE);
    precond_apply(p, bk.r, bk.Z, st, 0, 0);  // mpk.cpp:50-52
  }
  mpk_steps(p, bk, s, lo, hi, /*pending=*/0, st, mode == CS_MODE_FAST && fast_mpk);
  std::swap(bk.Q, bk.Z);  // q = basis.z ; aq = basis.p.columns(1, s)
  std::swap(bk.AQ, bk.P);
  ua.q = bk.Q;
  ua.aq = bk.AQ;
  ua.z = bk.Z;
  ua.p = bk.P;
  if (pz_on) {  // after the setup MPK the P block is free: it holds z_s from now on
    pz.zs = bk.P;
    // true residual: r is not stored, the pack forms it as D z_0 (CS_VAR_STORED_R keeps it)
    pz.r_from_z0 = tr_on && (var & CS_VAR_STORED_R) == 0 ? 1 : 0;
    ua.pz = pz;
  }
  if (mode == CS_MODE_FAST) {
    std::swap(bk.P, bk.AQ);  // pack wants P = A Q here
    packed_reduce(bk.Q, bk.Q);
    std::swap(bk.P, bk.AQ);
    small(launch_fast_setup);
  }

  // ---- outer iterations
  // multi-GPU fast algebra: halo planes move by NVLink peer stores from the
  // producing kernels (no NCCL on the SpMV path); collective, every rank calls it
  const bool p2p = mode == CS_MODE_FAST && fast_mpk && !general_pc && !hooks.any() &&
                   c->nranks > 1 && p2p_setup(p, bk.Z);
  // x's column in the workspace, counted in ld strides from Z (the same on every
  // rank): where the true-residual update pushes x's boundary rows
  const int x_col = static_cast<int>((bk.x - bk.Z) / ld);
  // r_k = b - A x_k and z_0 = M^-1 r_k in one SpMV (true-residual schedule)
  auto residual_z0 = [&](bool peer) {
    SpmvArgs g;
    g.x = bk.x;
    g.y = pz.r_from_z0 ? nullptr : bk.r;
    g.b = bk.b;
    g.zout = bk.Z;
    g.col = 0;
    g.pending = 1;
    g.st = st;
    if (peer) spmv_p2p(p, kResidF, g, 0);  // z_0's boundary rows to the neighbours
    else spmv_halo(p, kResidF, g, bk.x);
  };
  auto outer_fast = [&](bool first) {
    ua.zw = general_pc ? bk.zpA : bk.Z;  // z_0 = M^-1 r_k for the next MPK
    if (p2p) {  // z_0's (true residual: x's) boundary rows go to the neighbours from the update pass
      SpmvArgs pa;
      fill_push_args(p, pa, tr_on ? x_col : 0);
      ua.push_lo = pa.push_lo;
      ua.push_hi = pa.push_hi;
      ua.send_lo = pa.send_lo;
      ua.hi_begin = pa.hi_begin;
    }
    update_pass(first);
    if (p2p) p->p2p_pending = true;  // released by the next SpMV's interior launch
    if (tr_on) residual_z0(p2p);
    mpk_steps(p, bk, s, lo, hi, /*pending=*/1, st, fast_mpk, p2p, pz_on ? bk.P : nullptr);
    packed_reduce(bk.Q, bk.Z, pz);
    small(launch_fast_step);
  };
  auto outer_ref = [&]() {
    gram(bk.Q, s, bk.AQ, s, raw);          // assemble_gram, solver.cpp:139-147
    gram(bk.Q, s, bk.r, 1, raw + q);       // b1 = Q^T p_0, :153-154
    small(launch_ref_alpha);               // :155-157
    {
      Launch L(c, CS_PHASE_UPDATE);
      launch_ref_xr_update(ua, c->stream); // :159-163
    }
    gram(bk.r, 1, bk.r, 1, raw + q + s);   // ||r||, :165
    {
      Launch L(c, CS_PHASE_SMALL);
      launch_ref_test(sa, c->stream);      // :166-171
    }
    {
      Launch L(c, CS_PHASE_UPDATE);
      precond_apply(p, bk.r, bk.Z, st, 0, 0);
    }
    mpk_steps(p, bk, s, lo, hi, 0, st);    // :173-176
    gram(bk.Q, s, bk.P, s, raw + q + s + 1);  // b2, :178-179
    small(launch_ref_beta);                // :180-182
    ua.beta = beta_d;
    Launch L(c, CS_PHASE_UPDATE);
    launch_ref_block_update(ua, c->stream);  // :184-185
  };

  const int batch = cfg.check_every > 0 ? cfg.check_every : (n < (1 << 22) ? 16 : 4);
  volatile int* flag = static_cast<volatile int*>(c->pinned);
  cudaEvent_t ev[2];
  CS_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CS_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  int issued = 0, slot = 0;
  bool have_prev = false;
  if (hooks.any()) {  // per-outer host records: one outer at a time
    for (int k = 1; k <= cfg.max_outer; ++k) {
      if (mode == CS_MODE_FAST) {
        ua.zw = general_pc ? bk.zpA : bk.Z;
        update_pass(k == 1);
        if (tr_on) residual_z0(false);
        if (read_state(c).done) break;
        hooks.record_gram(W);  // W_k (the one this outer's alpha was solved with)
        hooks.record_x(bk.x);
        mpk_steps(p, bk, s, lo, hi, /*pending=*/1, st, fast_mpk, false, pz_on ? bk.P : nullptr);
        packed_reduce(bk.Q, bk.Z, pz);
        small(launch_fast_step);
      } else {
        outer_ref();
        const DevState hs = read_state(c);
        if (hs.outer_iters == k && hs.err == 0ull) {
          hooks.record_gram(W);
          hooks.record_x(bk.x);
        }
        if (hs.done) break;
      }
    }
    issued = cfg.max_outer;
  }
  // Single-GPU fast solves replay whole batches of outer iterations as one CUDA
  // graph: after the first (eager) batch, the next batch is captured once and
  // relaunched -- every launch of an outer has the same arguments (state lives
  // on the device), so the graph is exact; it removes the per-kernel launch
  // gaps that dominate small (L2-resident) problems. Not with timing spans,
  // hooks, several ranks (NCCL / peer-halo epochs) or CS_GRAPHS=0.
  static const bool graphs_env = [] {
    const char* e = std::getenv("CS_GRAPHS");
    return e == nullptr || std::atoi(e) != 0;
  }();
  const bool use_graph = graphs_env && mode == CS_MODE_FAST && c->nranks == 1 && !c->timing &&
                         !hooks.any();
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launches = 0;
  NvtxRange nvtx_loop("cs:outer iterations");
  for (; issued < cfg.max_outer;) {
    if (use_graph && issued > 0 && issued + batch <= cfg.max_outer) {
      if (gexec == nullptr) {
        const int64_t l0 = c->launches;
        cudaGraph_t g = nullptr;
        CS_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int bi = 0; bi < batch; ++bi) outer_fast(false);
        CS_CUDA(cudaStreamEndCapture(c->stream, &g));
        CS_CUDA(cudaGraphInstantiate(&gexec, g, 0));
        CS_CUDA(cudaGraphDestroy(g));
        graph_launches = c->launches - l0;
      } else {
        c->launches += graph_launches;
      }
      CS_CUDA(cudaGraphLaunch(gexec, c->stream));
      issued += batch;
    } else {
      for (int bi = 0; bi < batch && issued < cfg.max_outer; ++bi, ++issued) {
        if (mode == CS_MODE_FAST) outer_fast(issued == 0);
        else outer_ref();
      }
    }
    CS_CUDA(cudaMemcpyAsync(const_cast<int*>(&flag[slot]), &st->done, sizeof(int),
                            cudaMemcpyDeviceToHost, c->stream));
    CS_CUDA(cudaEventRecord(ev[slot], c->stream));
    if (issued >= cfg.max_outer) break;
    if (have_prev) {
      CS_CUDA(cudaEventSynchronize(ev[slot ^ 1]));
      if (flag[slot ^ 1]) break;
    }
    have_prev = true;
    slot ^= 1;
  }
  const double t_solve = timer.stop();
  trace.mark("setup+outer loop");
  if (gexec) cudaGraphExecDestroy(gexec);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  collect_timing(c);
  const DevState h = read_state(c);
  raise_device_error(h, s);

  CS_CUDA(cudaMemcpyAsync(x_dev, bk.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  // report, reference semantics (solver.cpp:120-188)
  rep->converged = h.converged;
  rep->outer_iters = h.outer_iters;
  const int64_t mpks = 1 + (h.converged ? h.outer_iters - 1 : h.outer_iters);
  rep->spmv_count = 1 + static_cast<int64_t>(s) * mpks;
  rep->precond_count = static_cast<int64_t>(s) * mpks;
  rep->allreduce_count = 2 * static_cast<int64_t>(h.outer_iters);
  const double lflops = 3.5 * (static_cast<double>(s) * s + s) * nglob;
  const double gflops = cfg.gram == CS_GRAM_FGS
                            ? static_cast<double>(cfg.nu) * (static_cast<double>(s) * s + 2.0 * s)
                            : static_cast<double>(s) * s * s / 3.0 + 2.0 * s * s * (s + 1.0);
  for (int k = 0; k < h.outer_iters; ++k) rep->local_update_flops += lflops;
  for (int k = 0; k < h.n_da + h.n_db; ++k) rep->gram_solve_flops += gflops;
  rep->n_rel = h.n_rel;
  rep->n_da = h.n_da;
  rep->n_db = h.n_db;
  auto copy_hist = [&](double* dst, const double* src, int len) {
    if (dst && rep->cap > 0 && len > 0)
      CS_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * std::min(len, rep->cap),
                              cudaMemcpyDeviceToHost, c->stream));
  };
  copy_hist(rep->rel_residual, rel, h.n_rel);
  copy_hist(rep->delta_alpha, da, h.n_da);
  copy_hist(rep->delta_beta, db, h.n_db);
  CS_CUDA(cudaStreamSynchronize(c->stream));
  // global reductions of the iterations that executed: ||b||, the setup
  // block, then one packed block per outer (fast) or W|b1, ||r||, b2 (reference)
  rep->device_allreduces =
      mode == CS_MODE_FAST
          ? 2 + static_cast<int64_t>(h.outer_iters)
          : 2 + 3 * static_cast<int64_t>(h.outer_iters) - (h.converged ? 1 : 0);
  (void)allred0;
  rep->kernel_launches = c->launches - launches0;
  rep->t_lanczos_ms = t_lz;
  rep->t_solve_ms = t_solve;
  rep->schedule = (pz_on ? CS_SCHED_P_FROM_Z : 0) | (explicit_w ? CS_SCHED_EXPLICIT_W : 0) |
                  (tr_on ? CS_SCHED_TRUE_R : 0) | (pz.r_from_z0 ? CS_SCHED_R_FROM_Z0 : 0) |
                  (p2p && p->xred_ok ? CS_SCHED_P2P_ALLREDUCE : 0);
  trace.mark("report");
}

// ====================================================================== classical PCG

void pcg_solve_dev(cs_problem* p, const double* b_dev, const double* x0_dev, double tol,
                   int max_iter, int mode, double* x_dev, cs_report* rep, const cs_config* hk) {
  cs_ctx* c = p->ctx;
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  if (!(tol >= 0.0) || max_iter < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "pcg_solve: bad tol/max_iter");
  if (mode == CS_MODE_REFERENCE && c->nranks > 1)
    fail(CS_ERR_INVALID_ARGUMENT, 0, "reference mode is single-GPU");
  const int64_t n = p->n_local, ld = p->ld;
  const int64_t launches0 = c->launches, allred0 = c->allreduces;
  // vectors: x, r, b, p, q, z  (reuse the s=1 workspace slots)
  Blocks bk = workspace(p, 1);
  double* xv = bk.x;
  double* rv = bk.r;
  double* bv = bk.b;
  double* pv = bk.Q;   // p needs ghost slots
  double* qv = bk.AQ;
  double* zv = bk.Z;
  const int hist = max_iter + 2;
  const size_t partial_n =
      std::max(static_cast<size_t>(std::max<int64_t>(spmv_dot_blocks(p->nslices), (n + 255) / 256)) * 2,
               tree_gram_partial_doubles(n, 1, 1)) + 64;
  char* scr = static_cast<char*>(
      ctx_scratch(c, sizeof(double) * (static_cast<size_t>(hist) + partial_n + 64) + 16 * 256));
  Arena ar{scr};
  double* dots = ar.take<double>(4);
  double* rel = ar.take<double>(hist);
  double* partial = ar.take<double>(partial_n);
  unsigned* ticket = ar.take<unsigned>(4);
  CS_CUDA(cudaMemsetAsync(ticket, 0, 4 * sizeof(unsigned), c->stream));
  DevState* st = c->state.as<DevState>();
  const double* inv = p->view().inv_diag;
  const bool serial = mode == CS_MODE_REFERENCE;
  CS_CUDA(cudaMemcpyAsync(xv, x0_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  CS_CUDA(cudaMemcpyAsync(bv, b_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  std::memset(rep, 0, offsetof(cs_report, cap));
  rep->schedule = 0;
  rep->n_rel = rep->n_da = rep->n_db = 0;
  const double bnorm = host_norm(p, bv, mode);
  if (bnorm == 0.0) {
    CS_CUDA(cudaMemsetAsync(x_dev, 0, sizeof(double) * n, c->stream));
    CS_CUDA(cudaStreamSynchronize(c->stream));
    rep->converged = 1;
    rep->n_rel = 1;
    if (rep->rel_residual && rep->cap > 0) rep->rel_residual[0] = 0.0;
    return;
  }
  cs_config hcfg;
  std::memset(&hcfg, 0, sizeof hcfg);
  if (hk) {  // PcgConfig hooks: error_reference, collect_iterates (solver.hpp:85-90)
    hcfg.error_reference = hk->error_reference;
    hcfg.collect_iterates = hk->collect_iterates;
  }
  hcfg.mode = mode;
  Hooks hooks(p, rep, hcfg, 1, bv);
  hooks.bnorm = bnorm;
  init_state(c, bnorm, 0);
  auto serial_dot = [&](const double* u, const double* v, double* out) {
    Launch L(c, CS_PHASE_REDUCE);
    launch_serial_gram(n, 1, 1, u, ld, v, ld, out, st, c->stream);
  };
  // general preconditioner (block Jacobi, device plugin): z = M^-1 r by its own
  // apply, the dots by separate reductions, p = z + beta p from z
  const bool gen = p->precond_general();
  auto vec = [&](int which, bool dots_on) {
    Launch L(c, CS_PHASE_UPDATE);
    launch_axpby_pcg(which, n, xv, gen && which == 2 ? zv : rv, pv, qv, gen ? nullptr : inv, st,
                     partial, ticket, dots, dots_on ? 0 : 1, c->stream);
  };
  auto gen_dots = [&]() {  // rr, rz after z = M^-1 r
    {
      Launch L(c, CS_PHASE_UPDATE);
      precond_apply(p, rv, zv, st, -1, 0);
    }
    if (serial) {
      serial_dot(rv, rv, dots);
      serial_dot(rv, zv, dots + 1);
    } else {
      Launch L(c, CS_PHASE_REDUCE);
      launch_tree_gram(n, 1, 1, rv, ld, rv, ld, dots, partial, ticket + 2, st, c->stream);
      launch_tree_gram(n, 1, 1, rv, ld, zv, ld, dots + 1, partial, ticket + 2, st, c->stream);
    }
  };
  auto scalar = [&](int which) {
    Launch L(c, CS_PHASE_SMALL);
    launch_pcg_scalar(which, tol, max_iter, st, dots, rel, c->stream);
  };
  Timer timer(c->stream);
  {  // r = b - A x0
    SpmvArgs g;
    g.x = xv;
    g.y = rv;
    g.b = bv;
    g.st = st;
    spmv_halo(p, kResid, g, xv);
  }
  if (hooks.any()) hooks.record_x(xv);
  if (gen) {
    gen_dots();
  } else if (serial) {
    serial_dot(rv, rv, dots);
    {
      Launch L(c, CS_PHASE_UPDATE);
      launch_precond_apply(n, inv, rv, zv, st, -1, 0, c->stream);
    }
    serial_dot(rv, zv, dots + 1);
  } else {
    vec(3, true);
  }
  allreduce_sum(c, dots, 2);
  scalar(0);
  if (gen)  // p = z
    CS_CUDA(cudaMemcpyAsync(pv, zv, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  else
    vec(0, false);  // p = z
  auto iteration = [&]() {
    SpmvArgs g;
    g.x = pv;
    g.y = qv;
    g.st = st;
    if (serial) {
      spmv_halo(p, kPlain, g, pv);
      serial_dot(pv, qv, dots);
    } else {
      g.partial = partial;
      g.ticket = ticket + 1;
      g.result = dots;
      spmv_halo(p, kDot, g, pv);
    }
    allreduce_sum(c, dots, 1);
    scalar(1);
    if (gen) {
      vec(1, false);
      gen_dots();
    } else if (serial) {
      vec(1, false);
      serial_dot(rv, rv, dots);
      {
        Launch L(c, CS_PHASE_UPDATE);
        launch_precond_apply(n, inv, rv, zv, st, -1, 0, c->stream);
      }
      serial_dot(rv, zv, dots + 1);
    } else {
      vec(1, true);
    }
    allreduce_sum(c, dots, 2);
    scalar(2);
    vec(2, false);
  };
  const int batch = hooks.any() ? 1 : (n < (1 << 22) ? 32 : 8);
  volatile int* flag = static_cast<volatile int*>(c->pinned);
  cudaEvent_t ev[2];
  CS_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CS_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  int issued = 0, slot = 0;
  bool have_prev = false;
  for (;;) {
    for (int bi = 0; bi < batch && issued < max_iter; ++bi, ++issued) {
      iteration();
      if (hooks.any()) {  // record_extras() after the x/r update (solver.cpp:245-246)
        const DevState hs = read_state(c);
        if (hs.outer_iters == issued + 1 && hs.err == 0ull) hooks.record_x(xv);
      }
    }
    CS_CUDA(cudaMemcpyAsync(const_cast<int*>(&flag[slot]), &st->done, sizeof(int),
                            cudaMemcpyDeviceToHost, c->stream));
    CS_CUDA(cudaEventRecord(ev[slot], c->stream));
    if (issued >= max_iter) break;
    if (have_prev) {
      CS_CUDA(cudaEventSynchronize(ev[slot ^ 1]));
      if (flag[slot ^ 1]) break;
    }
    have_prev = true;
    slot ^= 1;
  }
  const double t_solve = timer.stop();
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  collect_timing(c);
  const DevState h = read_state(c);
  raise_device_error(h, 1);
  CS_CUDA(cudaMemcpyAsync(x_dev, xv, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  rep->converged = h.converged;
  rep->outer_iters = h.outer_iters;
  rep->spmv_count = 1 + h.outer_iters;
  rep->precond_count = 1 + (h.converged ? h.outer_iters - 1 : h.outer_iters);
  rep->allreduce_count = 2 * static_cast<int64_t>(h.outer_iters);
  for (int k = 0; k < h.outer_iters; ++k) rep->local_update_flops += 8.0 * static_cast<double>(p->n_global);
  rep->n_rel = h.n_rel;
  if (rep->rel_residual && rep->cap > 0 && h.n_rel > 0)
    CS_CUDA(cudaMemcpyAsync(rep->rel_residual, rel, sizeof(double) * std::min(h.n_rel, rep->cap),
                            cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  rep->device_allreduces = c->allreduces - allred0;
  rep->kernel_launches = c->launches - launches0;
  rep->t_solve_ms = t_solve;
}

}  // namespace csg
