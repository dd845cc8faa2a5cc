// capi.cu -- the extern "C" boundary (include/chebstep_gpu.h). Every entry
// catches library / CUDA errors and returns a CS_* status with a thread-local
// message and payload, mirroring the reference's exception types
// (errors.hpp:9-56) so the C++ and Python layers can re-raise them.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <algorithm>
#include <cmath>
#include <string>

#include "lanczos.cuh"
#include "mmio.hpp"
#include "runtime.cuh"

namespace csg {
cs_ctx* ctx_create(int device);
void ctx_destroy(cs_ctx* c);
void comm_init(cs_ctx* c, int nranks, int rank, const unsigned char id[128]);
cs_problem* problem_generate(cs_ctx* c, int kind, int64_t nx, int64_t ny, int64_t nz,
                             const double* coef);
cs_problem* problem_upload_csr(cs_ctx* c, int64_t n, const int64_t* rowptr, const int64_t* col,
                               const double* val);
cs_problem* problem_upload_block(cs_ctx* c, int64_t n_global, int64_t row_begin, int64_t row_end,
                                 const int64_t* rowptr, const int64_t* col, const double* val);
void problem_set_precond(cs_problem* p, int kind);
void problem_download_csr(cs_problem* p, int64_t* rowptr, int64_t* col, double* val);
}  // namespace csg

using namespace csg;

namespace {
thread_local std::string t_msg;
thread_local int t_payload = 0;

template <class F>
int guard(F&& f) {
  t_msg.clear();
  t_payload = 0;
  try {
    f();
    return CS_OK;
  } catch (const LibError& e) {
    t_msg = e.msg;
    t_payload = e.payload;
    return e.code;
  } catch (const CudaError& e) {
    t_msg = e.what;
    return CS_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    t_msg = "host out of memory";
    return CS_ERR_GENERIC;
  } catch (const std::exception& e) {
    t_msg = e.what();
    return CS_ERR_GENERIC;
  }
}

void need(const void* p, const char* what) {
  if (p == nullptr) fail(CS_ERR_INVALID_ARGUMENT, 0, std::string("null ") + what);
}

// device copy of a host array
constexpr size_t kLargeCopy = size_t{32} << 20;  // staged above this (runtime.cu)

struct HostIn {
  DBuf d;
  HostIn(cs_ctx* c, const void* h, size_t bytes) : d(bytes) {
    if (bytes >= kLargeCopy) h2d_large(c, d.p, h, bytes);
    else if (bytes) CS_CUDA(cudaMemcpyAsync(d.p, h, bytes, cudaMemcpyHostToDevice, c->stream));
  }
};

void to_host(cs_ctx* c, void* h, const void* d, size_t bytes) {
  if (bytes >= kLargeCopy) d2h_large(c, h, d, bytes);
  else if (bytes) CS_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c->stream));
}

void sync(cs_ctx* c) { CS_CUDA(cudaStreamSynchronize(c->stream)); }

// CS_TRACE=1: host-side phase timestamps of the drop-in entries on stderr
struct Trace {
  const char* what;
  cudaStream_t st;
  bool on;
  std::chrono::steady_clock::time_point t0;
  Trace(const char* w, cudaStream_t s) : what(w), st(s), on(std::getenv("CS_TRACE") != nullptr) {
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cs-trace] %s %s %.1f ms\n", what, phase,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

void small_status(int st) {
  if (st == 0) return;
  const int code = st & 0xff, sub = st >> 8;
  if (code == 2) fail(CS_ERR_INVALID_MATRIX, 0, "gram_from_matrix: matrix not symmetric");
  if (sub == 1) fail(CS_ERR_NOT_SPD, 0, "gram: non-positive diagonal (basis degeneracy)");
  if (sub == 2) fail(CS_ERR_NOT_SPD, 0, "fgs: zero diagonal");
  fail(CS_ERR_NOT_SPD, 0, "cholesky: non-positive pivot (basis breakdown)");
}

}  // namespace

extern "C" {

const char* cs_last_error(int* payload) {
  if (payload) *payload = t_payload;
  return t_msg.c_str();
}

int cs_version(void) { return 100; }

int cs_device_count(int* count) {
  return guard([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    *count = n;
  });
}

int cs_ctx_create(int device, cs_ctx** out) {
  return guard([&] { *out = ctx_create(device); });
}

int cs_ctx_destroy(cs_ctx* ctx) {
  return guard([&] { ctx_destroy(ctx); });
}

int cs_ctx_set_timing(cs_ctx* ctx, int enable) {
  return guard([&] { ctx->timing = enable != 0; });
}

int cs_ctx_reset_timing(cs_ctx* ctx) {
  return guard([&] {
    collect_timing(ctx);
    ctx->phase_ms.fill(0.0);
    ctx->phase_launches.fill(0);
  });
}

int cs_ctx_get_timing(cs_ctx* ctx, int phase, double* ms, int64_t* launches) {
  return guard([&] {
    if (phase < 0 || phase >= CS_NUM_PHASES) fail(CS_ERR_INVALID_ARGUMENT, 0, "bad phase");
    collect_timing(ctx);
    *ms = ctx->phase_ms[phase];
    *launches = ctx->phase_launches[phase];
  });
}

int cs_ctx_launch_count(cs_ctx* ctx, int64_t* launches) {
  return guard([&] { *launches = ctx->launches; });
}

int cs_ctx_synchronize(cs_ctx* ctx) {
  return guard([&] { sync(ctx); });
}

int cs_ctx_stream(cs_ctx* ctx, void** stream) {
  return guard([&] { *stream = static_cast<void*>(ctx->stream); });
}

int cs_comm_unique_id(unsigned char id[128]) {
  return guard([&] {
    ncclUniqueId uid;
    const ncclResult_t r = ncclGetUniqueId(&uid);
    if (r != ncclSuccess) fail(CS_ERR_NCCL, 0, ncclGetErrorString(r));
    std::memcpy(id, uid.internal, 128);
  });
}

int cs_ctx_comm_init(cs_ctx* ctx, int nranks, int rank, const unsigned char id[128]) {
  return guard([&] { comm_init(ctx, nranks, rank, id); });
}

int cs_ctx_allreduce_max(cs_ctx* ctx, double* value) {
  return guard([&] {
    if (ctx->nranks == 1) return;
    DBuf d(sizeof(double));
    CS_CUDA(cudaMemcpyAsync(d.p, value, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const ncclResult_t r =
        ncclAllReduce(d.p, d.p, 1, ncclDouble, ncclMax, ctx->comm, ctx->stream);
    if (r != ncclSuccess) fail(CS_ERR_NCCL, 0, ncclGetErrorString(r));
    to_host(ctx, value, d.p, sizeof(double));
    sync(ctx);
  });
}

// ------------------------------------------------------------------ problems

int cs_problem_generate(cs_ctx* ctx, int kind, int64_t nx, int64_t ny, int64_t nz,
                        const double* coef, cs_problem** out) {
  return guard([&] { *out = problem_generate(ctx, kind, nx, ny, nz, coef); });
}

int cs_problem_upload_csr(cs_ctx* ctx, int64_t n, const int64_t* rowptr, const int64_t* col,
                          const double* val, cs_problem** out) {
  return guard([&] {
    need(rowptr, "rowptr");
    *out = problem_upload_csr(ctx, n, rowptr, col, val);
  });
}

int cs_problem_upload_csr_block(cs_ctx* ctx, int64_t n_global, int64_t row_begin,
                                int64_t row_end, const int64_t* rowptr_local,
                                const int64_t* col_global, const double* val, cs_problem** out) {
  return guard([&] {
    need(rowptr_local, "rowptr");
    *out = problem_upload_block(ctx, n_global, row_begin, row_end, rowptr_local, col_global, val);
  });
}

int cs_fgs_rate(int s, const double* w, double* spectral_norm, double* spectral_radius) {
  return guard([&] {
    need(w, "w");
    if (s < 1 || s > kMaxS) fail(CS_ERR_INVALID_ARGUMENT, 0, "fgs_rate: bad order");
    const size_t ss = static_cast<size_t>(s);
    auto W = [&](int i, int j) { return w[i + j * ss]; };
    // X solves (I + L) X = I column by column (gram.cpp:153-162)
    std::vector<double> x(ss * ss, 0.0), it(ss * ss, 0.0);
    for (int c = 0; c < s; ++c) {
      x[c + c * ss] = 1.0;
      for (int i = 0; i < s; ++i) {
        double acc = x[i + c * ss];
        for (int j = 0; j < i; ++j) acc -= W(i, j) * x[j + c * ss];
        x[i + c * ss] = acc;
      }
    }
    for (int c = 0; c < s; ++c)  // iteration matrix L^T X (gram.cpp:163-169)
      for (int i = 0; i < s; ++i) {
        double acc = 0.0;
        for (int j = i + 1; j < s; ++j) acc += W(j, i) * x[j + c * ss];
        it[i + c * ss] = acc;
      }
    *spectral_norm = max_singular_value(s, it.data());
    std::vector<double> mods(ss);
    general_eig_moduli(s, it.data(), mods.data());
    *spectral_radius = *std::max_element(mods.begin(), mods.end());
  });
}

int cs_kappa_sym(int s, const double* w, double* kappa) {
  return guard([&] {
    need(w, "w");
    if (s < 1 || s > kMaxS) fail(CS_ERR_INVALID_ARGUMENT, 0, "kappa: bad order");
    std::vector<double> ev(static_cast<size_t>(s));
    sym_eigenvalues(s, w, ev.data());
    // solver.cpp:69-74: largest / smallest eigenvalue, inf unless the smallest is > 0
    *kappa = ev[0] > 0.0 ? ev[s - 1] / ev[0] : std::numeric_limits<double>::infinity();
  });
}

int cs_mm_read(const char* path, int require_spd, cs_csr_host** out, int64_t* n, int64_t* nnz) {
  return guard([&] {
    need(path, "path");
    std::unique_ptr<HostCsr> h(mm_read(path, require_spd != 0));
    *n = h->n;
    *nnz = static_cast<int64_t>(h->col.size());
    *out = reinterpret_cast<cs_csr_host*>(h.release());
  });
}

int cs_csr_host_rows(const cs_csr_host* hh, int64_t row_begin, int64_t row_end,
                     int64_t* rowptr_local, int64_t* col, double* val) {
  return guard([&] {
    const HostCsr* h = reinterpret_cast<const HostCsr*>(hh);
    need(h, "csr");
    if (row_begin < 0 || row_end < row_begin || row_end > h->n)
      fail(CS_ERR_DIMENSION, 0, "bad row range");
    const int64_t b = h->rowptr[row_begin];
    for (int64_t i = row_begin; i <= row_end; ++i) rowptr_local[i - row_begin] = h->rowptr[i] - b;
    const int64_t cnt = h->rowptr[row_end] - b;
    if (col) std::memcpy(col, h->col.data() + b, sizeof(int64_t) * cnt);
    if (val) std::memcpy(val, h->val.data() + b, sizeof(double) * cnt);
  });
}

int cs_csr_host_free(cs_csr_host* h) {
  return guard([&] { delete reinterpret_cast<HostCsr*>(h); });
}

int cs_mm_write(const char* path, int64_t n, const int64_t* rowptr, const int64_t* col,
                const double* val) {
  return guard([&] {
    need(path, "path");
    mm_write(path, n, rowptr, col, val);
  });
}

int cs_csr_validate(int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                    int check) {
  return guard([&] {
    need(rowptr, "rowptr");
    if (check == CS_CHECK_STRUCTURE) validate_structure_host(n, rowptr, col, val, n + 1, rowptr[n]);
    else if (check == CS_CHECK_SYMMETRIC) validate_symmetric_host(n, rowptr, col, val);
    else if (check == CS_CHECK_SPD_DIAGONAL) validate_spd_diagonal_host(n, rowptr, col, val);
    else fail(CS_ERR_INVALID_ARGUMENT, 0, "unknown check");
  });
}

int cs_problem_read_mm(cs_ctx* ctx, const char* path, int require_spd, cs_problem** out) {
  return guard([&] {
    need(path, "path");
    std::unique_ptr<HostCsr> h(mm_read(path, require_spd != 0));
    int64_t b = 0, e = h->n;
    if (ctx->nranks > 1 && cs_partition_rows(h->n, 1, ctx->nranks, ctx->rank, &b, &e) != CS_OK)
      fail(CS_ERR_INVALID_ARGUMENT, 0, "matrix has fewer rows than ranks");
    std::vector<int64_t> rp(static_cast<size_t>(e - b) + 1);
    const int64_t off = h->rowptr[b];
    for (int64_t i = b; i <= e; ++i) rp[i - b] = h->rowptr[i] - off;
    *out = problem_upload_block(ctx, h->n, b, e, rp.data(), h->col.data() + off,
                                h->val.data() + off);
  });
}

int cs_problem_destroy(cs_problem* p) {
  return guard([&] {
    if (p) {
      cs_ctx* c = p->ctx;
      cudaSetDevice(c->device);
      cudaStreamSynchronize(c->stream);
      p2p_teardown(p);
      delete p;  // ~cs_problem: buffers freed on c->stream, c->live_problems decremented
    }
  });
}

int cs_problem_info(cs_problem* p, int64_t* info) {
  return guard([&] {
    info[0] = p->n_global;
    info[1] = p->n_local;
    info[2] = p->nnz_local;
    info[3] = p->row_begin;
    info[4] = p->n_ghost;
    info[5] = static_cast<int64_t>(p->vals.bytes + p->cols.bytes + p->pat.bytes + p->pval.bytes + p->pkey.bytes + p->pbits.bytes +
                                   p->meta.bytes + p->slice_ptr.bytes);
    info[6] = p->nslices;
    info[7] = p->compressed_slices;
    info[8] = p->uniform_slices;
    info[9] = p->pattern_entries;
    info[10] = static_cast<int64_t>(p->cdia.size());
    bool ud = !p->cdia.empty(), zu = !p->cdia.empty();
    for (const auto& k : p->cdia) {
      ud = ud && k.t.diag != 0.0;
      zu = zu && k.zuni;
    }
    info[11] = (ud ? 1 : 0) | (zu ? 2 : 0);
  });
}

int cs_problem_halo_mode(cs_problem* p, int* mode) {
  return guard([&] { *mode = p->ctx->nranks == 1 ? 0 : p->p2p ? 2 : 1; });
}

int cs_problem_download_csr(cs_problem* p, int64_t* rowptr, int64_t* col, double* val) {
  return guard([&] { problem_download_csr(p, rowptr, col, val); });
}

int cs_problem_ghosts(cs_problem* p, int64_t* ghost_cols) {
  return guard([&] {
    std::memcpy(ghost_cols, p->ghosts_host.data(), sizeof(int64_t) * p->ghosts_host.size());
  });
}

int cs_problem_set_precond(cs_problem* p, int kind) {
  return guard([&] { problem_set_precond(p, kind); });
}

int cs_problem_set_precond_block_jacobi(cs_problem* p, int bs, const double* blocks) {
  return guard([&] { problem_set_precond_block_jacobi(p, bs, blocks); });
}

int cs_problem_set_precond_fn(cs_problem* p, cs_precond_fn fn, void* user) {
  return guard([&] { problem_set_precond_fn(p, fn, user); });
}

int cs_problem_inv_diag(cs_problem* p, double* out) {
  return guard([&] {
    if (p->precond != CS_PRECOND_JACOBI) fail(CS_ERR_INVALID_ARGUMENT, 0, "not Jacobi");
    to_host(p->ctx, out, p->inv_diag.p, sizeof(double) * p->n_local);
    sync(p->ctx);
  });
}

// ------------------------------------------------------------------ unit entries

int cs_spmv(cs_problem* p, const double* x, double* y) {
  return guard([&] {
    cs_ctx* c = p->ctx;
    CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
    DBuf dx(sizeof(double) * p->ld), dy(sizeof(double) * p->ld);
    CS_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * p->n_local, cudaMemcpyHostToDevice, c->stream));
    SpmvArgs g;
    g.x = dx.as<double>();
    g.y = dy.as<double>();
    spmv_halo(p, kPlain, g, dx.as<double>());
    to_host(c, y, dy.p, sizeof(double) * p->n_local);
    sync(c);
  });
}

namespace {
// kind 5: the z_0 push kernel alone; kind 6: one fast-MPK middle step through the
// peer-memory halo (interior + release, wait + boundary). Both on the solve
// workspace's Z columns, with the exchange re-armed by p2p_setup (collective).
void bench_p2p(cs_problem* p, int kind, int reps, double* ms) {
  cs_ctx* c = p->ctx;
  if (p->ws.p == nullptr || p->ws_s < 2) fail(CS_ERR_INVALID_ARGUMENT, 0, "run a solve first");
  const int64_t ld = p->ld;
  double* Z = p->ws.as<double>() + 2 * p->ws_s * ld;  // workspace(): Q, AQ, Z, P, ...
  if (!p2p_setup(p, Z)) fail(CS_ERR_INVALID_ARGUMENT, 0, "peer-memory halo unavailable");
  std::function<void()> run;
  SpmvArgs g;
  if (kind == 5) {
    run = [&] {
      Launch L(c, CS_PHASE_COMM);
      SpmvArgs a;
      fill_push_args(p, a, 0);
      launch_halo_push(a, Z, p->n_local, nullptr, c->stream);
    };
  } else {
    g.x = Z;
    g.y = Z + 3 * ld;  // scratch columns of the basis
    g.zp2 = Z + ld;
    g.zout = Z + 2 * ld;
    g.ca = 1.0;
    g.cb = -0.5;
    g.cc = -1.0;
    p2p_push(p, Z, 0, nullptr);  // epoch 1's ghost planes (the z_0 push of a solve)
    run = [&] { spmv_p2p(p, kMpkMidF, g, 0); };
  }
  cudaEvent_t a, b;
  CS_CUDA(cudaEventCreate(&a));
  CS_CUDA(cudaEventCreate(&b));
  run();
  CS_CUDA(cudaEventRecord(a, c->stream));
  for (int i = 0; i < reps; ++i) run();
  CS_CUDA(cudaEventRecord(b, c->stream));
  CS_CUDA(cudaEventSynchronize(b));
  float t = 0.f;
  CS_CUDA(cudaEventElapsedTime(&t, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms = t / reps;
  // leave no push unreleased / no stale epoch: re-arm (collective)
  CS_CUDA(cudaStreamSynchronize(c->stream));
  p2p_setup(p, Z);
}
}  // namespace

int cs_bench_spmv(cs_problem* p, int kind, int reps, double* ms_per_launch) {
  return guard([&] {
    cs_ctx* c = p->ctx;
    CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
    if (reps < 1 || kind < 0 || kind > 6) fail(CS_ERR_INVALID_ARGUMENT, 0, "bad bench args");
    if (kind >= 5) {  // multi-GPU halo transport probes (collective; after one solve)
      bench_p2p(p, kind, reps, ms_per_launch);
      return;
    }
    const int64_t ld = p->ld, n = p->n_local;
    constexpr int S = 8;
    const int nvec = kind <= 2 ? 6 : 4 * S + 4;
    DBuf buf(sizeof(double) * ld * nvec), small(sizeof(double) * (4 * S * S + 4096) + 4096);
    double* v = buf.as<double>();
    {
      Launch L(c, CS_PHASE_OTHER);
      launch_random_vector(ld * nvec, 0, 99, v, c->stream);
    }
    double* sm = small.as<double>();
    CS_CUDA(cudaMemsetAsync(sm, 0, small.bytes, c->stream));
    DBuf part(sizeof(double) * (pack_partial_doubles(S, n) + 64));
    std::function<void()> run;
    SpmvArgs g;
    UpdateArgs ua{};
    if (kind <= 2) {
      g.x = v;
      g.y = v + ld;
      g.zp1 = v + 2 * ld;
      g.zp2 = v + 3 * ld;
      g.zpout = p->precond == CS_PRECOND_JACOBI ? v + 4 * ld : nullptr;
      g.zout = v + 5 * ld;
      g.ca = 1.0;
      g.cb = -0.5;
      g.cc = -1.0;
      const int k = kind == 0 ? kPlain : kind == 1 ? kMpkMid : kMpkMidF;
      if (k == kMpkMidF && std::getenv("CS_BENCH_NOP")) g.y = nullptr;  // PZ-schedule step
      run = [&, k] { launch_spmv(k, p->view(), g, 0, p->nslices, c->stream); };
    } else if (kind == 3) {
      unsigned* ticket = reinterpret_cast<unsigned*>(sm + 4 * S * S + 2048);
      PzArgs pz;
      if (std::getenv("CS_BENCH_PZ")) {
        pz.zs = v + 2 * S * ld;
        pz.sig1 = 1.0, pz.sig2 = 2.0, pz.k1 = 0.5, pz.k2 = 0.25, pz.dconst = 26.0;
      }
      run = [&, ticket, pz] {
        launch_pack(S, n, ld, v, v + S * ld, v + 2 * S * ld, v + 3 * S * ld, sm, part.as<double>(),
                    ticket, nullptr, nullptr, c->stream, pz);
      };
    } else {
      ua.s = S;
      ua.n = n;
      ua.ld = ld;
      ua.q = v;
      ua.aq = v + S * ld;
      ua.z = v + 2 * S * ld;
      ua.zw = v + 2 * S * ld;
      ua.p = v + 3 * S * ld;
      ua.x = v + 4 * S * ld;
      ua.r = v + (4 * S + 1) * ld;
      ua.inv_diag = p->view().inv_diag;
      ua.alpha = sm;
      ua.beta = sm + S;
      ua.st = c->state.as<DevState>();
      if (std::getenv("CS_BENCH_PZ")) {  // the PZ schedule's pass (P derived from Z)
        ua.pz.zs = v + 3 * S * ld;
        ua.pz.sig1 = 1.0, ua.pz.sig2 = 2.0, ua.pz.k1 = 0.5, ua.pz.k2 = 0.25, ua.pz.dconst = 26.0;
        ua.inv_const = 1.0 / 26.0;
      }
      CS_CUDA(cudaMemsetAsync(c->state.p, 0, sizeof(DevState), c->stream));
      run = [&] { launch_fast_update(ua, c->stream); };
    }
    cudaEvent_t a, b;
    CS_CUDA(cudaEventCreate(&a));
    CS_CUDA(cudaEventCreate(&b));
    run();  // warm-up
    CS_CUDA(cudaEventRecord(a, c->stream));
    for (int i = 0; i < reps; ++i) {
      Launch L(c, kind <= 2 ? CS_PHASE_SPMV : kind == 3 ? CS_PHASE_REDUCE : CS_PHASE_UPDATE);
      run();
    }
    CS_CUDA(cudaEventRecord(b, c->stream));
    CS_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    CS_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_per_launch = ms / reps;
  });
}

int cs_mpk(cs_problem* p, const double* r, int s, double lo, double hi, double* z, double* pblk) {
  return guard([&] {
    cs_ctx* c = p->ctx;
    CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
    if (s < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "mpk: s must be >= 1");
    if (!(hi > lo) || !(lo > 0.0) || !std::isfinite(hi))
      fail(CS_ERR_INVALID_ARGUMENT, 0, "ChebyshevParams: need lambda_max > lambda_min > 0");
    const int64_t n = p->n_local, ld = p->ld;
    DBuf Zb(sizeof(double) * ld * s), Pb(sizeof(double) * ld * s), rb(sizeof(double) * ld),
        za(sizeof(double) * ld), zb(sizeof(double) * ld), st(sizeof(DevState));
    CS_CUDA(cudaMemsetAsync(st.p, 0, sizeof(DevState), c->stream));
    CS_CUDA(cudaMemcpyAsync(rb.p, r, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    DevState* dst = st.as<DevState>();
    {
      Launch L(c, CS_PHASE_UPDATE);
      precond_apply(p, rb.as<double>(), Zb.as<double>(), dst, 0, 0);
    }
    mpk_unit(p, Zb.as<double>(), Pb.as<double>(), rb.as<double>(), za.as<double>(),
             zb.as<double>(), s, lo, hi, dst);
    DevState h;
    CS_CUDA(cudaMemcpyAsync(&h, dst, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    for (int j = 0; j < s; ++j) {
      to_host(c, z + j * n, Zb.as<double>() + j * ld, sizeof(double) * n);
      to_host(c, pblk + (j + 1) * n, Pb.as<double>() + j * ld, sizeof(double) * n);
    }
    sync(c);
    std::memcpy(pblk, r, sizeof(double) * n);  // P column 0 carries r (mpk.cpp:49)
    if (h.err) {
      const int payload = static_cast<int>(h.err & 0xffffffffu);
      fail(CS_ERR_BASIS_BREAKDOWN, payload, format_device_error(h.err, s));
    }
  });
}

int cs_block_gram(cs_ctx* ctx, int64_t n, int ku, int kv, const double* u, const double* v,
                  double* g, int mode) {
  return guard([&] {
    CS_CUDA(cudaSetDevice(ctx->device));
    StreamBind bind_stream_(ctx->stream);
    if (ku < 0 || kv < 0 || ku > kMaxS || kv > kMaxS)
      fail(CS_ERR_DIMENSION, 0, "SmallDense: dimensions must be in [0, 64]");
    if (ku == 0 || kv == 0) return;
    HostIn du(ctx, u, sizeof(double) * n * ku), dv(ctx, v, sizeof(double) * n * kv);
    DBuf dg(sizeof(double) * ku * kv), part(sizeof(double) * tree_gram_partial_doubles(n, ku, kv)),
        tk(sizeof(unsigned));
    CS_CUDA(cudaMemsetAsync(tk.p, 0, sizeof(unsigned), ctx->stream));
    {
      Launch L(ctx, CS_PHASE_REDUCE);
      if (mode == CS_MODE_REFERENCE)
        launch_serial_gram(n, ku, kv, du.d.as<double>(), n, dv.d.as<double>(), n, dg.as<double>(),
                           nullptr, ctx->stream);
      else
        launch_tree_gram(n, ku, kv, du.d.as<double>(), n, dv.d.as<double>(), n, dg.as<double>(),
                         part.as<double>(), tk.as<unsigned>(), nullptr, ctx->stream);
    }
    to_host(ctx, g, dg.p, sizeof(double) * ku * kv);
    sync(ctx);
  });
}

int cs_block_update(cs_ctx* ctx, int64_t n, int m, int k, const double* y, const double* x,
                    const double* c, double* out) {
  return guard([&] {
    CS_CUDA(cudaSetDevice(ctx->device));
    StreamBind bind_stream_(ctx->stream);
    if (m > kMaxS || k > kMaxS) fail(CS_ERR_DIMENSION, 0, "SmallDense: dimensions must be in [0, 64]");
    HostIn dy(ctx, y, sizeof(double) * n * k), dx(ctx, x, sizeof(double) * n * m),
        dc(ctx, c, sizeof(double) * m * k);
    DBuf dout(sizeof(double) * n * k);
    {
      Launch L(ctx, CS_PHASE_UPDATE);
      launch_block_update(n, m, k, dy.d.as<double>(), dx.d.as<double>(), dc.d.as<double>(),
                          dout.as<double>(), ctx->stream);
    }
    to_host(ctx, out, dout.p, sizeof(double) * n * k);
    sync(ctx);
  });
}

int cs_assemble_gram(cs_ctx* ctx, int64_t n, int k, const double* q, const double* aq, double* w,
                     int mode) {
  return guard([&] {
    CS_CUDA(cudaSetDevice(ctx->device));
    StreamBind bind_stream_(ctx->stream);
    if (k < 1 || k > kMaxS) fail(CS_ERR_DIMENSION, 0, "SmallDense: dimensions must be in [0, 64]");
    HostIn dq(ctx, q, sizeof(double) * n * k), da(ctx, aq, sizeof(double) * n * k);
    DBuf dw(sizeof(double) * k * k), part(sizeof(double) * tree_gram_partial_doubles(n, k, k)),
        tk(sizeof(unsigned)), st(sizeof(int));
    CS_CUDA(cudaMemsetAsync(tk.p, 0, sizeof(unsigned), ctx->stream));
    {
      Launch L(ctx, CS_PHASE_REDUCE);
      if (mode == CS_MODE_REFERENCE)
        launch_serial_gram(n, k, k, dq.d.as<double>(), n, da.d.as<double>(), n, dw.as<double>(),
                           nullptr, ctx->stream);
      else
        launch_tree_gram(n, k, k, dq.d.as<double>(), n, da.d.as<double>(), n, dw.as<double>(),
                         part.as<double>(), tk.as<unsigned>(), nullptr, ctx->stream);
    }
    {
      Launch L(ctx, CS_PHASE_SMALL);
      launch_unit_assemble(k, dw.as<double>(), st.as<int>(), ctx->stream);
    }
    int hs = 0;
    to_host(ctx, &hs, st.p, sizeof(int));
    to_host(ctx, w, dw.p, sizeof(double) * k * k);
    sync(ctx);
    small_status(hs);
  });
}

int cs_fgs_solve(cs_ctx* ctx, int s, const double* w, int k, const double* rhs, int nu,
                 double* x, double* delta) {
  return guard([&] {
    CS_CUDA(cudaSetDevice(ctx->device));
    StreamBind bind_stream_(ctx->stream);
    if (s < 1 || k < 1 || s > kMaxS || k > kMaxS)
      fail(CS_ERR_DIMENSION, 0, "SmallDense: dimensions must be in [0, 64]");
    if (nu < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "fgs: nu must be >= 1");
    HostIn dw(ctx, w, sizeof(double) * s * s), dr(ctx, rhs, sizeof(double) * s * k);
    DBuf dx(sizeof(double) * s * k), dd(sizeof(double)), st(sizeof(int));
    {
      Launch L(ctx, CS_PHASE_SMALL);
      launch_unit_fgs(s, dw.d.as<double>(), k, dr.d.as<double>(), nu, dx.as<double>(),
                      dd.as<double>(), st.as<int>(), ctx->stream);
    }
    int hs = 0;
    to_host(ctx, &hs, st.p, sizeof(int));
    sync(ctx);
    small_status(hs);
    to_host(ctx, x, dx.p, sizeof(double) * s * k);
    to_host(ctx, delta, dd.p, sizeof(double));
    sync(ctx);
  });
}

int cs_cholesky_solve(cs_ctx* ctx, int s, const double* w, int k, const double* rhs, double* x) {
  return guard([&] {
    CS_CUDA(cudaSetDevice(ctx->device));
    StreamBind bind_stream_(ctx->stream);
    if (s < 1 || k < 1 || s > kMaxS || k > kMaxS)
      fail(CS_ERR_DIMENSION, 0, "SmallDense: dimensions must be in [0, 64]");
    HostIn dw(ctx, w, sizeof(double) * s * s), dr(ctx, rhs, sizeof(double) * s * k);
    DBuf dx(sizeof(double) * s * k), st(sizeof(int));
    {
      Launch L(ctx, CS_PHASE_SMALL);
      launch_unit_chol(s, dw.d.as<double>(), k, dr.d.as<double>(), dx.as<double>(), st.as<int>(),
                       ctx->stream);
    }
    int hs = 0;
    to_host(ctx, &hs, st.p, sizeof(int));
    sync(ctx);
    small_status(hs);
    to_host(ctx, x, dx.p, sizeof(double) * s * k);
    sync(ctx);
  });
}

int cs_random_vector(cs_ctx* ctx, int64_t n, uint64_t seed, double* out) {
  return guard([&] {
    CS_CUDA(cudaSetDevice(ctx->device));
    StreamBind bind_stream_(ctx->stream);
    DBuf d(sizeof(double) * n);
    {
      Launch L(ctx, CS_PHASE_OTHER);
      launch_random_vector(n, 0, seed, d.as<double>(), ctx->stream);
    }
    to_host(ctx, out, d.p, sizeof(double) * n);
    sync(ctx);
  });
}

int cs_tridiag_eigvals(int m, const double* diag, const double* off, double* out) {
  return guard([&] { tridiag_eigenvalues(m, diag, off, out); });
}

int cs_estimate_interval(cs_problem* p, int steps, uint64_t seed, int mode, double* lo,
                         double* hi) {
  return guard([&] { estimate_interval_dev(p, steps, seed, mode, lo, hi, nullptr); });
}

// ------------------------------------------------------------------ solves

void cs_config_default(cs_config* cfg) {
  std::memset(cfg, 0, sizeof *cfg);
  cfg->s = 4;  // solver.hpp:17-28 defaults
  cfg->tol = 1e-6;
  cfg->max_outer = 500;
  cfg->nu = 30;
  cfg->gram = CS_GRAM_FGS;
  cfg->lanczos_steps = 40;
  cfg->seed = 1234;
  cfg->mode = CS_MODE_FAST;
}

int cs_pcg_s_solve_device(cs_problem* p, const double* b, const double* x0, const cs_config* cfg,
                          double* x, cs_report* rep) {
  return guard([&] { pcgs_solve_dev(p, b, x0, *cfg, x, rep); });
}

int cs_pcg_solve_device(cs_problem* p, const double* b, const double* x0, double tol,
                        int max_iter, int mode, double* x, cs_report* rep) {
  return guard([&] { pcg_solve_dev(p, b, x0, tol, max_iter, mode, x, rep); });
}

int cs_pcg_s_solve(cs_problem* p, const double* b, const double* x0, const cs_config* cfg,
                   double* x, cs_report* rep) {
  return guard([&] {
    cs_ctx* c = p->ctx;
    CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
    const size_t bytes = sizeof(double) * p->n_local;
    HostIn db(c, b, bytes), dx0(c, x0, bytes);
    DBuf dx(bytes);
    pcgs_solve_dev(p, db.d.as<double>(), dx0.d.as<double>(), *cfg, dx.as<double>(), rep);
    to_host(c, x, dx.p, bytes);
    sync(c);
  });
}

int cs_pcg_solve(cs_problem* p, const double* b, const double* x0, double tol, int max_iter,
                 int mode, double* x, cs_report* rep) {
  return guard([&] {
    cs_ctx* c = p->ctx;
    CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
    const size_t bytes = sizeof(double) * p->n_local;
    HostIn db(c, b, bytes), dx0(c, x0, bytes);
    DBuf dx(bytes);
    pcg_solve_dev(p, db.d.as<double>(), dx0.d.as<double>(), tol, max_iter, mode, dx.as<double>(),
                  rep);
    to_host(c, x, dx.p, bytes);
    sync(c);
  });
}

int cs_pcg_solve_cfg(cs_problem* p, const double* b, const double* x0, const cs_config* cfg,
                     double* x, cs_report* rep) {
  return guard([&] {
    cs_ctx* c = p->ctx;
    CS_CUDA(cudaSetDevice(c->device));
    StreamBind bind_stream_(c->stream);
    const size_t bytes = sizeof(double) * p->n_local;
    HostIn db(c, b, bytes), dx0(c, x0, bytes);
    DBuf dx(bytes);
    pcg_solve_dev(p, db.d.as<double>(), dx0.d.as<double>(), cfg->tol, cfg->max_outer, cfg->mode,
                  dx.as<double>(), rep, cfg);
    to_host(c, x, dx.p, bytes);
    sync(c);
  });
}

int cs_pcg_s_solve_csr(cs_ctx* ctx, int64_t n, const int64_t* rowptr, const int64_t* col,
                       const double* val, int precond, const double* b, const double* x0,
                       const cs_config* cfg, double* x, cs_report* rep) {
  return guard([&] {
    // solver.cpp:15-22 validation precedes everything else in the reference
    if (cfg->s < 1 || cfg->s > kMaxS)
      fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: s must be in [1, 64]");
    if (!(cfg->tol > 0.0)) fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: tol must be > 0");
    if (cfg->max_outer < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: max_outer must be >= 1");
    if (cfg->nu < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "SolverConfig: nu must be >= 1");
    CS_CUDA(cudaSetDevice(ctx->device));
    StreamBind bind_stream_(ctx->stream);
    Trace tr("cs_pcg_s_solve_csr", ctx->stream);
    std::unique_ptr<cs_problem> p(problem_upload_csr(ctx, n, rowptr, col, val));
    tr.mark("upload+SELL-32P");
    problem_set_precond(p.get(), precond);
    const size_t bytes = sizeof(double) * n;
    HostIn db(ctx, b, bytes), dx0(ctx, x0, bytes);
    DBuf dx(bytes);
    tr.mark("precond+vectors");
    pcgs_solve_dev(p.get(), db.d.as<double>(), dx0.d.as<double>(), *cfg, dx.as<double>(), rep);
    tr.mark("solve");
    to_host(ctx, x, dx.p, bytes);
    sync(ctx);
    tr.mark("download");
    p.reset();
    tr.mark("release");
  });
}

int cs_pcg_solve_csr(cs_ctx* ctx, int64_t n, const int64_t* rowptr, const int64_t* col,
                     const double* val, int precond, const double* b, const double* x0,
                     double tol, int max_iter, double* x, cs_report* rep) {
  return guard([&] {
    if (!(tol >= 0.0) || max_iter < 1) fail(CS_ERR_INVALID_ARGUMENT, 0, "pcg_solve: bad tol/max_iter");
    std::unique_ptr<cs_problem> p(problem_upload_csr(ctx, n, rowptr, col, val));
    problem_set_precond(p.get(), precond);
    const size_t bytes = sizeof(double) * n;
    HostIn db(ctx, b, bytes), dx0(ctx, x0, bytes);
    DBuf dx(bytes);
    pcg_solve_dev(p.get(), db.d.as<double>(), dx0.d.as<double>(), tol, max_iter, CS_MODE_FAST,
                  dx.as<double>(), rep);
    to_host(ctx, x, dx.p, bytes);
    sync(ctx);
  });
}

}  // extern "C"
