// runtime.cu -- device context, device-resident problems, halo exchange,
// collectives and launch/timing accounting.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <atomic>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "runtime.cuh"

namespace csg {

thread_local cudaStream_t g_alloc_stream = nullptr;

[[noreturn]] void fail(int code, int payload, const std::string& msg) {
  throw LibError{code, payload, msg};
}

#define CS_NCCL(call)                                                                   \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      ::csg::fail(CS_ERR_NCCL, 0, std::string("NCCL: ") + ncclGetErrorString(r_) + " in " #call); \
  } while (0)

// ------------------------------------------------------------------ accounting

cudaEvent_t pooled_event(cs_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CS_CUDA(cudaEventCreate(&e));
  return e;
}

Launch::Launch(cs_ctx* ctx, int ph) : c(ctx), phase(ph) {
  ++c->launches;
  ++c->phase_launches[ph];
  if (c->timing) {
    a = pooled_event(c);
    CS_CUDA(cudaEventRecord(a, c->stream));
  }
}

Launch::~Launch() {
  if (c->timing && a != nullptr) {
    cudaEvent_t b = pooled_event(c);
    cudaEventRecord(b, c->stream);
    c->spans.push_back({phase, a, b});
  }
}

void collect_timing(cs_ctx* c) {
  if (c->spans.empty()) return;
  CS_CUDA(cudaStreamSynchronize(c->stream));
  static const bool trace = std::getenv("CS_TIMING_TRACE") != nullptr;  // diagnostics
  for (const auto& s : c->spans) {
    float ms = 0.f;
    CS_CUDA(cudaEventElapsedTime(&ms, s.a, s.b));
    if (trace) std::fprintf(stderr, "[trace r%d] phase %d %.4f ms\n", c->rank, s.phase, ms);
    c->phase_ms[s.phase] += ms;
    c->event_pool.push_back(s.a);
    c->event_pool.push_back(s.b);
  }
  c->spans.clear();
}

void* ctx_scratch(cs_ctx* c, size_t bytes) {
  if (c->scratch_bytes < bytes) {
    CS_CUDA(cudaStreamSynchronize(c->stream));
    c->scratch.alloc(bytes);
    c->scratch_bytes = bytes;
  }
  return c->scratch.p;
}

// ------------------------------------------------------------------ communication

void halo_exchange_on(cs_problem* p, double* col, cudaStream_t st) {
  cs_ctx* c = p->ctx;
  if (p->general_halo) {
    double* buf = p->send_buf.as<double>();
    launch_halo_gather(p->send_off.back(), p->send_idx.as<int32_t>(), col, buf, st);
    CS_NCCL(ncclGroupStart());
    for (int q = 0; q < c->nranks; ++q) {
      const int64_t rc = p->recv_off[q + 1] - p->recv_off[q];
      const int64_t sc = p->send_off[q + 1] - p->send_off[q];
      if (rc) CS_NCCL(ncclRecv(col + p->n_local + p->recv_off[q], rc, ncclDouble, q, c->comm, st));
      if (sc) CS_NCCL(ncclSend(buf + p->send_off[q], sc, ncclDouble, q, c->comm, st));
    }
    CS_NCCL(ncclGroupEnd());
    return;
  }
  CS_NCCL(ncclGroupStart());
  if (p->ghost_lo > 0) {
    CS_NCCL(ncclRecv(col + p->n_local, p->ghost_lo, ncclDouble, c->rank - 1, c->comm, st));
    CS_NCCL(ncclSend(col, p->send_lo, ncclDouble, c->rank - 1, c->comm, st));
  }
  if (p->ghost_hi > 0) {
    CS_NCCL(ncclRecv(col + p->n_local + p->ghost_lo, p->ghost_hi, ncclDouble, c->rank + 1,
                     c->comm, st));
    CS_NCCL(ncclSend(col + p->n_local - p->send_hi, p->send_hi, ncclDouble, c->rank + 1, c->comm,
                     st));
  }
  CS_NCCL(ncclGroupEnd());
}

void halo_exchange(cs_problem* p, double* col) {
  cs_ctx* c = p->ctx;
  if (c->nranks == 1 || !p->has_halo()) return;
  Launch L(c, CS_PHASE_COMM);
  halo_exchange_on(p, col, c->stream);
}

void spmv_halo(cs_problem* p, int kind, SpmvArgs g, double* operand) {
  cs_ctx* c = p->ctx;
  const SellView A = p->view();
  const bool halo = c->nranks > 1 && p->has_halo();
  const bool overlap = halo && kind != kDot && p->slice_int_end > p->slice_int_begin;
  if (!overlap) {
    if (halo) halo_exchange(p, operand);
    Launch L(c, CS_PHASE_SPMV);
    launch_spmv(kind, A, g, 0, p->nslices, c->stream);
    return;
  }
  // halo on the comm stream, interior slices meanwhile, then the boundary
  CS_CUDA(cudaEventRecord(c->ev_ready, c->stream));
  CS_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
  ++c->launches;
  ++c->phase_launches[CS_PHASE_COMM];
  halo_exchange_on(p, operand, c->comm_stream);
  CS_CUDA(cudaEventRecord(c->ev_halo, c->comm_stream));
  {
    Launch L(c, CS_PHASE_SPMV);
    launch_spmv(kind, A, g, p->slice_int_begin, p->slice_int_end, c->stream);
  }
  CS_CUDA(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
  {
    Launch L(c, CS_PHASE_SPMV);
    // both boundary ranges [ie, nslices) and [0, ib) in one wrapped launch
    launch_spmv(kind, A, g, p->slice_int_end, p->nslices + p->slice_int_begin, c->stream);
  }
}

int kernel_setup(const void* func, int threads, int smem) {
  struct Key {
    int dev;
    const void* f;
    int threads, smem;
    bool operator<(const Key& o) const {
      return std::tie(dev, f, threads, smem) < std::tie(o.dev, o.f, o.threads, o.smem);
    }
  };
  static std::mutex mu;
  static std::map<Key, int> cache;
  static std::map<std::pair<int, const void*>, int> opted;  // attribute value per (device, kernel)
  int dev = 0;
  CS_CUDA(cudaGetDevice(&dev));
  const Key k{dev, func, threads, smem};
  std::lock_guard<std::mutex> lock(mu);
  const auto it = cache.find(k);
  if (it != cache.end()) return it->second;
  // the attribute is a per-kernel upper bound: only ever raise it (a later,
  // smaller launch must not lower the bound an earlier, larger one relies on)
  int& cur = opted[{dev, func}];
  if (smem > 48 * 1024 && smem > cur) {
    CS_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cur = smem;
  }
  int per_sm = 0;
  CS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem));
  per_sm = std::max(per_sm, 1);
  cache.emplace(k, per_sm);
  return per_sm;
}

void allreduce_sum(cs_ctx* c, double* dev, size_t count) {
  ++c->allreduces;
  if (c->nranks == 1) return;
  Launch L(c, CS_PHASE_COMM);
  CS_NCCL(ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, c->comm, c->stream));
}

// ------------------------------------------------------------------ NVLink peer-memory halo

namespace {
struct PeerInfo {
  cudaIpcMemHandle_t ws, sig;
  uint64_t gen;
  int64_t z_off, ld, n_local, ghost_lo;
  unsigned char uuid[16];
  int32_t ok, pad;
};

void fill_push(const cs_problem* p, SpmvArgs& g, int col);
}  // namespace

void fill_push_args(const cs_problem* p, SpmvArgs& g, int col) { fill_push(p, g, col); }

namespace {
void fill_push(const cs_problem* p, SpmvArgs& g, int col) {
  if (p->ghost_lo > 0) {  // my first plane -> rank-1's upper ghost plane
    const cs_problem::PeerMap& m = p->peer[0];
    g.push_lo = static_cast<double*>(m.ws) + m.ghost_off + static_cast<int64_t>(col) * m.ld;
    g.send_lo = p->send_lo;

  }
  if (p->ghost_hi > 0) {  // my last plane -> rank+1's lower ghost plane
    const cs_problem::PeerMap& m = p->peer[1];
    g.push_hi = static_cast<double*>(m.ws) + m.ghost_off + static_cast<int64_t>(col) * m.ld;
    g.hi_begin = p->n_local - p->send_hi;

  }
}
}  // namespace

void p2p_teardown(cs_problem* p) {
  for (auto& m : p->peer) {
    if (m.ws) cudaIpcCloseMemHandle(m.ws);
    if (m.sig) cudaIpcCloseMemHandle(m.sig);
    m = cs_problem::PeerMap{};
  }
  for (auto& x : p->xpeer) {
    if (x) cudaIpcCloseMemHandle(x);
    x = nullptr;
  }
  cudaGetLastError();
  p->p2p = false;
  p->xred_ok = false;
}

namespace {
size_t xred_bytes(int nranks) {
  return sizeof(double) * 2 * static_cast<size_t>(nranks) * kXredSlot +
         sizeof(unsigned long long) * kXredMaxRanks;
}

// Collective (every rank, after the neighbour mapping): map every rank's
// exchange buffer; flags restart at 0 for this solve (the all-gather orders the
// reset before any peer's first store). false on every rank if any rank cannot.
bool xred_setup(cs_problem* p, bool ok_in) {
  cs_ctx* c = p->ctx;
  const int N = c->nranks, me = c->rank;
  const char* env = std::getenv("CS_P2P_ALLREDUCE");
  int ok = ok_in && N <= kXredMaxRanks && (env == nullptr || std::atoi(env) != 0);
  if (ok && p->xred.p == nullptr) {
    StreamBind plain(nullptr);  // IPC export needs a cudaMalloc allocation
    p->xred.alloc(xred_bytes(N));
  }
  if (ok) {
    CS_CUDA(cudaMemsetAsync(p->xred.p, 0, xred_bytes(N), c->stream));
    if (!p->xred_exported) {
      p->xred_exported = cudaIpcGetMemHandle(&p->ipc_xred, p->xred.p) == cudaSuccess;
      cudaGetLastError();
    }
    ok = p->xred_exported;
  }
  struct XInfo {
    cudaIpcMemHandle_t h;
    unsigned char uuid[16];
    int32_t ok, pad;
  };
  XInfo mine{};
  mine.h = p->ipc_xred;
  std::memcpy(mine.uuid, c->uuid, 16);
  mine.ok = ok;
  DBuf dev(sizeof(XInfo) * (N + 1));
  XInfo* d = dev.as<XInfo>();
  CS_CUDA(cudaMemcpyAsync(d + N, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
  CS_NCCL(ncclAllGather(d + N, d, sizeof(XInfo), ncclChar, c->comm, c->stream));
  std::vector<XInfo> all(N);
  CS_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(XInfo) * N, cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  for (int r = 0; r < N && ok; ++r) {
    if (r == me) continue;
    // ranks sharing a GPU must not spin on each other: the NCCL allreduce instead
    if (!all[r].ok || std::memcmp(all[r].uuid, mine.uuid, 16) == 0) {
      ok = 0;
      break;
    }
    if (p->xpeer[r] == nullptr &&
        cudaIpcOpenMemHandle(&p->xpeer[r], all[r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      p->xpeer[r] = nullptr;
      ok = 0;
    }
  }
  DBuf e(sizeof(int));
  CS_CUDA(cudaMemcpyAsync(e.p, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CS_NCCL(ncclAllReduce(e.p, e.p, 1, ncclInt32, ncclMin, c->comm, c->stream));
  int all_ok = 0;
  CS_CUDA(cudaMemcpyAsync(&all_ok, e.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  p->xred_epoch = 0;
  if (std::getenv("CS_TRACE"))
    std::fprintf(stderr, "[cs-trace] rank %d xred_setup ok_in %d local %d all %d exported %d\n", me,
                 static_cast<int>(ok_in), ok, all_ok, static_cast<int>(p->xred_exported));
  return all_ok != 0;
}
}  // namespace

XredArgs xred_next(cs_problem* p, int npack) {
  XredArgs x;
  if (!p->xred_ok || npack > kXredSlot) return x;
  cs_ctx* c = p->ctx;
  x.nranks = c->nranks;
  x.rank = c->rank;
  x.npack = npack;
  x.epoch = ++p->xred_epoch;
  x.slots = p->xred.as<double>();
  x.flags = reinterpret_cast<unsigned long long*>(x.slots + 2 * static_cast<size_t>(x.nranks) * kXredSlot);
  for (int r = 0; r < x.nranks; ++r) {
    if (r == x.rank) continue;
    x.peer_slots[r] = static_cast<double*>(p->xpeer[r]);
    x.peer_flags[r] = reinterpret_cast<unsigned long long*>(
        x.peer_slots[r] + 2 * static_cast<size_t>(x.nranks) * kXredSlot);
  }
  return x;
}

bool p2p_setup(cs_problem* p, double* Z) {
  cs_ctx* c = p->ctx;
  p->p2p = false;
  p->p2p_epoch = 0;
  p->p2p_pending = false;
  if (c->nranks == 1 || p->general_halo) return false;
  const char* env = std::getenv("CS_P2P_HALO");
  int ok = (env == nullptr || std::atoi(env) != 0) && !p->ws.pooled && p->ws.p != nullptr;
  if (ok && p->sig.p == nullptr) {
    StreamBind plain(nullptr);  // IPC export needs a cudaMalloc allocation
    p->sig.alloc(64);
  }
  // receive counters restart at 0 for this solve; the exchange below orders the
  // reset before any peer's first push
  if (p->sig.p) CS_CUDA(cudaMemsetAsync(p->sig.p, 0, 64, c->stream));
  PeerInfo mine{};
  if (ok && p->ipc_gen != p->ws_gen) {  // export handles once per workspace generation
    ok = cudaIpcGetMemHandle(&p->ipc_ws, p->ws.p) == cudaSuccess &&
         cudaIpcGetMemHandle(&p->ipc_sig, p->sig.p) == cudaSuccess;
    cudaGetLastError();
    if (ok) p->ipc_gen = p->ws_gen;
  }
  if (ok) {
    mine.ws = p->ipc_ws;
    mine.sig = p->ipc_sig;
  }
  mine.gen = p->ws_gen;
  mine.z_off = Z - p->ws.as<double>();
  mine.ld = p->ld;
  mine.n_local = p->n_local;
  mine.ghost_lo = p->ghost_lo;
  if (!c->uuid_known) {  // cudaGetDeviceProperties costs milliseconds: once per context
    cudaDeviceProp prop;
    CS_CUDA(cudaGetDeviceProperties(&prop, c->device));
    std::memcpy(c->uuid, prop.uuid.bytes, 16);
    c->uuid_known = true;
  }
  std::memcpy(mine.uuid, c->uuid, 16);
  mine.ok = ok;
  DBuf dev(3 * sizeof(PeerInfo));
  PeerInfo* d = dev.as<PeerInfo>();
  CS_CUDA(cudaMemcpyAsync(d, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
  CS_NCCL(ncclGroupStart());
  if (p->ghost_lo > 0) {
    CS_NCCL(ncclSend(d, sizeof(PeerInfo), ncclChar, c->rank - 1, c->comm, c->stream));
    CS_NCCL(ncclRecv(d + 1, sizeof(PeerInfo), ncclChar, c->rank - 1, c->comm, c->stream));
  }
  if (p->ghost_hi > 0) {
    CS_NCCL(ncclSend(d, sizeof(PeerInfo), ncclChar, c->rank + 1, c->comm, c->stream));
    CS_NCCL(ncclRecv(d + 2, sizeof(PeerInfo), ncclChar, c->rank + 1, c->comm, c->stream));
  }
  CS_NCCL(ncclGroupEnd());
  PeerInfo got[3];
  CS_CUDA(cudaMemcpyAsync(got, d, sizeof got, cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  for (int side = 0; side < 2 && ok; ++side) {
    const bool present = side == 0 ? p->ghost_lo > 0 : p->ghost_hi > 0;
    if (!present) continue;
    const PeerInfo& in = got[1 + side];
    // ranks sharing one GPU must not spin on each other (no co-scheduling
    // guarantee between their kernels): those fall back to NCCL
    if (!in.ok || std::memcmp(in.uuid, mine.uuid, 16) == 0) {
      ok = 0;
      break;
    }
    cs_problem::PeerMap& m = p->peer[side];
    if (m.ws == nullptr || m.gen != in.gen) {
      if (m.ws) cudaIpcCloseMemHandle(m.ws);
      if (m.sig) cudaIpcCloseMemHandle(m.sig);
      m = cs_problem::PeerMap{};
      if (cudaIpcOpenMemHandle(&m.ws, in.ws, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
          cudaIpcOpenMemHandle(&m.sig, in.sig, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      m.gen = in.gen;
    }
    m.ld = in.ld;
    // rank-1 holds my first plane in its upper ghost slots; rank+1 my last in its lower
    m.ghost_off = in.z_off + in.n_local + (side == 0 ? in.ghost_lo : 0);
  }
  // every rank takes the same path
  DBuf e(sizeof(int));
  CS_CUDA(cudaMemcpyAsync(e.p, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CS_NCCL(ncclAllReduce(e.p, e.p, 1, ncclInt32, ncclMin, c->comm, c->stream));
  int all = 0;
  CS_CUDA(cudaMemcpyAsync(&all, e.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  p->p2p = all != 0;
  // the packed-block allreduce over peer memory (collective on every rank)
  p->xred_ok = xred_setup(p, p->p2p);
  return p->p2p;
}

// release args for the pushes of the previous kernel (if it pushed)
void fill_release(cs_problem* p, SpmvArgs& g) {
  if (!p->p2p_pending) return;
  if (p->ghost_lo > 0) {  // rank-1's "from upper" counter
    g.rel_lo = static_cast<unsigned long long*>(p->peer[0].sig) + 1;
    g.rel_lo_n = static_cast<unsigned long long>(p->send_lo);
  }
  if (p->ghost_hi > 0) {  // rank+1's "from lower" counter
    g.rel_hi = static_cast<unsigned long long*>(p->peer[1].sig) + 0;
    g.rel_hi_n = static_cast<unsigned long long>(p->send_hi);
  }
  p->p2p_pending = false;
}

void spmv_p2p(cs_problem* p, int kind, SpmvArgs g, int push_col) {
  cs_ctx* c = p->ctx;
  const SellView A = p->view();
  ++p->p2p_epoch;
  if (push_col >= 0) fill_push(p, g, push_col);
  {
    SpmvArgs gi = g;  // the interior launch releases the previous kernel's pushes
    fill_release(p, gi);
    if (p->slice_int_end > p->slice_int_begin) {
      Launch L(c, CS_PHASE_SPMV);
      launch_spmv(kind, A, gi, p->slice_int_begin, p->slice_int_end, c->stream);
    } else if (gi.rel_lo || gi.rel_hi) {
      Launch L(c, CS_PHASE_COMM);
      launch_halo_release(gi, g.st, c->stream);
    }
  }
  g.wait_ctr = p->sig.as<unsigned long long>();
  g.want_lo = p->p2p_epoch * static_cast<unsigned long long>(p->ghost_lo);
  g.want_hi = p->p2p_epoch * static_cast<unsigned long long>(p->ghost_hi);
  Launch L(c, CS_PHASE_SPMV);
  launch_spmv(kind, A, g, p->slice_int_end, p->nslices + p->slice_int_begin, c->stream);
  p->p2p_pending = push_col >= 0;
}

void p2p_push(cs_problem* p, const double* src, int col, DevState* st) {
  SpmvArgs g;
  fill_push(p, g, col);
  fill_release(p, g);  // (nothing pending here in practice)
  if (g.rel_lo || g.rel_hi) launch_halo_release(g, st, p->ctx->stream);
  Launch L(p->ctx, CS_PHASE_COMM);
  launch_halo_push(g, src, p->n_local, st, p->ctx->stream);
  p->p2p_pending = true;
}

std::string format_device_error(unsigned long long word, int) {
  const int code = static_cast<int>((word >> 32) & 0xff);
  const int sub = static_cast<int>((word >> 40) & 0xff);
  const int payload = static_cast<int>(word & 0xffffffffu);
  const std::string k = std::to_string(payload);
  switch (code) {
    case CS_ERR_BASIS_BREAKDOWN:
      return "mpk: non-finite basis column " + std::to_string(payload + 1);
    case CS_ERR_SOLVER_BREAKDOWN:
      if (sub == 1)
        return "Gram assembly degenerate at outer iteration " + k +
               ": gram: non-positive diagonal (basis degeneracy)";
      if (sub == 2) return "gram solve failed at outer iteration " + k + ": fgs: zero diagonal";
      if (sub == 3)
        return "gram solve failed at outer iteration " + k +
               ": cholesky: non-positive pivot (basis breakdown)";
      return "pcg: non-positive curvature at iteration " + k;
    case CS_ERR_NCCL:
      if (sub == 1 || payload == 1)
        return "allreduce: a peer's packed block did not arrive (peer-memory allreduce timeout)";
      return "halo exchange: peer ghost planes did not arrive (peer-memory halo timeout)";
    case CS_ERR_GENERIC:
      if (sub == 1) return "estimate_interval: degenerate start vector";
      return "estimate_interval: non-finite value";
    default:
      return "device error";
  }
}

}  // namespace csg

using namespace csg;

// ------------------------------------------------------------------ context (C++ side of the ABI)

namespace csg {

cs_ctx* ctx_create(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    fail(CS_ERR_CUDA, 0, "no CUDA device available (libchebstep_gpu has no CPU fallback)");
  if (device < 0 || device >= count) fail(CS_ERR_INVALID_ARGUMENT, 0, "bad device ordinal");
  CS_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<cs_ctx>();
  c->device = device;
  CS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CS_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  CS_CUDA(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  CS_CUDA(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  // keep freed pool memory cached for reuse (repeated solves / uploads)
  cudaMemPool_t pool;
  CS_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = ~uint64_t{0};
  CS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  c->state.alloc(sizeof(DevState));
  CS_CUDA(cudaMallocHost(&c->pinned, 4096));
  return c.release();
}

void ctx_destroy(cs_ctx* c) {
  if (c == nullptr) return;
  // a problem's buffers are freed on this context's stream: destroying the
  // context first would leave cs_problem_destroy a dangling stream
  if (c->live_problems.load() > 0)
    fail(CS_ERR_INVALID_ARGUMENT, c->live_problems.load(),
         "cs_ctx_destroy: " + std::to_string(c->live_problems.load()) +
             " problem(s) of this context are still alive; destroy them first");
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& s : c->spans) {
    cudaEventDestroy(s.a);
    cudaEventDestroy(s.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  // pooled buffers are freed on the context stream: release them before it goes
  c->scratch.release();
  c->normbuf.release();
  c->state.release();
  c->lz.release();
  cudaStreamSynchronize(c->stream);
  if (c->comm) ncclCommDestroy(c->comm);
  cudaEventDestroy(c->ev_ready);
  cudaEventDestroy(c->ev_halo);
  cudaStreamDestroy(c->stream);
  cudaStreamDestroy(c->comm_stream);
  cudaFreeHost(c->pinned);
  if (c->host_stage) cudaFreeHost(c->host_stage);
  delete c;
}

void comm_init(cs_ctx* c, int nranks, int rank, const unsigned char id[128]) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(CS_ERR_INVALID_ARGUMENT, 0, "bad rank");
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  if (c->comm) {
    ncclCommDestroy(c->comm);
    c->comm = nullptr;
  }
  c->nranks = nranks;
  c->rank = rank;
  if (nranks == 1) return;
  ncclUniqueId uid;
  static_assert(sizeof(uid.internal) == 128, "nccl id size");
  std::memcpy(uid.internal, id, 128);
  CS_NCCL(ncclCommInitRank(&c->comm, nranks, uid, rank));
}

// ------------------------------------------------------------------ problems

namespace {

int64_t stencil_nnz_planes(int kind, int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1) {
  int64_t total = 0;
  for (int64_t z = z0; z < z1; ++z) {
    const int64_t cz = 1 + (z > 0) + (z + 1 < nz);
    if (kind == CS_GEN_POISSON27) {
      const int64_t fx = nx > 1 ? 3 * nx - 2 : 1, fy = ny > 1 ? 3 * ny - 2 : 1;
      total += fx * fy * cz;
    } else {
      total += nx * ny * cz + 2 * ((nx - 1) * ny + nx * (ny - 1));
    }
  }
  return total;
}

void finish_sell(cs_problem* p, int64_t* widths_dev) {
  cs_ctx* c = p->ctx;
  size_t tmp_bytes = 0;
  scan_slice_ptr(widths_dev, p->nslices, p->slice_ptr.as<int64_t>(), nullptr, &tmp_bytes,
                 c->stream);
  DBuf tmp(tmp_bytes);
  scan_slice_ptr(widths_dev, p->nslices, p->slice_ptr.as<int64_t>(), tmp.p, &tmp_bytes, c->stream);
}

int64_t read_i64(cs_ctx* c, const int64_t* dev) {
  int64_t v = 0;
  CS_CUDA(cudaMemcpyAsync(&v, dev, sizeof v, cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  return v;
}

// Convert the freshly assembled explicit SELL-32 into SELL-32P (common.cuh):
// pattern-compressed slices drop their 4 B/slot column stream.
// Constant-diagonal classes over an all-uniform matrix (see CdiaClass): greedy
// left-to-right merge of consecutive slices' tables while the union stays
// <= 32 offsets with one value each; then per-row participation words.
void build_cdia(cs_problem* p) {
  cs_ctx* c = p->ctx;
  p->cdia.clear();
  p->pbits.release();
  const int64_t ns = p->nslices;
  const char* env = std::getenv("CS_SELL_CDIA");
  if (ns == 0 || p->uniform_slices != ns || (env && std::atoi(env) == 0)) return;
  std::vector<int64_t> meta(ns);
  std::vector<int2> pat(p->table_entries);
  std::vector<double> pval(p->table_entries);
  std::vector<int64_t> pkey(p->table_entries);
  CS_CUDA(cudaMemcpyAsync(meta.data(), p->meta.p, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost,
                          c->stream));
  CS_CUDA(cudaMemcpyAsync(pat.data(), p->pat.p, sizeof(int2) * pat.size(), cudaMemcpyDeviceToHost,
                          c->stream));
  CS_CUDA(cudaMemcpyAsync(pval.data(), p->pval.p, sizeof(double) * pval.size(),
                          cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaMemcpyAsync(pkey.data(), p->pkey.p, sizeof(int64_t) * pkey.size(),
                          cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  constexpr int kMaxClasses = 64;
  // class entries (global key, local offset, value), kept in key order = the
  // stored order of every row (rows are ascending in global columns)
  struct Ent {
    int64_t key;
    int off;
    double v;
  };
  std::vector<CdiaClass> cls;
  std::vector<std::vector<int64_t>> cls_keys;
  std::vector<Ent> cur;
  int64_t s0 = 0, last_tab = -1;
  auto flush = [&](int64_t s1) {
    CdiaClass k{};
    k.s0 = s0;
    k.s1 = s1;
    k.t.n = static_cast<int>(cur.size());
    std::vector<int64_t> keys;
    for (size_t j = 0; j < cur.size(); ++j) {
      k.t.off[j] = cur[j].off;
      k.t.v[j] = cur[j].v;
      keys.push_back(cur[j].key);
    }
    cls.push_back(k);
    cls_keys.push_back(keys);
  };
  const char* split_env = std::getenv("CS_CDIA_SPLIT");  // diagnostics: forced class break
  const int64_t split_at = split_env ? std::atoll(split_env) : -1;
  for (int64_t sl = 0; sl < ns; ++sl) {
    const int64_t ti = pat_index(meta[sl]);
    if (sl == split_at && sl > s0) {
      flush(sl);
      s0 = sl;
      cur.clear();
      last_tab = -1;
    }
    if (ti == last_tab) continue;  // same table as the previous slice
    const int U = pat_uniform(meta[sl]);
    std::vector<Ent> merged = cur;
    bool ok = true;
    for (int k = 0; k < U && ok; ++k) {
      const Ent e{pkey[ti + k], pat[ti + k].x, pval[ti + k]};
      auto it = std::lower_bound(merged.begin(), merged.end(), e,
                                 [](const Ent& a, const Ent& b) { return a.key < b.key; });
      if (it != merged.end() && it->key == e.key) {  // same entry: same offset, same value bits
        if (it->off != e.off || std::memcmp(&it->v, &e.v, sizeof e.v) != 0) ok = false;
      } else {
        merged.insert(it, e);
      }
    }
    if (ok && merged.size() <= static_cast<size_t>(kCdiaMax)) {
      cur.swap(merged);
    } else {
      if (U > kCdiaMax) return;  // one table alone does not fit
      flush(sl);
      if (static_cast<int>(cls.size()) >= kMaxClasses) return;
      s0 = sl;
      cur.clear();
      for (int k = 0; k < U; ++k) cur.push_back({pkey[ti + k], pat[ti + k].x, pval[ti + k]});
    }
    last_tab = ti;
  }
  flush(ns);
  // participation words on the device
  std::vector<int64_t> starts(cls.size());
  std::vector<int64_t> keys(cls.size() * kCdiaMax, INT64_MIN);
  std::vector<int32_t> nofs(cls.size());
  for (size_t k = 0; k < cls.size(); ++k) {
    starts[k] = cls[k].s0;
    nofs[k] = cls[k].t.n;
    for (int j = 0; j < cls[k].t.n; ++j) keys[k * kCdiaMax + j] = cls_keys[k][j];
  }
  DBuf d_starts(sizeof(int64_t) * starts.size()), d_keys(sizeof(int64_t) * keys.size()),
      d_n(sizeof(int32_t) * nofs.size());
  CS_CUDA(cudaMemcpyAsync(d_starts.p, starts.data(), d_starts.bytes, cudaMemcpyHostToDevice,
                          c->stream));
  CS_CUDA(cudaMemcpyAsync(d_keys.p, keys.data(), d_keys.bytes, cudaMemcpyHostToDevice, c->stream));
  CS_CUDA(cudaMemcpyAsync(d_n.p, nofs.data(), d_n.bytes, cudaMemcpyHostToDevice, c->stream));
  p->pbits.alloc(sizeof(uint32_t) * ns * kSliceRows);
  DBuf flags(sizeof(int) * (1 + cls.size()));
  CS_CUDA(cudaMemsetAsync(flags.p, 0, flags.bytes, c->stream));
  launch_cdia_bits(ns, p->n_local, static_cast<int>(cls.size()), d_starts.as<int64_t>(),
                   d_keys.as<int64_t>(), d_n.as<int32_t>(), p->meta.as<int64_t>(),
                   p->pkey.as<int64_t>(), p->pat.as<int2>(), p->pbits.as<uint32_t>(),
                   flags.as<int>(), flags.as<int>() + 1, c->stream);
  std::vector<int> hf(1 + cls.size());
  CS_CUDA(cudaMemcpyAsync(hf.data(), flags.p, flags.bytes, cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  if (hf[0]) {
    p->pbits.release();
    return;
  }
  for (size_t k = 0; k < cls.size(); ++k) {  // z-blocking structure (sell_zb_kernel)
    const CdiaTable& t = cls[k].t;
    cls[k].zstride = 0;
    if (t.n != 27) continue;
    const int64_t P = static_cast<int64_t>(t.off[9]) - t.off[0];
    bool box = P > 0;
    for (int i = 0; i < 9 && box; ++i)
      box = static_cast<int64_t>(t.off[9 + i]) - t.off[i] == P &&
            static_cast<int64_t>(t.off[18 + i]) - t.off[9 + i] == P;
    // measured (tools/spmv_micro.py, 240^3..272^3): pairing two planes per lane pays
    // only where the plane stride is a power of two -- there the three planes of
    // a row's neighbours alias in L1 and the row-wise kernel loses ~10%;
    // elsewhere the row-wise kernel is ~7% faster
    if (box && P % kSliceRows == 0 && (P & (P - 1)) == 0) cls[k].zstride = P;
    cls[k].boxP = cls[k].boxL = 0;
    const int64_t L = static_cast<int64_t>(t.off[3]) - t.off[0];
    bool box3 = box && L >= 3 && P >= 3 * L && P % 4 == 0 && t.off[13] == 0;
    for (int g = 0; g < 3 && box3; ++g)
      for (int i = 0; i < 3 && box3; ++i)
        for (int j = 0; j < 3 && box3; ++j)
          box3 = t.off[9 * g + 3 * i + j] == g * P + i * L + j - (P + L + 1);
    if (box3) {
      cls[k].boxP = P;
      cls[k].boxL = L;
    }
  }
  {  // geometric participation of the box classes (separable fast SpMV)
    DBuf geo(sizeof(int) * std::max<size_t>(cls.size(), 1));
    CS_CUDA(cudaMemsetAsync(geo.p, 0, geo.bytes, c->stream));
    for (size_t k = 0; k < cls.size(); ++k)
      if (cls[k].boxL > 0)
        launch_cdia_geo_check(p->pbits.as<uint32_t>(), cls[k].s0 * kSliceRows,
                              std::min(cls[k].s1 * kSliceRows, p->n_local), cls[k].boxP,
                              geo.as<int>() + k, c->stream);
    std::vector<int> hg(cls.size());
    CS_CUDA(cudaMemcpyAsync(hg.data(), geo.p, sizeof(int) * cls.size(), cudaMemcpyDeviceToHost,
                            c->stream));
    CS_CUDA(cudaStreamSynchronize(c->stream));
    for (size_t k = 0; k < cls.size(); ++k) {
      cls[k].geo = cls[k].boxL > 0 && (hg[k] & 1) == 0;
      cls[k].zuni = cls[k].geo && (hg[k] & 2) == 0;
      if (!cls[k].zuni) continue;
      const int64_t r0 = cls[k].s0 * kSliceRows, r1 = std::min(cls[k].s1 * kSliceRows, p->n_local);
      const int64_t last = r0 + (r1 - r0 - 1) / cls[k].boxP * cls[k].boxP;
      uint32_t w[2];
      CS_CUDA(cudaMemcpyAsync(&w[0], p->pbits.as<uint32_t>() + r0, 4, cudaMemcpyDeviceToHost, c->stream));
      CS_CUDA(cudaMemcpyAsync(&w[1], p->pbits.as<uint32_t>() + last, 4, cudaMemcpyDeviceToHost, c->stream));
      CS_CUDA(cudaStreamSynchronize(c->stream));
      cls[k].zl0 = (w[0] >> 4) & 1u;
      cls[k].zuN = (w[1] >> 22) & 1u;
    }
  }
  for (size_t k = 0; k < cls.size(); ++k) {
    cls[k].t.diag = 0.0;
    if (hf[1 + k]) continue;
    for (int j = 0; j < cls[k].t.n; ++j)
      if (cls_keys[k][j] == 0) cls[k].t.diag = cls[k].t.v[j];
  }
  p->cdia = std::move(cls);
}

void compress_sell(cs_problem* p, int dedupe = 1) {
  cs_ctx* c = p->ctx;
  const int64_t ns = p->nslices;
  const int64_t nn = std::max<int64_t>(ns, 1);
  DBuf cnt(sizeof(int64_t) * 7 * nn);
  DBuf ptrs(sizeof(int64_t) * 4 * (ns + 1));
  DBuf keys(sizeof(unsigned long long) * 2 * nn), slcs(sizeof(int32_t) * 3 * nn);
  int64_t* val_cnt = cnt.as<int64_t>();
  int64_t* pat_cnt = val_cnt + nn;
  int64_t* col_cnt = pat_cnt + nn;
  int64_t* kind = col_cnt + nn;
  int64_t* tab_cnt = kind + nn;
  int64_t* headpos = tab_cnt + nn;
  int64_t* slice_tab = headpos + nn;
  int64_t* new_ptr = ptrs.as<int64_t>();
  int64_t* pat_ptr = new_ptr + (ns + 1);
  int64_t* col_ptr = pat_ptr + (ns + 1);
  int64_t* tab_ptr = col_ptr + (ns + 1);
  unsigned long long* hash = keys.as<unsigned long long>();
  unsigned long long* hash_sorted = hash + nn;
  int32_t* iota = slcs.as<int32_t>();
  int32_t* slc_sorted = iota + nn;
  int32_t* slice_rep = slc_sorted + nn;
  const ColMap cm{p->row_begin, p->n_local, p->ghost_global.as<int64_t>()};
  launch_compress_plan(ns, p->slice_ptr.as<int64_t>(), p->cols.as<int32_t>(), p->vals.as<double>(),
                       cm, val_cnt, pat_cnt, col_cnt, kind, hash, dedupe, c->stream);
  // uniform tables: sort (hash, slice), one table per group of equal hashes
  launch_iota_i32(ns, iota, c->stream);
  size_t tb = 0, tm = 0, ts = 0;
  scan_slice_ptr(val_cnt, ns, new_ptr, nullptr, &tb, c->stream);
  if (ns > 0) {
    scan_max_i64(headpos, ns, headpos, nullptr, &tm, c->stream);
    sort_tables(hash, hash_sorted, iota, slc_sorted, ns, nullptr, &ts, c->stream);
  }
  DBuf tmp(std::max({tb, tm, ts}));
  if (ns > 0) {
    sort_tables(hash, hash_sorted, iota, slc_sorted, ns, tmp.p, &ts, c->stream);
    launch_table_heads(ns, hash_sorted, slc_sorted, kind, tab_cnt, headpos, c->stream);
    scan_max_i64(headpos, ns, headpos, tmp.p, &tm, c->stream);
  }
  for (int64_t* pair : {val_cnt, pat_cnt, col_cnt, tab_cnt}) {
    int64_t* out = pair == val_cnt ? new_ptr : pair == pat_cnt ? pat_ptr
                 : pair == col_cnt ? col_ptr : tab_ptr;
    if (ns > 0) scan_slice_ptr(pair, ns, out, tmp.p, &tb, c->stream);
    else CS_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), c->stream));
  }
  // tab_ptr is indexed by sorted position: exclusive offsets of the heads
  launch_table_assign(ns, hash_sorted, slc_sorted, headpos, tab_ptr, slice_tab, slice_rep,
                      c->stream);
  const int64_t nval = read_i64(c, new_ptr + ns);
  const int64_t nvpat = read_i64(c, pat_ptr + ns);
  const int64_t ncol = read_i64(c, col_ptr + ns);
  const int64_t ntab = read_i64(c, tab_ptr + ns);
  const int64_t npat = ntab + nvpat;  // [uniform tables | value-pattern slices]
  DBuf nvals(sizeof(double) * std::max<int64_t>(nval, 1));
  DBuf ncols(sizeof(int32_t) * std::max<int64_t>(ncol, 1));
  DBuf npatb(sizeof(int2) * std::max<int64_t>(npat, 1));
  DBuf npval(sizeof(double) * std::max<int64_t>(npat, 1));
  DBuf npkey(sizeof(int64_t) * std::max<int64_t>(npat, 1));
  DBuf nmeta(sizeof(int64_t) * nn);
  launch_compress_fill(ns, p->slice_ptr.as<int64_t>(), p->cols.as<int32_t>(), p->vals.as<double>(),
                       cm, kind, slice_tab, slice_rep, new_ptr, pat_ptr, ntab, col_ptr,
                       nvals.as<double>(), ncols.as<int32_t>(), npatb.as<int2>(),
                       npval.as<double>(), npkey.as<int64_t>(), nmeta.as<int64_t>(), c->stream);
  DBuf bad(sizeof(int));
  CS_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
  launch_compress_verify(ns, p->slice_ptr.as<int64_t>(), p->cols.as<int32_t>(),
                         p->vals.as<double>(), cm, kind, slice_tab, npatb.as<int2>(),
                         npval.as<double>(), npkey.as<int64_t>(), bad.as<int>(), c->stream);
  int hbad = 0;
  CS_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  if (hbad) {
    if (!dedupe) fail(CS_ERR_GENERIC, 0, "SELL-32PU conversion failed verification");
    compress_sell(p, 0);  // hash collision: one table per uniform slice
    return;
  }
  DBuf nptr(sizeof(int64_t) * (ns + 1));
  CS_CUDA(cudaMemcpyAsync(nptr.p, new_ptr, sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToDevice,
                          c->stream));
  int64_t nc = 0, nu = 0, wmax = 0;
  {
    std::vector<int64_t> k(ns), w(ns);
    if (ns) {
      CS_CUDA(cudaMemcpyAsync(k.data(), kind, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost,
                              c->stream));
      CS_CUDA(cudaMemcpyAsync(w.data(), val_cnt, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost,
                              c->stream));
    }
    CS_CUDA(cudaStreamSynchronize(c->stream));
    for (int64_t v : k) {
      nc += (v & 0xff) != 0;
      nu += (v & 0xff) == 2;
    }
    for (int64_t v : w) wmax = std::max(wmax, v / kSliceRows);
  }
  p->vals = std::move(nvals);
  p->cols = std::move(ncols);
  p->pat = std::move(npatb);
  p->pval = std::move(npval);
  p->pkey = std::move(npkey);
  p->meta = std::move(nmeta);
  p->slice_ptr = std::move(nptr);
  p->compressed_slices = nc;
  p->uniform_slices = nu;
  p->pattern_entries = npat;
  p->table_entries = ntab;
  p->max_width = static_cast<int>(wmax);
  build_cdia(p);
}

}  // namespace

cs_problem* problem_generate(cs_ctx* c, int kind, int64_t nx, int64_t ny, int64_t nz,
                             const double* coef) {
  if (kind != CS_GEN_POISSON27 && kind != CS_GEN_STENCIL7)
    fail(CS_ERR_INVALID_ARGUMENT, 0, "unknown generator kind");
  if (nx < 1 || ny < 1 || nz < 1)
    fail(CS_ERR_INVALID_ARGUMENT, 0, "poisson27: grid dimensions must be >= 1");
  constexpr int64_t kMaxN = int64_t{1} << 31;  // problems.cpp:18-20
  if (nx > kMaxN / ny || nx * ny > kMaxN / nz)
    fail(CS_ERR_INVALID_ARGUMENT, 0, "poisson27: grid size overflow");
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  auto p = std::make_unique<cs_problem>();
  p->attach(c);
  p->gen_kind = kind;
  p->nx = nx, p->ny = ny, p->nz = nz;
  const int64_t plane = nx * ny;
  int64_t r0 = 0, r1 = plane * nz;
  if (c->nranks > 1) {
    if (cs_partition_rows(plane * nz, plane, c->nranks, c->rank, &r0, &r1) != CS_OK)
      fail(CS_ERR_INVALID_ARGUMENT, 0, "grid has fewer z-planes than ranks");
  }
  StencilDesc d{kind, nx, ny, nz, r0 / plane, r1 / plane, 1.0, 1.0, 1.0};
  if (coef != nullptr) d.cx = coef[0], d.cy = coef[1], d.cz = coef[2];
  p->n_global = plane * nz;
  p->row_begin = r0;
  p->n_local = r1 - r0;
  p->ghost_lo = d.z0 > 0 ? plane : 0;
  p->ghost_hi = d.z1 < nz ? plane : 0;
  p->send_lo = p->ghost_lo;
  p->send_hi = p->ghost_hi;
  p->n_ghost = p->ghost_lo + p->ghost_hi;
  if (p->n_local + p->n_ghost >= (int64_t{1} << 31))
    fail(CS_ERR_INVALID_ARGUMENT, 0, "rank block exceeds int32 column range");
  p->ld = round_up(p->n_local + p->n_ghost, 32);
  p->nslices = (p->n_local + kSliceRows - 1) / kSliceRows;
  p->nnz_local = stencil_nnz_planes(kind, nx, ny, nz, d.z0, d.z1);
  // interior slices: rows whose stencils stay inside the owned planes
  p->slice_int_begin = p->ghost_lo ? (plane + kSliceRows - 1) / kSliceRows : 0;
  p->slice_int_end = p->ghost_hi ? (p->n_local - plane) / kSliceRows : p->nslices;
  if (p->slice_int_end < p->slice_int_begin) p->slice_int_begin = p->slice_int_end = 0;

  p->slice_ptr.alloc(sizeof(int64_t) * (p->nslices + 1));
  {
    DBuf widths(sizeof(int64_t) * p->nslices);
    launch_stencil_widths(d, p->n_local, p->nslices, widths.as<int64_t>(), c->stream);
    finish_sell(p.get(), widths.as<int64_t>());
  }
  const int64_t total = read_i64(c, p->slice_ptr.as<int64_t>() + p->nslices);
  p->vals.alloc(sizeof(double) * total);
  p->cols.alloc(sizeof(int32_t) * total);
  p->diag.alloc(sizeof(double) * std::max<int64_t>(p->n_local, 1));
  launch_stencil_fill(d, p->n_local, p->nslices, p->slice_ptr.as<int64_t>(), p->vals.as<double>(),
                      p->cols.as<int32_t>(), p->diag.as<double>(), c->stream);
  // ghost global ids: plane z0-1 then plane z1 (the compression's merge keys need them)
  for (int64_t i = 0; i < p->ghost_lo; ++i) p->ghosts_host.push_back(r0 - plane + i);
  for (int64_t i = 0; i < p->ghost_hi; ++i) p->ghosts_host.push_back(r1 + i);
  p->ghost_global.alloc(sizeof(int64_t) * std::max<int64_t>(p->n_ghost, 1));
  if (p->n_ghost)
    CS_CUDA(cudaMemcpyAsync(p->ghost_global.p, p->ghosts_host.data(), sizeof(int64_t) * p->n_ghost,
                            cudaMemcpyHostToDevice, c->stream));
  compress_sell(p.get());
  CS_CUDA(cudaStreamSynchronize(c->stream));
  return p.release();
}

namespace {

// Collective halo plan of a general CSR row block (all ranks call): owner
// ranges by allgather, then every rank tells each owner which of its rows it
// needs (counts, then the global row ids) -- point-to-point over NCCL.
void plan_general_halo(cs_problem* p) {
  cs_ctx* c = p->ctx;
  const int P = c->nranks, me = c->rank;
  p->general_halo = true;
  p->send_off.assign(P + 1, 0);
  p->recv_off.assign(P + 1, 0);
  if (P == 1) {
    if (p->n_ghost) fail(CS_ERR_INVALID_MATRIX, 0, "column index out of range");
    p->send_idx.alloc(8);
    p->send_buf.alloc(8);
    return;
  }
  DBuf ranges(sizeof(int64_t) * 2 * (P + 1));
  const int64_t mine[2] = {p->row_begin, p->row_begin + p->n_local};
  int64_t* dr = ranges.as<int64_t>();
  CS_CUDA(cudaMemcpyAsync(dr + 2 * P, mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
  CS_NCCL(ncclAllGather(dr + 2 * P, dr, 2, ncclInt64, c->comm, c->stream));
  std::vector<int64_t> r(2 * P);
  CS_CUDA(cudaMemcpyAsync(r.data(), dr, sizeof(int64_t) * 2 * P, cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  for (int q = 0; q < P; ++q)
    if (r[2 * q] != (q ? r[2 * q - 1] : 0) || r[2 * q + 1] < r[2 * q])
      fail(CS_ERR_INVALID_ARGUMENT, 0, "row blocks must be contiguous and ordered by rank");
  if (r[2 * P - 1] != p->n_global)
    fail(CS_ERR_INVALID_ARGUMENT, 0, "row blocks must cover all rows");
  // ghosts are sorted, owners own ascending row ranges: one segment per owner
  const std::vector<int64_t>& g = p->ghosts_host;
  for (int q = 0; q < P; ++q) {
    const auto hi = std::lower_bound(g.begin(), g.end(), r[2 * q + 1]);
    p->recv_off[q + 1] = hi - g.begin();
  }
  if (p->recv_off[me + 1] != p->recv_off[me])
    fail(CS_ERR_INVALID_MATRIX, 0, "ghost column inside the owned block");
  std::vector<int64_t> rcnt(P), scnt(P);
  for (int q = 0; q < P; ++q) rcnt[q] = p->recv_off[q + 1] - p->recv_off[q];
  DBuf cnt(sizeof(int64_t) * 2 * P);
  int64_t* dc = cnt.as<int64_t>();
  CS_CUDA(cudaMemcpyAsync(dc, rcnt.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, c->stream));
  CS_NCCL(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    CS_NCCL(ncclSend(dc + q, 1, ncclInt64, q, c->comm, c->stream));
    CS_NCCL(ncclRecv(dc + P + q, 1, ncclInt64, q, c->comm, c->stream));
  }
  CS_NCCL(ncclGroupEnd());
  CS_CUDA(cudaMemcpyAsync(scnt.data(), dc + P, sizeof(int64_t) * P, cudaMemcpyDeviceToHost,
                          c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  scnt[me] = 0;
  for (int q = 0; q < P; ++q) p->send_off[q + 1] = p->send_off[q] + scnt[q];
  const int64_t ns = p->send_off[P], nr = p->recv_off[P];
  DBuf req(sizeof(int64_t) * std::max<int64_t>(nr, 1)), got(sizeof(int64_t) * std::max<int64_t>(ns, 1));
  if (nr)
    CS_CUDA(cudaMemcpyAsync(req.p, g.data(), sizeof(int64_t) * nr, cudaMemcpyHostToDevice,
                            c->stream));
  CS_NCCL(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (rcnt[q]) CS_NCCL(ncclSend(req.as<int64_t>() + p->recv_off[q], rcnt[q], ncclInt64, q, c->comm, c->stream));
    if (scnt[q]) CS_NCCL(ncclRecv(got.as<int64_t>() + p->send_off[q], scnt[q], ncclInt64, q, c->comm, c->stream));
  }
  CS_NCCL(ncclGroupEnd());
  std::vector<int64_t> rows(ns);
  if (ns)
    CS_CUDA(cudaMemcpyAsync(rows.data(), got.p, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost,
                            c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<int32_t> idx(ns);
  for (int64_t k = 0; k < ns; ++k) {
    const int64_t l = rows[k] - p->row_begin;
    if (l < 0 || l >= p->n_local) fail(CS_ERR_GENERIC, 0, "halo request outside the owned block");
    idx[k] = static_cast<int32_t>(l);
  }
  p->send_idx.alloc(sizeof(int32_t) * std::max<int64_t>(ns, 1));
  p->send_buf.alloc(sizeof(double) * std::max<int64_t>(ns, 1));
  if (ns)
    CS_CUDA(cudaMemcpyAsync(p->send_idx.p, idx.data(), sizeof(int32_t) * ns,
                            cudaMemcpyHostToDevice, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
}

// longest run of slices without ghost columns: computed while the halo flies
void interior_range(cs_problem* p) {
  cs_ctx* c = p->ctx;
  p->slice_int_begin = 0;
  p->slice_int_end = p->nslices;
  if (p->n_ghost == 0 || p->nslices == 0) return;
  DBuf flag(static_cast<size_t>(p->nslices));
  launch_slice_ghost_flag(p->n_local, p->nslices, p->slice_ptr.as<int64_t>(), p->cols.as<int32_t>(),
                          flag.as<unsigned char>(), c->stream);
  std::vector<unsigned char> f(p->nslices);
  CS_CUDA(cudaMemcpyAsync(f.data(), flag.p, f.size(), cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  int64_t best_b = 0, best_e = 0;
  for (int64_t s = 0; s < p->nslices;) {
    if (f[s]) {
      ++s;
      continue;
    }
    int64_t e = s;
    while (e < p->nslices && !f[e]) ++e;
    if (e - s > best_e - best_b) best_b = s, best_e = e;
    s = e;
  }
  p->slice_int_begin = best_b;
  p->slice_int_end = best_e;
}

}  // namespace

namespace {
// CS_TRACE=1: per-phase wall times of the CSR upload (stream-synchronised; diagnostics only)
struct UploadTrace {
  cudaStream_t st;
  bool on = std::getenv("CS_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit UploadTrace(cudaStream_t s) : st(s) {}
  void mark(const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cs-trace]   upload %s %.1f ms\n", phase,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};
}  // namespace

// Column/value upload of a CSR row block, streamed: slice-aligned row chunks
// of <= kChunkNnz entries go host -> device on the copy stream through two
// staging buffers while the SELL-32 fill of the previous chunk runs on the
// compute stream. Device memory: 2 chunks instead of the whole int64 CSR
// (58.8 GB at 27-pt 512^3); the host arrays may be pageable (the caller's
// std::vector), each chunk is one cudaMemcpyAsync per array.
// Host copy of `bytes` split over `threads` workers (pageable -> page-locked
// staging: one thread's memcpy reaches ~11 GB/s, the DMA from page-locked
// memory ~55 GB/s).
void parallel_copy(void* dst, const void* src, size_t bytes, int threads) {
  if (threads <= 1 || bytes < (size_t{8} << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t part = (bytes / threads + 4095) & ~size_t{4095};
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) {
    const size_t b0 = t * part;
    if (b0 >= bytes) break;
    const size_t len = std::min(part, bytes - b0);
    pool.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + b0, static_cast<const char*>(src) + b0, len);
    });
  }
  std::memcpy(dst, src, std::min(part, bytes));
  for (auto& th : pool) th.join();
}

int upload_threads() {
  const char* e = std::getenv("CS_UPLOAD_THREADS");
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  return e ? std::max(1, std::atoi(e)) : std::min(hw, 16);
}

// two page-locked staging buffers of `bytes` each, cached on the context
char* host_stage(cs_ctx* c, size_t bytes) {
  if (c->host_stage_bytes < bytes) {
    if (c->host_stage) cudaFreeHost(c->host_stage);
    c->host_stage = nullptr;
    c->host_stage_bytes = 0;
    CS_CUDA(cudaHostAlloc(&c->host_stage, 2 * bytes, cudaHostAllocPortable));
    c->host_stage_bytes = bytes;
  }
  return static_cast<char*>(c->host_stage);
}

// Large host<->device copies of caller (pageable) memory through the context's
// page-locked staging: 64 MB chunks, host threads fill / drain one buffer while
// the DMA of the other runs. Both are ordered on c->stream.
constexpr size_t kStageChunk = size_t{64} << 20;

void h2d_large(cs_ctx* c, void* dev, const void* host, size_t bytes) {
  char* hs = host_stage(c, std::max(c->host_stage_bytes, kStageChunk));
  const size_t chunk = c->host_stage_bytes;
  const int nt = upload_threads();
  cudaEvent_t ev[2];
  for (auto& e : ev) CS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (size_t off = 0, k = 0; off < bytes; off += chunk, ++k) {
    const int b = static_cast<int>(k & 1);
    const size_t len = std::min(chunk, bytes - off);
    if (k >= 2) CS_CUDA(cudaEventSynchronize(ev[b]));
    parallel_copy(hs + b * chunk, static_cast<const char*>(host) + off, len, nt);
    CS_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + off, hs + b * chunk, len,
                            cudaMemcpyHostToDevice, c->stream));
    CS_CUDA(cudaEventRecord(ev[b], c->stream));
  }
  CS_CUDA(cudaStreamSynchronize(c->stream));  // the staging may be reused right after
  for (auto& e : ev) cudaEventDestroy(e);
}

void d2h_large(cs_ctx* c, void* host, const void* dev, size_t bytes) {
  char* hs = host_stage(c, std::max(c->host_stage_bytes, kStageChunk));
  const size_t chunk = c->host_stage_bytes;
  const int nt = upload_threads();
  cudaEvent_t ev[2];
  for (auto& e : ev) CS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const size_t nk = (bytes + chunk - 1) / chunk;
  auto issue = [&](size_t k) {
    const size_t off = k * chunk, len = std::min(chunk, bytes - off);
    CS_CUDA(cudaMemcpyAsync(hs + (k & 1) * chunk, static_cast<const char*>(dev) + off, len,
                            cudaMemcpyDeviceToHost, c->stream));
    CS_CUDA(cudaEventRecord(ev[k & 1], c->stream));
  };
  if (nk) issue(0);
  for (size_t k = 0; k < nk; ++k) {
    CS_CUDA(cudaEventSynchronize(ev[k & 1]));
    if (k + 1 < nk) issue(k + 1);  // the next DMA runs while this chunk drains
    const size_t off = k * chunk, len = std::min(chunk, bytes - off);
    parallel_copy(static_cast<char*>(host) + off, hs + (k & 1) * chunk, len, nt);
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

void stream_csr_fill(cs_problem* p, const int64_t* rowptr, const int64_t* col, const double* val,
                     const int64_t* drp, int* bad) {
  cs_ctx* c = p->ctx;
  const int64_t n = p->n_local;
  if (n == 0) return;
  // staged (default): host threads copy each chunk into page-locked memory while
  // the previous chunk's DMA and SELL fill run; CS_UPLOAD_STAGED=0: one
  // cudaMemcpyAsync per array per chunk straight from the caller's memory
  const char* senv = std::getenv("CS_UPLOAD_STAGED");
  const bool staged = senv == nullptr || std::atoi(senv) != 0;
  const char* env = std::getenv("CS_UPLOAD_CHUNK_NNZ");
  const int64_t kChunkNnz = env ? std::max<int64_t>(std::atoll(env), 1)
                                : (staged ? int64_t{1} << 23 : int64_t{1} << 25);
  std::vector<int64_t> cut{0};
  int64_t most = 0;
  for (int64_t r = 0; r < n;) {
    int64_t e = std::min(n, r + kSliceRows);
    while (e < n && rowptr[std::min(n, e + kSliceRows)] - rowptr[r] <= kChunkNnz)
      e = std::min(n, e + kSliceRows);
    most = std::max(most, rowptr[e] - rowptr[r]);
    cut.push_back(e);
    r = e;
  }
  const size_t cap = static_cast<size_t>(std::max<int64_t>(most, 1));
  DBuf stage[2];
  for (auto& b : stage) b.alloc(16 * cap);
  cudaEvent_t ready, copied[2], filled[2];
  CS_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    CS_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    CS_CUDA(cudaEventCreateWithFlags(&filled[i], cudaEventDisableTiming));
  }
  CS_CUDA(cudaEventRecord(ready, c->stream));  // staging allocations are stream-ordered
  CS_CUDA(cudaStreamWaitEvent(c->comm_stream, ready, 0));
  char* hs = staged ? host_stage(c, 16 * cap) : nullptr;
  const int nthreads = upload_threads();
  for (size_t k = 0; k + 1 < cut.size(); ++k) {
    const int b = static_cast<int>(k & 1);
    const int64_t r0 = cut[k], r1 = cut[k + 1];
    const int64_t e0 = rowptr[r0], cnt = rowptr[r1] - e0;
    int64_t* scol = stage[b].as<int64_t>();
    double* sval = reinterpret_cast<double*>(scol + cap);
    if (k >= 2) CS_CUDA(cudaStreamWaitEvent(c->comm_stream, filled[b], 0));
    if (cnt > 0 && staged) {
      char* hb = hs + static_cast<size_t>(b) * 16 * cap;
      if (k >= 2) CS_CUDA(cudaEventSynchronize(copied[b]));  // its last DMA has drained
      parallel_copy(hb, col + e0, sizeof(int64_t) * cnt, nthreads);
      parallel_copy(hb + 8 * cap, val + e0, sizeof(double) * cnt, nthreads);
      CS_CUDA(cudaMemcpyAsync(scol, hb, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice,
                              c->comm_stream));
      CS_CUDA(cudaMemcpyAsync(sval, hb + 8 * cap, sizeof(double) * cnt, cudaMemcpyHostToDevice,
                              c->comm_stream));
    } else if (cnt > 0) {
      CS_CUDA(cudaMemcpyAsync(scol, col + e0, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice,
                              c->comm_stream));
      CS_CUDA(cudaMemcpyAsync(sval, val + e0, sizeof(double) * cnt, cudaMemcpyHostToDevice,
                              c->comm_stream));
    }
    CS_CUDA(cudaEventRecord(copied[b], c->comm_stream));
    CS_CUDA(cudaStreamWaitEvent(c->stream, copied[b], 0));
    launch_csr_fill(n, p->row_begin, p->n_global, p->ghost_global.as<int64_t>(), p->n_ghost, drp,
                    scol, sval, e0, r0, r1, p->slice_ptr.as<int64_t>(), p->vals.as<double>(),
                    p->cols.as<int32_t>(), p->diag.as<double>(), bad, c->stream);
    CS_CUDA(cudaEventRecord(filled[b], c->stream));
  }
  CS_CUDA(cudaStreamSynchronize(c->stream));
  CS_CUDA(cudaStreamSynchronize(c->comm_stream));
  cudaEventDestroy(ready);
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(filled[i]);
  }
}

cs_problem* problem_upload_block(cs_ctx* c, int64_t n_global, int64_t row_begin, int64_t row_end,
                                 const int64_t* rowptr, const int64_t* col, const double* val) {
  if (n_global < 0 || row_begin < 0 || row_end < row_begin || row_end > n_global)
    fail(CS_ERR_DIMENSION, 0, "bad row block");
  if (c->nranks == 1 && (row_begin != 0 || row_end != n_global))
    fail(CS_ERR_INVALID_ARGUMENT, 0, "single rank must own every row");
  const int64_t n = row_end - row_begin;
  if (rowptr[0] != 0) fail(CS_ERR_INVALID_MATRIX, 0, "row_offsets[0] must be 0");
  const int64_t nnz = rowptr[n];
  if (nnz < 0) fail(CS_ERR_INVALID_MATRIX, 0, "row_offsets[n] must equal nnz");
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  NvtxRange nvtx_("cs:upload CSR (streamed) + SELL/CDIA conversion");
  UploadTrace ut(c->stream);
  auto p = std::make_unique<cs_problem>();
  p->attach(c);
  p->n_global = n_global;
  p->row_begin = row_begin;
  p->n_local = n;
  if (c->nranks > 1) {
    // sorted unique off-block columns (partition.cpp numbering)
    std::vector<int64_t>& g = p->ghosts_host;
    for (int64_t k = 0; k < nnz; ++k)
      if (col[k] < row_begin || col[k] >= row_end)
        if (col[k] >= 0 && col[k] < n_global) g.push_back(col[k]);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
  }
  p->n_ghost = static_cast<int64_t>(p->ghosts_host.size());
  if (n + p->n_ghost >= (int64_t{1} << 31))
    fail(CS_ERR_INVALID_ARGUMENT, 0, "rank block exceeds int32 column range");
  p->ld = round_up(std::max<int64_t>(n + p->n_ghost, 1), 32);
  p->nslices = (n + kSliceRows - 1) / kSliceRows;
  p->nnz_local = nnz;
  p->ghost_global.alloc(sizeof(int64_t) * std::max<int64_t>(p->n_ghost, 1));
  if (p->n_ghost)
    CS_CUDA(cudaMemcpyAsync(p->ghost_global.p, p->ghosts_host.data(), sizeof(int64_t) * p->n_ghost,
                            cudaMemcpyHostToDevice, c->stream));
  // rowptr first: the slice widths validate it on the device before any
  // column/value byte moves
  DBuf drp(sizeof(int64_t) * (n + 1)), bad(sizeof(int));
  CS_CUDA(cudaMemcpyAsync(drp.p, rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice,
                          c->stream));
  CS_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
  p->slice_ptr.alloc(sizeof(int64_t) * (p->nslices + 1));
  if (p->nslices > 0) {
    DBuf widths(sizeof(int64_t) * p->nslices);
    launch_csr_widths(n, drp.as<int64_t>(), p->nslices, widths.as<int64_t>(), bad.as<int>(),
                      c->stream);
    finish_sell(p.get(), widths.as<int64_t>());
  } else {
    CS_CUDA(cudaMemsetAsync(p->slice_ptr.p, 0, sizeof(int64_t), c->stream));
  }
  int hbad = 0;
  CS_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  const int64_t total = read_i64(c, p->slice_ptr.as<int64_t>() + p->nslices);
  ut.mark("rowptr h2d+widths");
  // a local validation failure must not leave peers waiting in the halo plan
  int local_err = hbad ? 1 : 0;
  if (!local_err) {
    p->vals.alloc(sizeof(double) * std::max<int64_t>(total, 1));
    p->cols.alloc(sizeof(int32_t) * std::max<int64_t>(total, 1));
    p->diag.alloc(sizeof(double) * std::max<int64_t>(n, 1));
    stream_csr_fill(p.get(), rowptr, col, val, drp.as<int64_t>(), bad.as<int>());
    CS_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CS_CUDA(cudaStreamSynchronize(c->stream));
    ut.mark("col/val h2d+fill (streamed)");
    local_err = hbad ? 2 : 0;
  }
  if (c->nranks > 1) {
    // agree on failure before any point-to-point traffic
    DBuf e(sizeof(int));
    CS_CUDA(cudaMemcpyAsync(e.p, &local_err, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CS_NCCL(ncclAllReduce(e.p, e.p, 1, ncclInt32, ncclMax, c->comm, c->stream));
    int any = 0;
    CS_CUDA(cudaMemcpyAsync(&any, e.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CS_CUDA(cudaStreamSynchronize(c->stream));
    if (any && !local_err) fail(CS_ERR_INVALID_MATRIX, 0, "invalid row block on another rank");
  }
  if (local_err == 1) fail(CS_ERR_INVALID_MATRIX, 0, "row_offsets must be nondecreasing");
  if (local_err == 2) fail(CS_ERR_INVALID_MATRIX, 0, "column index out of range");
  interior_range(p.get());
  plan_general_halo(p.get());
  ut.mark("halo plan");
  compress_sell(p.get());
  ut.mark("compress");
  return p.release();
}

cs_problem* problem_upload_csr(cs_ctx* c, int64_t n, const int64_t* rowptr, const int64_t* col,
                               const double* val) {
  if (c->nranks > 1)
    fail(CS_ERR_INVALID_ARGUMENT, 0,
         "CSR upload of a whole matrix is single-rank; use cs_problem_upload_csr_block for P>1");
  if (n < 0) fail(CS_ERR_DIMENSION, 0, "negative dimension");
  if (n >= (int64_t{1} << 31)) fail(CS_ERR_INVALID_ARGUMENT, 0, "n exceeds int32 column range");
  return problem_upload_block(c, n, 0, n, rowptr, col, val);
}

// Block Jacobi: the caller's dense diagonal blocks are uploaded
// and factorised on the device; apply = two triangular solves per block.
void problem_set_precond_block_jacobi(cs_problem* p, int bs, const double* blocks) {
  cs_ctx* c = p->ctx;
  if (bs < 1 || bs > 16) fail(CS_ERR_INVALID_ARGUMENT, 0, "block_jacobi: bs must be in [1, 16]");
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  const int64_t nb = (p->n_local + bs - 1) / bs;
  const size_t bytes = sizeof(double) * static_cast<size_t>(nb) * bs * bs;
  DBuf f(std::max<size_t>(bytes, 8)), bad(sizeof(int));
  if (bytes)
    CS_CUDA(cudaMemcpyAsync(f.p, blocks, bytes, cudaMemcpyHostToDevice, c->stream));
  const int big = INT_MAX;
  CS_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  {
    Launch L(c, CS_PHASE_OTHER);
    launch_bj_factor(nb, bs, f.as<double>(), bad.as<int>(), c->stream);
  }
  int hbad = big;
  CS_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  if (hbad != big)
    fail(CS_ERR_NOT_SPD, hbad,
         "block_jacobi: diagonal block " + std::to_string(hbad) + " is not positive definite");
  p->pc_factor = std::move(f);
  p->pc_bs = bs;
  p->pc_fn = nullptr;
  p->precond = CS_PRECOND_BLOCK_JACOBI;
}

void problem_set_precond_fn(cs_problem* p, cs_precond_fn fn, void* user) {
  if (fn == nullptr) fail(CS_ERR_INVALID_ARGUMENT, 0, "precond fn must not be NULL");
  p->pc_fn = fn;
  p->pc_user = user;
  p->pc_factor.release();
  p->pc_bs = 0;
  p->precond = CS_PRECOND_DEVICE_FN;
}

// out = M^-1 in on the context stream for every preconditioner kind, with the
// basis-breakdown check of column `col` (col < 0: none; pending: record in
// st->pending, the fast algebra's speculative MPK). The caller accounts the
// launch (Launch scope).
void precond_apply(cs_problem* p, const double* in, double* out, DevState* st, int col,
                   int pending) {
  cs_ctx* c = p->ctx;
  const int64_t n = p->n_local;
  switch (p->precond) {
    case CS_PRECOND_BLOCK_JACOBI:
      launch_bj_apply(n, p->pc_bs, p->pc_factor.as<double>(), in, out, st, col, pending,
                      c->stream);
      return;
    case CS_PRECOND_DEVICE_FN:
      if (p->pc_fn(p->pc_user, in, out, n, c->stream) != 0)
        fail(CS_ERR_GENERIC, 0, "device preconditioner apply failed");
      CS_CUDA(cudaGetLastError());
      if (col >= 0) launch_precond_apply(n, nullptr, out, out, st, col, pending, c->stream);
      return;
    default:
      launch_precond_apply(n, p->view().inv_diag, in, out, st, col, pending, c->stream);
  }
}

void problem_set_precond(cs_problem* p, int kind) {
  cs_ctx* c = p->ctx;
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  if (kind == CS_PRECOND_IDENTITY) {
    p->precond = kind;
    return;
  }
  if (kind == CS_PRECOND_BLOCK_JACOBI || kind == CS_PRECOND_DEVICE_FN)
    fail(CS_ERR_INVALID_ARGUMENT, 0,
         "set the block-Jacobi / device preconditioner with its own entry point");
  if (kind != CS_PRECOND_JACOBI) fail(CS_ERR_INVALID_ARGUMENT, 0, "unknown preconditioner");
  if (!p->inv_diag.p) p->inv_diag.alloc(sizeof(double) * std::max<int64_t>(p->n_local, 1));
  DBuf bad(sizeof(int));
  CS_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
  {
    Launch L(c, CS_PHASE_OTHER);
    launch_inv_diag(p->n_local, p->diag.as<double>(), p->inv_diag.as<double>(), bad.as<int>(),
                    c->stream);
  }
  int hbad = 0;
  CS_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  if (hbad) fail(CS_ERR_NOT_SPD, 0, "jacobi: diagonal must be strictly positive");
  p->precond = kind;
}

void problem_download_csr(cs_problem* p, int64_t* rowptr, int64_t* col, double* val) {
  cs_ctx* c = p->ctx;
  CS_CUDA(cudaSetDevice(c->device));
  StreamBind bind_stream_(c->stream);
  const int64_t n = p->n_local;
  DBuf len(sizeof(int64_t) * std::max<int64_t>(n, 1)), rp(sizeof(int64_t) * (n + 1));
  const SellView A = p->view();
  if (n > 0) {
    launch_sell_row_len(A, len.as<int64_t>(), c->stream);
    size_t tb = 0;
    scan_rowptr(len.as<int64_t>(), n, rp.as<int64_t>(), nullptr, &tb, c->stream);
    DBuf tmp(tb);
    scan_rowptr(len.as<int64_t>(), n, rp.as<int64_t>(), tmp.p, &tb, c->stream);
  } else {
    CS_CUDA(cudaMemsetAsync(rp.p, 0, sizeof(int64_t), c->stream));
  }
  CS_CUDA(cudaMemcpyAsync(rowptr, rp.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, c->stream));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t nnz = rowptr[n];
  if (nnz == 0) return;
  // slice-aligned row chunks of <= 32M entries through two device stages: the
  // conversion of chunk k+1 overlaps the download of chunk k, and device memory
  // stays at 2 chunks (the whole int64 CSR is 58.8 GB at 27-pt 512^3)
  constexpr int64_t kChunk = int64_t{1} << 25;
  std::vector<int64_t> cut{0};
  int64_t most = 0;
  for (int64_t r = 0; r < n;) {
    int64_t e = std::min(n, r + kSliceRows);
    while (e < n && rowptr[std::min(n, e + kSliceRows)] - rowptr[r] <= kChunk)
      e = std::min(n, e + kSliceRows);
    most = std::max(most, rowptr[e] - rowptr[r]);
    cut.push_back(e);
    r = e;
  }
  const size_t cap = static_cast<size_t>(std::max<int64_t>(most, 1));
  DBuf stage[2];
  for (auto& b : stage) b.alloc(16 * cap);
  cudaEvent_t conv[2], dl[2];
  for (int i = 0; i < 2; ++i) {
    CS_CUDA(cudaEventCreateWithFlags(&conv[i], cudaEventDisableTiming));
    CS_CUDA(cudaEventCreateWithFlags(&dl[i], cudaEventDisableTiming));
  }
  const size_t nk = cut.size() - 1;
  auto stage_ptr = [&](size_t k) { return stage[k & 1].as<int64_t>(); };
  auto convert = [&](size_t k) {
    const int b = static_cast<int>(k & 1);
    if (k >= 2) CS_CUDA(cudaStreamWaitEvent(c->stream, dl[b], 0));  // stage's last download
    int64_t* dc = stage_ptr(k);
    launch_sell_to_csr(A, p->row_begin, p->ghost_global.as<int64_t>(), rp.as<int64_t>(), dc,
                       reinterpret_cast<double*>(dc + cap), cut[k], cut[k + 1], rowptr[cut[k]],
                       c->stream);
    CS_CUDA(cudaEventRecord(conv[b], c->stream));
  };
  // software pipeline: chunk k+1 converts on the GPU while the host drains chunk
  // k (a copy into pageable memory returns when it has landed)
  convert(0);
  for (size_t k = 0; k < nk; ++k) {
    if (k + 1 < nk) convert(k + 1);
    const int b = static_cast<int>(k & 1);
    const int64_t e0 = rowptr[cut[k]], cnt = rowptr[cut[k + 1]] - e0;
    CS_CUDA(cudaStreamWaitEvent(c->comm_stream, conv[b], 0));
    if (cnt) {
      int64_t* dc = stage_ptr(k);
      CS_CUDA(cudaMemcpyAsync(col + e0, dc, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost,
                              c->comm_stream));
      CS_CUDA(cudaMemcpyAsync(val + e0, reinterpret_cast<double*>(dc + cap), sizeof(double) * cnt,
                              cudaMemcpyDeviceToHost, c->comm_stream));
    }
    CS_CUDA(cudaEventRecord(dl[b], c->comm_stream));
  }
  CS_CUDA(cudaStreamSynchronize(c->comm_stream));
  CS_CUDA(cudaStreamWaitEvent(c->stream, dl[0], 0));  // the stages are freed on c->stream
  CS_CUDA(cudaStreamWaitEvent(c->stream, dl[1], 0));
  CS_CUDA(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(conv[i]);
    cudaEventDestroy(dl[i]);
  }
}

}  // namespace csg
