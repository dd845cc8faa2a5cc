// runtime.cuh -- host-side runtime objects behind the C ABI: device context
// (streams, NCCL communicator, per-phase CUDA-event timing, launch counts),
// device-resident problems (SELL matrix + preconditioner + halo layout) and
// the cached per-problem solve workspace.
#pragma once
#include <atomic>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <array>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "chebstep_gpu.h"
#include "common.cuh"
#include "kernels.cuh"
#include "lanczos.cuh"

namespace csg {

// Stream the current library call allocates on (set by bind_stream for the
// duration of a context/problem operation). With a stream bound, buffers come
// from the device's stream-ordered memory pool (cudaMallocAsync), which the
// context configures to retain freed memory -- so repeated solves/uploads reuse
// HBM instead of cudaMalloc/cudaFree-ing tens of GB per call.
extern thread_local cudaStream_t g_alloc_stream;
struct StreamBind {
  cudaStream_t prev;
  explicit StreamBind(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
  ~StreamBind() { g_alloc_stream = prev; }
};

// RAII device buffer
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;  // allocation stream (pool) or nullptr (cudaMalloc)
  bool pooled = false;
  DBuf() = default;
  explicit DBuf(size_t b) { alloc(b); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes), stream(o.stream), pooled(o.pooled) {
    o.p = nullptr, o.bytes = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, bytes = o.bytes, stream = o.stream, pooled = o.pooled;
      o.p = nullptr, o.bytes = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t b) {
    release();
    if (b == 0) b = 8;
    if (g_alloc_stream != nullptr) {
      CS_CUDA(cudaMallocAsync(&p, b, g_alloc_stream));
      stream = g_alloc_stream;
      pooled = true;
    } else {
      CS_CUDA(cudaMalloc(&p, b));
      pooled = false;
    }
    bytes = b;
  }
  void release() {
    if (p) {
      if (pooled) cudaFreeAsync(p, stream);
      else cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct TimedSpan {
  int phase;
  cudaEvent_t a, b;
};

}  // namespace csg

struct cs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;       // compute
  cudaStream_t comm_stream = nullptr;  // halo exchange
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  // multi-GPU
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // accounting
  int64_t launches = 0;
  std::array<int64_t, CS_NUM_PHASES> phase_launches{};
  std::array<double, CS_NUM_PHASES> phase_ms{};
  bool timing = false;
  std::vector<csg::TimedSpan> spans;
  std::vector<cudaEvent_t> event_pool;
  int64_t allreduces = 0;
  std::atomic<int> live_problems{0};  // problems created on this context, not yet destroyed
  // scratch
  csg::DBuf state;      // DevState
  csg::DBuf scratch;    // partials / tickets / scalars
  csg::DBuf normbuf;    // ||b|| reduction scratch
  // Lanczos basis (2 x steps vectors + 3) of the last estimate, reused by every
  // problem of this context (one solve at a time): 86 GB at 512^3, so a fresh
  // problem per call (the reference-signature entry) must not re-map it
  csg::DBuf lz;
  size_t scratch_bytes = 0;
  void* pinned = nullptr;  // pinned host staging for flags
  void* host_stage = nullptr;    // 2 x host_stage_bytes page-locked upload staging
  size_t host_stage_bytes = 0;
  unsigned char uuid[16] = {};
  bool uuid_known = false;
};

struct cs_problem {
  cs_ctx* ctx = nullptr;
  // every problem is counted on its context from creation to destruction: its
  // pooled buffers are freed on the context's stream (see ctx_destroy)
  void attach(cs_ctx* c) {
    ctx = c;
    ++c->live_problems;
  }
  cs_problem() = default;
  cs_problem(const cs_problem&) = delete;
  cs_problem& operator=(const cs_problem&) = delete;
  ~cs_problem() {
    if (ctx) --ctx->live_problems;
  }
  int64_t n_global = 0, row_begin = 0, n_local = 0, n_ghost = 0, ld = 0, nnz_local = 0;
  int64_t nslices = 0;
  int64_t slice_int_begin = 0, slice_int_end = 0;  // interior slices (no ghost columns)
  // halo: ghosts = [lower plane (from rank-1) | upper plane (from rank+1)]
  int64_t ghost_lo = 0, ghost_hi = 0, send_lo = 0, send_hi = 0;
  // general CSR blocks: ghosts grouped by owner rank (ascending global order);
  // peer q receives x[send_idx[send_off[q] .. send_off[q+1])] and sends its
  // rows into ghost slots [recv_off[q], recv_off[q+1])
  bool general_halo = false;
  std::vector<int64_t> send_off, recv_off;  // nranks + 1 each
  csg::DBuf send_idx, send_buf;
  bool has_halo() const {
    if (!general_halo) return ghost_lo > 0 || ghost_hi > 0;
    return send_off.back() > 0 || recv_off.back() > 0;
  }
  int gen_kind = -1;
  int64_t nx = 0, ny = 0, nz = 0;
  csg::DBuf slice_ptr, vals, cols, meta, pat, pval, pkey, pbits, diag, inv_diag, ghost_global;
  std::vector<csg::CdiaClass> cdia;
  int64_t compressed_slices = 0, uniform_slices = 0, pattern_entries = 0, table_entries = 0;
  int max_width = 0;
  std::vector<int64_t> ghosts_host;
  int precond = CS_PRECOND_IDENTITY;
  // general (non-diagonal) preconditioners, SURVEY 8f4
  int pc_bs = 0;              // block Jacobi: rows per block
  csg::DBuf pc_factor;        // block Jacobi: Cholesky factors, bs*bs per block
  cs_precond_fn pc_fn = nullptr;
  void* pc_user = nullptr;
  bool precond_general() const {
    return precond == CS_PRECOND_BLOCK_JACOBI || precond == CS_PRECOND_DEVICE_FN;
  }
  // cached solve workspace and Lanczos basis (reused across solves)
  int ws_s = -1;
  uint64_t ws_gen = 0;  // bumped whenever ws is (re)allocated
  csg::DBuf ws;
  // NVLink peer-memory halo of the fast MPK (z-slab problems):
  // the neighbours' workspaces and receive counters mapped by CUDA IPC
  struct PeerMap {
    uint64_t gen = 0;               // peer ws generation of the mapping
    void* ws = nullptr;             // mapped peer workspace base
    void* sig = nullptr;            // mapped peer receive counters
    int64_t ghost_off = 0;          // element offset of my plane in the peer's Z column 0
    int64_t ld = 0;                 // peer column stride (elements)
  };
  PeerMap peer[2];                  // [rank-1, rank+1]
  csg::DBuf sig;                    // my receive counters [from rank-1, from rank+1] (IPC-exported)
  int64_t z_off = 0;                // element offset of Z in ws
  bool p2p = false;                 // peer mappings valid for the current ws
  uint64_t ipc_gen = 0;             // ws generation of ipc_ws
  cudaIpcMemHandle_t ipc_ws{}, ipc_sig{};
  unsigned long long p2p_epoch = 0; // halo exchanges consumed in the current solve
  bool p2p_pending = false;         // the last kernel pushed rows not yet released
  // fused NVLink allreduce of the packed block (csg::XredArgs): my exchange
  // buffer [2][nranks][kXredSlot] doubles + [nranks] flags, every rank's mapped
  csg::DBuf xred;
  cudaIpcMemHandle_t ipc_xred{};
  bool xred_exported = false;
  void* xpeer[csg::kXredMaxRanks] = {};
  bool xred_ok = false;
  unsigned long long xred_epoch = 0;
  csg::SellView view() const {
    csg::SellView v;
    v.n_local = n_local;
    v.nslices = nslices;
    v.slice_ptr = slice_ptr.as<int64_t>();
    v.vals = vals.as<double>();
    v.cols = cols.as<int32_t>();
    v.meta = meta.as<int64_t>();
    v.pat = pat.as<int2>();
    v.pval = pval.as<double>();
    v.uniform = uniform_slices > 0;
    v.uniform_all = uniform_slices == nslices && nslices > 0;
    v.table_entries = table_entries;
    v.pbits = cdia.empty() ? nullptr : pbits.as<uint32_t>();
    v.cdia = cdia.data();
    v.ncdia = static_cast<int>(cdia.size());
    v.max_width = max_width;
    v.xlen = (n_local + n_ghost + 1) / 2 * 2;
    v.inv_diag = precond == CS_PRECOND_JACOBI ? inv_diag.as<double>() : nullptr;
    return v;
  }
};

namespace csg {

// launch accounting + optional CUDA-event timing of every kernel
// NVTX range for Nsight timelines (header-only NVTX v3: no link dependency,
// a no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Launch {
  cs_ctx* c;
  int phase;
  cudaEvent_t a = nullptr;
  Launch(cs_ctx* ctx, int ph);
  ~Launch();
};
cudaEvent_t pooled_event(cs_ctx* c);
void collect_timing(cs_ctx* c);

// SpMV with halo exchange (interior rows overlap the transfer)
void spmv_halo(cs_problem* p, int kind, SpmvArgs g, double* operand_col);
void halo_exchange(cs_problem* p, double* col);
void allreduce_sum(cs_ctx* c, double* dev, size_t count);
// large pageable host <-> device copies through page-locked staging (host
// threads + DMA overlapped); complete when they return
void h2d_large(cs_ctx* c, void* dev, const void* host, size_t bytes);
void d2h_large(cs_ctx* c, void* host, const void* dev, size_t bytes);
// out = M^-1 in for every preconditioner kind (+ the breakdown check of column
// col >= 0, recorded as pending when `pending`); general kinds: block Jacobi,
// device plugin
void precond_apply(cs_problem* p, const double* in, double* out, DevState* st, int col,
                   int pending);
void problem_set_precond_block_jacobi(cs_problem* p, int bs, const double* blocks);
void problem_set_precond_fn(cs_problem* p, cs_precond_fn fn, void* user);
// NVLink halo: map the neighbours' workspaces (collective over the communicator;
// every rank calls it once per solve after its workspace is final). Returns
// whether the peer-memory path is on for this solve (all ranks agree).
bool p2p_setup(cs_problem* p, double* Z);
// arguments of the fused allreduce for the next pack (advances the epoch)
csg::XredArgs xred_next(cs_problem* p, int npack);
void p2p_teardown(cs_problem* p);
// SpMV of the fast MPK through the peer-memory halo: interior slices, then the
// boundary slices after this exchange's ghost planes arrived; push_col (or
// nullptr) is the Z column whose boundary rows the epilogue pushes.
void spmv_p2p(cs_problem* p, int kind, SpmvArgs g, int push_col);
// push Z column `col`'s boundary rows (the z_0 halo after the update pass)
void p2p_push(cs_problem* p, const double* src, int col, DevState* st);
// the push arguments of Z column `col` (diagnostics)
void fill_push_args(const cs_problem* p, SpmvArgs& g, int col);
// scratch region of the context, grown on demand
void* ctx_scratch(cs_ctx* c, size_t bytes);

// solver entry points (solver.cu)
void estimate_interval_dev(cs_problem* p, int steps, uint64_t seed, int mode, double* lo,
                           double* hi, double* t_ms);
void pcgs_solve_dev(cs_problem* p, const double* b, const double* x0, const cs_config& cfg,
                    double* x, cs_report* rep);
void mpk_unit(cs_problem* p, double* Z, double* P, double* r, double* zpA, double* zpB, int s,
              double lo, double hi, DevState* st);
void pcg_solve_dev(cs_problem* p, const double* b, const double* x0, double tol, int max_iter,
                   int mode, double* x, cs_report* rep, const cs_config* hooks = nullptr);

// error helpers
[[noreturn]] void fail(int code, int payload, const std::string& msg);
std::string format_device_error(unsigned long long word, int s);

}  // namespace csg
