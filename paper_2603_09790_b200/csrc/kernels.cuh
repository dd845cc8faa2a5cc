// kernels.cuh -- host launchers of every device kernel (internal interface).
#pragma once
#include "common.cuh"

namespace csg {

// ------------------------------------------------------------------ problems (sell.cu)
struct StencilDesc {
  int kind;  // CS_GEN_*
  int64_t nx, ny, nz;
  int64_t z0, z1;  // owned z-planes [z0, z1)
  double cx, cy, cz;
};
// Per-slice widths of a generated slab (analytic row lengths), then fill.
void launch_stencil_widths(const StencilDesc& d, int64_t n_local, int64_t nslices, int64_t* widths,
                           cudaStream_t st);
void launch_stencil_fill(const StencilDesc& d, int64_t n_local, int64_t nslices,
                         const int64_t* slice_ptr, double* vals, int32_t* cols, double* diag,
                         cudaStream_t st);
// exclusive scan of widths*32 -> slice_ptr[0..nslices]
void scan_slice_ptr(const int64_t* widths, int64_t nslices, int64_t* slice_ptr, void* tmp,
                    size_t* tmp_bytes, cudaStream_t st);
// CSR (device, int64) -> SELL-32; validates offsets and column range into *bad.
void launch_csr_widths(int64_t n, const int64_t* rowptr, int64_t nslices, int64_t* widths,
                       int* bad, cudaStream_t st);
// row block [row_begin, row_begin+n) of an n_global CSR with global columns
// (ghosts: sorted off-block columns, local n + index)
// (streamed) rows [r0, r1) of the block, r0 % 32 == 0; col/val hold entries
// [nnz_base, ...) of the block (the chunk's part of the host arrays)
void launch_csr_fill(int64_t n, int64_t row_begin, int64_t n_global, const int64_t* ghosts,
                     int64_t n_ghost, const int64_t* rowptr, const int64_t* col, const double* val,
                     int64_t nnz_base, int64_t r0, int64_t r1, const int64_t* slice_ptr,
                     double* vals, int32_t* cols, double* diag, int* bad, cudaStream_t st);
void launch_slice_ghost_flag(int64_t n_local, int64_t nslices, const int64_t* slice_ptr,
                             const int32_t* cols, unsigned char* flag, cudaStream_t st);
void launch_halo_gather(int64_t count, const int32_t* idx, const double* x, double* buf,
                        cudaStream_t st);
// SELL -> CSR row lengths and fill (global columns via row_begin / ghost map)
void launch_sell_row_len(const SellView& a, int64_t* len, cudaStream_t st);
// rows [r0, r1) (r0 % 32 == 0), entries written at col/val[rowptr[row] - base]
void launch_sell_to_csr(const SellView& a, int64_t row_begin, const int64_t* ghost_global,
                        const int64_t* rowptr, int64_t* col, double* val, int64_t r0, int64_t r1,
                        int64_t base, cudaStream_t st);
void scan_rowptr(const int64_t* len, int64_t n, int64_t* rowptr, void* tmp, size_t* tmp_bytes,
                 cudaStream_t st);
// SELL-32 -> SELL-32P(U) conversion (see SellView): plan per-slice kinds, sizes
// and uniform-table hashes; sort the hashes into shared tables; fill; verify.
// Local -> global column map of a rank block (the merge key is the global
// relative offset: rows store their entries in ascending global column order).
struct ColMap {
  int64_t row_begin, n_local;
  const int64_t* ghost;  // ghost_global (device), n_ghost entries
};
void launch_compress_plan(int64_t nslices, const int64_t* slice_ptr, const int32_t* cols,
                          const double* vals, ColMap cm, int64_t* val_cnt, int64_t* pat_cnt,
                          int64_t* col_cnt, int64_t* kind, unsigned long long* hash, int dedupe,
                          cudaStream_t st);
// inclusive max-scan (tmp == nullptr: query *tmp_bytes)
void scan_max_i64(const int64_t* in, int64_t n, int64_t* out, void* tmp, size_t* tmp_bytes,
                  cudaStream_t st);
// radix sort of (hash, slice) pairs (tmp == nullptr: query *tmp_bytes)
void sort_tables(const unsigned long long* key_in, unsigned long long* key_out,
                 const int32_t* val_in, int32_t* val_out, int64_t n, void* tmp, size_t* tmp_bytes,
                 cudaStream_t st);
void launch_table_heads(int64_t n, const unsigned long long* key, const int32_t* slc,
                        const int64_t* kind, int64_t* tab_cnt, int64_t* headpos, cudaStream_t st);
void launch_table_assign(int64_t n, const unsigned long long* key, const int32_t* slc,
                         const int64_t* headpos, const int64_t* tab_ptr, int64_t* slice_tab,
                         int32_t* slice_rep, cudaStream_t st);
void launch_iota_i32(int64_t n, int32_t* out, cudaStream_t st);
// CDIA participation words (see CdiaClass); *bad = 1 if a table key is missing;
// nodiag[c] = 1 if some owned row of class c lacks key 0 (its diagonal)
void launch_cdia_bits(int64_t nslices, int64_t n_local, int ncls, const int64_t* starts,
                      const int64_t* ckeys, const int32_t* nofs, const int64_t* meta,
                      const int64_t* pkey, const int2* pat, uint32_t* bits, int* bad,
                      int* nodiag, cudaStream_t st);
// 3x3x3 box class rows [r0, r1) with plane stride P: *bad = 1 unless every
// participation word is geometric (see sell.cu cdia_geo_kernel)
void launch_cdia_geo_check(const uint32_t* bits, int64_t r0, int64_t r1, int64_t P, int* bad,
                           cudaStream_t st);
void launch_compress_fill(int64_t nslices, const int64_t* slice_ptr, const int32_t* cols,
                          const double* vals, ColMap cm, const int64_t* kind,
                          const int64_t* slice_tab, const int32_t* slice_rep,
                          const int64_t* new_ptr, const int64_t* pat_ptr, int64_t pat_base,
                          const int64_t* col_ptr, double* nvals, int32_t* ncols, int2* pat,
                          double* pval, int64_t* pkey, int64_t* meta, cudaStream_t st);
void launch_compress_verify(int64_t nslices, const int64_t* slice_ptr, const int32_t* cols,
                            const double* vals, ColMap cm, const int64_t* kind,
                            const int64_t* slice_tab, const int2* pat, const double* pval,
                            const int64_t* pkey, int* bad, cudaStream_t st);
// inv_diag[i] = 1/diag[i]; *bad = 1 if any diag <= 0 (precond.cpp:17-22)
void launch_inv_diag(int64_t n, const double* diag, double* inv_diag, int* bad, cudaStream_t st);

// ------------------------------------------------------------------ SpMV family (spmv.cu)
enum SpmvKind {
  kPlain = 0, kResid = 1, kMpkFirst = 2, kMpkMid = 3, kMpkLast = 4, kDot = 5,
  // fast algebra: z_q = ca*D^-1 p_q + cb*z_{q-1} + cc*z_{q-2}, no zp vectors, D from the row
  kMpkFirstF = 6, kMpkMidF = 7,
  // true-residual schedule (CS_VAR_TRUE_R): r = b - A x and z_0 = M^-1 r in one
  // pass (breakdown check on z_0 as basis column 0, NVLink push of z_0)
  kResidF = 8
};
struct SpmvArgs {
  const double* x = nullptr;   // operand (owned + ghost slots)
  double* y = nullptr;         // A x (p column, r, ...)
  const double* b = nullptr;   // kResid: y = b - A x
  const double* zp1 = nullptr; // zp_{q-1}
  const double* zp2 = nullptr; // zp_{q-2}
  double* zpout = nullptr;     // zp_q (Jacobi only)
  double* zout = nullptr;      // z_q = M^-1 zp_q
  double ca = 0, cb = 0, cc = 0;
  int col = 0;                 // basis column for the breakdown payload
  int pending = 0;             // record breakdown in st->pending instead of st->err
  DevState* st = nullptr;
  double* partial = nullptr;   // kDot: per-block partials of x.y
  unsigned* ticket = nullptr;  // kDot: last-block finalisation
  double* result = nullptr;    // kDot: finalised sum
  // NVLink peer-memory halo (z-slab problems, fast MPK). Producer:
  // z rows [0, send_lo) also go to push_lo[row] (rank-1's upper ghost plane) and
  // rows [hi_begin, n_local) to push_hi[row - hi_begin] (rank+1's lower ghost
  // plane), plain remote stores. Signal: the NEXT kernel on the producer's
  // stream (its predecessor has completed, so every remote store of it is
  // visible) adds the known row counts to the peers' receive counters with one
  // release reduction each (rel_*), from block 0 before anything else.
  // Consumer: before the first slice every block waits until wait_ctr[0] >=
  // want_lo and wait_ctr[1] >= want_hi (acquire).
  double* push_lo = nullptr;
  double* push_hi = nullptr;
  int64_t send_lo = 0, hi_begin = 0;
  unsigned long long* rel_lo = nullptr;
  unsigned long long* rel_hi = nullptr;
  unsigned long long rel_lo_n = 0, rel_hi_n = 0;
  const unsigned long long* wait_ctr = nullptr;
  unsigned long long want_lo = 0, want_hi = 0;
};
void launch_spmv(int kind, const SellView& a, const SpmvArgs& g, int64_t slice_begin,
                 int64_t slice_end, cudaStream_t st);
int spmv_dot_blocks(int64_t nslices);
// Push rows [0, send_lo) and [hi_begin, n_local) of col into the neighbours'
// ghost slots (the z_0 halo of the fast MPK; signalled by the next kernel).
void launch_halo_push(const SpmvArgs& g, const double* col, int64_t n_local, DevState* st,
                      cudaStream_t s);
// Release a previous kernel's pushes when no SpMV launch follows to do it.
void launch_halo_release(const SpmvArgs& g, DevState* st, cudaStream_t s);

// ------------------------------------------------------------------ vector kernels (vec.cu)
void launch_precond_apply(int64_t n, const double* inv_diag, const double* in, double* out,
                          DevState* st, int col, int pending, cudaStream_t s);
void launch_random_vector(int64_t n, int64_t offset, uint64_t seed, double* out, cudaStream_t s);
// block Jacobi: in-place Cholesky of nblocks bs x bs blocks
// (*bad_block = min failing block, caller initialises to INT_MAX); apply
// out = M^-1 in with the breakdown check of launch_precond_apply
void launch_bj_factor(int64_t nblocks, int bs, double* f, int* bad_block, cudaStream_t s);
void launch_bj_apply(int64_t n, int bs, const double* f, const double* in, double* out,
                     DevState* st, int col, int pending, cudaStream_t s);
// serial ascending-order Gram: g[i + j*ku] = sum_l u_i[l] v_j[l]; one thread per entry.
void launch_serial_gram(int64_t n, int ku, int kv, const double* u, int64_t ldu, const double* v,
                        int64_t ldv, double* g, DevState* st, cudaStream_t s);
// deterministic block-tree Gram (generic, any ku/kv <= 64), finalised by the last block.
void launch_tree_gram(int64_t n, int ku, int kv, const double* u, int64_t ldu, const double* v,
                      int64_t ldv, double* g, double* partial, unsigned* ticket, DevState* st,
                      cudaStream_t s);
size_t tree_gram_partial_doubles(int64_t n, int ku, int kv);
// Fast algebra with P derived from Z ("PZ" schedule, diagonal preconditioners):
// the fast MPK epilogue z_q = ca D^-1 p_q + cb z_{q-1} + cc z_{q-2} is inverted
// instead of storing p_q = A z_{q-1}: column j of P (p_{j+1}) is
//   j = 0: (z_1 + sigma z_0) * k1 ;  j >= 1: ((z_{j+1} + 2 sigma z_j) + z_{j-1}) * k2
// times a_ii (diag[i], or the uniform value; 1 for identity), k1 = 1/alpha, k2 = 1/(2 alpha).
// The MPK's last step writes the virtual z_s (instead of p_s) to `zs`. Saves the
// s P columns' write in the MPK and their reads in the pack and update passes.
struct PzArgs {
  const double* zs = nullptr;    // z_s; nullptr: P is streamed (non-PZ)
  double sig1 = 0.0, sig2 = 0.0;  // sigma, 2 sigma
  double k1 = 0.0, k2 = 0.0;      // 1/alpha, 1/(2 alpha)
  double dconst = 1.0;            // the uniform diagonal a_ii (Jacobi), 1 (identity)
  const double* diag = nullptr;   // non-uniform Jacobi: the diagonal a_ii (else nullptr)
  // true-residual schedule: the pack forms r = D z_0 (z_0 = D^-1 r, Z column 0)
  // instead of reading r, which the residual SpMV then does not store
  int r_from_z0 = 0;
};
#ifdef __CUDACC__
// zz[0..S] = z_0 .. z_S of one row; p[j] = column j of P; the same arithmetic
// wherever P is derived (pack, update), so both see the same bits
template <int S>
__device__ __forceinline__ void p_from_z(const double (&zz)[S + 1], const PzArgs& a, double di,
                                         double (&p)[S]) {
#pragma unroll
  for (int j = 0; j < S; ++j) {
    double t;
    if (j == 0) t = fma(a.sig1, zz[0], zz[1]) * a.k1;
    else t = (fma(a.sig2, zz[j], zz[j + 1]) + zz[j - 1]) * a.k2;
    p[j] = t * di;  // di = a_ii of the row (diag[i] or the uniform value): format-independent
  }
}
#endif
// Fused NVLink allreduce of the packed block (multi-GPU fast algebra, DESIGN.md
// 7): the pack's last block stores its rank-local block into slot [epoch & 1]
// [rank] of EVERY rank's exchange buffer (peer memory mapped by CUDA IPC),
// releases a per-source flag in each, waits for all flags of this epoch and sums
// the slots in rank order 0..N-1 -- the same bits on every rank, no NCCL call.
constexpr int kXredMaxRanks = 8;
constexpr int kXredSlot = 1024;  // doubles per slot (>= the packed block for s <= 16)
struct XredArgs {
  int nranks = 0, rank = 0, npack = 0;
  unsigned long long epoch = 0;
  double* slots = nullptr;              // mine: [2][nranks][kXredSlot]
  unsigned long long* flags = nullptr;  // mine: [nranks] (flag r written by rank r)
  double* peer_slots[kXredMaxRanks] = {};
  unsigned long long* peer_flags[kXredMaxRanks] = {};
};
// fast packed reduction {Q^T P, Z^T P, Z^T r, Q^T r, r^T r} (2s^2+2s+1 doubles)
bool pack_supported(int s);
// flags (multi-rank, or nullptr): s rank-local basis-breakdown column flags
// written by the last block (see launch_pending_flags). pz.zs != nullptr: P is
// derived from Z (p unused).
void launch_pack(int s, int64_t n, int64_t ld, const double* q, const double* z, const double* p,
                 const double* r, double* packed, double* partial, unsigned* ticket,
                 DevState* st, double* flags, cudaStream_t strm, const PzArgs& pz = PzArgs{},
                 const XredArgs& xr = XredArgs{});
// flags[j] = 1.0 iff this rank's pending basis breakdown is in column j
void launch_pending_flags(int s, const DevState* st, double* flags, cudaStream_t strm);
size_t pack_partial_doubles(int s, int64_t n);
// x/r/Q/AQ updates
struct UpdateArgs {
  int s;
  int64_t n, ld;
  double* q;             // Q block (in place)
  double* aq;            // AQ block (in place)
  const double* z;       // Z block (beta path); z column 0 is overwritten with M^-1 r (fast)
  double* zw;            // where to write M^-1 r (fast), nullptr = skip
  const double* p;       // P block = A Z columns 1..s
  double* x;
  double* r;
  const double* inv_diag;  // nullptr = identity
  double inv_const = 0.0;  // != 0: every row's 1/a_ii (uniform diagonal): no D^-1 stream
  const double* alpha;   // device s
  const double* beta;    // device s x s, nullptr = no block update
  DevState* st;
  // NVLink peer halo of z_0 (fast MPK, see SpmvArgs): rows [0, send_lo) also to
  // push_lo[row], rows [hi_begin, n) to push_hi[row - hi_begin]; released by
  // the next kernel on the stream
  double* push_lo = nullptr;
  double* push_hi = nullptr;
  int64_t send_lo = 0, hi_begin = 0;
  PzArgs pz;  // pz.zs != nullptr: P derived from Z (p unused)
};
void launch_fast_update(const UpdateArgs& a, cudaStream_t s);  // beta block update + x/r + z0
// true-residual schedule: Q <- Z + Q beta (beta != nullptr), x += Q alpha; no AQ
// block, no r (the next residual SpMV forms r and z_0); push_* carry x's rows.
// false: s has no specialised order (nothing launched).
bool launch_fast_update_tr(const UpdateArgs& a, cudaStream_t s);
// The same beta pass fused with the explicit Gram W = Q_new^T AQ_new of the
// vectors it writes (raw, unsymmetrised s x s into wout via per-block partials
// and last-block finalisation). false: s not supported, nothing launched.
bool update_gram_supported(int s);
size_t update_gram_partial_doubles(int s);
bool launch_fast_update_gram(const UpdateArgs& a, double* partial, unsigned* ticket, double* wout,
                             cudaStream_t s);
void launch_ref_xr_update(const UpdateArgs& a, cudaStream_t s);   // solver.cpp:159-162
void launch_ref_block_update(const UpdateArgs& a, cudaStream_t s);  // dense_ops.cpp:29-42 x2
// generic block_update (unit entry)
void launch_block_update(int64_t n, int m, int k, const double* y, const double* x,
                         const double* c, double* out, cudaStream_t s);
void launch_axpby_pcg(int which, int64_t n, double* x, double* r, double* p, const double* q,
                      const double* inv_diag, DevState* st, double* partial, unsigned* ticket,
                      double* result, int serial, cudaStream_t s);
// lanczos helpers
void launch_scale2(int64_t n, double* v, double* g, const double* src_v, const double* src_g,
                   const double* denom, DevState* st, cudaStream_t s);

// ------------------------------------------------------------------ small single-CTA kernels (small.cu)
struct SmallArgs {
  int s;
  int nu;
  int gram;        // CS_GRAM_*
  int max_outer;
  double tol;
  DevState* st;
  double* W;       // s x s symmetric Gram (persistent)
  double* alpha;   // s
  double* beta;    // s x s
  double* raw;     // reference mode: raw products (W, b1, b2, rr) / fast: packed block
  double* rel;     // history arrays
  double* da;
  double* db;
  const double* Wexp = nullptr;  // fast: raw Q_k^T AQ_k of this outer (explicit W), or null
  const double* flags = nullptr; // fast, multi-rank: allreduced basis-breakdown column flags
  int fast_fgs = 1;              // fast: reassociated FGS sweeps (0 = reference sequence)
};
void launch_fast_setup(const SmallArgs& a, cudaStream_t s);   // W_1, alpha_1 from packed
void launch_fast_step(const SmallArgs& a, cudaStream_t s);    // stop test, beta, recurrence, alpha
void launch_ref_alpha(const SmallArgs& a, cudaStream_t s);    // symmetrise W, alpha solve
void launch_ref_test(const SmallArgs& a, cudaStream_t s);     // rel residual + stop test
void launch_ref_beta(const SmallArgs& a, cudaStream_t s);     // beta solve, k++
void launch_unit_fgs(int s, const double* w, int k, const double* rhs, int nu, double* x,
                     double* delta, int* status, cudaStream_t st);
void launch_unit_chol(int s, const double* w, int k, const double* rhs, double* x, int* status,
                      cudaStream_t st);
void launch_unit_assemble(int k, double* w, int* status, cudaStream_t st);
// classical PCG scalar steps
void launch_pcg_scalar(int which, double tol, int max_iter, DevState* st, const double* dots,
                       double* rel, cudaStream_t s);
void launch_set_state(DevState* st, double bnorm, int k, cudaStream_t s);

}  // namespace csg
