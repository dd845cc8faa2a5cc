/* chebstep_gpu.h -- C ABI of the B200-native Chebyshev s-step PCG solve path.
 *
 * libchebstep_gpu.so (paper_2603_09790_b200/lib/) implements every function
 * below with hand-written sm_100a CUDA kernels; there is no CPU fallback: on a
 * machine without a usable CUDA device every compute entry returns CS_ERR_CUDA.
 * The C++ drop-in (include/chebstep/*.hpp, namespace chebstep) and the Python
 * mirror (paper_2603_09790_b200/__init__.py) are both layered on this ABI.
 *
 * Reference interface each entry replaces (paths relative to
 * /root/reference/proj):
 *   cs_pcg_s_solve_csr   chebstep::pcg_s_solve            include/chebstep/solver.hpp:81-83
 *   cs_pcg_solve_csr     chebstep::pcg_solve              include/chebstep/solver.hpp:95-100
 *   cs_spmv              chebstep::spmv_into              include/chebstep/csr.hpp:52-53
 *   cs_mpk               chebstep::mpk_chebyshev          include/chebstep/mpk.hpp:43-44
 *   cs_block_gram        chebstep::block_gram             include/chebstep/dense_ops.hpp:17
 *   cs_block_update      chebstep::block_update           include/chebstep/dense_ops.hpp:20-21
 *   cs_assemble_gram     chebstep::assemble_gram          include/chebstep/gram.hpp:27
 *   cs_fgs_solve         chebstep::fgs_solve              include/chebstep/gram.hpp:49-50
 *   cs_cholesky_solve    chebstep::small_cholesky_solve   include/chebstep/dense_ops.hpp:28
 *   cs_estimate_interval chebstep::estimate_interval      include/chebstep/spectral.hpp:49-50
 *   cs_random_vector     chebstep::random_vector          include/chebstep/util.hpp:42
 *   cs_problem_generate  chebstep::poisson27 (+ the new 7-point generators)
 *                                                         include/chebstep/problems.hpp:26
 *   cs_problem_set_precond  Identity/JacobiPreconditioner include/chebstep/precond.hpp:25-41
 *
 * Conventions: all sizes int64; blocks are column-major n x k (block.hpp:13-20);
 * small dense matrices column-major (block.hpp:35-55). Host pointers unless a
 * function name ends in _device. Every function returns a CS_* status; on
 * failure cs_last_error() gives the message and the payload (basis column for
 * CS_ERR_BASIS_BREAKDOWN, outer iteration for CS_ERR_SOLVER_BREAKDOWN), which
 * the C++ layer rethrows as the matching errors.hpp exception type.
 */
#ifndef CHEBSTEP_GPU_H
#define CHEBSTEP_GPU_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define CS_OK 0
#define CS_ERR_DIMENSION 1          /* DimensionError        errors.hpp:15-18 */
#define CS_ERR_INVALID_MATRIX 2     /* InvalidMatrixError    errors.hpp:20-23 */
#define CS_ERR_NOT_SPD 3            /* NotSpdError           errors.hpp:25-30 */
#define CS_ERR_BASIS_BREAKDOWN 4    /* BasisBreakdownError   errors.hpp:32-37 */
#define CS_ERR_SOLVER_BREAKDOWN 5   /* SolverBreakdownError  errors.hpp:39-44 */
#define CS_ERR_GUARD_EXCEEDED 6     /* GuardExceededError    errors.hpp:46-49 */
#define CS_ERR_PARSE 7              /* ParseError            errors.hpp:51-54 */
#define CS_ERR_INVALID_ARGUMENT 8   /* InvalidArgumentError  errors.hpp:56-59 */
#define CS_ERR_GENERIC 9            /* Error                 errors.hpp:9-13  */
#define CS_ERR_CUDA 10              /* device/runtime failure (no CPU fallback) */
#define CS_ERR_NCCL 11              /* collective failure */

/* ------------------------------------------------------------ enums */
#define CS_PRECOND_IDENTITY 0
#define CS_PRECOND_JACOBI 1
#define CS_PRECOND_BLOCK_JACOBI 2 /* bs consecutive rows per block, Cholesky solves */
#define CS_PRECOND_DEVICE_FN 3    /* caller-supplied device apply (cs_problem_set_precond_fn) */

#define CS_GEN_POISSON27 0 /* problems.cpp:13-53 */
#define CS_GEN_STENCIL7 1  /* 7-point, coefficients (cx,cy,cz): poisson7 = (1,1,1), aniso = (1,1,100) */

#define CS_GRAM_FGS 0
#define CS_GRAM_CHOLESKY 1

/* Arithmetic mode of a solve.
 *  CS_MODE_FAST:      one packed reduction (one allreduce) per outer iteration via the
 *                     Gram product recurrence, deterministic tree reductions, fused passes.
 *  CS_MODE_REFERENCE: the reference's algebra and operation order (explicit W, b1, b2;
 *                     serial ascending-index reductions; no FMA); bitwise equal to the
 *                     CPU reference on one GPU given the same spectrum. */
#define CS_MODE_FAST 0
#define CS_MODE_REFERENCE 1

/* timing phases (cs_ctx_get_timing) */
#define CS_PHASE_SPMV 0      /* SpMV / fused MPK step kernels */
#define CS_PHASE_REDUCE 1    /* tall-skinny Gram / projection reductions */
#define CS_PHASE_SMALL 2     /* single-CTA Gram-solve kernels */
#define CS_PHASE_UPDATE 3    /* fused block / vector update passes */
#define CS_PHASE_LANCZOS 4   /* spectrum estimation, all kernels */
#define CS_PHASE_COMM 5      /* halo exchange + allreduce */
#define CS_PHASE_OTHER 6
#define CS_NUM_PHASES 7

typedef struct cs_ctx cs_ctx;
typedef struct cs_problem cs_problem;

typedef struct {
  int s;              /* SolverConfig::s                 solver.hpp:17 */
  double tol;         /* SolverConfig::tol               solver.hpp:18 */
  int max_outer;      /* SolverConfig::max_outer         solver.hpp:19 */
  int nu;             /* FgsConfig::nu                   gram.hpp:36   */
  int gram;           /* CS_GRAM_*                       solver.hpp:21 */
  int has_spectrum;   /* SolverConfig::spectrum present  solver.hpp:26 */
  double lambda_min, lambda_max;
  int lanczos_steps;  /* solver.hpp:27 */
  uint64_t seed;      /* solver.hpp:28 */
  int mode;           /* CS_MODE_* */
  int check_every;    /* outer iterations per host convergence poll (0 = auto) */
  /* analysis hooks (solver.hpp:30-34); none changes the iterate sequence.
   * Enabling any of them syncs with the host once per outer iteration. */
  int collect_gram;          /* W_k and kappa_2(W_k) per outer iteration */
  int track_true_residual;   /* ||b - A x_k|| / ||b|| (initial + per outer) */
  const double* error_reference; /* host x* (n_local): A-norm errors, or NULL */
  int collect_iterates;      /* x_k (initial + per outer) */
  /* CS_VAR_* bit set: arithmetic variants of a mode, for attributing and
   * bounding the outer-count sensitivity (tools/count_band.py). 0 = the mode's
   * shipped arithmetic. */
  int variant;
} cs_config;

/* cs_config.variant bits */
#define CS_VAR_EXPLICIT_W 1   /* fast: W_k = sym(Q_k^T AQ_k) from the vectors each outer (in the
                                 same single allreduce) instead of the product recurrence */
#define CS_VAR_RECUR_W 2      /* fast: force the pure W recurrence (round-1 algebra) */
#define CS_VAR_REF_FGS 4      /* fast: the reference's FGS operation sequence */
#define CS_VAR_REF_MPK 8      /* fast: the reference's MPK epilogue (zp streams, no FMA); 1 GPU */
#define CS_VAR_TREE 16        /* reference: fixed-shape tree reductions instead of serial chains */
#define CS_VAR_P_FROM_Z 32    /* fast: P columns derived from Z (no P stream) --
                                 the default wherever it applies; the bit is accepted */
#define CS_VAR_P_STORED 64    /* fast: the stored-P schedule (round-1 default) */
#define CS_VAR_TRUE_R 128     /* fast, PZ schedule: r_{k+1} = b - A x_{k+1} from one residual
                                 SpMV instead of r_k - AQ alpha (no AQ block) --
                                 the default wherever the PZ schedule runs; the bit is accepted */
#define CS_VAR_RECUR_R 256    /* fast: the recursive residual r_k - AQ alpha (AQ block kept) */
#define CS_VAR_STORED_R 512   /* fast, true residual: store r (default: the pack forms r = D z_0) */

typedef struct {
  /* SolveReport (solver.hpp:39-68), reference semantics */
  int converged;
  int outer_iters;
  int64_t spmv_count, precond_count, allreduce_count;
  double local_update_flops, gram_solve_flops;
  double lambda_min, lambda_max; /* spectrum_used */
  int cap;                        /* capacity of the caller's history arrays */
  int n_rel, n_da, n_db;
  double* rel_residual;           /* caller-owned, may be NULL */
  double* delta_alpha;
  double* delta_beta;
  /* device-side facts */
  int64_t device_allreduces;      /* collectives actually issued (fast mode: 1 per outer) */
  int64_t kernel_launches;        /* kernels launched by this solve */
  double t_lanczos_ms, t_solve_ms;/* CUDA-event times on the solve stream */
  /* analysis-hook outputs, caller-owned (NULL = not wanted), `cap` entries each;
   * gram_history holds cap * s*s doubles, iterates cap * n_local doubles. */
  int n_kappa, n_true, n_aerr, n_iter;
  double* kappa_w;
  double* gram_history;
  double* true_rel_residual;
  double* a_norm_error;
  double* iterates;
  int schedule;                   /* CS_SCHED_* bits of the fast schedule that ran */
} cs_report;

/* cs_report.schedule bits */
#define CS_SCHED_P_FROM_Z 1   /* P derived from Z (no P stream) */
#define CS_SCHED_EXPLICIT_W 2 /* W_k reduced from the vectors each outer */
#define CS_SCHED_TRUE_R 4     /* r from b - A x each outer (no AQ block) */
#define CS_SCHED_R_FROM_Z0 8  /* r not stored: the pack forms r = D z_0 */
#define CS_SCHED_P2P_ALLREDUCE 16 /* multi-GPU: the packed block's allreduce fused into the
                                     pack over NVLink peer memory (no NCCL call per outer) */

/* ------------------------------------------------------------ errors / info */
const char* cs_last_error(int* payload);
int cs_version(void);
int cs_device_count(int* count);

/* ------------------------------------------------------------ context */
int cs_ctx_create(int device, cs_ctx** out);
int cs_ctx_destroy(cs_ctx* ctx);
int cs_ctx_set_timing(cs_ctx* ctx, int enable);
int cs_ctx_reset_timing(cs_ctx* ctx);
int cs_ctx_get_timing(cs_ctx* ctx, int phase, double* ms, int64_t* launches);
int cs_ctx_launch_count(cs_ctx* ctx, int64_t* launches);
int cs_ctx_synchronize(cs_ctx* ctx);
/* the cudaStream_t every solve kernel of this context is launched on */
int cs_ctx_stream(cs_ctx* ctx, void** stream);

/* Multi-GPU (one process per GPU). Rank 0 creates the id and the host
 * transports its 128 bytes to the other ranks (torch.distributed, files...). */
int cs_comm_unique_id(unsigned char id[128]);
int cs_ctx_comm_init(cs_ctx* ctx, int nranks, int rank, const unsigned char id[128]);
int cs_ctx_allreduce_max(cs_ctx* ctx, double* value); /* host scalar max over ranks */

/* ------------------------------------------------------------ partitioning (host only, no GPU) */
/* Contiguous, plane-aligned row partition: rows [begin, end) of rank `rank`.
 * `plane` rows are kept together (nx*ny for z-slabs, 1 for general CSR). */
int cs_partition_rows(int64_t n_rows, int64_t plane, int nranks, int rank, int64_t* begin,
                      int64_t* end);
/* Halo map of one rank's row block [row_begin, row_end) of a CSR matrix given
 * its local rows (rowptr relative, global columns). Ghost columns are the
 * sorted unique off-block columns; local numbering is owned rows
 * 0..n_loc-1 then ghosts in ascending global order. Writes n_ghost, the
 * ghost list (cap entries) and the remapped int32 local columns. Pass
 * ghost_cols = NULL to query n_ghost only. */
int cs_halo_map_csr(int64_t row_begin, int64_t row_end, const int64_t* rowptr_local,
                    const int64_t* col_global, int64_t* n_ghost, int64_t* ghost_cols,
                    int64_t ghost_cap, int32_t* col_local);

/* ------------------------------------------------------------ small dense analysis (host) */
/* chebstep::fgs_rate (gram.hpp:58-66, gram.cpp:148-174) of a NORMALIZED s x s
 * Gram matrix w (column-major, unit diagonal): largest singular value and
 * spectral radius of the FGS residual iteration matrix L^T (I+L)^{-1}.
 * Host eigen/singular solvers replace the reference's dgesvd/dgeev
 * (agreement ~1e-13 relative). */
int cs_fgs_rate(int s, const double* w, double* spectral_norm, double* spectral_radius);
/* kappa_2 of a symmetric s x s matrix (solver.cpp:69-74: dsyevd there). */
int cs_kappa_sym(int s, const double* w, double* kappa);

/* ------------------------------------------------------------ host CSR ingestion (no GPU) */
/* Library-owned host CSR (int64 offsets/columns, FP64 values). */
typedef struct cs_csr_host cs_csr_host;
/* chebstep::read_matrix_market (problems.hpp:28-31, problems.cpp:55-109):
 * coordinate real symmetric, 1-based, expanded to the full pattern, rows
 * sorted by column; CS_ERR_PARSE / CS_ERR_INVALID_MATRIX / CS_ERR_NOT_SPD with
 * the reference's messages. The entry section is parsed by all host cores. */
int cs_mm_read(const char* path, int require_spd, cs_csr_host** out, int64_t* n, int64_t* nnz);
/* Rows [row_begin, row_end) of a host CSR: rowptr_local (row_end-row_begin+1,
 * starting at 0), global columns and values. col/val may be NULL (offsets only). */
int cs_csr_host_rows(const cs_csr_host* h, int64_t row_begin, int64_t row_end,
                     int64_t* rowptr_local, int64_t* col, double* val);
int cs_csr_host_free(cs_csr_host* h);
/* chebstep::write_matrix_market (problems.hpp:33-34, problems.cpp:111-127):
 * lower triangle, %.17g values. */
int cs_mm_write(const char* path, int64_t n, const int64_t* rowptr, const int64_t* col,
                const double* val);
/* validate_structure / validate_symmetric / validate_spd_diagonal (csr.hpp:41-47) */
#define CS_CHECK_STRUCTURE 0
#define CS_CHECK_SYMMETRIC 1
#define CS_CHECK_SPD_DIAGONAL 2
int cs_csr_validate(int64_t n, const int64_t* rowptr, const int64_t* col, const double* val,
                    int check);

/* ------------------------------------------------------------ problems (device-resident) */
/* Generate a stencil operator directly on the device as SELL-32. With an
 * initialised communicator the rank gets its z-slab of the global nx*ny*nz
 * grid; otherwise the whole grid. coef = (cx,cy,cz) for CS_GEN_STENCIL7. */
int cs_problem_generate(cs_ctx* ctx, int kind, int64_t nx, int64_t ny, int64_t nz,
                        const double* coef, cs_problem** out);
/* Upload a host CSR (int64 offsets/columns, FP64 values; reference CsrMatrix
 * layout csr.hpp:12-19) and convert it to SELL-32 on the device. Single rank. */
int cs_problem_upload_csr(cs_ctx* ctx, int64_t n, const int64_t* rowptr, const int64_t* col,
                          const double* val, cs_problem** out);
/* Collective over the context's ranks: this rank's row block [row_begin,
 * row_end) of an n_global x n_global CSR (rowptr_local starts at 0, GLOBAL
 * column indices). Blocks must be contiguous and ordered by rank. Builds the
 * ghost list (sorted off-block columns, partition.cpp numbering), the
 * owner-grouped halo plan (NCCL point-to-point) and the interior slice range
 * that overlaps the halo. With one rank it equals cs_problem_upload_csr. */
int cs_problem_upload_csr_block(cs_ctx* ctx, int64_t n_global, int64_t row_begin,
                                int64_t row_end, const int64_t* rowptr_local,
                                const int64_t* col_global, const double* val, cs_problem** out);
/* Matrix Market file -> device problem: every rank parses the file, keeps
 * its cs_partition_rows(n, 1, nranks, rank) block and uploads it (collective). */
int cs_problem_read_mm(cs_ctx* ctx, const char* path, int require_spd, cs_problem** out);
int cs_problem_destroy(cs_problem* p);
/* info12: n_global, n_local, nnz_local, row_begin, n_ghost, device bytes of the
 * SELL arrays, slices, pattern-compressed slices, uniform-value slices, pattern
 * table entries, constant-diagonal (CDIA) classes, CDIA flags: bit 0 every class
 * has a uniform diagonal, bit 1 every class is a geometric box with plane-uniform
 * z faces (the separable SpMV reads no participation words) */
int cs_problem_info(cs_problem* p, int64_t* info12);
/* Local rows back as CSR with GLOBAL column indices (bit-exact assembly check). */
int cs_problem_download_csr(cs_problem* p, int64_t* rowptr, int64_t* col, double* val);
/* Ghost global column list of this rank (n_ghost entries). */
int cs_problem_ghosts(cs_problem* p, int64_t* ghost_cols);
/* Halo transport of the last solve on this problem: 0 none (single rank),
 * 1 NCCL send/recv, 2 NVLink peer-memory stores from the producing kernels. */
int cs_problem_halo_mode(cs_problem* p, int* mode);
int cs_problem_set_precond(cs_problem* p, int kind);
int cs_problem_inv_diag(cs_problem* p, double* out);

/* Pluggable preconditioners beyond the reference's two (the
 * reference accepts any `const Preconditioner&`, precond.hpp:12-23). Neither
 * has a CPU fallback: the apply runs on the device inside the solve.
 *
 * Block Jacobi: M = blockdiag(A_11, A_22, ...), blocks of bs consecutive local
 * rows (the last may be shorter). `blocks` (host) holds ceil(n_local/bs) dense
 * bs x bs column-major diagonal blocks of A (a short last block padded with the
 * identity). They are factorised on the device, L L^T = A_bb, left-looking
 * like small_cholesky_solve (dense_ops.cpp:55-88); CS_ERR_NOT_SPD (payload =
 * block) if a pivot is not positive and finite. apply: out_b = L^-T L^-1 in_b,
 * forward then back substitution in the reference's loop order. 1 <= bs <= 16. */
int cs_problem_set_precond_block_jacobi(cs_problem* p, int bs, const double* blocks);
/* Device plugin: out = M^-1 in for n_local doubles, both device pointers,
 * enqueued on `stream` (a cudaStream_t) by the callee; return 0 or nonzero on
 * failure (the solve then fails with CS_ERR_GENERIC). Called s times per outer
 * iteration, plus once per Lanczos step and once at setup. */
typedef int (*cs_precond_fn)(void* user, const double* in, double* out, int64_t n_local,
                             void* stream);
int cs_problem_set_precond_fn(cs_problem* p, cs_precond_fn fn, void* user);

/* ------------------------------------------------------------ kernel-level entries (host buffers) */
int cs_spmv(cs_problem* p, const double* x, double* y);
int cs_mpk(cs_problem* p, const double* r, int s, double lambda_min, double lambda_max,
           double* z, double* pblk);
/* mode: CS_MODE_REFERENCE = serial ascending order (bitwise), CS_MODE_FAST = tree */
int cs_block_gram(cs_ctx* ctx, int64_t n, int ku, int kv, const double* u, const double* v,
                  double* g, int mode);
int cs_block_update(cs_ctx* ctx, int64_t n, int m, int k, const double* y, const double* x,
                    const double* c, double* out);
int cs_assemble_gram(cs_ctx* ctx, int64_t n, int k, const double* q, const double* aq,
                     double* w, int mode);
int cs_fgs_solve(cs_ctx* ctx, int s, const double* w, int k, const double* rhs, int nu,
                 double* x, double* delta);
int cs_cholesky_solve(cs_ctx* ctx, int s, const double* w, int k, const double* rhs, double* x);
int cs_random_vector(cs_ctx* ctx, int64_t n, uint64_t seed, double* out);
int cs_tridiag_eigvals(int m, const double* diag, const double* off, double* out);
int cs_estimate_interval(cs_problem* p, int steps, uint64_t seed, int mode, double* lambda_min,
                         double* lambda_max);

/* Time one solve kernel alone on device-resident data (CUDA events), for
 * roofline measurements: kind 0 = y = A x, 1 = fused MPK middle step
 * (reference recurrence), 2 = fused MPK middle step (fast recurrence),
 * 3 = packed one-allreduce reduction (s = 8), 4 = fused update pass (s = 8).
 * Average ms per launch. */
/* Kernel micro-benchmarks (CUDA events, ms per launch): 0 SpMV, 1 reference MPK
 * step, 2 fast MPK step, 3 packed reduction (s=8), 4 update pass (s=8); multi-GPU
 * (collective, after one solve): 5 peer-memory z_0 push, 6 fast MPK step through
 * the peer-memory halo. */
int cs_bench_spmv(cs_problem* p, int kind, int reps, double* ms_per_launch);

/* ------------------------------------------------------------ solves */
void cs_config_default(cs_config* cfg);
/* b, x0, x are host arrays of the rank's n_local rows. */
int cs_pcg_s_solve(cs_problem* p, const double* b, const double* x0, const cs_config* cfg,
                   double* x, cs_report* rep);
int cs_pcg_solve(cs_problem* p, const double* b, const double* x0, double tol, int max_iter,
                 int mode, double* x, cs_report* rep);
/* Classical PCG with the PcgConfig fields of a cs_config: tol, max_outer (as
 * max_iter), mode, error_reference, collect_iterates (solver.hpp:85-90). */
int cs_pcg_solve_cfg(cs_problem* p, const double* b, const double* x0, const cs_config* cfg,
                     double* x, cs_report* rep);
/* Device-resident variants: b, x0, x are device pointers (n_local doubles). */
int cs_pcg_s_solve_device(cs_problem* p, const double* b, const double* x0,
                          const cs_config* cfg, double* x, cs_report* rep);
int cs_pcg_solve_device(cs_problem* p, const double* b, const double* x0, double tol,
                        int max_iter, int mode, double* x, cs_report* rep);
/* The reference-signature drop-in: host CSR + host vectors in, host x out;
 * upload, SELL conversion, preconditioner setup, spectrum estimate, solve and
 * download all happen inside (what chebstep::pcg_s_solve does). */
int cs_pcg_s_solve_csr(cs_ctx* ctx, int64_t n, const int64_t* rowptr, const int64_t* col,
                       const double* val, int precond, const double* b, const double* x0,
                       const cs_config* cfg, double* x, cs_report* rep);
int cs_pcg_solve_csr(cs_ctx* ctx, int64_t n, const int64_t* rowptr, const int64_t* col,
                     const double* val, int precond, const double* b, const double* x0,
                     double tol, int max_iter, double* x, cs_report* rep);

#ifdef __cplusplus
}
#endif
#endif
