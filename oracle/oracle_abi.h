/* oracle_abi.h -- TEST INFRASTRUCTURE ONLY.
 *
 * One C ABI, implemented twice:
 *   ref_*  oracle/ref_capi.cpp: thin extern "C" wrappers over the UNMODIFIED
 *          reference library (/root/reference/proj/src, compiled in place with
 *          -Dchebstep=chebstep_ref by oracle/Makefile into oracle/_ref/).
 *   orc_*  oracle/cs_oracle.c: plain-C restatement of the same algorithms,
 *          each function citing the reference file:line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load either library, and only as the checker / CPU baseline. The
 * product (paper_2603_09790_b200) never links or calls anything here.
 *
 * Status codes match include/chebstep_gpu.h (CS_OK ...). Matrices are CSR
 * with int64 offsets/columns and FP64 values (reference util.hpp:10,
 * csr.hpp:12-19); blocks are column-major n x k (block.hpp:13-20).
 */
#ifndef CHEBSTEP_ORACLE_ABI_H
#define CHEBSTEP_ORACLE_ABI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int s;
  double tol;
  int max_outer;
  int nu;
  int gram;          /* 0 = fgs, 1 = cholesky (solver.hpp:14) */
  int has_spectrum;  /* inject SolverConfig::spectrum (solver.hpp:26) */
  double lambda_min, lambda_max;
  int lanczos_steps;
  uint64_t seed;
} oc_cfg;

typedef struct {
  int converged;
  int outer_iters;
  int64_t spmv_count, precond_count, allreduce_count;
  double local_update_flops, gram_solve_flops;
  double lambda_min, lambda_max;
  int cap;                 /* capacity of the three history arrays */
  int n_rel, n_da, n_db;   /* filled lengths */
  double* rel_residual;
  double* delta_alpha;
  double* delta_beta;
} oc_report;

/* analysis hooks (solver.hpp:30-34), reference library only */
typedef struct {
  int collect_gram, track_true_residual, collect_iterates;
  const double* error_reference;
  int cap;                      /* entries per history (gram: cap*s*s, iterates: cap*n) */
  double* kappa_w;
  double* gram_history;
  double* true_rel_residual;
  double* a_norm_error;
  double* iterates;
  int n_kappa, n_true, n_aerr, n_iter;
} oc_hooks;

int ref_pcg_s_solve_hooks(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                          const double* b, const double* x0, int precond, const oc_cfg* cfg,
                          oc_hooks* hk, double* x, oc_report* rep);
int ref_pcg_solve_hooks(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        const double* b, const double* x0, int precond, double tol, int max_iter,
                        oc_hooks* hk, double* x, oc_report* rep);

/* Matrix Market I/O and CSR validation (problems.cpp:55-127, csr.cpp:58-110),
 * reference library only. ref_mm_read: call with rp == NULL for n / nnz. */
int ref_mm_read(const char* path, int require_spd, int64_t* n, int64_t* nnz, int64_t* rp,
                int64_t* ci, double* v);
int ref_mm_write(const char* path, int64_t n, const int64_t* rp, const int64_t* ci,
                 const double* v);
int ref_csr_validate(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     int64_t nnz, int check);

/* fgs_rate(normalize_gram(gram_from_matrix(w))) (gram.cpp:60-76,148-174) and
 * kappa_of via dsyevd (solver.cpp:69-74), reference library only */
int ref_fgs_rate_normalized(int s, const double* w, double* norm, double* radius);
int ref_sym_eigvals(int s, const double* w, double* out);

#define OC_DECLARE(P)                                                                  \
  int P##poisson27_fill(int64_t nx, int64_t ny, int64_t nz, int64_t* rowptr,           \
                        int64_t* col, double* val);                                   \
  int P##spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,        \
              const double* x, double* y);                                            \
  int P##jacobi_invdiag(int64_t n, const int64_t* rp, const int64_t* ci,               \
                        const double* v, double* out);                                \
  int P##mpk(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,         \
             int precond, const double* r, int s, double lo, double hi, double* z,    \
             double* p);                                                              \
  int P##block_gram(int64_t n, int ku, int kv, const double* u, const double* w,       \
                    double* g);                                                       \
  int P##block_update(int64_t n, int m, int k, const double* y, const double* x,       \
                      const double* c, double* out);                                  \
  int P##assemble_gram(int64_t n, int k, const double* q, const double* aq,            \
                       double* w);                                                    \
  int P##fgs_solve(int s, const double* w, int k, const double* rhs, int nu,           \
                   double* x, double* delta);                                         \
  int P##cholesky_solve(int s, const double* w, int k, const double* rhs, double* x);  \
  int P##random_vector(int64_t n, uint64_t seed, double* out);                         \
  int P##tridiag_eigvals(int m, const double* diag, const double* off, double* out);   \
  int P##estimate_interval(int64_t n, const int64_t* rp, const int64_t* ci,            \
                           const double* v, int precond, int steps, uint64_t seed,    \
                           double* lo, double* hi);                                   \
  int P##pcg_s_solve(int64_t n, const int64_t* rp, const int64_t* ci,                  \
                     const double* v, const double* b, const double* x0, int precond, \
                     const oc_cfg* cfg, double* x, oc_report* rep);                   \
  int P##pcg_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,   \
                   const double* b, const double* x0, int precond, double tol,        \
                   int max_iter, double* x, oc_report* rep);                          \
  const char* P##last_error(int* payload);

OC_DECLARE(ref_)
OC_DECLARE(orc_)

/* reference monitor_inexact (solver.cpp:275-282) over (outer_iters, delta_alpha) */
int ref_monitor_inexact(int outer_iters, int n_da, const double* delta_alpha, double delta_cap,
                        double* max_delta, double* budget, int* pass);

/* restatement-only generators for problems the reference does not ship
 * (SURVEY a22): 7-point stencil with coefficients (cx, cy, cz); poisson7 is
 * (1,1,1) and the anisotropic config-4 operator is (1,1,100). */
int orc_stencil7_fill(int64_t nx, int64_t ny, int64_t nz, double cx, double cy, double cz,
                      int64_t* rowptr, int64_t* col, double* val);

#ifdef __cplusplus
}
#endif
#endif
