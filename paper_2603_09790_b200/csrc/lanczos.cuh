// lanczos.cuh -- device scalars and launchers of the spectrum estimate.
#pragma once
#include "common.cuh"

namespace csg {

constexpr int kLanczosMax = 256;  // steps cap (reference default 40)

struct LanczosScalars {
  double alpha[kLanczosMax];
  double beta[kLanczosMax];
  double proj[kLanczosMax];
  double dot;    // last reduced scalar
  double denom;  // normaliser of the next basis pair
  double rdenom; // 1 / denom (the fast G-only scale multiplies)
  int count;     // completed alpha entries
};

// r = M^-1 t - a v_j - b v_{j-1}, gr = t - a g_j - b g_{j-1}; M^-1 t from inv_diag,
// or precomputed in mt (general preconditioners; r may alias mt)
void lz_resid(int64_t n, const double* t, const double* inv_diag, const double* mt,
              const double* vj, const double* gj, const double* vp, const double* gp, double* r,
              double* gr, const LanczosScalars* sc, int j, DevState* st, cudaStream_t s);
void lz_axpy2(int64_t n, const double* v, const double* g, double* r, double* gr,
              const double* proj, DevState* st, cudaStream_t s);
int lz_cgs_blocks(int64_t n);
void lz_cgs(int64_t n, int64_t ld, int m, const double* V, const double* G, double* r, double* gr,
            const double* proj, double* partial, unsigned* ticket, double* result, DevState* st,
            cudaStream_t s);
// fast CGS projections proj[i] = G_i . r (i < m <= 40) in one pass over r and G
bool lz_proj_supported(int m);
size_t lz_proj_partial_doubles(int m);
void lz_proj(int64_t n, int64_t ld, int m, const double* G, const double* r, double* proj,
             double* partial, unsigned* ticket, DevState* st, cudaStream_t s);
// G-only fast Lanczos for diagonal M (v = D^-1 g, r = D^-1 gr never stored);
// dinv = a_ii^-1 vector or nullptr with the uniform dconst (1 for identity)
void lz2_resid_proj(int64_t n, int64_t ld, int m, const double* t, const double* G,
                    const double* dinv, double dconst, double* gr, const LanczosScalars* sc, int j,
                    double* proj, double* partial, unsigned* ticket, DevState* st, cudaStream_t s);
void lz2_cgs(int64_t n, int64_t ld, int m, const double* G, const double* dinv, double dconst,
             double* gr, const double* proj, double* partial, unsigned* ticket, double* result,
             DevState* st, cudaStream_t s);
void lz2_scale(int64_t n, const double* gr, const double* dinv, double dconst, double* g, double* v,
               const LanczosScalars* sc, DevState* st, cudaStream_t s);
void lz_scalar(int which, int j, int steps, LanczosScalars* sc, DevState* st, cudaStream_t s);

// host: eigenvalues of the symmetric tridiagonal (d[m], e[m-1]) ascending
void tridiag_eigenvalues(int m, const double* d, const double* e, double* out);
// host: eigenvalues of a small dense symmetric matrix (column-major s x s), ascending
void sym_eigenvalues(int s, const double* w, double* out);
// host: largest singular value / eigenvalue moduli of a general s x s matrix
double max_singular_value(int s, const double* m);
void general_eig_moduli(int n, const double* m, double* out);

}  // namespace csg
