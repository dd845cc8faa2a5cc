// small.cu -- single-CTA kernels for the s x s Gram systems and the solver
// control (stop test, breakdown detection) -- no host round trip.
//
// Every GPU runs these redundantly on identical (allreduced) inputs, so all
// ranks take identical decisions. FGS and Cholesky keep the reference loop
// order and rounding exactly (gram.cpp:78-119, dense_ops.cpp:55-88,
// solver.cpp:33-44): given equal inputs the results are bitwise equal.
// Right-hand-side columns are independent in the reference, so they run on
// separate threads here.
#include "kernels.cuh"

namespace csg {
namespace {

constexpr int kSmallThreads = 128;
// error sub-codes (host formats the reference's messages from them)
constexpr int kSubAssembly = 1, kSubFgs = 2, kSubChol = 3, kSubPcg = 4;

__device__ __forceinline__ void raise(DevState* st, int code, int sub, int payload) {
  atomicCAS(&st->err, 0ull, make_err(code | (sub << 8), payload));
  st->done = 1;
}

// Frobenius norm, block.cpp:53-57 (serial over column-major data)
__device__ double frob_serial(int len, const double* m) {
  double acc = 0.0;
  for (int i = 0; i < len; ++i) acc = __dadd_rn(acc, __dmul_rn(m[i], m[i]));
  return __dsqrt_rn(acc);
}

// Residual ||rhs - W x||_F / ||rhs||_F with the reference order; tmp >= s*k.
__device__ double gram_residual(int s, const double* W, int k, const double* rhs, const double* x,
                                double rn, double* tmp) {
  for (int e = threadIdx.x; e < s * k; e += blockDim.x) {
    const int i = e % s, col = e / s;
    double acc = rhs[e];
    for (int j = 0; j < s; ++j) acc = __dsub_rn(acc, __dmul_rn(W[i + j * s], x[j + col * s]));
    tmp[e] = acc;
  }
  __syncthreads();
  __shared__ double res;
  if (threadIdx.x == 0) {
    double r2 = 0.0;
    for (int e = 0; e < s * k; ++e) r2 = __dadd_rn(r2, __dmul_rn(tmp[e], tmp[e]));
    res = rn == 0.0 ? 0.0 : __ddiv_rn(__dsqrt_rn(r2), rn);
  }
  __syncthreads();
  return res;
}

// One thread per right-hand-side column, W and the iterate in registers.
template <int S>
__device__ void fgs_columns_reg(const double* W, int k, const double* rhs, int nu, double* x) {
  for (int col = threadIdx.x; col < k; col += blockDim.x) {
    double w[S][S], b[S], xc[S];
#pragma unroll
    for (int i = 0; i < S; ++i) {
      b[i] = rhs[i + col * S];
      xc[i] = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) w[i][j] = W[i + j * S];
    }
    for (int sweep = 0; sweep < nu; ++sweep) {
#pragma unroll
      for (int i = 0; i < S; ++i) {
        double acc = b[i];
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j != i) acc = __dsub_rn(acc, __dmul_rn(w[i][j], xc[j]));
        xc[i] = __ddiv_rn(acc, w[i][i]);
      }
    }
#pragma unroll
    for (int i = 0; i < S; ++i) x[i + col * S] = xc[i];
  }
}

// Fast-mode FGS (same sweep order, reassociated arithmetic): reciprocal of
// the diagonal instead of a division, and each row's sum is started at the
// sweep's beginning from the not-yet-updated x_j (j > i) and finished by one
// FMA per freshly updated x_j -- the dependent chain per row is one FMA plus
// one multiply instead of s-1 sub/mul pairs and a division.
template <int S>
__device__ void fgs_fast_reg(const double* W, int k, const double* rhs, int nu, double* x) {
  for (int col = threadIdx.x; col < k; col += blockDim.x) {
    double w[S][S], inv[S], b[S], xc[S], acc[S];
#pragma unroll
    for (int i = 0; i < S; ++i) {
      b[i] = rhs[i + col * S];
      xc[i] = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) w[i][j] = W[i + j * S];
      inv[i] = 1.0 / w[i][i];
    }
    for (int sweep = 0; sweep < nu; ++sweep) {
#pragma unroll
      for (int i = 0; i < S; ++i) {
        acc[i] = b[i];
#pragma unroll
        for (int j = i + 1; j < S; ++j) acc[i] = fma(-w[i][j], xc[j], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < S; ++i) {
        xc[i] = acc[i] * inv[i];
#pragma unroll
        for (int r = i + 1; r < S; ++r) acc[r] = fma(-w[r][i], xc[i], acc[r]);
      }
    }
#pragma unroll
    for (int i = 0; i < S; ++i) x[i + col * S] = xc[i];
  }
}

__device__ void fgs_fast_generic(int s, const double* W, int k, const double* rhs, int nu,
                                 double* x) {
  for (int col = threadIdx.x; col < k; col += blockDim.x) {
    const double* b = rhs + col * s;
    double* xc = x + col * s;
    for (int sweep = 0; sweep < nu; ++sweep)
      for (int i = 0; i < s; ++i) {
        double a0 = b[i], a1 = 0.0;
        int j = 0;
        for (; j + 1 < s; j += 2) {
          if (j != i) a0 = fma(-W[i + j * s], xc[j], a0);
          if (j + 1 != i) a1 = fma(-W[i + (j + 1) * s], xc[j + 1], a1);
        }
        if (j < s && j != i) a0 = fma(-W[i + j * s], xc[j], a0);
        xc[i] = (a0 + a1) / W[i + i * s];
      }
  }
}

// gram.cpp:78-119. Returns 0 or the NotSpd sub-code. x, tmp: s*k.
// fast = reassociated sweeps (fast algebra only); otherwise the reference's
// exact operation sequence.
// S > 0: the order is known at compile time and only that register variant is
// instantiated (the runtime switch inlines every variant: ~14k SASS instructions
// in one kernel, whose instruction-cache misses ncu showed as the top stall).
template <int S = 0>
__device__ int fgs_dev(int s, const double* W, int k, const double* rhs, int nu, double* x,
                       double* delta, double* tmp, bool fast = false) {
  for (int i = 0; i < s; ++i)
    if (!(W[i + i * s] > 0.0)) return kSubFgs;
  __shared__ double rn_sh;
  if (threadIdx.x == 0) rn_sh = frob_serial(s * k, rhs);
  for (int e = threadIdx.x; e < s * k; e += blockDim.x) x[e] = 0.0;
  __syncthreads();
  const double rn = rn_sh;
  if (rn == 0.0) {
    *delta = 0.0;
    return 0;
  }
  if constexpr (S > 0) {
    if (fast) fgs_fast_reg<S>(W, k, rhs, nu, x);
    else fgs_columns_reg<S>(W, k, rhs, nu, x);
    __syncthreads();
    *delta = gram_residual(s, W, k, rhs, x, rn, tmp);
    return 0;
  }
  if (fast) {
    switch (s) {
      case 2: fgs_fast_reg<2>(W, k, rhs, nu, x); break;
      case 3: fgs_fast_reg<3>(W, k, rhs, nu, x); break;
      case 4: fgs_fast_reg<4>(W, k, rhs, nu, x); break;
      case 5: fgs_fast_reg<5>(W, k, rhs, nu, x); break;
      case 6: fgs_fast_reg<6>(W, k, rhs, nu, x); break;
      case 8: fgs_fast_reg<8>(W, k, rhs, nu, x); break;
      default: fgs_fast_generic(s, W, k, rhs, nu, x);
    }
    __syncthreads();
    *delta = gram_residual(s, W, k, rhs, x, rn, tmp);
    return 0;
  }
  switch (s) {  // register-resident sweeps for small orders, same operation sequence
    case 2: fgs_columns_reg<2>(W, k, rhs, nu, x); break;
    case 3: fgs_columns_reg<3>(W, k, rhs, nu, x); break;
    case 4: fgs_columns_reg<4>(W, k, rhs, nu, x); break;
    case 5: fgs_columns_reg<5>(W, k, rhs, nu, x); break;
    case 6: fgs_columns_reg<6>(W, k, rhs, nu, x); break;
    case 8: fgs_columns_reg<8>(W, k, rhs, nu, x); break;
    default:
      for (int col = threadIdx.x; col < k; col += blockDim.x) {
        const double* b = rhs + col * s;
        double* xc = x + col * s;
        for (int sweep = 0; sweep < nu; ++sweep)
          for (int i = 0; i < s; ++i) {
            double acc = b[i];
            for (int j = 0; j < s; ++j)
              if (j != i) acc = __dsub_rn(acc, __dmul_rn(W[i + j * s], xc[j]));
            xc[i] = __ddiv_rn(acc, W[i + i * s]);
          }
      }
  }
  __syncthreads();
  *delta = gram_residual(s, W, k, rhs, x, rn, tmp);
  return 0;
}

// dense_ops.cpp:55-88 + solver.cpp:33-44. L in lmat (s*s).
__device__ int chol_dev(int s, const double* W, int k, const double* rhs, double* x,
                        double* delta, double* lmat, double* tmp) {
  __shared__ int fail;
  if (threadIdx.x == 0) {
    fail = 0;
    for (int e = 0; e < s * s; ++e) lmat[e] = 0.0;
    for (int j = 0; j < s && !fail; ++j) {
      double d = W[j + j * s];
      for (int q = 0; q < j; ++q) d = __dsub_rn(d, __dmul_rn(lmat[j + q * s], lmat[j + q * s]));
      if (!(d > 0.0) || !isfinite(d)) {
        fail = 1;
        break;
      }
      const double dg = __dsqrt_rn(d);
      lmat[j + j * s] = dg;
      for (int i = j + 1; i < s; ++i) {
        double v = W[i + j * s];
        for (int q = 0; q < j; ++q) v = __dsub_rn(v, __dmul_rn(lmat[i + q * s], lmat[j + q * s]));
        lmat[i + j * s] = __ddiv_rn(v, dg);
      }
    }
  }
  __syncthreads();
  if (fail) return kSubChol;
  for (int col = threadIdx.x; col < k; col += blockDim.x) {
    double* xc = x + col * s;
    for (int i = 0; i < s; ++i) xc[i] = rhs[i + col * s];
    for (int i = 0; i < s; ++i) {
      double v = xc[i];
      for (int q = 0; q < i; ++q) v = __dsub_rn(v, __dmul_rn(lmat[i + q * s], xc[q]));
      xc[i] = __ddiv_rn(v, lmat[i + i * s]);
    }
    for (int i = s - 1; i >= 0; --i) {
      double v = xc[i];
      for (int q = i + 1; q < s; ++q) v = __dsub_rn(v, __dmul_rn(lmat[q + i * s], xc[q]));
      xc[i] = __ddiv_rn(v, lmat[i + i * s]);
    }
  }
  __syncthreads();
  __shared__ double rn_sh;
  if (threadIdx.x == 0) rn_sh = frob_serial(s * k, rhs);
  __syncthreads();
  *delta = gram_residual(s, W, k, rhs, x, rn_sh, tmp);
  return 0;
}

template <int S = 0>
__device__ int solve_dev(const SmallArgs& a, const double* W, int k, const double* rhs, double* x,
                         double* delta, double* scratch, bool fast = false) {
  if (a.gram == 0) return fgs_dev<S>(a.s, W, k, rhs, a.nu, x, delta, scratch, fast);
  return chol_dev(a.s, W, k, rhs, x, delta, scratch, scratch + a.s * a.s);
}

// gram.cpp:38-49 symmetrisation + finish_assembly diagonal test (gram.cpp:22-35)
__device__ bool symmetrise_check(int s, double* W) {
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int i = e % s, j = e / s;
    if (i < j) {
      const double v = __dmul_rn(0.5, __dadd_rn(W[i + j * s], W[j + i * s]));
      W[i + j * s] = v;  // (i,j) and (j,i) are written by the same thread
      W[j + i * s] = v;
    }
  }
  __syncthreads();
  bool ok = true;
  for (int i = 0; i < s; ++i) {
    const double d = W[i + i * s];
    if (!(d > 0.0) || !isfinite(d)) ok = false;
  }
  return ok;
}

// dynamic shared memory layout for the solver kernels
struct SmallSmem {
  double* W;    // s*s working Gram
  double* Wn;   // s*s next Gram
  double* rhs;  // s*s
  double* x;    // s*s
  double* t1;   // s*s
  double* scr;  // 2*s*s scratch (Cholesky L + residual)
};
__device__ SmallSmem carve(int s) {
  extern __shared__ double sm[];
  const int q = s * s;
  return {sm, sm + q, sm + 2 * q, sm + 3 * q, sm + 4 * q, sm + 5 * q};
}

__device__ __forceinline__ bool halted(const DevState* st) {
  return *(volatile const int*)&st->done != 0;
}

// ---------------------------------------------------------------- fast mode

// After setup MPK(r0) and the packed reduction with Q = Z: W_1 = sym(Z^T P),
// b1 = Z^T r0, rel[0] = sqrt(r0.r0)/||b||; alpha_1.
template <int S>
__global__ void fast_setup_kernel(SmallArgs a) {
  DevState* st = a.st;
  if (halted(st)) return;
  const int s = a.s, q = s * s;
  const double* pk = a.raw;
  SmallSmem m = carve(s);
  for (int e = threadIdx.x; e < q; e += blockDim.x) m.W[e] = pk[q + e];
  for (int e = threadIdx.x; e < s; e += blockDim.x) m.rhs[e] = pk[2 * q + e];
  if (threadIdx.x == 0) {
    a.rel[0] = __ddiv_rn(__dsqrt_rn(pk[2 * q + 2 * s]), st->bnorm);
    st->n_rel = 1;
  }
  __syncthreads();
  if (!symmetrise_check(s, m.W)) {
    if (threadIdx.x == 0) raise(st, 5, kSubAssembly, 1);
    return;
  }
  double delta;
  const int bad = solve_dev<S>(a, m.W, 1, m.rhs, m.x, &delta, m.scr, a.fast_fgs != 0);
  if (bad) {
    if (threadIdx.x == 0) raise(st, 5, bad, 1);
    return;
  }
  for (int e = threadIdx.x; e < q; e += blockDim.x) a.W[e] = m.W[e];
  for (int e = threadIdx.x; e < s; e += blockDim.x) a.alpha[e] = m.x[e];
  if (threadIdx.x == 0) {
    a.da[0] = delta;
    st->n_da = 1;
    st->k = 1;
  }
}

// End of outer k: stop test on r_k, beta_k = FGS(W_k, -G1), then the
// one-allreduce recurrence W_{k+1} = G2 + G1^T b + b^T G1 + b^T W_k b,
// b1_{k+1} = c1 + b^T c2 and alpha_{k+1}.
template <int S>
__global__ void fast_step_kernel(SmallArgs a) {
  DevState* st = a.st;
  if (halted(st)) return;
  const int s = a.s, q = s * s;
  const int k = st->k;
  const double* pk = a.raw;
  const double* G1 = pk;
  const double* G2 = pk + q;
  const double* c1 = pk + 2 * q;
  const double* c2 = pk + 2 * q + s;
  SmallSmem m = carve(s);
  __shared__ int stop;
  if (threadIdx.x == 0) {
    const double rel = __ddiv_rn(__dsqrt_rn(pk[2 * q + 2 * s]), st->bnorm);
    a.rel[k] = rel;
    st->n_rel = k + 1;
    st->outer_iters = k;
    stop = 0;
    if (rel <= a.tol) {
      st->converged = 1;
      st->done = 1;
      stop = 1;
    } else if (a.flags) {  // multi-rank: the lowest breakdown column of any rank
      for (int j = 0; j < s; ++j)
        if (a.flags[j] != 0.0) {
          st->err = make_err(4, j);
          st->done = 1;
          stop = 1;
          break;
        }
    } else if (st->pending != 0ull) {
      st->err = st->pending;
      st->done = 1;
      stop = 1;
    }
  }
  for (int e = threadIdx.x; e < q; e += blockDim.x) {
    m.W[e] = a.Wexp ? a.Wexp[e] : a.W[e];
    m.rhs[e] = -G1[e];
  }
  __syncthreads();
  if (stop) return;
  // explicit W_k: assembled from this outer's vectors like assemble_gram
  // (gram.cpp:38-49), it replaces the recurrence's W_k for beta_k and as the
  // base of W_{k+1}, so the recurrence error never compounds past one step
  if (a.Wexp && !symmetrise_check(s, m.W)) {
    if (threadIdx.x == 0) raise(st, 5, kSubAssembly, k);
    return;
  }
  double delta;
  int bad = solve_dev<S>(a, m.W, s, m.rhs, m.x, &delta, m.scr, a.fast_fgs != 0);
  if (bad) {
    if (threadIdx.x == 0) raise(st, 5, bad, k);
    return;
  }
  double* beta = m.x;
  for (int e = threadIdx.x; e < q; e += blockDim.x) a.beta[e] = beta[e];
  if (threadIdx.x == 0) {
    a.db[k - 1] = delta;
    st->n_db = k;
  }
  if (k >= a.max_outer) {
    __syncthreads();
    if (threadIdx.x == 0) st->done = 1;
    return;
  }
  // t1 = W_k beta + G1 (so W_{k+1} = G2 + G1^T b + b^T t1)
  for (int e = threadIdx.x; e < q; e += blockDim.x) {
    const int i = e % s, j = e / s;
    double acc = G1[e];
    for (int l = 0; l < s; ++l) acc = fma(m.W[i + l * s], beta[l + j * s], acc);
    m.t1[e] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < q; e += blockDim.x) {
    const int i = e % s, j = e / s;
    double acc = G2[e];
    for (int l = 0; l < s; ++l) acc = fma(G1[l + i * s], beta[l + j * s], acc);
    for (int l = 0; l < s; ++l) acc = fma(beta[l + i * s], m.t1[l + j * s], acc);
    m.Wn[e] = acc;
  }
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    double acc = c1[i];
    for (int l = 0; l < s; ++l) acc = fma(beta[l + i * s], c2[l], acc);
    m.rhs[i] = acc;
  }
  __syncthreads();
  if (!symmetrise_check(s, m.Wn)) {
    if (threadIdx.x == 0) raise(st, 5, kSubAssembly, k + 1);
    return;
  }
  bad = solve_dev<S>(a, m.Wn, 1, m.rhs, m.x, &delta, m.scr, a.fast_fgs != 0);
  if (bad) {
    if (threadIdx.x == 0) raise(st, 5, bad, k + 1);
    return;
  }
  for (int e = threadIdx.x; e < q; e += blockDim.x) a.W[e] = m.Wn[e];
  for (int e = threadIdx.x; e < s; e += blockDim.x) a.alpha[e] = m.x[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    a.da[k] = delta;
    st->n_da = k + 1;
    st->k = k + 1;
  }
}

// ---------------------------------------------------------------- reference mode
// raw layout: [W raw s*s | b1 s | rr 1 | b2 raw s*s]

__global__ void ref_alpha_kernel(SmallArgs a) {
  DevState* st = a.st;
  if (halted(st)) return;
  const int s = a.s, q = s * s, k = st->k;
  SmallSmem m = carve(s);
  for (int e = threadIdx.x; e < q; e += blockDim.x) m.W[e] = a.raw[e];
  for (int e = threadIdx.x; e < s; e += blockDim.x) m.rhs[e] = a.raw[q + e];
  __syncthreads();
  if (!symmetrise_check(s, m.W)) {
    if (threadIdx.x == 0) raise(st, 5, kSubAssembly, k);
    return;
  }
  double delta;
  const int bad = solve_dev(a, m.W, 1, m.rhs, m.x, &delta, m.scr);
  if (bad) {
    if (threadIdx.x == 0) raise(st, 5, bad, k);
    return;
  }
  for (int e = threadIdx.x; e < q; e += blockDim.x) a.W[e] = m.W[e];
  for (int e = threadIdx.x; e < s; e += blockDim.x) a.alpha[e] = m.x[e];
  if (threadIdx.x == 0) {
    a.da[k - 1] = delta;
    st->n_da = k;
  }
}

// rel[k] = ||r_k|| / ||b|| and the stop test (solver.cpp:164-171); k = 0 records rel[0].
__global__ void ref_test_kernel(SmallArgs a) {
  DevState* st = a.st;
  if (halted(st)) return;
  const int s = a.s, k = st->k;
  const double rr = a.raw[s * s + s];
  const double rel = __ddiv_rn(__dsqrt_rn(rr), st->bnorm);
  a.rel[k] = rel;
  st->n_rel = k + 1;
  if (k == 0) {
    st->k = 1;
    return;
  }
  st->outer_iters = k;
  if (rel <= a.tol) {
    st->converged = 1;
    st->done = 1;
  }
}

__global__ void ref_beta_kernel(SmallArgs a) {
  DevState* st = a.st;
  if (halted(st)) return;
  const int s = a.s, q = s * s, k = st->k;
  SmallSmem m = carve(s);
  for (int e = threadIdx.x; e < q; e += blockDim.x) {
    m.W[e] = a.W[e];
    m.rhs[e] = -a.raw[q + s + 1 + e];
  }
  __syncthreads();
  double delta;
  const int bad = solve_dev(a, m.W, s, m.rhs, m.x, &delta, m.scr);
  if (bad) {
    if (threadIdx.x == 0) raise(st, 5, bad, k);
    return;
  }
  for (int e = threadIdx.x; e < q; e += blockDim.x) a.beta[e] = m.x[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    a.db[k - 1] = delta;
    st->n_db = k;
    if (k >= a.max_outer) st->done = 1;
    else st->k = k + 1;
  }
}

// ---------------------------------------------------------------- unit entries

__global__ void unit_fgs_kernel(int s, const double* w, int k, const double* rhs, int nu,
                                double* x, double* delta, int* status) {
  extern __shared__ double sm[];
  double* W = sm;
  double* R = W + s * s;
  double* X = R + s * k;
  double* T = X + s * k;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) W[e] = w[e];
  for (int e = threadIdx.x; e < s * k; e += blockDim.x) R[e] = rhs[e];
  __syncthreads();
  // gram_from_matrix (gram.cpp:51-58): exact symmetry, then finish_assembly
  bool sym = true;
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < j; ++i)
      if (W[i + j * s] != W[j + i * s]) sym = false;
  if (!sym) {
    if (threadIdx.x == 0) *status = 2;
    return;
  }
  for (int i = 0; i < s; ++i) {
    const double d = W[i + i * s];
    if (!(d > 0.0) || !isfinite(d)) {
      if (threadIdx.x == 0) *status = 3 | (kSubAssembly << 8);
      return;
    }
  }
  double dl;
  const int bad = fgs_dev(s, W, k, R, nu, X, &dl, T);
  if (bad) {
    if (threadIdx.x == 0) *status = 3 | (bad << 8);
    return;
  }
  for (int e = threadIdx.x; e < s * k; e += blockDim.x) x[e] = X[e];
  if (threadIdx.x == 0) {
    *delta = dl;
    *status = 0;
  }
}

__global__ void unit_chol_kernel(int s, const double* w, int k, const double* rhs, double* x,
                                 int* status) {
  extern __shared__ double sm[];
  double* W = sm;
  double* R = W + s * s;
  double* X = R + s * k;
  double* L = X + s * k;
  double* T = L + s * s;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) W[e] = w[e];
  for (int e = threadIdx.x; e < s * k; e += blockDim.x) R[e] = rhs[e];
  __syncthreads();
  double dl;
  const int bad = chol_dev(s, W, k, R, X, &dl, L, T);
  if (bad) {
    if (threadIdx.x == 0) *status = 3 | (bad << 8);
    return;
  }
  for (int e = threadIdx.x; e < s * k; e += blockDim.x) x[e] = X[e];
  if (threadIdx.x == 0) *status = 0;
}

__global__ void unit_assemble_kernel(int k, double* w, int* status) {
  extern __shared__ double sm[];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) sm[e] = w[e];
  __syncthreads();
  const bool ok = symmetrise_check(k, sm);
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) w[e] = sm[e];
  if (threadIdx.x == 0) *status = ok ? 0 : (3 | (kSubAssembly << 8));
}

// ---------------------------------------------------------------- classical PCG scalars
// which 0: setup (rel[0], rho); 1: step = rho/pq with the curvature test;
// 2: rel, stop test, beta = rho_new/rho.   dots: [0] pq or rr, [1] rz
__global__ void pcg_scalar_kernel(int which, double tol, int max_iter, DevState* st,
                                  const double* dots, double* rel) {
  if (halted(st)) return;
  const int it = st->k;
  if (which == 0) {
    rel[0] = __ddiv_rn(__dsqrt_rn(dots[0]), st->bnorm);
    st->n_rel = 1;
    st->rho = dots[1];
    st->k = 1;
  } else if (which == 1) {
    const double pq = dots[0];
    if (!(pq > 0.0)) {
      raise(st, 5, kSubPcg, it);
      return;
    }
    st->scal[0] = __ddiv_rn(st->rho, pq);
  } else {
    const double r = __ddiv_rn(__dsqrt_rn(dots[0]), st->bnorm);
    rel[it] = r;
    st->n_rel = it + 1;
    st->outer_iters = it;
    if (r <= tol) {
      st->converged = 1;
      st->done = 1;
      return;
    }
    const double rho_new = dots[1];
    st->scal[1] = __ddiv_rn(rho_new, st->rho);
    st->rho = rho_new;
    if (it >= max_iter) st->done = 1;
    else st->k = it + 1;
  }
}

size_t small_smem(int s) { return static_cast<size_t>(7) * s * s * sizeof(double); }

template <class K>
void launch_small(K kern, const SmallArgs& a, cudaStream_t st) {
  const size_t sm = small_smem(a.s);
  if (sm > 48 * 1024)
    CS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sm)));
  kern<<<1, kSmallThreads, sm, st>>>(a);
  CS_CUDA(cudaGetLastError());
}

}  // namespace

#define CSG_SMALL_DISPATCH(KERNEL, a, st)                    \
  switch ((a).s) {                                          \
    case 2: launch_small(KERNEL<2>, a, st); break;          \
    case 3: launch_small(KERNEL<3>, a, st); break;          \
    case 4: launch_small(KERNEL<4>, a, st); break;          \
    case 5: launch_small(KERNEL<5>, a, st); break;          \
    case 6: launch_small(KERNEL<6>, a, st); break;          \
    case 8: launch_small(KERNEL<8>, a, st); break;          \
    default: launch_small(KERNEL<0>, a, st);                \
  }
void launch_fast_setup(const SmallArgs& a, cudaStream_t s) { CSG_SMALL_DISPATCH(fast_setup_kernel, a, s); }
void launch_fast_step(const SmallArgs& a, cudaStream_t s) { CSG_SMALL_DISPATCH(fast_step_kernel, a, s); }
#undef CSG_SMALL_DISPATCH
void launch_ref_alpha(const SmallArgs& a, cudaStream_t s) { launch_small(ref_alpha_kernel, a, s); }
void launch_ref_test(const SmallArgs& a, cudaStream_t s) {
  ref_test_kernel<<<1, 1, 0, s>>>(a);
  CS_CUDA(cudaGetLastError());
}
void launch_ref_beta(const SmallArgs& a, cudaStream_t s) { launch_small(ref_beta_kernel, a, s); }

void launch_unit_fgs(int s, const double* w, int k, const double* rhs, int nu, double* x,
                     double* delta, int* status, cudaStream_t st) {
  const size_t sm = sizeof(double) * (static_cast<size_t>(s) * s + 3 * static_cast<size_t>(s) * k);
  if (sm > 48 * 1024)
    CS_CUDA(cudaFuncSetAttribute(unit_fgs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sm)));
  unit_fgs_kernel<<<1, kSmallThreads, sm, st>>>(s, w, k, rhs, nu, x, delta, status);
  CS_CUDA(cudaGetLastError());
}

void launch_unit_chol(int s, const double* w, int k, const double* rhs, double* x, int* status,
                      cudaStream_t st) {
  const size_t sm =
      sizeof(double) * (2 * static_cast<size_t>(s) * s + 3 * static_cast<size_t>(s) * k);
  if (sm > 48 * 1024)
    CS_CUDA(cudaFuncSetAttribute(unit_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sm)));
  unit_chol_kernel<<<1, kSmallThreads, sm, st>>>(s, w, k, rhs, x, status);
  CS_CUDA(cudaGetLastError());
}

void launch_unit_assemble(int k, double* w, int* status, cudaStream_t st) {
  unit_assemble_kernel<<<1, kSmallThreads, sizeof(double) * k * k, st>>>(k, w, status);
  CS_CUDA(cudaGetLastError());
}

void launch_pcg_scalar(int which, double tol, int max_iter, DevState* st, const double* dots,
                       double* rel, cudaStream_t s) {
  pcg_scalar_kernel<<<1, 1, 0, s>>>(which, tol, max_iter, st, dots, rel);
  CS_CUDA(cudaGetLastError());
}

}  // namespace csg
