// lanczos.cu -- device kernels of the spectrum estimate (estimate_interval,
// spectral.cpp:60-132): Lanczos on M^-1 A in the M inner product with full
// reorthogonalisation. The basis pairs (v_j, g_j = M v_j) live in two device
// blocks; the Ritz values of the <= 40 x 40 tridiagonal are computed on the
// host from the downloaded coefficients (tridiag.cpp).
//
// Two variants share the kernels:
//  * reference: modified Gram-Schmidt, one serial-order dot + axpy pair per
//    stored vector, exactly the reference operation sequence;
//  * fast: classical Gram-Schmidt -- all projections g_i . r from one pass,
//    the correction from a second pass fused with the r.gr reduction.
#include "kernels.cuh"
#include "lanczos.cuh"

namespace csg {
namespace {

constexpr int kThreads = 256;
inline unsigned grid_for(int64_t n) { return static_cast<unsigned>((n + kThreads - 1) / kThreads); }

__device__ __forceinline__ bool halted(const DevState* st) {
  return *(volatile const int*)&st->done != 0;
}

// r = M^-1 t - a v_j - b v_{j-1}; gr = t - a g_j - b g_{j-1}  (spectral.cpp:93-102)
__global__ void resid_kernel(int64_t n, const double* __restrict__ t,
                             const double* __restrict__ inv_diag, const double* __restrict__ vj,
                             const double* __restrict__ gj, const double* __restrict__ vp,
                             const double* __restrict__ gp, double* r, double* gr,
                             const LanczosScalars* sc, int j, DevState* st) {
  if (halted(st)) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = sc->alpha[j];
  const double tv = t[i];
  double rv = inv_diag ? __dmul_rn(inv_diag[i], tv) : tv;
  double gv = tv;
  rv = __dadd_rn(rv, __dmul_rn(-a, vj[i]));
  gv = __dadd_rn(gv, __dmul_rn(-a, gj[i]));
  if (j > 0) {
    const double b = sc->beta[j - 1];
    rv = __dadd_rn(rv, __dmul_rn(-b, vp[i]));
    gv = __dadd_rn(gv, __dmul_rn(-b, gp[i]));
  }
  r[i] = rv;
  gr[i] = gv;
}

// reference MGS step: r += (-p) v_i ; gr += (-p) g_i with p = sc->proj[0]
__global__ void axpy2_kernel(int64_t n, const double* __restrict__ v, const double* __restrict__ g,
                             double* r, double* gr, const double* proj, DevState* st) {
  if (halted(st)) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double p = *proj;
  r[i] = __dadd_rn(r[i], __dmul_rn(-p, v[i]));
  gr[i] = __dadd_rn(gr[i], __dmul_rn(-p, g[i]));
}

// fast CGS correction over all stored pairs, fused with the r.gr block sums
__global__ void __launch_bounds__(kThreads)
    cgs_kernel(int64_t n, int64_t ld, int m, const double* __restrict__ V,
               const double* __restrict__ G, double* r, double* gr, const double* proj,
               double* partial, unsigned* ticket, double* result, DevState* st) {
  if (halted(st)) return;
  __shared__ double sp[kLanczosMax];
  __shared__ double red[kThreads / 32];
  __shared__ bool last;
  for (int t = threadIdx.x; t < m; t += blockDim.x) sp[t] = proj[t];
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double d = 0.0;
  if (i < n) {
    double rv = r[i], gv = gr[i];
    for (int c = 0; c < m; ++c) {
      rv = fma(-sp[c], V[c * ld + i], rv);
      gv = fma(-sp[c], G[c * ld + i], gv);
    }
    r[i] = rv;
    gr[i] = gv;
    d = rv * gv;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) d += __shfl_down_sync(0xffffffffu, d, off);
  if (lane == 0) red[warp] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    finalize_partials(partial, gridDim.x, 1, result);
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

// scalar steps: 0 normalise start (nrm = sqrt(v.g) > 0), 1 alpha_j (finite),
// 2 beta_j = sqrt(max(0, r.gr)) with the invariant-subspace exit.
__global__ void scalar_kernel(int which, int j, int steps, LanczosScalars* sc, DevState* st) {
  if (halted(st)) return;
  const double d = sc->dot;
  if (which == 0) {
    const double nrm = __dsqrt_rn(d);
    if (!(nrm > 0.0)) {
      atomicCAS(&st->err, 0ull, make_err(9 | (1 << 8), 0));
      st->done = 1;
      return;
    }
    sc->denom = nrm;
  } else if (which == 1) {
    if (!isfinite(d)) {
      atomicCAS(&st->err, 0ull, make_err(9 | (2 << 8), j));
      st->done = 1;
      return;
    }
    sc->alpha[j] = d;
    sc->count = j + 1;
  } else {
    const double bj = __dsqrt_rn(0.0 < d ? d : 0.0);  // std::max(0.0, d)
    if (!isfinite(bj)) {
      atomicCAS(&st->err, 0ull, make_err(9 | (2 << 8), j));
      st->done = 1;
      return;
    }
    if (bj == 0.0) {
      st->done = 1;  // invariant subspace: use the completed steps
      return;
    }
    if (j + 1 < steps) {
      sc->beta[j] = bj;
      sc->denom = bj;
    } else {
      st->done = 1;
    }
  }
}

}  // namespace

void lz_resid(int64_t n, const double* t, const double* inv_diag, const double* vj,
              const double* gj, const double* vp, const double* gp, double* r, double* gr,
              const LanczosScalars* sc, int j, DevState* st, cudaStream_t s) {
  if (n == 0) return;
  resid_kernel<<<grid_for(n), kThreads, 0, s>>>(n, t, inv_diag, vj, gj, vp, gp, r, gr, sc, j, st);
  CS_CUDA(cudaGetLastError());
}

void lz_axpy2(int64_t n, const double* v, const double* g, double* r, double* gr,
              const double* proj, DevState* st, cudaStream_t s) {
  if (n == 0) return;
  axpy2_kernel<<<grid_for(n), kThreads, 0, s>>>(n, v, g, r, gr, proj, st);
  CS_CUDA(cudaGetLastError());
}

int lz_cgs_blocks(int64_t n) { return static_cast<int>(grid_for(n > 0 ? n : 1)); }

void lz_cgs(int64_t n, int64_t ld, int m, const double* V, const double* G, double* r, double* gr,
            const double* proj, double* partial, unsigned* ticket, double* result, DevState* st,
            cudaStream_t s) {
  cgs_kernel<<<grid_for(n > 0 ? n : 1), kThreads, 0, s>>>(n, ld, m, V, G, r, gr, proj, partial,
                                                         ticket, result, st);
  CS_CUDA(cudaGetLastError());
}

void lz_scalar(int which, int j, int steps, LanczosScalars* sc, DevState* st, cudaStream_t s) {
  scalar_kernel<<<1, 1, 0, s>>>(which, j, steps, sc, st);
  CS_CUDA(cudaGetLastError());
}

}  // namespace csg
