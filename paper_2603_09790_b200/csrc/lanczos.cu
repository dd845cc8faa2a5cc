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
#include <algorithm>
#include <cstdlib>

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
// mt != nullptr: M^-1 t was applied already (general preconditioners), r may alias it
__global__ void resid_kernel(int64_t n, const double* __restrict__ t,
                             const double* __restrict__ inv_diag, const double* mt,
                             const double* __restrict__ vj, const double* __restrict__ gj,
                             const double* __restrict__ vp, const double* __restrict__ gp,
                             double* r, double* gr, const LanczosScalars* sc, int j, DevState* st) {
  if (halted(st)) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = sc->alpha[j];
  const double tv = t[i];
  double rv = mt ? mt[i] : inv_diag ? __dmul_rn(inv_diag[i], tv) : tv;
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

// fast CGS correction over all stored pairs, fused with the r.gr block sums.
// MB > 0: at most MB pairs, the loop unrolled so every row's 2m loads are in
// flight together (a runtime-bounded loop issued them two at a time).
template <int MB>
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
    if constexpr (MB > 0) {
      // chunks of 8 pairs: 16 loads in flight per thread at a register count
      // that keeps several blocks resident (all 2m at once needed ~200 registers)
      constexpr int kC = 8;  // 16 measured slower (Lanczos 59.5 -> 75.5 ms at 256^3)
#pragma unroll 1
      for (int c0 = 0; c0 < MB; c0 += kC) {
        if (c0 >= m) break;
        double vv[kC], gg[kC];
#pragma unroll
        for (int c = 0; c < kC; ++c)
          if (c0 + c < m) {
            vv[c] = __ldcs(V + (c0 + c) * ld + i);
            gg[c] = __ldcs(G + (c0 + c) * ld + i);
          }
#pragma unroll
        for (int c = 0; c < kC; ++c)
          if (c0 + c < m) {
            rv = fma(-sp[c0 + c], vv[c], rv);
            gv = fma(-sp[c0 + c], gg[c], gv);
          }
      }
    } else {
      for (int c = 0; c < m; ++c) {
        rv = fma(-sp[c], V[c * ld + i], rv);
        gv = fma(-sp[c], G[c * ld + i], gv);
      }
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

// fast CGS projections proj[i] = g_i . r for i < m in ONE pass: r is read
// once, each g_i once; every thread keeps m accumulators over a grid-stride
// row sweep (fixed grid: deterministic), then a fixed warp/block tree and
// last-block finalisation in block order.
// Grid: one wave of resident blocks at the kernel's occupancy (a fixed 296-block
// grid left the 60-80-register instances at 16 warps/SM with too few loads in
// flight: 1.7 TB/s at m = 12..20, profiles/r02h_launches_head_256_summary.txt).
// Fixed per device and kernel, so the reduction order is run-to-run identical.
constexpr int kProjBlocks = 296;      // legacy fixed grid (CS_LZ_GRID=0)
constexpr int kProjMaxBlocks = 148 * 8;

template <typename K>
int proj_grid(K kern) {
  static const bool fixed = [] {
    const char* e = std::getenv("CS_LZ_GRID");
    return e != nullptr && std::atoi(e) == 0;
  }();
  if (fixed) return kProjBlocks;
  const int per_sm = kernel_setup(reinterpret_cast<const void*>(kern), kThreads, 0);
  return std::min(148 * per_sm, kProjMaxBlocks);
}

template <int MB>
__global__ void __launch_bounds__(kThreads)
    proj_kernel(int64_t n, int64_t ld, int m, const double* __restrict__ G,
                const double* __restrict__ r, double* proj, double* partial, unsigned* ticket,
                DevState* st) {
  if (halted(st)) return;
  __shared__ double red[MB][kThreads / 32];
  __shared__ bool last;
  double acc[MB];
#pragma unroll
  for (int c = 0; c < MB; ++c) acc[c] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    double gg[MB];  // every load of the row in flight before the FMA chain
#pragma unroll
    for (int c = 0; c < MB; ++c) gg[c] = c < m ? __ldcs(G + c * ld + i) : 0.0;
    const double rv = __ldcs(r + i);
#pragma unroll
    for (int c = 0; c < MB; ++c)
      if (c < m) acc[c] = fma(gg[c], rv, acc[c]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < MB; ++c) {
    if (c < m) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[c] += __shfl_down_sync(0xffffffffu, acc[c], off);
      if (lane == 0) red[c][warp] = acc[c];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < m; c += kThreads) {
    double sum = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) sum += red[c][w];
    partial[static_cast<int64_t>(blockIdx.x) * m + c] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_partials(partial, gridDim.x, m, proj);
  if (threadIdx.x == 0) *ticket = 0u;
}

// ---- G-only Lanczos (fast mode, diagonal M = D: identity or Jacobi). The M
// inner-product pairs satisfy v = D^-1 g and r = D^-1 gr exactly in exact
// arithmetic, so only the g_j are stored (half the basis: 43 GB at 512^3) and
// v, r are formed per row where needed (dinv: a_ii^-1 vector, or the uniform
// constant dconst when dinv is null).

// gr = t - a g_j - b g_{j-1} (spectral.cpp:93-102 on the g side), written, and
// in the same pass proj_i = g_i . (D^-1 gr) for i < m = j + 1
template <int MB>
__global__ void __launch_bounds__(kThreads)
    lz2_resid_proj_kernel(int64_t n, int64_t ld, int m, const double* __restrict__ t,
                          const double* __restrict__ G, const double* __restrict__ dinv,
                          double dconst, double* gr, const LanczosScalars* sc, int j,
                          double* proj, double* partial, unsigned* ticket, DevState* st) {
  if (halted(st)) return;
  __shared__ double red[MB][kThreads / 32];
  __shared__ bool last;
  const double a = sc->alpha[j], b = j > 0 ? sc->beta[j - 1] : 0.0;
  double acc[MB];
#pragma unroll
  for (int c = 0; c < MB; ++c) acc[c] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    // every basis load of the row first (ncu: with the loads interleaved into
    // the FMA chain one load was in flight per thread, 2.2 TB/s)
    double gg[MB];
    const double* gi = G + i;
#pragma unroll
    for (int c = 0; c < MB; ++c) gg[c] = c < m ? __ldcs(gi + c * ld) : 0.0;
    const double tv = __ldcs(t + i);
    const double di = dinv ? __ldg(dinv + i) : dconst;
    const double gj = __ldg(gi + j * ld), gj1 = j > 0 ? __ldg(gi + (j - 1) * ld) : 0.0;
    double gv = fma(-a, gj, tv);
    if (j > 0) gv = fma(-b, gj1, gv);
    gr[i] = gv;
    const double rv = gv * di;
#pragma unroll
    for (int c = 0; c < MB; ++c)
      if (c < m) acc[c] = fma(gg[c], rv, acc[c]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < MB; ++c) {
    if (c < m) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[c] += __shfl_down_sync(0xffffffffu, acc[c], off);
      if (lane == 0) red[c][warp] = acc[c];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < m; c += kThreads) {
    double sum = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) sum += red[c][w];
    partial[static_cast<int64_t>(blockIdx.x) * m + c] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_partials(partial, gridDim.x, m, proj);
  if (threadIdx.x == 0) *ticket = 0u;
}

// gr -= sum_i proj_i g_i (8-column chunks), fused with the dot (D^-1 gr) . gr
__global__ void __launch_bounds__(kThreads)
    lz2_cgs_kernel(int64_t n, int64_t ld, int m, const double* __restrict__ G,
                   const double* __restrict__ dinv, double dconst, double* gr, const double* proj,
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
    double gv = gr[i];
    constexpr int kC = 8;  // 16 measured slower (Lanczos 59.5 -> 75.5 ms at 256^3)
#pragma unroll 1
    for (int c0 = 0; c0 < m; c0 += kC) {
      double gg[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c)
        if (c0 + c < m) gg[c] = __ldcs(G + (c0 + c) * ld + i);
#pragma unroll
      for (int c = 0; c < kC; ++c)
        if (c0 + c < m) gv = fma(-sp[c0 + c], gg[c], gv);
    }
    gr[i] = gv;
    d = gv * (dinv ? __ldg(dinv + i) : dconst) * gv;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) d += __shfl_down_sync(0xffffffffu, d, off);
  if (lane == 0) red[warp] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) sum += red[w];
    partial[blockIdx.x] = sum;
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

// g_{j+1} = gr / beta_j, v = D^-1 g_{j+1}
__global__ void lz2_scale_kernel(int64_t n, const double* __restrict__ gr,
                                 const double* __restrict__ dinv, double dconst, double* g,
                                 double* v, const LanczosScalars* sc, DevState* st) {
  if (halted(st)) return;
  // one reciprocal per step, not a division per row (fast mode only; the
  // reference-order Lanczos keeps its divisions); a grid-stride sweep so the
  // state and scalar loads are paid once per thread, not once per row
  const double rd = sc->rdenom;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double gv = gr[i] * rd;
    g[i] = gv;
    v[i] = gv * (dinv ? dinv[i] : dconst);
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
    sc->rdenom = 1.0 / nrm;
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
      sc->rdenom = 1.0 / bj;
    } else {
      st->done = 1;
    }
  }
}

}  // namespace

void lz_resid(int64_t n, const double* t, const double* inv_diag, const double* mt,
              const double* vj, const double* gj, const double* vp, const double* gp, double* r,
              double* gr, const LanczosScalars* sc, int j, DevState* st, cudaStream_t s) {
  if (n == 0) return;
  resid_kernel<<<grid_for(n), kThreads, 0, s>>>(n, t, inv_diag, mt, vj, gj, vp, gp, r, gr, sc, j,
                                                st);
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
  const unsigned grid = grid_for(n > 0 ? n : 1);
#define CSG_CGS(MB) \
  cgs_kernel<MB><<<grid, kThreads, 0, s>>>(n, ld, m, V, G, r, gr, proj, partial, ticket, result, st)
  if (m <= 8) CSG_CGS(8);
  else if (m <= 16) CSG_CGS(16);
  else if (m <= 24) CSG_CGS(24);
  else if (m <= 32) CSG_CGS(32);
  else if (m <= 40) CSG_CGS(40);
  else CSG_CGS(0);
#undef CSG_CGS
  CS_CUDA(cudaGetLastError());
}

void lz2_resid_proj(int64_t n, int64_t ld, int m, const double* t, const double* G,
                    const double* dinv, double dconst, double* gr, const LanczosScalars* sc, int j,
                    double* proj, double* partial, unsigned* ticket, DevState* st, cudaStream_t s) {
#define CSG_RP(MB)                                                                          \
  lz2_resid_proj_kernel<MB><<<proj_grid(lz2_resid_proj_kernel<MB>), kThreads, 0, s>>>(      \
      n, ld, m, t, G, dinv, dconst, gr, sc, j, proj, partial, ticket, st)
  if (m <= 8) CSG_RP(8);
  else if (m <= 16) CSG_RP(16);
  else if (m <= 24) CSG_RP(24);
  else if (m <= 32) CSG_RP(32);
  else CSG_RP(40);
#undef CSG_RP
  CS_CUDA(cudaGetLastError());
}

void lz2_cgs(int64_t n, int64_t ld, int m, const double* G, const double* dinv, double dconst,
             double* gr, const double* proj, double* partial, unsigned* ticket, double* result,
             DevState* st, cudaStream_t s) {
  lz2_cgs_kernel<<<grid_for(n > 0 ? n : 1), kThreads, 0, s>>>(n, ld, m, G, dinv, dconst, gr, proj,
                                                             partial, ticket, result, st);
  CS_CUDA(cudaGetLastError());
}

void lz2_scale(int64_t n, const double* gr, const double* dinv, double dconst, double* g, double* v,
               const LanczosScalars* sc, DevState* st, cudaStream_t s) {
  if (n == 0) return;
  const unsigned grid = std::min<unsigned>(grid_for(n), 148u * 8u);
  lz2_scale_kernel<<<grid, kThreads, 0, s>>>(n, gr, dinv, dconst, g, v, sc, st);
  CS_CUDA(cudaGetLastError());
}

bool lz_proj_supported(int m) { return m >= 1 && m <= 40; }

size_t lz_proj_partial_doubles(int m) { return static_cast<size_t>(kProjMaxBlocks) * m; }

void lz_proj(int64_t n, int64_t ld, int m, const double* G, const double* r, double* proj,
             double* partial, unsigned* ticket, DevState* st, cudaStream_t s) {
#define CSG_PROJ(MB)                                                               \
  proj_kernel<MB><<<proj_grid(proj_kernel<MB>), kThreads, 0, s>>>(n, ld, m, G, r, proj, \
                                                                  partial, ticket, st)
  if (m <= 8) CSG_PROJ(8);
  else if (m <= 16) CSG_PROJ(16);
  else if (m <= 24) CSG_PROJ(24);
  else if (m <= 32) CSG_PROJ(32);
  else CSG_PROJ(40);
#undef CSG_PROJ
  CS_CUDA(cudaGetLastError());
}

void lz_scalar(int which, int j, int steps, LanczosScalars* sc, DevState* st, cudaStream_t s) {
  scalar_kernel<<<1, 1, 0, s>>>(which, j, steps, sc, st);
  CS_CUDA(cudaGetLastError());
}

}  // namespace csg
