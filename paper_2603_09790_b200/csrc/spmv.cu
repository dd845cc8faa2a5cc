// spmv.cu -- SELL-32 FP64 SpMV fused with the Chebyshev matrix-power-kernel
// epilogue (the dominant kernel of the solve).
//
// One warp owns one slice (32 consecutive rows, lane = row). Per slot k a
// warp streams 256 B of values and 128 B of int32 columns with
// evict-first (ld.global.cs) loads so the L2 keeps the x planes resident,
// gathers x[col] through the read-only path, and accumulates the row with
// separate multiply and add roundings in the stored column order:
// acc = acc + v*x exactly as csr.cpp:116-121 (no FMA), so y is bitwise the
// reference SpMV. Padding slots carry col = -1 and are skipped.
//
// Epilogues (each basis vector is written exactly once):
//   kPlain     y = A x
//   kResid     r = b - A x                               (solver.cpp:119-121)
//   kMpkFirst  p_1 = A z_0; zp_1 = lincomb3(a, p_1, -s, zp_0, 0, zp_0);
//              z_1 = M^-1 zp_1; finite check                (mpk.cpp:55-59)
//   kMpkMid    p_q = A z_{q-1}; zp_q = lincomb3(2a, p_q, -2s, zp_{q-1}, -g, zp_{q-2});
//              z_q = M^-1 zp_q; finite check                (mpk.cpp:60-66)
//   kMpkLast   p_s = A z_{s-1}; finite check on p_s (label s-1, mpk.cpp:68-69)
//   kDot       y = A x and the deterministic block sum of x.y (classical PCG p.q)
//   kMpkFirstF/kMpkMidF (fast algebra only): with Jacobi zp_j = D z_j, so
//              z_q = 2a D^-1 p_q - 2s z_{q-1} - z_{q-2}  (first step: a, -s, no z_{q-2});
//              D = a_ii and z_{q-1}[row] are picked up by the row loop itself, so
//              the step reads/writes 24n fewer bytes than the reference recurrence.
#include "kernels.cuh"

namespace csg {
namespace {

constexpr int kWarps = 8;  // slices per 256-thread block

__device__ __forceinline__ void report(const SpmvArgs& g, int col) {
  if (g.st == nullptr) return;
  unsigned long long* w = g.pending ? &g.st->pending : &g.st->err;
  atomicCAS(w, 0ull, make_err(4 /*CS_ERR_BASIS_BREAKDOWN*/, col));
  if (!g.pending) g.st->done = 1;
}

template <int KIND, bool JAC>
__global__ void __launch_bounds__(kWarps * 32)
    sell_kernel(SellView a, SpmvArgs g, int64_t slice_begin, int64_t slice_end) {
  if (g.st != nullptr && *(volatile int*)&g.st->done) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t slice = slice_begin + static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  const bool active = slice < slice_end;
  double acc = 0.0, dval = 1.0, xd = 0.0;
  int64_t row = 0;
  if (active) {
    row = slice * kSliceRows + lane;
    const int64_t base = a.slice_ptr[slice];
    const int width = static_cast<int>((a.slice_ptr[slice + 1] - base) >> 5);
    const double* vp = a.vals + base + lane;
    const double* __restrict__ x = g.x;
    auto term = [&](int32_t c, double v) {
      const double xv = __ldg(x + c);
      acc = __dadd_rn(acc, __dmul_rn(v, xv));
      if constexpr (KIND == kMpkFirstF || KIND == kMpkMidF) {
        if (c == row) {
          dval = v;
          xd = xv;
        }
      }
    };
    const int64_t m = a.meta[slice];
    if (m >= 0) {  // explicit int32 columns
      const int32_t* cp = a.cols + m + lane;
#pragma unroll 9
      for (int k = 0; k < width; ++k) {
        const int32_t c = __ldcs(cp + k * kSliceRows);
        const double v = __ldcs(vp + k * kSliceRows);
        if (c >= 0) term(c, v);
      }
    } else {  // shared relative-offset pattern: column = row + off_k where lane bit set
      const int2* pp = a.pat + (-m - 1);
#pragma unroll 9
      for (int k = 0; k < width; ++k) {
        const int2 e = __ldg(pp + k);
        const double v = __ldcs(vp + k * kSliceRows);
        if ((e.y >> lane) & 1) term(static_cast<int32_t>(row + e.x), v);
      }
    }
  }
  const bool own = active && row < a.n_local;
  double dotv = 0.0;
  if (own) {
    if constexpr (KIND == kPlain) {
      g.y[row] = acc;
    } else if constexpr (KIND == kResid) {
      g.y[row] = __dsub_rn(g.b[row], acc);
    } else if constexpr (KIND == kMpkFirst || KIND == kMpkMid) {
      g.y[row] = acc;
      const double y1 = g.zp1[row];
      const double y2 = (KIND == kMpkFirst) ? y1 : g.zp2[row];
      const double t = __dadd_rn(__dmul_rn(g.ca, acc), __dmul_rn(g.cb, y1));
      const double zp = __dadd_rn(t, __dmul_rn(g.cc, y2));
      double z = zp;
      if constexpr (JAC) {
        g.zpout[row] = zp;
        z = __dmul_rn(a.inv_diag[row], zp);
      }
      g.zout[row] = z;
      if (!isfinite(z)) report(g, g.col);
    } else if constexpr (KIND == kMpkFirstF || KIND == kMpkMidF) {
      g.y[row] = acc;
      if constexpr (!JAC) xd = g.x[row];  // identity: z_{q-1}[row] even without a stored diagonal
      const double dp = JAC ? acc / dval : acc;
      double z = fma(g.cb, xd, g.ca * dp);
      if constexpr (KIND == kMpkMidF) z = fma(g.cc, g.zp2[row], z);
      g.zout[row] = z;
      if (!isfinite(z)) report(g, g.col);
    } else if constexpr (KIND == kMpkLast) {
      g.y[row] = acc;
      if (!isfinite(acc)) report(g, g.col);
    } else if constexpr (KIND == kDot) {
      g.y[row] = acc;
      dotv = g.x[row] * acc;
    }
  }
  if constexpr (KIND == kDot) {
    // fixed-shape tree: warp shuffle, then warp 0 over the 8 warp sums
    __shared__ double red[kWarps];
    __shared__ bool last;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dotv += __shfl_down_sync(0xffffffffu, dotv, off);
    if (lane == 0) red[warp] = dotv;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += red[w];
      g.partial[blockIdx.x] = s;
      __threadfence();
      const unsigned t = atomicAdd(g.ticket, 1u);
      last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      finalize_partials(g.partial, gridDim.x, 1, g.result);
      if (threadIdx.x == 0) *g.ticket = 0u;
    }
  }
}

template <int KIND>
void launch_kind(bool jac, const SellView& a, const SpmvArgs& g, int64_t sb, int64_t se,
                 cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((se - sb + kWarps - 1) / kWarps);
  if (jac)
    sell_kernel<KIND, true><<<grid, kWarps * 32, 0, st>>>(a, g, sb, se);
  else
    sell_kernel<KIND, false><<<grid, kWarps * 32, 0, st>>>(a, g, sb, se);
}

}  // namespace

int spmv_dot_blocks(int64_t nslices) { return static_cast<int>((nslices + kWarps - 1) / kWarps); }

void launch_spmv(int kind, const SellView& a, const SpmvArgs& g, int64_t sb, int64_t se,
                 cudaStream_t st) {
  if (se <= sb) return;
  const bool jac = a.inv_diag != nullptr;
  switch (kind) {
    case kPlain: launch_kind<kPlain>(false, a, g, sb, se, st); break;
    case kResid: launch_kind<kResid>(false, a, g, sb, se, st); break;
    case kMpkFirst: launch_kind<kMpkFirst>(jac, a, g, sb, se, st); break;
    case kMpkMid: launch_kind<kMpkMid>(jac, a, g, sb, se, st); break;
    case kMpkLast: launch_kind<kMpkLast>(false, a, g, sb, se, st); break;
    case kDot: launch_kind<kDot>(false, a, g, sb, se, st); break;
    case kMpkFirstF: launch_kind<kMpkFirstF>(jac, a, g, sb, se, st); break;
    case kMpkMidF: launch_kind<kMpkMidF>(jac, a, g, sb, se, st); break;
    default: throw LibError{9, 0, "bad spmv kind"};
  }
  CS_CUDA(cudaGetLastError());
}

}  // namespace csg
