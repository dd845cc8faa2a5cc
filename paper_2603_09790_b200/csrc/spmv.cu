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
#include <algorithm>
#include <cstdint>
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"

namespace csg {
namespace {

constexpr int kWarps = 8;  // warps per 256-thread block
#ifndef CS_SPMV_MINB
#define CS_SPMV_MINB 8  // 32 registers: full occupancy (64 warps / SM)
#endif
#ifndef CS_CD_KB
#define CS_CD_KB 9  // CDIA gathers in flight per batch
#endif
#ifndef CS_SPMV_ZB
#define CS_SPMV_ZB 1
#endif
#ifndef CS_SPMV_ZB_MINB
#define CS_SPMV_ZB_MINB 3  // z-blocked kernel: two planes of gathers in flight
#endif
#ifndef CS_SPMV_CD_MINB
#define CS_SPMV_CD_MINB 4  // CDIA kernel: 64 registers (all x gathers of a row in flight)
#endif
#ifndef CS_SPMV_PERSIST
#define CS_SPMV_PERSIST 1
#endif

__device__ __forceinline__ void report(const SpmvArgs& g, int col) {
  if (g.st == nullptr || col < 0) return;  // col < 0: checked after a separate apply
  unsigned long long* w = g.pending ? &g.st->pending : &g.st->err;
  atomicCAS(w, 0ull, make_err(4 /*CS_ERR_BASIS_BREAKDOWN*/, col));
  if (!g.pending) g.st->done = 1;
}

struct SliceMeta {
  int64_t base, end, meta;
};

template <bool UNI = false>
__device__ __forceinline__ SliceMeta load_meta(const SellView& a, int64_t slice, int64_t se) {
  SliceMeta m{0, 0, make_pat_meta(0, 0)};
  if (slice < se) {
    if constexpr (!UNI) {  // uniform slices have no value slots
      m.base = a.slice_ptr[slice];
      m.end = a.slice_ptr[slice + 1];
    }
    m.meta = a.meta[slice];
  }
  return m;
}

constexpr int kStabMax = 1024;  // uniform-table entries staged per block (16 KB)

__device__ __forceinline__ int stage_tables(const SellView& a, SlotRec* stab) {
  const int staged = a.table_entries < kStabMax ? static_cast<int>(a.table_entries) : kStabMax;
  for (int i = threadIdx.x; i < staged; i += blockDim.x) {
    const int2 e = __ldg(a.pat + i);
    stab[i] = SlotRec{e.x, static_cast<unsigned>(e.y), __ldg(a.pval + i)};
  }
  __syncthreads();
  return staged;
}

// One row of one slice: sum_k v_k * x[c_k] in stored order, acc = acc + v*x.
// CDIA row: the class table is a kernel parameter, so t.off[k] / t.v[k] are
// immediate constant-bank operands of the unrolled loop (no table loads at all;
// ncu showed shared-memory table broadcasts costing as many L1 wavefronts as
// the x gathers, and register-indexed constant loads saturating the ADU pipe).
// N > 0: the class has exactly N offsets (compile time: no per-slot bound
// tests; the common stencils, 7 and 27). N == 0: runtime t.n.
// Gathers are issued in batches of kB (a batch's loads in flight together),
// then the batch's products are added in slot order. Slices whose 32 rows all
// hold every entry (a stencil's interior) skip the per-slot predicates; bits at
// or above t.n are zero by construction.
template <int N>
__device__ __forceinline__ double row_sum_cdia(const CdiaTable& t, const double* __restrict__ x,
                                               int r32, uint32_t bits) {
  constexpr int kB = N > 0 ? (CS_CD_KB < N ? CS_CD_KB : N) : 8;
  constexpr int kMax = N > 0 ? N : kCdiaMax;
  const int n = N > 0 ? N : t.n;
  double acc = 0.0;
  const uint32_t full = n >= 32 ? 0xffffffffu : (1u << n) - 1u;
  if (__all_sync(0xffffffffu, bits == full)) {
#pragma unroll
    for (int c = 0; c < kMax; c += kB) {
      if (N == 0 && c >= n) break;
      double xv[kB];
#pragma unroll
      for (int j = 0; j < kB; ++j)
        if (c + j < kMax && (N > 0 || c + j < n)) xv[j] = __ldg(x + (r32 + t.off[c + j]));
#pragma unroll
      for (int j = 0; j < kB; ++j)
        if (c + j < kMax && (N > 0 || c + j < n))
          acc = __dadd_rn(acc, __dmul_rn(t.v[c + j], xv[j]));
    }
    return acc;
  }
#pragma unroll
  for (int c = 0; c < kMax; c += kB) {
    if (N == 0 && c >= n) break;
    double xv[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const bool on = c + j < kMax && ((bits >> (c + j)) & 1u);
      xv[j] = on ? __ldg(x + (r32 + t.off[c + j])) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kB; ++j)
      if (c + j < kMax && ((bits >> (c + j)) & 1u))
        acc = __dadd_rn(acc, __dmul_rn(t.v[c + j], xv[j]));
  }
  return acc;
}

__device__ __forceinline__ double row_sum(const SellView& a, const double* __restrict__ x,
                                          const SliceMeta& sm, int64_t row, int lane,
                                          const SlotRec* stab, int staged) {
  double acc = 0.0;
  const int width = static_cast<int>((sm.end - sm.base) >> 5);
  const double* vp = a.vals + sm.base + lane;
  if (sm.meta >= 0) {  // explicit int32 columns
    const int32_t* cp = a.cols + sm.meta + lane;
#pragma unroll 9
    for (int k = 0; k < width; ++k) {
      const int32_t c = __ldcs(cp + k * kSliceRows);
      const double v = __ldcs(vp + k * kSliceRows);
      if (c >= 0) acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + c)));
    }
  } else if (const int U = pat_uniform(sm.meta); U > 0) {  // uniform values, no value slots
    const int64_t pi = pat_index(sm.meta);
    if (pi + U <= staged) {  // table in shared memory
      const SlotRec* t = stab + pi;
      const double* xr = x + row;
#pragma unroll 9
      for (int k = 0; k < U; ++k) {
        const SlotRec e = t[k];
        if ((e.mask >> lane) & 1u) acc = __dadd_rn(acc, __dmul_rn(e.v, __ldg(xr + e.off)));
      }
    } else if (U <= 32) {
      // lane k holds table entry k; {off, mask, value} of every slot arrive by shuffle
      const int2 pl = lane < U ? __ldg(a.pat + pi + lane) : make_int2(0, 0);
      const double pv = lane < U ? __ldg(a.pval + pi + lane) : 0.0;
#pragma unroll 9
      for (int k = 0; k < U; ++k) {
        const int off = __shfl_sync(0xffffffffu, pl.x, k);
        const unsigned msk = static_cast<unsigned>(__shfl_sync(0xffffffffu, pl.y, k));
        const double v = __shfl_sync(0xffffffffu, pv, k);
        if ((msk >> lane) & 1u) acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + row + off)));
      }
    } else {
      for (int k = 0; k < U; ++k) {
        const int2 e = __ldg(a.pat + pi + k);
        const double v = __ldg(a.pval + pi + k);
        if ((e.y >> lane) & 1) acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + row + e.x)));
      }
    }
  } else if (width <= 32) {  // shared relative-offset pattern: column = row + off_k
    // lane k holds pattern entry k; every slot's {off, mask} arrives by shuffle
    const int2* pp = a.pat + pat_index(sm.meta);
    const int2 pl = lane < width ? __ldg(pp + lane) : make_int2(0, 0);
#pragma unroll 9
    for (int k = 0; k < width; ++k) {
      const int off = __shfl_sync(0xffffffffu, pl.x, k);
      const unsigned msk = static_cast<unsigned>(__shfl_sync(0xffffffffu, pl.y, k));
      const double v = __ldcs(vp + k * kSliceRows);
      if ((msk >> lane) & 1u) acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + row + off)));
    }
  } else {  // wide pattern: broadcast entry loads
    const int2* pp = a.pat + pat_index(sm.meta);
    for (int k = 0; k < width; ++k) {
      const int2 e = __ldg(pp + k);
      const double v = __ldcs(vp + k * kSliceRows);
      if ((e.y >> lane) & 1) acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + row + e.x)));
    }
  }
  return acc;
}

// ------------------------------------------------------------------ shared pieces

struct EpiOps {
  double e1 = 0.0, e2 = 0.0, einv = 1.0, exd = 0.0;
};

// epilogue operands of one row, loaded ahead of (independent of) the row sum
// cinv != 0: the CDIA class's uniform Jacobi scale 1/a_ii (bitwise the
// inv_diag entry, precond.cpp:22), so the D^-1 vector is not streamed.
template <int KIND, bool JAC>
__device__ __forceinline__ EpiOps epi_load(const SellView& a, const SpmvArgs& g, int64_t row,
                                           double cinv = 0.0) {
  EpiOps e;
  if constexpr (KIND == kResid) e.e1 = g.b[row];
  if constexpr (KIND == kResidF) {
    e.e1 = g.b[row];
    if constexpr (JAC) e.einv = cinv != 0.0 ? cinv : a.inv_diag[row];
  }
  if constexpr (KIND == kMpkFirst || KIND == kMpkMid) {
    e.e1 = g.zp1[row];
    if constexpr (KIND == kMpkMid) e.e2 = g.zp2[row];
    if constexpr (JAC) e.einv = cinv != 0.0 ? cinv : a.inv_diag[row];
  }
  if constexpr (KIND == kMpkFirstF || KIND == kMpkMidF) {
    e.exd = g.x[row];
    if constexpr (KIND == kMpkMidF) e.e2 = g.zp2[row];
    if constexpr (JAC) e.einv = cinv != 0.0 ? cinv : a.inv_diag[row];
  }
  if constexpr (KIND == kDot) e.exd = g.x[row];
  return e;
}

template <int KIND, bool JAC>
__device__ __forceinline__ void epi_store(const SpmvArgs& g, int64_t row, double acc,
                                          const EpiOps& e, double& dotv, double& zv) {
  if constexpr (KIND == kPlain) {
    g.y[row] = acc;
  } else if constexpr (KIND == kResid) {
    g.y[row] = __dsub_rn(e.e1, acc);
  } else if constexpr (KIND == kResidF) {
    const double r = e.e1 - acc;
    if (g.y) g.y[row] = r;  // nullptr: the pack forms r = D z_0
    const double z = JAC ? r * e.einv : r;
    g.zout[row] = z;
    zv = z;
    if (!isfinite(z)) report(g, g.col);
  } else if constexpr (KIND == kMpkFirst || KIND == kMpkMid) {
    g.y[row] = acc;
    const double y2 = (KIND == kMpkFirst) ? e.e1 : e.e2;
    const double t = __dadd_rn(__dmul_rn(g.ca, acc), __dmul_rn(g.cb, e.e1));
    const double zp = __dadd_rn(t, __dmul_rn(g.cc, y2));
    double z = zp;
    if constexpr (JAC) {
      g.zpout[row] = zp;
      z = __dmul_rn(e.einv, zp);
    }
    g.zout[row] = z;
    if (!isfinite(z)) report(g, g.col);
  } else if constexpr (KIND == kMpkFirstF || KIND == kMpkMidF) {
    if (g.y) g.y[row] = acc;  // nullptr: P derived from Z later (PZ schedule)
    const double dp = JAC ? acc * e.einv : acc;
    double z = fma(g.cb, e.exd, g.ca * dp);
    if constexpr (KIND == kMpkMidF) z = fma(g.cc, e.e2, z);
    g.zout[row] = z;
    zv = z;
    if (!isfinite(z)) report(g, g.col);
  } else if constexpr (KIND == kMpkLast) {
    g.y[row] = acc;
    if (!isfinite(acc)) report(g, g.col);
  } else if constexpr (KIND == kDot) {
    g.y[row] = acc;
    dotv += e.exd * acc;
  }
}

// kDot: fixed-shape block tree, then last-block finalisation in block order
template <int NW = kWarps>
__device__ __forceinline__ void dot_finish(const SpmvArgs& g, double dotv) {
  __shared__ double red[NW];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) dotv += __shfl_down_sync(0xffffffffu, dotv, off);
  if (lane == 0) red[warp] = dotv;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[w];
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

// ------------------------------------------------------------------ NVLink halo
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// thread 0 of every block: wait for this step's ghost planes (bounded: a peer
// that never signals turns into a CS_ERR_NCCL error instead of a hung GPU)
__device__ __noinline__ void halo_wait(const unsigned long long* ctr, unsigned long long want_lo,
                                       unsigned long long want_hi, DevState* st) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(ctr) < want_lo || ld_acquire_sys(ctr + 1) < want_hi) {
    __nanosleep(100);
    if (globaltimer() - t0 > 20ull * 1000000000ull) {
      if (st != nullptr) {
        atomicCAS(&st->err, 0ull, make_err(11 /*CS_ERR_NCCL*/, 0));
        st->done = 1;
      }
      return;
    }
  }
}

// signal side: the previous kernel's pushes are complete (stream order), so one
// thread releases them. __threadfence_system() per pushing warp/block instead
// compiled to MEMBAR.SC.SYS (+ CCTL.IVALL, wiping L1) hundreds of times per
// launch and cost ~0.25 ms per exchange on B200.
__device__ __forceinline__ void halo_release(const SpmvArgs& g) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (g.rel_lo) red_release_sys(g.rel_lo, g.rel_lo_n);
    if (g.rel_hi) red_release_sys(g.rel_hi, g.rel_hi_n);
  }
}

// producer side, per row: copy z into the neighbour's ghost slot
__device__ __forceinline__ void halo_push_row(const SpmvArgs& g, int64_t row, double z) {
  if (g.push_lo != nullptr && row < g.send_lo) g.push_lo[row] = z;
  if (g.push_hi != nullptr && row >= g.hi_begin) g.push_hi[row - g.hi_begin] = z;
}

__global__ void __launch_bounds__(256) halo_push_kernel(SpmvArgs g, const double* __restrict__ col,
                                                        int64_t n_local, DevState* st) {
  if (st != nullptr && *(volatile int*)&st->done) return;
  const int64_t nlo = g.push_lo ? g.send_lo : 0;
  const int64_t nhi = g.push_hi ? n_local - g.hi_begin : 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nlo + nhi;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < nlo) g.push_lo[i] = col[i];
    else g.push_hi[i - nlo] = col[g.hi_begin + i - nlo];
  }
}

__global__ void halo_release_kernel(SpmvArgs g, DevState* st) {
  if (st != nullptr && *(volatile int*)&st->done) return;
  halo_release(g);
}

// ------------------------------------------------------------------ LDG kernel
// Persistent warps walk slices with a grid stride; the next slice's metadata
// and the epilogue operands of the current rows are loaded ahead of the row
// sums so that their latency overlaps the value/x stream.
template <int KIND, bool JAC, int CDN>
__global__ void __launch_bounds__(kWarps * 32, CDN != 0 ? CS_SPMV_CD_MINB : CS_SPMV_MINB)
    sell_kernel(SellView a, SpmvArgs g, int64_t slice_begin, int64_t slice_end,
                const __grid_constant__ CdiaTable t) {
  if (g.st != nullptr && *(volatile int*)&g.st->done) return;
  halo_release(g);
  if (g.wait_ctr != nullptr) {
    if (threadIdx.x == 0) halo_wait(g.wait_ctr, g.want_lo, g.want_hi, g.st);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * kWarps;
  constexpr bool kPush = KIND == kMpkFirstF || KIND == kMpkMidF || KIND == kResidF;
  const bool push = kPush && (g.push_lo != nullptr || g.push_hi != nullptr);
  constexpr bool CD = CDN != 0;
  __shared__ SlotRec stab[CD ? 1 : kStabMax];
  const int staged = !CD && a.uniform ? stage_tables(a, stab) : 0;
  // virtual slice indices past nslices wrap to the start, so [ie, nslices + ib)
  // covers both boundary ranges of a halo'd SpMV in one launch
  const auto phys = [&](int64_t v) { return v >= a.nslices ? v - a.nslices : v; };
  // The next slice's metadata (table path) or participation word (CDIA path:
  // ncu put 20% of the stall samples on the first test of a just-loaded word)
  // is loaded one iteration ahead, so its latency overlaps this slice.
  int64_t slice = slice_begin + static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  double dotv = 0.0;
  SliceMeta sm{};
  uint32_t bits = 0;
  if constexpr (!CD) sm = load_meta(a, phys(slice), slice < slice_end ? a.nslices : 0);
  else if (slice < slice_end) bits = __ldcs(a.pbits + phys(slice) * kSliceRows + lane);
  for (; slice < slice_end; slice += wstride) {
    const int64_t vn = slice + wstride;
    SliceMeta next{};
    uint32_t bits_next = 0;
    if constexpr (!CD) next = load_meta(a, phys(vn), vn < slice_end ? a.nslices : 0);
    else if (vn < slice_end) bits_next = __ldcs(a.pbits + phys(vn) * kSliceRows + lane);
    const int64_t row = phys(slice) * kSliceRows + lane;
    const bool own = row < a.n_local;
    EpiOps e;
    if (own) e = epi_load<KIND, JAC>(a, g, row, CD ? t.inv : 0.0);
    double acc;
    if constexpr (CD)
      acc = row_sum_cdia<(CDN > 0 ? CDN : 0)>(t, g.x, static_cast<int>(row), bits);
    else acc = row_sum(a, g.x, sm, row, lane, stab, staged);
    if (own) {
      double zv = 0.0;
      epi_store<KIND, JAC>(g, row, acc, e, dotv, zv);
      if constexpr (kPush) {
        if (push) halo_push_row(g, row, zv);
      }
    }
    sm = next;
    bits = bits_next;
  }
  if constexpr (KIND == kDot) dot_finish(g, dotv);
}

// ------------------------------------------------------------------ z-blocked CDIA kernel
// A 27-entry class whose table is three groups of nine offsets a plane apart
// (off[9+i] = off[i] + P, off[18+i] = off[9+i] + P: a box stencil in natural
// ordering) lets one lane compute the rows r and r + P together: their 54
// neighbours are only 36 distinct x values (planes z-1, z, z+1, z+2), so each
// is gathered once and feeds both rows' sums, each row still adding its
// entries in its own stored order (group 0, 1, 2). Slice pairs (s, s + P/32)
// tile a range of whole plane pairs.
template <int KIND, bool JAC>
__global__ void __launch_bounds__(kWarps * 32, CS_SPMV_ZB_MINB)
    sell_zb_kernel(SellView a, SpmvArgs g, int64_t lo, int64_t npairs, int64_t sp,
                   const __grid_constant__ CdiaTable t) {
  if (g.st != nullptr && *(volatile int*)&g.st->done) return;
  halo_release(g);
  if (g.wait_ctr != nullptr) {
    if (threadIdx.x == 0) halo_wait(g.wait_ctr, g.want_lo, g.want_hi, g.st);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * kWarps;
  constexpr bool kPush = KIND == kMpkFirstF || KIND == kMpkMidF || KIND == kResidF;
  const bool push = kPush && (g.push_lo != nullptr || g.push_hi != nullptr);
  const int P = static_cast<int>(sp * kSliceRows);
  const double* __restrict__ x = g.x;
  double dotv = 0.0;
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * kWarps + warp; v < npairs; v += wstride) {
    const int64_t q = v / sp, w = v - q * sp;
    const int64_t s1 = lo + 2 * q * sp + w;
    const int ra = static_cast<int>(s1 * kSliceRows + lane), rb = ra + P;
    const bool own_a = ra < a.n_local, own_b = rb < a.n_local;
    const uint32_t ba = __ldcs(a.pbits + ra), bb = __ldcs(a.pbits + rb);
    EpiOps ea, eb;
    if (own_a) ea = epi_load<KIND, JAC>(a, g, ra, t.inv);
    if (own_b) eb = epi_load<KIND, JAC>(a, g, rb, t.inv);
    double acc_a = 0.0, acc_b = 0.0;
    double L0[9], L1[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      L0[i] = ((ba >> i) & 1u) ? __ldg(x + (ra + t.off[i])) : 0.0;
      L1[i] = (((ba >> (9 + i)) | (bb >> i)) & 1u) ? __ldg(x + (ra + t.off[9 + i])) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if ((ba >> i) & 1u) acc_a = __dadd_rn(acc_a, __dmul_rn(t.v[i], L0[i]));
#pragma unroll
    for (int i = 0; i < 9; ++i)
      L0[i] = (((ba >> (18 + i)) | (bb >> (9 + i))) & 1u) ? __ldg(x + (ra + t.off[18 + i])) : 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if ((ba >> (9 + i)) & 1u) acc_a = __dadd_rn(acc_a, __dmul_rn(t.v[9 + i], L1[i]));
      if ((bb >> i) & 1u) acc_b = __dadd_rn(acc_b, __dmul_rn(t.v[i], L1[i]));
    }
#pragma unroll
    for (int i = 0; i < 9; ++i)
      L1[i] = ((bb >> (18 + i)) & 1u) ? __ldg(x + (rb + t.off[18 + i])) : 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if ((ba >> (18 + i)) & 1u) acc_a = __dadd_rn(acc_a, __dmul_rn(t.v[18 + i], L0[i]));
      if ((bb >> (9 + i)) & 1u) acc_b = __dadd_rn(acc_b, __dmul_rn(t.v[9 + i], L0[i]));
    }
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if ((bb >> (18 + i)) & 1u) acc_b = __dadd_rn(acc_b, __dmul_rn(t.v[18 + i], L1[i]));
    if (own_a) {
      double zv = 0.0;
      epi_store<KIND, JAC>(g, ra, acc_a, ea, dotv, zv);
      if constexpr (kPush)
        if (push) halo_push_row(g, ra, zv);
    }
    if (own_b) {
      double zv = 0.0;
      epi_store<KIND, JAC>(g, rb, acc_b, eb, dotv, zv);
      if constexpr (kPush)
        if (push) halo_push_row(g, rb, zv);
    }
  }
  if constexpr (KIND == kDot) dot_finish(g, dotv);
}

// ------------------------------------------------------------------ TMA kernel
// A block owns tiles of kWarps consecutive slices; their value slots are one
// contiguous range of `vals`, streamed into shared memory by a single
// cp.async.bulk per tile (double-buffered, completion on an mbarrier) two tiles
// ahead. Meanwhile each thread resolves its row's columns (pattern shuffles or
// explicit column loads) and issues ALL of its x gathers into registers; after
// the tile lands the row sum runs in stored order from shared memory + registers.
constexpr int kXMax = 32;  // slice width served by this kernel

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

template <int KIND, bool JAC>
__global__ void __launch_bounds__(kWarps * 32, 2)
    sell_tma_kernel(SellView a, SpmvArgs g, int64_t sb, int64_t se, uint32_t stage_bytes) {
  if (g.st != nullptr && *(volatile int*)&g.st->done) return;
  extern __shared__ __align__(128) unsigned char tma_smem[];
  __shared__ __align__(8) uint64_t full[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ntiles = (se - sb + kWarps - 1) / kWarps;
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t t, int st) {
    const int64_t s0 = sb + t * kWarps;
    const int64_t s1 = s0 + kWarps < se ? s0 + kWarps : se;
    const int64_t vb = a.slice_ptr[s0], ve = a.slice_ptr[s1];
    const uint32_t bytes = static_cast<uint32_t>((ve - vb) * sizeof(double));
    mbar_expect_tx(&full[st], bytes);
    bulk_g2s(tma_smem + st * stage_bytes, a.vals + vb, bytes, &full[st]);
  };
  int64_t tile = blockIdx.x;
  if (threadIdx.x == 0) {
    if (tile < ntiles) issue(tile, 0);
    if (tile + gridDim.x < ntiles) issue(tile + gridDim.x, 1);
  }
  uint32_t phase0 = 0, phase1 = 0;
  int st = 0;
  double dotv = 0.0;
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t s0 = sb + tile * kWarps;
    const int64_t slice = s0 + warp;
    const bool active = slice < se;
    const int64_t row = slice * kSliceRows + lane;
    const bool own = active && row < a.n_local;
    int width = 0;
    int64_t voff = 0;
    double xv[kXMax];
    unsigned valid = 0;  // bit k: slot k contributes to this row
    EpiOps e;
    if (active) {
      const int64_t base = a.slice_ptr[slice];
      width = static_cast<int>((a.slice_ptr[slice + 1] - base) >> 5);
      voff = base - a.slice_ptr[s0];
      const int64_t m = a.meta[slice];
      if (own) e = epi_load<KIND, JAC>(a, g, row);
      if (m < 0) {
        const int2* pp = a.pat + pat_index(m);
        const int2 pl = lane < width ? __ldg(pp + lane) : make_int2(0, 0);
#pragma unroll
        for (int k = 0; k < kXMax; ++k) {
          const int off = __shfl_sync(0xffffffffu, pl.x, k);
          const unsigned msk = static_cast<unsigned>(__shfl_sync(0xffffffffu, pl.y, k));
          const bool on = k < width && ((msk >> lane) & 1u);
          xv[k] = on ? __ldg(g.x + row + off) : 0.0;
          valid |= on ? (1u << k) : 0u;
        }
      } else {
        const int32_t* cp = a.cols + m + lane;
#pragma unroll
        for (int k = 0; k < kXMax; ++k) {
          const int32_t c = k < width ? __ldcs(cp + k * kSliceRows) : -1;
          xv[k] = c >= 0 ? __ldg(g.x + c) : 0.0;
          valid |= c >= 0 ? (1u << k) : 0u;
        }
      }
    }
    if (st == 0) {
      mbar_wait(&full[0], phase0);
      phase0 ^= 1u;
    } else {
      mbar_wait(&full[1], phase1);
      phase1 ^= 1u;
    }
    if (active) {
      const double* vs = reinterpret_cast<const double*>(tma_smem + st * stage_bytes) + voff + lane;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < kXMax; ++k)
        if ((valid >> k) & 1u) acc = __dadd_rn(acc, __dmul_rn(vs[k * kSliceRows], xv[k]));
      double zv;
      if (own) epi_store<KIND, JAC>(g, row, acc, e, dotv, zv);
    }
    __syncthreads();  // every warp is done reading stage st
    if (threadIdx.x == 0 && tile + 2 * gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + 2 * gridDim.x, st);
    }
    st ^= 1;
  }
  if constexpr (KIND == kDot) dot_finish(g, dotv);
}

// ------------------------------------------------------------------ plane-streaming box kernel
// A 27-entry CDIA class whose table is a 3x3x3 box in natural ordering
// (off[9g + 3i + j] = g*P + i*L + j - (P + L + 1), so off[13] = 0: the
// generated 27-point operators, CdiaClass::boxL) is applied plane by plane
// from shared memory. Rows of a class range [R0, R1) are cut into columns of
// T consecutive rows per plane (row r = R0 + m*P + c*T + i); a block walks its
// columns upwards through the planes. Ring stage k of column c holds
//   x[S_k, S_k + T + 2L + 2), S_k = R0 + c*T + (k-1)*P - L - 1 (every x value
//     that group g of the rows of plane m = k - g reads),
//   the participation words of plane k's rows, z_{q-2} of plane k-2's rows,
// each one cp.async.bulk completing on the stage's mbarrier. At stage k a row
// position i loads its nine x values ONCE and feeds three rows: group 0 of
// plane k (a new sum), group 1 of plane k-1, group 2 of plane k-2 (complete:
// epilogue). Each row still adds its 27 entries in stored (ascending offset)
// order, each bit-tested exactly as row_sum_cdia, so the sum is bitwise the
// CDIA / CSR row sum. Per row: 9 shared loads instead of 27 L1 gathers, and
// every operand stream arrives by bulk copy, several planes ahead.
#ifndef CS_BOX_THREADS
#define CS_BOX_THREADS 512
#endif
#ifndef CS_BOX_ROWS
#define CS_BOX_ROWS 4  // rows per thread per plane: T = 2048
#endif
#ifndef CS_BOX_NS
#define CS_BOX_NS 4  // ring stages (planes in flight + 1)
#endif
constexpr int kBoxT = CS_BOX_THREADS * CS_BOX_ROWS;

struct BoxGeom {
  int64_t R0, R1;     // class rows of this launch (local row indices)
  int64_t P, L;       // plane stride, line stride
  int64_t nplanes;    // ceil((R1 - R0) / P)
  int64_t ncols;      // ceil(P / T)
  int64_t xlen;       // x elements that may be read (even)
  int64_t n_local;
  int xs;             // x doubles per stage (even)
  int ns;             // ring stages
  uint32_t stage_bytes;
  int sep = 0;        // separable plane sums (fast kinds, NEG1, geometric class)
  double dp1 = 0.0;   // centre value + 1 (separable: y = dp1 * x_c - sum of present x)
  // separable on a class with plane-uniform z face bits (CdiaClass::zuni): no
  // participation-word stream -- x / y face bits from one plane per column
  // segment, z bits from the plane index (the launch's first plane lacks its
  // lower neighbour iff !zl_first, its last plane its upper one iff !zu_last)
  int nobits = 0, zl_first = 1, zu_last = 1;
  int zplast = 0;     // nobits: the launch plane holding its last real row (R1 may be slice-padded)
  int64_t lseg = 1;   // planes per band of the item order (BoxIter)
  int vstrip = 0;     // separable path with vertical row strips (L divides the block size)
};

__device__ __forceinline__ uint32_t bk_of(const uint32_t* bs, int i, int lim) {
  return i < lim ? bs[i] : 0u;
}

// a block's stage sequence: items [i0, i1) (item = column * nplanes + plane)
// split into column segments of planes [m0, m1); a segment streams stages
// k = m0 .. m1 + 1
struct BoxIter {
  int64_t it, i1;
  int c = 0, k = 0, m0 = 0, m1 = 0;
  bool valid = false;
  // items in plane-band-major order: band s (planes [s*lseg, s*lseg + ls)),
  // then column, then plane. With lseg ~ one block's share, blocks on
  // neighbouring columns walk the same planes at the same time, so the halo
  // lines a column stages from its neighbours are L2 hits (column-major order:
  // +26 % DRAM reads at 512^3, profiles/r02h_ncu_sep512_*.txt)
  __device__ __forceinline__ void seg(const BoxGeom& b) {
    valid = it < i1;
    if (!valid) return;
    const int64_t band_items = b.ncols * b.lseg;
    const int64_t nb = (b.nplanes + b.lseg - 1) / b.lseg;
    int64_t s = it / band_items;
    if (s > nb - 1) s = nb - 1;
    const int64_t rem = it - s * band_items;
    const int64_t p0 = s * b.lseg;
    const int64_t ls = b.nplanes - p0 < b.lseg ? b.nplanes - p0 : b.lseg;
    const int64_t cc = rem / ls;
    c = static_cast<int>(cc);
    m0 = static_cast<int>(p0 + (rem - cc * ls));
    const int64_t end = p0 + ls;  // this column's band ends here
    m1 = static_cast<int>(m0 + (i1 - it) < end ? m0 + (i1 - it) : end);
    k = m0;
  }
  __device__ __forceinline__ void next(const BoxGeom& b) {
    if (++k > m1 + 1) {
      it += m1 - m0;
      seg(b);
    }
  }
};

// E2: one row-aligned epilogue stream of plane k-2 is staged too -- z_{q-2}
// (kMpkMidF) or b (kResidF, B_SRC)
template <bool E2, bool B_SRC = false>
__device__ __forceinline__ void box_issue(const BoxGeom& b, const SellView& a, const SpmvArgs& g,
                                          unsigned char* stage, uint64_t* bar, int64_t c,
                                          int64_t k, int64_t m1) {
  const int64_t cb = b.R0 + c * kBoxT;
  const int64_t width = b.P - c * kBoxT < kBoxT ? b.P - c * kBoxT : kBoxT;
  const int64_t S = cb + (k - 1) * b.P - b.L - 1;
  const int64_t E = S & ~int64_t{1};
  const int64_t xlo = E > 0 ? E : 0, xhi = E + b.xs < b.xlen ? E + b.xs : b.xlen;
  uint32_t bytes = 0;
  const uint32_t bx = xhi > xlo ? static_cast<uint32_t>((xhi - xlo) * 8) : 0u;
  bytes += bx;
  int64_t nb = 0, rb = cb + k * b.P;
  if (k < m1 && !b.nobits) {
    nb = b.R1 - rb < width ? b.R1 - rb : width;
    nb = nb > 0 ? (nb + 3) & ~int64_t{3} : 0;
  }
  bytes += static_cast<uint32_t>(nb * 4);
  int64_t nz = 0, rz = cb + (k - 2) * b.P;
  if constexpr (E2) {
    if (k >= 2 && k - 2 < m1) {
      nz = b.R1 - rz < width ? b.R1 - rz : width;
      nz = nz > 0 ? (nz + 1) & ~int64_t{1} : 0;
    }
    bytes += static_cast<uint32_t>(nz * 8);
  }
  mbar_expect_tx(bar, bytes);
  double* xs = reinterpret_cast<double*>(stage);
  if (bx) bulk_g2s(xs + (xlo - E), g.x + xlo, bx, bar);
  if (nb) bulk_g2s(stage + 8 * b.xs + 8 * kBoxT, a.pbits + rb, static_cast<uint32_t>(nb * 4), bar);
  if constexpr (E2)
    if (nz) bulk_g2s(stage + 8 * b.xs, (B_SRC ? g.b : g.zp2) + rz, static_cast<uint32_t>(nz * 8), bar);
}

// One row position of a stage: its nine x values (3 lines x 3) feed group 0 of
// the plane-k row, group 1 of the plane-(k-1) row and group 2 of the
// plane-(k-2) row, each sum in stored order. MODE 0: every row holds all 27
// entries. MODE 1: the three rows hold the same 9-entry sub-pattern m (an x or
// y face of the grid): absent entries read as 0.0 and are added -- bitwise the
// same as skipping them, because a running sum that starts at +0.0 is never
// -0.0 (round-to-nearest gives +0 on exact cancellation) and every table value
// is finite, so acc + v * 0.0 == acc. MODE 2: per-row, per-entry tests.
// NEG1: every off-centre value is -1.0 and acc + (-1.0 * x) is computed as the
// bitwise-equal acc - x.
template <int MODE, bool NEG1>
__device__ __forceinline__ void box_terms(const CdiaTable& t, const double* xs, int L,
                                          uint32_t bk, uint32_t b1, uint32_t b2, uint32_t m,
                                          double& acc0, double& acc1, double& acc2, double& cen) {
  double v[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    if (MODE == 0) {
      v[e] = xs[(e / 3) * L + (e % 3)];
    } else if (MODE == 1) {
      v[e] = e == 4 || ((m >> e) & 1u) ? xs[(e / 3) * L + (e % 3)] : 0.0;
    } else {
      // the centre is always loaded: it is also x[row] of the plane k-1 row
      const bool need = e == 4 || (((bk >> e) | (b1 >> (9 + e)) | (b2 >> (18 + e))) & 1u) != 0u;
      v[e] = need ? xs[(e / 3) * L + (e % 3)] : 0.0;
    }
  }
  cen = v[4];
  if (MODE == 1 && !((m >> 4) & 1u)) v[4] = 0.0;
  const auto term = [&](double& acc, int slot, double xv) {
    if (NEG1 && slot != 13) acc = __dsub_rn(acc, xv);
    else acc = __dadd_rn(acc, __dmul_rn(t.v[slot], xv));
  };
#pragma unroll
  for (int e = 0; e < 9; ++e)
    if (MODE < 2 || ((b2 >> (18 + e)) & 1u)) term(acc2, 18 + e, v[e]);
#pragma unroll
  for (int e = 0; e < 9; ++e)
    if (MODE < 2 || ((b1 >> (9 + e)) & 1u)) term(acc1, 9 + e, v[e]);
#pragma unroll
  for (int e = 0; e < 9; ++e)
    if (MODE < 2 || ((bk >> e) & 1u)) term(acc0, e, v[e]);
}

// Separable variant for the fast kinds (no bitwise-order requirement) on
// geometric classes whose off-centre values are all -1: the plane-(k-1) box
// sum B = sum of the present x in the 3x3 window is formed ONCE per row
// position from three masked line sums (8 adds instead of 27), then added to
// the plane-k row (its lower plane, if present), the plane-(k-1) row and the
// plane-(k-2) row (its upper plane, if present); the row's value is
// (a_ii + 1) x_c - S. fxy: any live row's word (x/y face bits agree across the
// planes of a geometric class).
__device__ __forceinline__ void box_terms_sep(const double* xs, int L, uint32_t fxy, bool zl,
                                              bool zu, double& acc0, double& acc1, double& acc2,
                                              double& cen) {
  const bool xl = (fxy >> 12) & 1u, xr = (fxy >> 14) & 1u;
  const bool yd = (fxy >> 10) & 1u, yu = (fxy >> 16) & 1u;
  double ls[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double a = xs[i * L], m = xs[i * L + 1], c = xs[i * L + 2];
    if (i == 1) cen = m;
    double t = xl ? a + m : m;
    ls[i] = xr ? t + c : t;
  }
  double bsum = ls[1];
  if (yd) bsum += ls[0];
  if (yu) bsum += ls[2];
  acc0 = zl ? bsum : 0.0;
  acc1 += bsum;
  if (zu) acc2 += bsum;
}

// Separable box SpMV, compile-time specialised (sell_boxsep_kernel): the fast
// kinds on a planar class (geometric box, every off-centre value -1, plane-
// uniform z faces: no participation-word stream) whose line length divides the
// block (vertical strips). The same sums in the same order as the separable
// path of sell_box_kernel -- bitwise the same z -- with the per-row overhead
// gone: face flags are decoded once per column segment (a warp whose lanes are
// all interior adds without selects), z faces are per-stage uniform, the
// finite check is one flag reported at the end (same error word), and the
// push test is per stage. ncu on the general kernel: 107 instructions per row,
// ALU pipe 56 %, issue-bound at 58 % of HBM (profiles/r02h_ncu_box_*.txt).
// WS: warp-specialised ring -- one extra producer warp issues the bulk copies
// as soon as every consumer warp has released the slot (an "empty" mbarrier per
// slot, one arrive per consumer warp) instead of thread 0 issuing them between
// block-wide barriers (ncu: barrier stalls and warp 0 lagging every stage).
// ring slots of the planar kernel: its stages carry no participation words, so
// up to kSepNS fit (CS_BOXSEP_NS); measured at 256^3: 4 slots 312 ms of SpMV per
// solve, 5: 317, 6: 328 (profiles/r02h_ab_ring_depth_256.txt) -- default 4
constexpr int kSepNS = 8;
// LC > 0: the line length as a compile-time constant (256, 512: the row offsets
// of a strip become immediate address offsets)
template <int KIND, bool JAC, bool WS, int LC>
__global__ void __launch_bounds__(CS_BOX_THREADS + (WS ? 32 : 0), 1)
    sell_boxsep_kernel(SellView a, SpmvArgs g, BoxGeom b, const __grid_constant__ CdiaTable t) {
  if (g.st != nullptr && *(volatile int*)&g.st->done) return;
  halo_release(g);
  if (g.wait_ctr != nullptr) {
    if (threadIdx.x == 0) halo_wait(g.wait_ctr, g.want_lo, g.want_hi, g.st);
    __syncthreads();
  }
  constexpr bool kE2 = KIND == kMpkMidF || KIND == kResidF;
  constexpr bool kBsrc = KIND == kResidF;
  constexpr bool kPush = KIND == kMpkFirstF || KIND == kMpkMidF || KIND == kResidF;
  constexpr int R = CS_BOX_ROWS;
  const bool push = kPush && (g.push_lo != nullptr || g.push_hi != nullptr);
  extern __shared__ __align__(128) unsigned char box_smem[];
  __shared__ __align__(8) uint64_t full[kSepNS];
  __shared__ __align__(8) uint64_t empty[WS ? kSepNS : 1];
  constexpr int kCW = CS_BOX_THREADS / 32;  // consumer warps
  const int64_t items = b.ncols * b.nplanes;
  const int64_t i0 = items * blockIdx.x / gridDim.x, i1 = items * (blockIdx.x + 1) / gridDim.x;
  BoxIter cur{i0, i1}, pre{i0, i1};
  cur.seg(b);
  pre.seg(b);
  int psl = 0;
  if (threadIdx.x == 0) {
    for (int sl = 0; sl < b.ns; ++sl) {
      mbar_init(&full[sl], 1);
      if constexpr (WS) mbar_init(&empty[sl], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (!WS)
      for (; psl < b.ns - 1 && pre.valid; ++psl, pre.next(b))
        box_issue<kE2, kBsrc>(b, a, g, box_smem + psl * b.stage_bytes, &full[psl], pre.c, pre.k, pre.m1);
  }
  __syncthreads();
  double dotv = 0.0;
  if constexpr (WS) {
    if (threadIdx.x >= CS_BOX_THREADS) {  // producer warp: lane 0 streams every stage
      if (threadIdx.x == CS_BOX_THREADS) {
        int slot = 0;
        uint32_t eph = 0;
        for (int n = 0; pre.valid; pre.next(b), ++n) {
          if (n >= b.ns) mbar_wait(&empty[slot], eph);  // all consumers left this slot
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          box_issue<kE2, kBsrc>(b, a, g, box_smem + slot * b.stage_bytes, &full[slot], pre.c, pre.k,
                                pre.m1);
          if (++slot == b.ns) {
            slot = 0;
            if (n >= b.ns) eph ^= 1u;
          }
        }
      }
      if constexpr (KIND == kDot) dot_finish<kCW + 1>(g, dotv);
      return;
    }
  }
  const int R0 = static_cast<int>(b.R0), R1 = static_cast<int>(b.R1), P = static_cast<int>(b.P);
  const int L = LC > 0 ? LC : static_cast<int>(b.L);
  const int end2 = static_cast<int>(b.R1 < b.n_local ? b.R1 : b.n_local);
  const int vx = static_cast<int>(threadIdx.x) % L, vg = static_cast<int>(threadIdx.x) / L;
  const int ib = vg * R * L + vx;  // column row of this thread's line j: ib + j L
  const double ca = g.ca, cb = g.cb, cc = g.cc, einv = JAC ? t.inv : 1.0, dp1 = b.dp1;
  double ap[R], ap2[R], cen2[R];
  bool xl = false, xr = false, inner = false;
  uint32_t ydm = 0u, yum = 0u;  // bit j: row j has its lower / upper line
  bool bad = false;
  int sl = 0;
  uint32_t phase = 0;
  for (; cur.valid; cur.next(b)) {
    if (!WS && threadIdx.x == 0 && pre.valid) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      box_issue<kE2, kBsrc>(b, a, g, box_smem + psl * b.stage_bytes, &full[psl], pre.c, pre.k, pre.m1);
      pre.next(b);
      psl = psl + 1 == b.ns ? 0 : psl + 1;
    }
    const int c = cur.c, k = cur.k, m0 = cur.m0;
    const int cbase = R0 + c * kBoxT;
    const int width = min(P - c * kBoxT, kBoxT);
    if (k == m0) {  // new column segment: face flags of the thread's positions
      uint32_t fx = 0u;
      ydm = yum = 0u;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        ap[j] = ap2[j] = cen2[j] = 0.0;
        const int i = ib + j * L, r = cbase + m0 * P + i;
        const uint32_t w = i < width && r < R1 ? __ldg(a.pbits + r) : 0u;
        fx |= w;
        ydm |= ((w >> 10) & 1u) << j;
        yum |= ((w >> 16) & 1u) << j;
      }
      xl = (fx >> 12) & 1u;
      xr = (fx >> 14) & 1u;
      inner = __all_sync(0xffffffffu, xl && xr && ydm == (1u << R) - 1u && yum == (1u << R) - 1u);
    }
    mbar_wait(&full[sl], phase);
    const unsigned char* stage = box_smem + sl * b.stage_bytes;
    const int slot = sl;
    if (++sl == b.ns) {
      sl = 0;
      phase ^= 1u;
    }
    const int S = cbase + (k - 1) * P - L - 1;
    const double* xb = reinterpret_cast<const double*>(stage) + (S & 1) + vg * R * L + vx;
    const double* es = reinterpret_cast<const double*>(stage + 8 * b.xs);
    const bool zl = k > 0 || b.zl_first, zu = k - 2 < b.zplast || b.zu_last;
    double ls[R + 2], cm[R + 2];
    if (inner) {
#pragma unroll
      for (int l = 0; l < R + 2; ++l) {
        const double x0 = xb[l * L], x1 = xb[l * L + 1], x2 = xb[l * L + 2];
        cm[l] = x1;
        ls[l] = (x0 + x1) + x2;
      }
    } else {
#pragma unroll
      for (int l = 0; l < R + 2; ++l) {
        const double x0 = xb[l * L], x1 = xb[l * L + 1], x2 = xb[l * L + 2];
        cm[l] = x1;
        const double tt = xl ? x0 + x1 : x1;
        ls[l] = xr ? tt + x2 : tt;
      }
    }
    double acc0[R], acc1[R], acc2[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      double bs = ls[j + 1];
      if (inner) {
        bs += ls[j];
        bs += ls[j + 2];
      } else {
        if ((ydm >> j) & 1u) bs += ls[j];
        if ((yum >> j) & 1u) bs += ls[j + 2];
      }
      acc0[j] = bs;
      acc1[j] = ap[j] + bs;
      acc2[j] = ap2[j] + bs;
    }
    if (!zl)  // the launch's first plane has no lower neighbour plane
#pragma unroll
      for (int j = 0; j < R; ++j) acc0[j] = 0.0;
    if (!zu)  // the plane k-2 row has no upper neighbour plane
#pragma unroll
      for (int j = 0; j < R; ++j) acc2[j] = ap2[j];
    // epilogue: rows of plane k-2 complete
    const int rb2 = cbase + (k - 2) * P;
    const int lim_2 = k - 2 >= m0 ? max(0, min(width, end2 - rb2)) : 0;
    const bool edge = push && (rb2 < g.send_lo || rb2 + width > g.hi_begin);
    // a full column of live rows (the common case): no per-row bound test
    const int lim = lim_2 == kBoxT ? 0x7fffffff : lim_2;
    double* const ybase = g.y != nullptr ? g.y + rb2 : nullptr;
    double* const zbase = g.zout + rb2;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int i = ib + j * L;
      const double y = fma(dp1, cen2[j], -acc2[j]);  // (a_ii + 1) x_c - S
      if (i < lim) {
        const int64_t row = rb2 + i;
        if constexpr (KIND == kDot) {
          g.y[row] = y;
          dotv += cen2[j] * y;
        } else {
          double z;
          if constexpr (KIND == kResidF) {
            const double r = es[i] - y;
            if (ybase) ybase[i] = r;  // nullptr: the pack forms r = D z_0
            z = JAC ? r * einv : r;
          } else {
            if (ybase) ybase[i] = y;
            const double dp = JAC ? y * einv : y;
            z = fma(cb, cen2[j], ca * dp);
            if constexpr (KIND == kMpkMidF) z = fma(cc, es[i], z);
          }
          zbase[i] = z;
          bad |= !isfinite(z);
          if constexpr (kPush)
            if (edge) halo_push_row(g, row, z);
        }
      }
      ap2[j] = acc1[j];
      cen2[j] = cm[j + 1];
      ap[j] = acc0[j];
    }
    if constexpr (WS) {  // this warp's reads of the slot are done (arrive = release)
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[slot]);
    } else {
      (void)slot;
      __syncthreads();
    }
  }
  if (bad) report(g, g.col);
  if constexpr (KIND == kDot) dot_finish<kCW + (WS ? 1 : 0)>(g, dotv);
}

#ifndef CS_BOX_MINB
#define CS_BOX_MINB 1
#endif
template <int KIND, bool JAC, bool NEG1>
__global__ void __launch_bounds__(CS_BOX_THREADS, CS_BOX_MINB)
    sell_box_kernel(SellView a, SpmvArgs g, BoxGeom b, const __grid_constant__ CdiaTable t) {
  if (g.st != nullptr && *(volatile int*)&g.st->done) return;
  halo_release(g);
  if (g.wait_ctr != nullptr) {
    if (threadIdx.x == 0) halo_wait(g.wait_ctr, g.want_lo, g.want_hi, g.st);
    __syncthreads();
  }
  constexpr bool kE2 = KIND == kMpkMidF || KIND == kResidF;
  constexpr bool kBsrc = KIND == kResidF;  // the staged stream is b, not z_{q-2}
  constexpr bool kPush = KIND == kMpkFirstF || KIND == kMpkMidF || KIND == kResidF;
  constexpr int R = CS_BOX_ROWS;
  const bool push = kPush && (g.push_lo != nullptr || g.push_hi != nullptr);
  extern __shared__ __align__(128) unsigned char box_smem[];
  __shared__ __align__(8) uint64_t full[CS_BOX_NS];
  const int64_t items = b.ncols * b.nplanes;
  const int64_t i0 = items * blockIdx.x / gridDim.x, i1 = items * (blockIdx.x + 1) / gridDim.x;
  BoxIter cur{i0, i1}, pre{i0, i1};
  cur.seg(b);
  pre.seg(b);
  int psl = 0;
  if (threadIdx.x == 0) {
    for (int sl = 0; sl < b.ns; ++sl) mbar_init(&full[sl], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (; psl < b.ns - 1 && pre.valid; ++psl, pre.next(b))
      box_issue<kE2, kBsrc>(b, a, g, box_smem + psl * b.stage_bytes, &full[psl], pre.c, pre.k, pre.m1);
  }
  __syncthreads();
  double ap[R], ap2[R], cen2[R];  // running sums of planes k-1, k-2; centre of plane k-2
  uint32_t bp[R], bp2[R];         // participation words of planes k-1, k-2
  uint32_t fxy[R];                // nobits: the x / y face bits of this column's positions
  // rows of a column held by this thread: i = tid + j * threads, or (vertical
  // strips, separable path) R consecutive lines at one x position, so the R + 2
  // three-point line sums of the strip are formed once and shared by its rows
  int ii[R];
  const int vx = b.vstrip ? static_cast<int>(threadIdx.x % b.L) : 0;
  const int vg = b.vstrip ? static_cast<int>(threadIdx.x / b.L) : 0;
#pragma unroll
  for (int j = 0; j < R; ++j)
    ii[j] = b.vstrip ? (vg * R + j) * static_cast<int>(b.L) + vx
                     : static_cast<int>(threadIdx.x) + j * CS_BOX_THREADS;
  double dotv = 0.0;
  const int R0 = static_cast<int>(b.R0), R1 = static_cast<int>(b.R1), P = static_cast<int>(b.P);
  const int L = static_cast<int>(b.L);
  const int end2 = static_cast<int>(b.R1 < b.n_local ? b.R1 : b.n_local);
  int sl = 0;
  uint32_t phase = 0;
  for (; cur.valid; cur.next(b)) {
    if (threadIdx.x == 0 && pre.valid) {  // refill the slot consumed last iteration
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      box_issue<kE2, kBsrc>(b, a, g, box_smem + psl * b.stage_bytes, &full[psl], pre.c, pre.k, pre.m1);
      pre.next(b);
      psl = psl + 1 == b.ns ? 0 : psl + 1;
    }
    const int c = cur.c, k = cur.k, m0 = cur.m0, m1 = cur.m1;
    mbar_wait(&full[sl], phase);
    const unsigned char* stage = box_smem + sl * b.stage_bytes;
    if (++sl == b.ns) {
      sl = 0;
      phase ^= 1u;
    }
    const int cb = R0 + c * kBoxT;
    const int S = cb + (k - 1) * P - L - 1;
    const double* xs = reinterpret_cast<const double*>(stage) + (S & 1);
    const double* zs = reinterpret_cast<const double*>(stage + 8 * b.xs);
    const uint32_t* bs = reinterpret_cast<const uint32_t*>(stage + 8 * b.xs + 8 * kBoxT);
    const int width = min(P - c * kBoxT, kBoxT);
    if (k == m0) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        ap[j] = ap2[j] = cen2[j] = 0.0;
        bp[j] = bp2[j] = 0u;
        const int i = ii[j];
        const int r = cb + m0 * P + i;  // plane-invariant on a geometric class
        fxy[j] = b.nobits && i < width && r < R1 ? __ldg(a.pbits + r) : 0u;
      }
    }
    // rows of planes k (new sums), k-1 and k-2 (complete) held by this column
    const int rbk = cb + k * P, rb1 = rbk - P, rb2 = rb1 - P;
    const int lim_k = k < m1 ? max(0, min(width, R1 - rbk)) : 0;
    const int lim_1 = k - 1 >= m0 && k - 1 < m1 ? max(0, min(width, R1 - rb1)) : 0;
    const int lim_2 = k - 2 >= m0 ? max(0, min(width, end2 - rb2)) : 0;
    constexpr bool kSepKind =
        NEG1 && (KIND == kMpkFirstF || KIND == kMpkMidF || KIND == kDot || KIND == kResidF);
    uint32_t bk[R], mk[R];
    double acc0[R], acc1[R], acc2[R], cen[R];
    if (kSepKind && b.sep) {
      const bool zl = k > 0 || b.zl_first, zu = k - 2 < b.zplast || b.zu_last;  // nobits
      if (b.vstrip) {
        // line sums of lines vg*R - 1 .. vg*R + R at x = vx (xs index of (line l,
        // x + dx) is (l + 1) L + x + dx + 1); each row adds its own line, then the
        // one below and the one above -- the order of box_terms_sep
        uint32_t fx = 0u;
#pragma unroll
        for (int j = 0; j < R; ++j) fx |= b.nobits ? fxy[j] : bk_of(bs, ii[j], lim_k) | bp[j] | bp2[j];
        const bool xl = (fx >> 12) & 1u, xr = (fx >> 14) & 1u;
        double ls[R + 2], cm[R + 2];
        const double* xb = xs + vg * R * L + vx;
#pragma unroll
        for (int l = 0; l < R + 2; ++l) {
          const double a = xb[l * L], m = xb[l * L + 1], c = xb[l * L + 2];
          cm[l] = m;
          const double t = xl ? a + m : m;
          ls[l] = xr ? t + c : t;
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
          bk[j] = !b.nobits && ii[j] < lim_k ? bs[ii[j]] : 0u;
          const uint32_t f = b.nobits ? fxy[j] : bk[j] | bp[j] | bp2[j];
          const bool zlj = b.nobits ? zl : ((bk[j] >> 4) & 1u) != 0u;
          const bool zuj = b.nobits ? zu : ((bp2[j] >> 22) & 1u) != 0u;
          double bsum = ls[j + 1];
          if ((f >> 10) & 1u) bsum += ls[j];
          if ((f >> 16) & 1u) bsum += ls[j + 2];
          cen[j] = cm[j + 1];
          acc0[j] = zlj ? bsum : 0.0;
          acc1[j] = ap[j] + bsum;
          acc2[j] = zuj ? ap2[j] + bsum : ap2[j];
          acc2[j] = fma(b.dp1, cen2[j], -acc2[j]);  // (a_ii + 1) x_c - S, completed rows only
        }
        goto epilogue;
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int i = ii[j];
        bk[j] = !b.nobits && i < lim_k ? bs[i] : 0u;
        acc1[j] = ap[j];
        acc2[j] = ap2[j];
        if (b.nobits)
          box_terms_sep(xs + i, L, fxy[j], zl, zu, acc0[j], acc1[j], acc2[j], cen[j]);
        else
          box_terms_sep(xs + i, L, bk[j] | bp[j] | bp2[j], (bk[j] >> 4) & 1u, (bp2[j] >> 22) & 1u,
                        acc0[j], acc1[j], acc2[j], cen[j]);
        acc2[j] = fma(b.dp1, cen2[j], -acc2[j]);  // (a_ii + 1) x_c - S, completed rows only
      }
      goto epilogue;
    }
    {
    bool agree = true, full = true;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int i = ii[j];
      bk[j] = i < lim_k ? bs[i] : 0u;
      // the 9-entry sub-pattern each live row uses from this stage (rows outside
      // the column/segment are never stored, so they do not constrain it)
      const uint32_t g0 = bk[j] & 0x1FFu, g1 = (bp[j] >> 9) & 0x1FFu, g2 = (bp2[j] >> 18) & 0x1FFu;
      const bool l0 = i < lim_k, l1 = i < lim_1, l2 = i < lim_2;
      const uint32_t m = (l0 ? g0 : 0u) | (l1 ? g1 : 0u) | (l2 ? g2 : 0u);
      mk[j] = m;
      agree = agree && (!l0 || g0 == m) && (!l1 || g1 == m) && (!l2 || g2 == m);
      full = full && m == 0x1FFu;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      acc0[j] = 0.0;
      acc1[j] = ap[j];
      acc2[j] = ap2[j];
    }
    const unsigned all_agree = __all_sync(0xffffffffu, agree);
    if (all_agree && __all_sync(0xffffffffu, full)) {  // interior: all 27 entries
#pragma unroll
      for (int j = 0; j < R; ++j)
        box_terms<0, NEG1>(t, xs + ii[j], L, bk[j], bp[j], bp2[j],
                           mk[j], acc0[j], acc1[j], acc2[j], cen[j]);
    } else if (all_agree) {  // x / y faces: one sub-pattern per row position
#pragma unroll
      for (int j = 0; j < R; ++j)
        box_terms<1, NEG1>(t, xs + ii[j], L, bk[j], bp[j], bp2[j],
                           mk[j], acc0[j], acc1[j], acc2[j], cen[j]);
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j)
        box_terms<2, NEG1>(t, xs + ii[j], L, bk[j], bp[j], bp2[j],
                           mk[j], acc0[j], acc1[j], acc2[j], cen[j]);
    }
    }
  epilogue:
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int i = ii[j];
      if (i < lim_2) {  // plane k-2 row complete
        const int64_t r2 = rb2 + i;
        EpiOps eo;
        eo.exd = cen2[j];
        eo.einv = JAC ? t.inv : 1.0;
        if constexpr (kE2 && !kBsrc) eo.e2 = zs[i];
        if constexpr (kBsrc) eo.e1 = zs[i];
        if constexpr (KIND == kResid) eo.e1 = g.b[r2];
        double zv = 0.0;
        epi_store<KIND, JAC>(g, r2, acc2[j], eo, dotv, zv);
        if constexpr (kPush)
          if (push) halo_push_row(g, r2, zv);
      }
      ap2[j] = acc1[j];
      bp2[j] = bp[j];
      cen2[j] = cen[j];  // x[row] of the plane k-1 row (off[13] = 0)
      ap[j] = acc0[j];
      bp[j] = bk[j];
    }
    __syncthreads();  // every thread is done with slot sl before it is refilled
  }
  if constexpr (KIND == kDot) dot_finish<CS_BOX_THREADS / 32>(g, dotv);
}

#ifndef CS_SPMV_TMA
#define CS_SPMV_TMA 0  // measured slower on B200 (16 warps/SM at 128 regs); DESIGN.md 3
#endif

int spmv_grid(int64_t nslices, bool cd = false) {
  const int64_t want = (nslices + kWarps - 1) / kWarps;
  if (!CS_SPMV_PERSIST) return static_cast<int>(want > 0 ? want : 1);
  // one wave of resident blocks at the kernel's occupancy
  const int64_t cap = 148 * (cd ? CS_SPMV_CD_MINB : CS_SPMV_MINB);
  return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

int tma_grid(int64_t nslices) {
  const int64_t tiles = (nslices + kWarps - 1) / kWarps;
  const int64_t cap = 148 * 2;  // 2 resident blocks per SM (2 x 2 stages of shared memory)
  return static_cast<int>(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
}

bool use_tma(const SellView& a) {
  return CS_SPMV_TMA && !a.uniform && a.max_width > 0 && a.max_width <= kXMax;
}

template <int KIND, bool JAC>
void tma_launch(const SellView& a, const SpmvArgs& g, int64_t sb, int64_t se, cudaStream_t st) {
  const uint32_t stage = static_cast<uint32_t>(kWarps) * a.max_width * kSliceRows * sizeof(double);
  kernel_setup(reinterpret_cast<const void*>(sell_tma_kernel<KIND, JAC>), kWarps * 32,
               static_cast<int>(2 * stage));
  sell_tma_kernel<KIND, JAC><<<tma_grid(se - sb), kWarps * 32, 2 * stage, st>>>(a, g, sb, se, stage);
}

// CS_SPMV_BOX=0 in the environment: box classes take the gather kernels (A/B runs)
bool box_enabled() {
  const char* e = std::getenv("CS_SPMV_BOX");
  return e == nullptr || std::atoi(e) != 0;
}

constexpr bool box_kind(int kind) {
  return kind == kPlain || kind == kResid || kind == kMpkFirstF || kind == kMpkMidF ||
         kind == kMpkLast || kind == kDot || kind == kResidF;
}

// Plane-streaming launch over the class rows [lo, hi) * 32; false: not applicable.
template <int KIND>
bool box_launch(bool jac, const SellView& a, const SpmvArgs& g, const CdiaClass& cl,
                const CdiaTable& t, int64_t lo, int64_t hi, cudaStream_t st) {
  if constexpr (!box_kind(KIND)) {
    return false;
  } else {
    if (!box_enabled() || cl.boxL == 0 || a.pbits == nullptr) return false;
    const auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
    if (!al16(g.x) || (KIND == kMpkMidF && !al16(g.zp2)) || (KIND == kResidF && !al16(g.b)))
      return false;
    BoxGeom b{};
    b.R0 = lo * kSliceRows;
    b.R1 = hi * kSliceRows;
    b.P = cl.boxP;
    b.L = cl.boxL;
    b.nplanes = (b.R1 - b.R0 + b.P - 1) / b.P;
    b.ncols = (b.P + kBoxT - 1) / kBoxT;
    b.xlen = a.xlen;
    b.n_local = a.n_local;
    b.xs = static_cast<int>((kBoxT + 2 * b.L + 4 + 1) / 2 * 2);
    b.stage_bytes = static_cast<uint32_t>(round_up(8 * b.xs + 12 * kBoxT, 128));
    constexpr int kSmemMax = 227 * 1024 - 1024;
    b.ns = std::min<int>(CS_BOX_NS, kSmemMax / static_cast<int>(b.stage_bytes));
    if (b.ns < 2) return false;
    const int smem = b.ns * static_cast<int>(b.stage_bytes);
    for (int e = 0; e < 27; ++e)  // box_terms MODE 1 adds 0.0 * v for absent entries
      if (!std::isfinite(t.v[e])) return false;
    bool neg1 = true;  // every off-centre value is -1.0 (the 27-point Poisson operators)
    for (int e = 0; e < 27; ++e) neg1 = neg1 && (e == 13 || t.v[e] == -1.0);
    auto kern = jac ? (neg1 ? sell_box_kernel<KIND, true, true> : sell_box_kernel<KIND, true, false>)
                    : (neg1 ? sell_box_kernel<KIND, false, true> : sell_box_kernel<KIND, false, false>);
    const int per_sm = kernel_setup(reinterpret_cast<const void*>(kern), CS_BOX_THREADS, smem);
    // separable plane sums for the fast kinds on geometric -1 classes (CS_BOX_SEP=0: off)
    const char* sep_e = std::getenv("CS_BOX_SEP");  // per launch, like CS_SPMV_BOX
    const bool sep_env = sep_e == nullptr || std::atoi(sep_e) != 0;
    b.sep = sep_env && neg1 && cl.geo &&
            (KIND == kMpkFirstF || KIND == kMpkMidF || KIND == kDot || KIND == kResidF);
    b.dp1 = t.v[13] + 1.0;
    {
      const int64_t cr0 = cl.s0 * kSliceRows;
      const int64_t cr1 = std::min(cl.s1 * kSliceRows, a.n_local);
      const char* nb_e = std::getenv("CS_BOX_NOBITS");
      const bool nb_env = nb_e == nullptr || std::atoi(nb_e) != 0;
      if (b.sep && cl.zuni && nb_env && (b.R0 - cr0) % b.P == 0 && std::min(b.R1, a.n_local) <= cr1) {
        const int64_t d = (b.R0 - cr0) / b.P, clast = (cr1 - cr0 - 1) / b.P;
        b.nobits = 1;
        b.zplast = static_cast<int>((std::min(b.R1, a.n_local) - 1 - b.R0) / b.P);
        b.zl_first = d > 0 || cl.zl0;
        b.zu_last = d + b.zplast < clast || cl.zuN;
      }
    }
    {
      const char* vs_e = std::getenv("CS_BOX_VSTRIP");
      const bool vs_env = vs_e == nullptr || std::atoi(vs_e) != 0;
      b.vstrip = vs_env && b.sep && b.L <= CS_BOX_THREADS && CS_BOX_THREADS % b.L == 0;
    }
    const int64_t items = b.ncols * b.nplanes;
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>(items, 148 * per_sm)));
    {  // band length ~ one block's share of the items (CS_BOX_BANDS=0: column-major)
      const char* bd_e = std::getenv("CS_BOX_BANDS");
      const bool bands = bd_e == nullptr || std::atoi(bd_e) != 0;
      const int64_t share = (items + grid - 1) / grid;
      b.lseg = bands ? std::max<int64_t>(1, std::min<int64_t>(b.nplanes, share)) : b.nplanes;
    }
    if constexpr (KIND == kMpkFirstF || KIND == kMpkMidF || KIND == kResidF || KIND == kDot) {
      const char* sk_e = std::getenv("CS_BOX_SEPK");
      const bool sk_env = sk_e == nullptr || std::atoi(sk_e) != 0;
      if (sk_env && b.sep && b.nobits && b.vstrip) {
        const char* ws_e = std::getenv("CS_BOX_WS");
        const bool ws = ws_e == nullptr || std::atoi(ws_e) != 0;
        const int lc = b.L == 512 ? 512 : b.L == 256 ? 256 : 0;
#define CSG_SK(W, LCV)                                                                 \
  (jac ? sell_boxsep_kernel<KIND, true, W, LCV> : sell_boxsep_kernel<KIND, false, W, LCV>)
        auto sk = ws ? (lc == 512 ? CSG_SK(true, 512) : lc == 256 ? CSG_SK(true, 256) : CSG_SK(true, 0))
                     : (lc == 512 ? CSG_SK(false, 512) : lc == 256 ? CSG_SK(false, 256) : CSG_SK(false, 0));
#undef CSG_SK
        const int nthr = CS_BOX_THREADS + (ws ? 32 : 0);
        // stage = x slice + the epilogue stream (no participation words): more slots
        const char* ns_e = std::getenv("CS_BOXSEP_NS");
        const int ns_want = std::min(kSepNS, std::max(2, ns_e ? std::atoi(ns_e) : 4));
        b.stage_bytes = static_cast<uint32_t>(round_up(8 * b.xs + 8 * kBoxT, 128));
        b.ns = std::min<int>(ns_want, kSmemMax / static_cast<int>(b.stage_bytes));
        const int ssmem = b.ns * static_cast<int>(b.stage_bytes);
        const int per = kernel_setup(reinterpret_cast<const void*>(sk), nthr, ssmem);
        const unsigned sgrid = static_cast<unsigned>(
            std::max<int64_t>(1, std::min<int64_t>(items, 148 * per)));
        const char* bd_e = std::getenv("CS_BOX_BANDS");
        if (bd_e == nullptr || std::atoi(bd_e) != 0)  // bands sized for this kernel's grid
          b.lseg = std::max<int64_t>(1, std::min<int64_t>(b.nplanes, (items + sgrid - 1) / sgrid));
        sk<<<sgrid, nthr, ssmem, st>>>(a, g, b, t);
        return true;
      }
    }
    kern<<<grid, CS_BOX_THREADS, smem, st>>>(a, g, b, t);
    return true;
  }
}

template <int KIND>
void launch_kind(bool jac, const SellView& a, const SpmvArgs& g, int64_t sb, int64_t se,
                 cudaStream_t st) {
  if (use_tma(a)) {
    if (jac) tma_launch<KIND, true>(a, g, sb, se, st);
    else tma_launch<KIND, false>(a, g, sb, se, st);
    return;
  }
  // CDIA: one launch per (class x physical range) piece -- z-blocked over whole
  // plane pairs where the class allows it, the rest row-wise. kDot finalises
  // one sum per launch, so a multi-launch kDot takes the table kernel instead.
  // Only the first launch releases the previous kernel's peer pushes.
  if (a.ncdia > 0) {
    struct Piece {
      int k;
      int64_t lo, hi, sp;  // sp > 0: z-blocked, hi - lo = 2 * pairs
    };
    Piece list[2 * 64 * 2];
    int np = 0;
    const int64_t ranges[2][2] = {{sb, se < a.nslices ? se : a.nslices}, {0, se - a.nslices}};
    for (const auto& r : ranges)
      for (int k = 0; k < a.ncdia; ++k) {
        int64_t lo = std::max(r[0], a.cdia[k].s0);
        const int64_t hi = std::min(r[1], a.cdia[k].s1);
        if (lo >= hi) continue;
        if (box_kind(KIND) && box_enabled() && a.cdia[k].boxL > 0) {
          list[np++] = {k, lo, hi, -1};
          continue;
        }
        const int64_t sp = CS_SPMV_ZB ? a.cdia[k].zstride / kSliceRows : 0;
        if (sp > 0 && hi - lo >= 2 * sp) {
          const int64_t span = (hi - lo) / (2 * sp) * (2 * sp);
          list[np++] = {k, lo, lo + span, sp};
          lo += span;
        }
        if (lo < hi) list[np++] = {k, lo, hi, 0};
      }
    if (KIND != kDot || np == 1) {
      SpmvArgs gg = g;
      for (int e = 0; e < np; ++e) {
        const Piece& pc = list[e];
        CdiaTable t = a.cdia[pc.k].t;
        t.inv = jac && t.diag != 0.0 ? 1.0 / t.diag : 0.0;  // IEEE, = inv_diag_kernel
        if (pc.sp < 0 && box_launch<KIND>(jac, a, gg, a.cdia[pc.k], t, pc.lo, pc.hi, st)) {
          gg.rel_lo = gg.rel_hi = nullptr;
          continue;
        }
        if (pc.sp < 0) {  // box launch not applicable after all: row-wise
          const unsigned grid = static_cast<unsigned>(spmv_grid(pc.hi - pc.lo, true));
          if (jac) sell_kernel<KIND, true, 27><<<grid, kWarps * 32, 0, st>>>(a, gg, pc.lo, pc.hi, t);
          else sell_kernel<KIND, false, 27><<<grid, kWarps * 32, 0, st>>>(a, gg, pc.lo, pc.hi, t);
          gg.rel_lo = gg.rel_hi = nullptr;
          continue;
        }
        if (pc.sp > 0) {
          const int64_t pairs = (pc.hi - pc.lo) / 2;
          const unsigned zg = static_cast<unsigned>(std::min<int64_t>(
              std::max<int64_t>((pairs + kWarps - 1) / kWarps, 1), 148 * CS_SPMV_ZB_MINB));
          if (jac) sell_zb_kernel<KIND, true><<<zg, kWarps * 32, 0, st>>>(a, gg, pc.lo, pairs, pc.sp, t);
          else sell_zb_kernel<KIND, false><<<zg, kWarps * 32, 0, st>>>(a, gg, pc.lo, pairs, pc.sp, t);
        } else {
          const unsigned grid = static_cast<unsigned>(spmv_grid(pc.hi - pc.lo, true));
#define CSG_CD(N)                                                                                \
  do {                                                                                           \
    if (jac) sell_kernel<KIND, true, N><<<grid, kWarps * 32, 0, st>>>(a, gg, pc.lo, pc.hi, t);   \
    else sell_kernel<KIND, false, N><<<grid, kWarps * 32, 0, st>>>(a, gg, pc.lo, pc.hi, t);      \
  } while (0)
          if (t.n == 27) CSG_CD(27);
          else if (t.n == 7) CSG_CD(7);
          else CSG_CD(-1);
#undef CSG_CD
        }
        gg.rel_lo = gg.rel_hi = nullptr;
      }
      return;
    }
  }
  const unsigned grid = static_cast<unsigned>(spmv_grid(se - sb));
  const CdiaTable none{};
  if (jac) sell_kernel<KIND, true, 0><<<grid, kWarps * 32, 0, st>>>(a, g, sb, se, none);
  else sell_kernel<KIND, false, 0><<<grid, kWarps * 32, 0, st>>>(a, g, sb, se, none);
}

}  // namespace

void launch_halo_push(const SpmvArgs& g, const double* col, int64_t n_local, DevState* st,
                      cudaStream_t s) {
  const int64_t rows = (g.push_lo ? g.send_lo : 0) + (g.push_hi ? n_local - g.hi_begin : 0);
  if (rows == 0) return;
  const int64_t blocks = std::min<int64_t>((rows + 255) / 256, 148 * 4);
  halo_push_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(g, col, n_local, st);
  CS_CUDA(cudaGetLastError());
}

void launch_halo_release(const SpmvArgs& g, DevState* st, cudaStream_t s) {
  halo_release_kernel<<<1, 32, 0, s>>>(g, st);
  CS_CUDA(cudaGetLastError());
}

int spmv_dot_blocks(int64_t nslices) {
  const int a = spmv_grid(nslices), b = tma_grid(nslices);
  return std::max({a, b, 148 * 4});  // the box kernel: <= 148 x resident blocks
}

void launch_spmv(int kind, const SellView& a, const SpmvArgs& g, int64_t sb, int64_t se,
                 cudaStream_t st) {
  if (se <= sb) return;
  if (se > a.nslices && use_tma(a)) {  // the TMA tiles need contiguous slices
    launch_spmv(kind, a, g, sb, a.nslices, st);
    launch_spmv(kind, a, g, a.nslices, se, st);
    return;
  }
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
    case kResidF: launch_kind<kResidF>(jac, a, g, sb, se, st); break;
    default: throw LibError{9, 0, "bad spmv kind"};
  }
  CS_CUDA(cudaGetLastError());
}

}  // namespace csg
