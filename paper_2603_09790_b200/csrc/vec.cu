#include <algorithm>
// vec.cu -- streaming vector/block kernels: tall-skinny reductions (serial
// reference order, deterministic tree, and the fused packed one-allreduce
// reduction on FP64 DMMA), the fused x/r/Q/AQ update pass, preconditioner
// apply, seeded start vectors and the classical-PCG vector steps.
//
// Arithmetic contracts:
//  * "reference" kernels keep the reference's per-element operation sequence
//    with explicit __dmul_rn/__dadd_rn (no FMA contraction):
//    axpy y = y + a*x (kernels_scalar.cpp:6-8), xpby y = x + b*y (:10-12),
//    block_update out_j = y_j + sum_q c_qj x_q in ascending q (dense_ops.cpp:29-42),
//    dot / Gram entries as ONE serial ascending chain (dense_ops.cpp:10-15,
//    kernels_scalar.cpp:22-33);
//  * "fast" reductions use fixed-shape trees (warp shuffles, fixed block
//    count, last-block finalisation in block order): deterministic run to run,
//    but not the serial order.
#include <climits>
#include <cstdio>

#include "kernels.cuh"

namespace csg {
namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t threads, int per = kThreads) {
  return static_cast<unsigned>((threads + per - 1) / per);
}

__device__ __forceinline__ bool halted(const DevState* st) {
  return st != nullptr && *(volatile const int*)&st->done;
}

// ------------------------------------------------------------------ precond / rng

__global__ void precond_kernel(int64_t n, const double* __restrict__ inv_diag,
                               const double* __restrict__ in, double* out, DevState* st, int col,
                               int pending) {
  if (halted(st)) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double z = inv_diag ? __dmul_rn(inv_diag[i], in[i]) : in[i];
  out[i] = z;
  if (col >= 0 && !isfinite(z) && st != nullptr) {
    atomicCAS(pending ? &st->pending : &st->err, 0ull, make_err(4, col));
    if (!pending) st->done = 1;
  }
}

// ------------------------------------------------------------------ block Jacobi
// One thread per diagonal block. Factor: left-looking Cholesky with the
// operation order of small_cholesky_solve (dense_ops.cpp:55-88), in place on the
// bs x bs column-major block (lower triangle = L). Apply: forward then back
// substitution, ascending/descending like its solve loops, separate roundings.
__global__ void bj_factor_kernel(int64_t nblocks, int bs, double* f, int* bad_block) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  double* L = f + b * bs * bs;
  for (int j = 0; j < bs; ++j) {
    double d = L[j + j * bs];
    for (int q = 0; q < j; ++q) d = __dsub_rn(d, __dmul_rn(L[j + q * bs], L[j + q * bs]));
    if (!(d > 0.0) || !isfinite(d)) {
      atomicMin(bad_block, static_cast<int>(b < INT_MAX ? b : INT_MAX - 1));
      return;
    }
    const double dg = __dsqrt_rn(d);
    L[j + j * bs] = dg;
    for (int i = j + 1; i < bs; ++i) {
      double v = L[i + j * bs];
      for (int q = 0; q < j; ++q) v = __dsub_rn(v, __dmul_rn(L[i + q * bs], L[j + q * bs]));
      L[i + j * bs] = __ddiv_rn(v, dg);
    }
    for (int i = 0; i < j; ++i) L[i + j * bs] = 0.0;  // upper triangle unused
  }
}

template <int BS>
__global__ void bj_apply_kernel(int64_t n, const double* __restrict__ f, const double* __restrict__ in,
                                double* out, DevState* st, int col, int pending) {
  if (halted(st)) return;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r0 = b * BS;
  if (r0 >= n) return;
  const double* L = f + b * BS * BS;
  double x[BS];
#pragma unroll
  for (int i = 0; i < BS; ++i) x[i] = r0 + i < n ? in[r0 + i] : 0.0;
#pragma unroll
  for (int i = 0; i < BS; ++i) {
    double v = x[i];
#pragma unroll
    for (int q = 0; q < i; ++q) v = __dsub_rn(v, __dmul_rn(__ldg(L + i + q * BS), x[q]));
    x[i] = __ddiv_rn(v, __ldg(L + i + i * BS));
  }
#pragma unroll
  for (int i = BS - 1; i >= 0; --i) {
    double v = x[i];
#pragma unroll
    for (int q = i + 1; q < BS; ++q) v = __dsub_rn(v, __dmul_rn(__ldg(L + q + i * BS), x[q]));
    x[i] = __ddiv_rn(v, __ldg(L + i + i * BS));
  }
  bool fin = true;
#pragma unroll
  for (int i = 0; i < BS; ++i)
    if (r0 + i < n) {
      out[r0 + i] = x[i];
      fin = fin && isfinite(x[i]);
    }
  if (col >= 0 && !fin && st != nullptr) {
    atomicCAS(pending ? &st->pending : &st->err, 0ull, make_err(4, col));
    if (!pending) st->done = 1;
  }
}

// util.hpp:25-40: the i-th SplitMix64 draw is a pure function of
// seed + (i+1)*golden, so the sequential generator parallelises exactly.
__global__ void random_kernel(int64_t n, int64_t offset, uint64_t seed, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t z = seed + static_cast<uint64_t>(offset + i + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z = z ^ (z >> 31);
  const double unit = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
  out[i] = __dsub_rn(__dmul_rn(2.0, unit), 1.0);
}

// ------------------------------------------------------------------ serial-order Gram

// One warp per Gram entry. Lanes load 32 consecutive (u_l, v_l) pairs
// coalesced and form the rounded products; the ONE ascending chain
// acc = acc + u_l*v_l then runs over the 32 products in lane order (shuffles are
// off the dependency chain), so the entry is bitwise the reference's serial
// sum while memory is streamed at full width. Next chunk is prefetched.
__global__ void __launch_bounds__(128)
    serial_gram_kernel(int64_t n, int ku, int kv, const double* __restrict__ u, int64_t ldu,
                       const double* __restrict__ v, int64_t ldv, double* g, DevState* st) {
  if (halted(st)) return;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (e >= ku * kv) return;
  const int i = e % ku, j = e / ku;
  const double* ui = u + i * ldu;
  const double* vj = v + j * ldv;
  double acc = 0.0;
  double pu = lane < n ? ui[lane] : 0.0, pv = lane < n ? vj[lane] : 0.0;
  for (int64_t l0 = 0; l0 < n; l0 += 32) {
    const double prod = __dmul_rn(pu, pv);
    const int64_t nx = l0 + 32 + lane;
    pu = nx < n ? ui[nx] : 0.0;  // prefetch the next chunk
    pv = nx < n ? vj[nx] : 0.0;
    const int cnt = n - l0 < 32 ? static_cast<int>(n - l0) : 32;
    if (cnt == 32) {
#pragma unroll
      for (int t = 0; t < 32; ++t) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, t));
    } else {
      for (int t = 0; t < cnt; ++t) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, t));
    }
  }
  if (lane == 0) g[e] = acc;
}

// ------------------------------------------------------------------ tree Gram (generic)

constexpr int kTreeBlocks = 296;  // 2 x 148 SMs

__global__ void __launch_bounds__(kThreads)
    tree_gram_kernel(int64_t n, int ku, int kv, const double* __restrict__ u, int64_t ldu,
                     const double* __restrict__ v, int64_t ldv, double* g, double* partial,
                     unsigned* ticket, DevState* st) {
  if (halted(st)) return;
  // kTreeGroup entries per pass over the block's rows: a row of v (and of u
  // when entries share it) is loaded once per group instead of once per entry.
  // Each entry keeps its own accumulator, thread stride and reduction tree, so
  // the result is bitwise the one-entry-per-pass order.
  constexpr int kTreeGroup = 8;
  __shared__ double red[kTreeGroup][kThreads / 32];
  __shared__ bool last;
  const int ne = ku * kv;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t b1 = min(n, b0 + chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e0 = 0; e0 < ne; e0 += kTreeGroup) {
    const int cnt = min(kTreeGroup, ne - e0);
    const double* ui[kTreeGroup];
    const double* vj[kTreeGroup];
    double acc[kTreeGroup];
#pragma unroll
    for (int g = 0; g < kTreeGroup; ++g) {
      const int e = min(e0 + g, ne - 1);
      ui[g] = u + (e % ku) * ldu;
      vj[g] = v + (e / ku) * ldv;
      acc[g] = 0.0;
    }
    for (int64_t l = b0 + threadIdx.x; l < b1; l += kThreads) {
#pragma unroll
      for (int g = 0; g < kTreeGroup; ++g)
        if (g < cnt) acc[g] += ui[g][l] * vj[g][l];
    }
#pragma unroll
    for (int g = 0; g < kTreeGroup; ++g) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[g] += __shfl_down_sync(0xffffffffu, acc[g], off);
      if (lane == 0) red[g][warp] = acc[g];
    }
    __syncthreads();
    if (threadIdx.x < cnt) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += red[threadIdx.x][w];
      partial[static_cast<int64_t>(blockIdx.x) * ne + e0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_partials(partial, gridDim.x, ne, g);
  if (threadIdx.x == 0) *ticket = 0u;
}

// ------------------------------------------------------------------ rank-global breakdown flags
// flags[j] = 1.0 when this rank's speculative MPK saw a non-finite value first
// in basis column j, else 0.0; summed by the packed block's allreduce, so every
// rank raises the same BasisBreakdownError (the lowest column of any rank).
__device__ __forceinline__ void write_pending_flags(int s, const DevState* st, double* flags) {
  const unsigned long long pw = *(volatile const unsigned long long*)&st->pending;
  const int col = pw ? static_cast<int>(pw & 0xffffffffull) : -1;
  for (int j = threadIdx.x; j < s; j += blockDim.x) flags[j] = j == col ? 1.0 : 0.0;
}

__global__ void pending_flags_kernel(int s, const DevState* st, double* flags) {
  write_pending_flags(s, st, flags);
}

// ------------------------------------------------------------------ packed DMMA reduction
//
// One pass over Q, Z, P (= A Z columns 1..s) and r produces the whole
// one-allreduce block {G1 = Q^T P, G2 = Z^T P, c1 = Z^T r, c2 = Q^T r, rr}.
// A warp streams 32-row chunks with coalesced loads (lane = row); the r
// products are plain per-lane FMAs, the (2s x s) Gram products run on the
// FP64 tensor cores (mma.sync m8n8k4, DMMA) from a warp-private shared-memory
// tile laid out [column][row] with a 36-double stride so the fragment loads
// are bank-conflict free. Per-warp partials are combined in a fixed order and
// the last block reduces the block partials in block order.

constexpr int kPackWarps = 8;
constexpr int kPackStride = 36;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int S>
struct PackShape {
  static constexpr int MT = (2 * S + 7) / 8;
  static constexpr int NT = (S + 7) / 8;
  static constexpr int UC = MT * 8;
  static constexpr int PC = NT * 8;
  static constexpr int NOUT = 2 * S * S + 2 * S + 1;
  static constexpr size_t smem_warp = static_cast<size_t>(UC + PC) * kPackStride;
  static constexpr size_t smem_bytes = smem_warp * kPackWarps * sizeof(double);
};

#ifndef CS_PACK_MINB
#define CS_PACK_MINB 2
#endif
__device__ __forceinline__ unsigned long long xr_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void xr_st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// the last block of the pack: exchange + fixed-order sum (see XredArgs)
__device__ __forceinline__ void xred_exchange(const XredArgs& x, double* packed, DevState* st) {
  const int N = x.nranks, me = x.rank, par = static_cast<int>(x.epoch & 1ull);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp r (< N) stores the block into rank r's slot, then its lane 0 fences once
  // (one MEMBAR.SYS per peer, not per thread) and releases the flag
  if (warp < N) {
    const int r = warp;
    double* dst = (r == me ? x.slots : x.peer_slots[r]) +
                  (static_cast<int64_t>(par) * N + me) * kXredSlot;
    for (int e = lane; e < x.npack; e += 32) dst[e] = packed[e];
    __syncwarp();
    if (lane == 0 && r != me) {
      __threadfence_system();
      xr_st_release(x.peer_flags[r] + me, x.epoch);
    }
  }
  if (warp == (N < 8 ? N : 0) && lane < N && lane != me) {  // wait for every source (bounded)
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (xr_ld_acquire(x.flags + lane) < x.epoch) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20ull * 1000000000ull) {
        atomicCAS(&st->err, 0ull, make_err(11 /*CS_ERR_NCCL*/, 1));
        st->done = 1;
        break;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < x.npack; e += blockDim.x) {
    double sum = 0.0;
    for (int r = 0; r < N; ++r)
      sum += __ldcg(x.slots + (static_cast<int64_t>(par) * N + r) * kXredSlot + e);
    packed[e] = sum;
  }
}

// XR: the multi-GPU instance with the fused allreduce (the single-GPU instance
// carries no exchange code: measured 35 % slower with it compiled in)
template <int S, bool PZ, bool XR>
__global__ void __launch_bounds__(kPackWarps * 32, CS_PACK_MINB)
    pack_kernel(int64_t n, int64_t ld, const double* __restrict__ Q, const double* __restrict__ Z,
                const double* __restrict__ P, const double* __restrict__ r, double* packed,
                double* partial, unsigned* ticket, DevState* st, double* flags, PzArgs pz,
                const __grid_constant__ XredArgs xr) {
  using Sh = PackShape<S>;
  if (halted(st)) return;
  extern __shared__ double smem[];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* sU = smem + warp * Sh::smem_warp;
  double* sP = sU + Sh::UC * kPackStride;
  for (int c = 2 * S; c < Sh::UC; ++c) sU[c * kPackStride + lane] = 0.0;
  for (int c = S; c < Sh::PC; ++c) sP[c * kPackStride + lane] = 0.0;

  double acc[Sh::MT][Sh::NT][2];
#pragma unroll
  for (int m = 0; m < Sh::MT; ++m)
#pragma unroll
    for (int q = 0; q < Sh::NT; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
  double c1[S], c2[S], rr = 0.0;
#pragma unroll
  for (int i = 0; i < S; ++i) c1[i] = c2[i] = 0.0;

  const int64_t nchunks = (n + 31) / 32;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kPackWarps;
  for (int64_t ch = static_cast<int64_t>(blockIdx.x) * kPackWarps + warp; ch < nchunks;
       ch += stride) {
    const int64_t row = ch * 32 + lane;
    const bool ok = row < n;
    double qv[S], zv[S], pv[S];
    if constexpr (PZ) {
      double zz[S + 1];
#pragma unroll
      for (int i = 0; i < S; ++i) {
        qv[i] = ok ? __ldcs(Q + i * ld + row) : 0.0;
        zz[i] = ok ? __ldcs(Z + i * ld + row) : 0.0;
        zv[i] = zz[i];
      }
      zz[S] = ok ? __ldcs(pz.zs + row) : 0.0;
      const double di = pz.diag ? (ok ? __ldg(pz.diag + row) : 1.0) : pz.dconst;
      p_from_z<S>(zz, pz, di, pv);
    } else {
#pragma unroll
      for (int i = 0; i < S; ++i) {
        qv[i] = ok ? __ldcs(Q + i * ld + row) : 0.0;
        zv[i] = ok ? __ldcs(Z + i * ld + row) : 0.0;
        pv[i] = ok ? __ldcs(P + i * ld + row) : 0.0;
      }
    }
    double rv;
    if constexpr (PZ) {
      const double di = pz.diag ? (ok ? __ldg(pz.diag + row) : 1.0) : pz.dconst;
      rv = pz.r_from_z0 ? (ok ? zv[0] * di : 0.0) : (ok ? __ldcs(r + row) : 0.0);
    } else {
      rv = ok ? __ldcs(r + row) : 0.0;
    }
    rr = fma(rv, rv, rr);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      c2[i] = fma(qv[i], rv, c2[i]);
      c1[i] = fma(zv[i], rv, c1[i]);
      sU[i * kPackStride + lane] = qv[i];
      sU[(S + i) * kPackStride + lane] = zv[i];
      sP[i * kPackStride + lane] = pv[i];
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double a[Sh::MT], b[Sh::NT];
#pragma unroll
      for (int m = 0; m < Sh::MT; ++m) a[m] = sU[(m * 8 + g) * kPackStride + kk * 4 + t];
#pragma unroll
      for (int q = 0; q < Sh::NT; ++q) b[q] = sP[(q * 8 + g) * kPackStride + kk * 4 + t];
#pragma unroll
      for (int m = 0; m < Sh::MT; ++m)
#pragma unroll
        for (int q = 0; q < Sh::NT; ++q) dmma(acc[m][q], a[m], b[q]);
    }
    __syncwarp();
  }
  // warp-level: plain accumulators by shuffle tree
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    rr += __shfl_down_sync(0xffffffffu, rr, off);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      c1[i] += __shfl_down_sync(0xffffffffu, c1[i], off);
      c2[i] += __shfl_down_sync(0xffffffffu, c2[i], off);
    }
  }
  __syncthreads();  // tiles are dead; reuse smem as [warp][NOUT]
  double* out = smem + warp * Sh::NOUT;
#pragma unroll
  for (int m = 0; m < Sh::MT; ++m)
#pragma unroll
    for (int q = 0; q < Sh::NT; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = m * 8 + g;       // U column: Q_i (i < S) or Z_{i-S}
        const int j = q * 8 + 2 * t + e;  // P column
        if (i < 2 * S && j < S) out[(i < S ? 0 : S * S) + (i % S) + j * S] = acc[m][q][e];
      }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) {
      out[2 * S * S + i] = c1[i];
      out[2 * S * S + S + i] = c2[i];
    }
    out[2 * S * S + 2 * S] = rr;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < Sh::NOUT; e += kPackWarps * 32) {
    double s = 0.0;
    for (int w = 0; w < kPackWarps; ++w) s += smem[w * Sh::NOUT + e];
    partial[static_cast<int64_t>(blockIdx.x) * Sh::NOUT + e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_partials(partial, gridDim.x, Sh::NOUT, packed);
  if (flags) write_pending_flags(S, st, flags);
  if (threadIdx.x == 0) *ticket = 0u;
  if constexpr (XR) {  // fused NVLink allreduce of packed[0, npack)
    __syncthreads();
    xred_exchange(xr, packed, st);
  }
}

int pack_grid(int64_t n) {
  const int64_t chunks = (n + 31) / 32;
  const int64_t want = (chunks + kPackWarps - 1) / kPackWarps;
  const int64_t cap = 148 * (CS_PACK_MINB > 2 ? CS_PACK_MINB : 3);
  return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

template <int S>
void pack_launch(int64_t n, int64_t ld, const double* q, const double* z, const double* p,
                 const double* r, double* packed, double* partial, unsigned* ticket, DevState* st,
                 double* flags, cudaStream_t strm, const PzArgs& pz, const XredArgs& xr) {
  using Sh = PackShape<S>;
  const bool pzm = pz.zs != nullptr;
  auto kern = xr.nranks > 1 ? (pzm ? pack_kernel<S, true, true> : pack_kernel<S, false, true>)
                            : (pzm ? pack_kernel<S, true, false> : pack_kernel<S, false, false>);
  // one wave of resident blocks (a grid past the resident count leaves a
  // half-occupied second wave: 444 blocks at 2 per SM measured 0.64 ms at 256^3)
  const int per_sm = kernel_setup(reinterpret_cast<const void*>(kern), kPackWarps * 32,
                                  static_cast<int>(Sh::smem_bytes));
  const int64_t want = pack_grid(n);
  const int grid = static_cast<int>(std::min<int64_t>(want, 148 * per_sm));
  kern<<<grid, kPackWarps * 32, Sh::smem_bytes, strm>>>(n, ld, q, z, p, r, packed, partial, ticket,
                                                        st, flags, pz, xr);
  CS_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ update pass
//
// Per row, in one read of each operand:
//   (beta)  Q_j <- Z_j + sum_q beta_qj Q_q ; AQ_j <- P_j + sum_q beta_qj AQ_q
//   (xr)    for j: x <- x + alpha_j Q_j ; r <- r + (-alpha_j) AQ_j
//   (z0)    z_0 <- M^-1 r (the next MPK's first column) + finite check
// with the reference operation order (block_update, then the interleaved axpys).

// per-column base pointers as kernel parameters: the column addresses become
// uniform-register operands instead of 64-bit per-thread address registers
template <int SM>
struct Cols {
  double* q[SM];
  double* aq[SM];
  const double* z[SM];
  const double* p[SM];
};

// Block = 8 warps over 128 rows: warps 0-3 take the Q role (Q_j <- Z_j + sum_q
// beta_qj Q_q, then x += sum_j alpha_j Q_j), warps 4-7 the AQ role (AQ_j <- P_j +
// sum_q beta_qj AQ_q, then r += sum_j (-alpha_j) AQ_j and z_0 = M^-1 r). The two
// halves are independent, so each thread holds 2s operands instead of 4s.
constexpr int kUpdRows = 128;

// AQ role of the PZ schedule: the new-basis part P of this row derived from Z
template <int S>
__device__ __forceinline__ void p_row_from_z(const UpdateArgs& a, const Cols<S>& c, int64_t i,
                                             double (&p)[S]) {
  double zz[S + 1];
#pragma unroll
  for (int q = 0; q < S; ++q) zz[q] = c.z[q][i];
  zz[S] = a.pz.zs[i];
  p_from_z<S>(zz, a.pz, a.pz.diag ? a.pz.diag[i] : a.pz.dconst, p);
}

#ifndef CS_UPD_FMA
#define CS_UPD_FMA 0  // 1: one FMA per term in the fast pass (measured slower: profiles/r02_update_pack_sweep.txt)
#endif
#ifndef CS_UPD_PAIRED
#define CS_UPD_PAIRED 1  // Q/AQ roles of a row in one warp (0: block halves + block barrier)
#endif
// Lanes 0-15 of a warp take the Q role of 16 rows, lanes 16-31 the AQ role of
// the SAME rows (each load instruction moves two full 128-byte segments). The
// AQ role overwrites Z column 0 with z_0 = M^-1 r, which the Q role of its row
// reads: the pair shares a warp, so a warp barrier (or, in the PZ schedule, the
// shuffle that hands the Q lane's Z row to its AQ lane) orders the load before
// the store -- no block-wide barrier.
template <int S, bool BETA, bool XR, bool Z0, bool PZ = false>
__global__ void __launch_bounds__(kThreads) update_kernel(UpdateArgs a, Cols<(S > 0 ? S : kMaxS)> c) {
  static_assert(!PZ || (S > 0 && BETA && Z0), "PZ: compile-time order, fast beta pass");
  if (halted(a.st)) return;
  constexpr int SM = S > 0 ? S : kMaxS;
  const int s = S > 0 ? S : a.s;
  __shared__ double sh_alpha[SM];
  __shared__ double sh_beta[BETA ? SM * SM : 1];
  for (int t = threadIdx.x; t < s; t += blockDim.x) sh_alpha[t] = XR ? a.alpha[t] : 0.0;
  if constexpr (BETA)
    for (int t = threadIdx.x; t < s * s; t += blockDim.x) sh_beta[t] = a.beta[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const bool aq_role = CS_UPD_PAIRED ? lane >= 16 : threadIdx.x >= kUpdRows;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kUpdRows +
                    (CS_UPD_PAIRED ? (threadIdx.x >> 5) * 16 + (lane & 15)
                                   : (threadIdx.x & (kUpdRows - 1)));
  const bool active = i < a.n;
  double* const* dst = aq_role ? c.aq : c.q;      // updated in place
  const double* const* src = aq_role ? c.p : c.z; // new basis part
  double acc = 0.0;
  double lo[SM], hi[SM];
#pragma unroll
  for (int q = 0; q < SM; ++q) lo[q] = hi[q] = 0.0;
  double zs_i = 0.0, d_i = 1.0;
  if (active) {
    if constexpr (XR) acc = aq_role ? a.r[i] : a.x[i];
#pragma unroll
    for (int q = 0; q < SM; ++q)
      if (q < s) {
        lo[q] = dst[q][i];
        if (BETA && !(PZ && aq_role)) hi[q] = src[q][i];
      }
    if constexpr (PZ)
      if (aq_role) {
        zs_i = a.pz.zs[i];
        d_i = a.pz.diag ? a.pz.diag[i] : a.pz.dconst;
      }
  }
  if constexpr (PZ && CS_UPD_PAIRED) {  // every lane: the Q lane's Z row to its AQ lane
    double zz[SM + 1];
#pragma unroll
    for (int q = 0; q < SM; ++q) zz[q] = __shfl_xor_sync(0xffffffffu, hi[q], 16);
    zz[SM] = zs_i;
    if (aq_role) p_from_z<SM>(zz, a.pz, d_i, hi);
  } else if constexpr (PZ) {
    if (aq_role && active) p_row_from_z<SM>(a, c, i, hi);
    __syncthreads();
  } else if constexpr (Z0) {
    if (CS_UPD_PAIRED) __syncwarp();
    else __syncthreads();
  }
  if (!active) return;  if constexpr (BETA) {
    // out_j = y_j + sum_q c_qj x_q, ascending q for every j (dense_ops.cpp:35-39);
    // the fast pass (Z0) contracts each term into one FMA (half the FP64 issue)
#pragma unroll
    for (int q = 0; q < SM; ++q)
      if (q < s) {
        const double xq = lo[q];
#pragma unroll
        for (int j = 0; j < SM; ++j)
          if (j < s) {
            if constexpr (Z0 && CS_UPD_FMA) hi[j] = fma(sh_beta[q + j * s], xq, hi[j]);
            else hi[j] = __dadd_rn(hi[j], __dmul_rn(sh_beta[q + j * s], xq));
          }
      }
#pragma unroll
    for (int j = 0; j < SM; ++j)
      if (j < s) dst[j][i] = hi[j];
  }
  if constexpr (XR) {
    // solver.cpp:159-162: x += alpha_j q_j ; r += (-alpha_j) aq_j, ascending j
    const double sign = aq_role ? -1.0 : 1.0;
#pragma unroll
    for (int j = 0; j < SM; ++j)
      if (j < s) {
        if constexpr (Z0 && CS_UPD_FMA) acc = fma(sign * sh_alpha[j], BETA ? hi[j] : lo[j], acc);
        else acc = __dadd_rn(acc, __dmul_rn(sign * sh_alpha[j], BETA ? hi[j] : lo[j]));
      }
    if (aq_role) a.r[i] = acc;
    else a.x[i] = acc;
  }
  if constexpr (Z0) {
    if (aq_role) {
      const double z = !a.inv_diag        ? acc
                       : a.inv_const != 0.0 ? __dmul_rn(a.inv_const, acc)
                                            : __dmul_rn(a.inv_diag[i], acc);
      a.zw[i] = z;
      if (a.push_lo != nullptr && i < a.send_lo) a.push_lo[i] = z;
      if (a.push_hi != nullptr && i >= a.hi_begin) a.push_hi[i - a.hi_begin] = z;
      if (!isfinite(z)) atomicCAS(&a.st->pending, 0ull, make_err(4, 0));
    }
  }
}

// update_kernel<S, true, true, true> fused with the explicit Gram of the new
// basis: a persistent grid walks 128-row tiles; each tile's new Q and AQ rows
// are also staged in shared memory ([column][row], stride 132 doubles: the
// DMMA fragment loads are conflict-free) and every warp folds 16 of its rows
// into its (Q^T AQ) accumulator tiles with FP64 mma.sync m8n8k4 (the pack
// kernel's fragment layout). No extra HBM traffic: the Gram reads only what
// the pass already holds. Per-warp tiles are summed in a fixed order into one
// partial per block; the last block reduces the partials in block order.
constexpr int kGramStride = 132;

template <int S, bool PZ>
__global__ void __launch_bounds__(kThreads)
    update_gram_kernel(UpdateArgs a, Cols<S> c, double* partial, unsigned* ticket, double* wout) {
  if (halted(a.st)) return;
  constexpr int MT = (S + 7) / 8;
  constexpr int SP = MT * 8;
  __shared__ double sh_alpha[S];
  __shared__ double sh_beta[S * S];
  __shared__ double tile[2][SP][kGramStride];
  // Q role's Z rows for the AQ role (static shared memory allows it up to s = 8;
  // larger orders reload Z from global memory)
  constexpr bool kShZ = PZ && S <= 8;
  __shared__ double sh_z[kShZ ? S : 1][kShZ ? kUpdRows : 1];
  __shared__ bool last;
  for (int t = threadIdx.x; t < S; t += blockDim.x) sh_alpha[t] = a.alpha[t];
  for (int t = threadIdx.x; t < S * S; t += blockDim.x) sh_beta[t] = a.beta[t];
  if constexpr (SP > S) {
    for (int t = threadIdx.x; t < 2 * (SP - S) * kGramStride; t += blockDim.x) {
      const int h = t / ((SP - S) * kGramStride), rem = t % ((SP - S) * kGramStride);
      tile[h][S + rem / kGramStride][rem % kGramStride] = 0.0;  // padded columns stay zero
    }
  }
  __syncthreads();
  const bool aq_role = threadIdx.x >= kUpdRows;
  const int rl = threadIdx.x & (kUpdRows - 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  double* const* dst = aq_role ? c.aq : c.q;
  const double* const* src = aq_role ? c.p : c.z;
  const double sign = aq_role ? -1.0 : 1.0;
  double acc[MT][MT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int q = 0; q < MT; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kUpdRows;
  for (int64_t t0 = static_cast<int64_t>(blockIdx.x) * kUpdRows; t0 < a.n; t0 += stride) {
    const int64_t i = t0 + rl;
    const bool active = i < a.n;
    double lo[S], hi[S];
    double xr = 0.0;
    double zs_i = 0.0, d_i = 1.0;
    if (active) {
      xr = aq_role ? a.r[i] : a.x[i];
#pragma unroll
      for (int q = 0; q < S; ++q) {
        lo[q] = dst[q][i];
        if (!(PZ && aq_role)) hi[q] = src[q][i];
      }
      if constexpr (kShZ) {
        if (!aq_role) {
#pragma unroll
          for (int q = 0; q < S; ++q) sh_z[q][rl] = hi[q];
        } else {
          zs_i = a.pz.zs[i];
          d_i = a.pz.diag ? a.pz.diag[i] : a.pz.dconst;
        }
      } else if constexpr (PZ) {
        if (aq_role) p_row_from_z<S>(a, c, i, hi);
      }
    } else {
#pragma unroll
      for (int q = 0; q < S; ++q) lo[q] = hi[q] = 0.0;
    }
    // the AQ role overwrites Z column 0 (z_0) that the Q role of the same rows
    // reads above; the previous tile's fragment loads also end here
    __syncthreads();
    if constexpr (kShZ) {
      if (aq_role && active) {
        double zz[S + 1];
#pragma unroll
        for (int q = 0; q < S; ++q) zz[q] = sh_z[q][rl];
        zz[S] = zs_i;
        p_from_z<S>(zz, a.pz, d_i, hi);
      }
    }
    // out_j = y_j + sum_q c_qj x_q, ascending q for every j (fused as in update_kernel)
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const double xq = lo[q];
#pragma unroll
      for (int j = 0; j < S; ++j) hi[j] = fma(sh_beta[q + j * S], xq, hi[j]);
    }
#pragma unroll
    for (int j = 0; j < S; ++j) tile[aq_role][j][rl] = active ? hi[j] : 0.0;
    if (active) {
#pragma unroll
      for (int j = 0; j < S; ++j) dst[j][i] = hi[j];
      // solver.cpp:159-162: x += alpha_j q_j ; r += (-alpha_j) aq_j, ascending j
#pragma unroll
      for (int j = 0; j < S; ++j) xr = fma(sign * sh_alpha[j], hi[j], xr);
      if (aq_role) {
        a.r[i] = xr;
        const double z = !a.inv_diag        ? xr
                         : a.inv_const != 0.0 ? __dmul_rn(a.inv_const, xr)
                                              : __dmul_rn(a.inv_diag[i], xr);
        a.zw[i] = z;
        if (a.push_lo != nullptr && i < a.send_lo) a.push_lo[i] = z;
        if (a.push_hi != nullptr && i >= a.hi_begin) a.push_hi[i - a.hi_begin] = z;
        if (!isfinite(z)) atomicCAS(&a.st->pending, 0ull, make_err(4, 0));
      } else {
        a.x[i] = xr;
      }
    }
    __syncthreads();
    // warp w: rows [16w, 16w + 16) of the tile, 4 k-steps of 4 rows
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k0 = warp * 16 + kk * 4 + t4;
      double fa[MT], fb[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        fa[m] = tile[0][m * 8 + g][k0];
        fb[m] = tile[1][m * 8 + g][k0];
      }
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int q = 0; q < MT; ++q) dmma(acc[m][q], fa[m], fb[q]);
    }
  }
  __syncthreads();  // tiles are dead: reuse as [warp][S*S]
  double* out = &tile[0][0][0];
  static_assert(2 * SP * kGramStride >= (kThreads / 32) * S * S, "reduction scratch");
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int q = 0; q < MT; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ii = m * 8 + g, jj = q * 8 + 2 * t4 + e;
        if (ii < S && jj < S) out[warp * S * S + ii + jj * S] = acc[m][q][e];
      }
  __syncthreads();
  for (int e = threadIdx.x; e < S * S; e += blockDim.x) {
    double sum = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) sum += out[w * S * S + e];
    partial[static_cast<int64_t>(blockIdx.x) * S * S + e] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_partials(partial, gridDim.x, S * S, wout);
  if (threadIdx.x == 0) *ticket = 0u;
}

// True-residual schedule (CS_VAR_TRUE_R): the pass keeps only the
// Q role -- Q_j <- Z_j + sum_q beta_qj Q_q, x <- x + sum_j alpha_j Q_j, in the
// fast pass's operation order -- and no AQ block or recursive r: the next
// launch forms r = b - A x and z_0 = M^-1 r (kResidF). One row per thread;
// x's boundary rows go to the neighbours' ghost slots for that residual.
// Bytes per row: 8 (3s + 2) instead of 8 (5s + 6).
template <int S, bool BETA>
__global__ void __launch_bounds__(kThreads) update_tr_kernel(UpdateArgs a, Cols<S> c) {
  if (halted(a.st)) return;
  __shared__ double sh_alpha[S];
  __shared__ double sh_beta[BETA ? S * S : 1];
  for (int t = threadIdx.x; t < S; t += blockDim.x) sh_alpha[t] = a.alpha[t];
  if constexpr (BETA)
    for (int t = threadIdx.x; t < S * S; t += blockDim.x) sh_beta[t] = a.beta[t];
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
  if (i >= a.n) return;
  double acc = a.x[i];
  double lo[S], hi[S];
#pragma unroll
  for (int q = 0; q < S; ++q) {
    lo[q] = c.q[q][i];
    if constexpr (BETA) hi[q] = c.z[q][i];
  }
  if constexpr (BETA) {
#pragma unroll
    for (int q = 0; q < S; ++q)
#pragma unroll
      for (int j = 0; j < S; ++j) hi[j] = __dadd_rn(hi[j], __dmul_rn(sh_beta[q + j * S], lo[q]));
#pragma unroll
    for (int j = 0; j < S; ++j) c.q[j][i] = hi[j];
  }
#pragma unroll
  for (int j = 0; j < S; ++j) acc = __dadd_rn(acc, __dmul_rn(sh_alpha[j], BETA ? hi[j] : lo[j]));
  a.x[i] = acc;
  if (a.push_lo != nullptr && i < a.send_lo) a.push_lo[i] = acc;
  if (a.push_hi != nullptr && i >= a.hi_begin) a.push_hi[i - a.hi_begin] = acc;
}

template <int S>
Cols<S> make_cols(const UpdateArgs& a) {
  Cols<S> c{};
  const int s = S == kMaxS ? a.s : S;
  for (int j = 0; j < s; ++j) {
    c.q[j] = a.q ? a.q + j * a.ld : nullptr;
    c.aq[j] = a.aq ? a.aq + j * a.ld : nullptr;
    c.z[j] = a.z ? a.z + j * a.ld : nullptr;
    c.p[j] = a.p ? a.p + j * a.ld : nullptr;
  }
  return c;
}

template <bool BETA, bool XR, bool Z0>
void update_dispatch(const UpdateArgs& a, cudaStream_t st) {
  const unsigned grid = grid_for(a.n, kUpdRows);
  if (a.n == 0) return;
#define CSG_UPD(SV)                                                                          \
  if constexpr (BETA && Z0 && SV > 0) {                                                      \
    if (a.pz.zs) {                                                                           \
      update_kernel<SV, BETA, XR, Z0, true><<<grid, kThreads, 0, st>>>(a, make_cols<SV>(a)); \
      break;                                                                                 \
    }                                                                                        \
  }                                                                                          \
  update_kernel<SV, BETA, XR, Z0><<<grid, kThreads, 0, st>>>(a, make_cols<SV ? SV : kMaxS>(a))
  switch (a.s) {
    case 1: CSG_UPD(1); break;
    case 2: CSG_UPD(2); break;
    case 3: CSG_UPD(3); break;
    case 4: CSG_UPD(4); break;
    case 5: CSG_UPD(5); break;
    case 6: CSG_UPD(6); break;
    case 8: CSG_UPD(8); break;
    case 10: CSG_UPD(10); break;
    case 12: CSG_UPD(12); break;
    case 16: CSG_UPD(16); break;
    default:
      if (BETA && a.pz.zs) throw LibError{9, 0, "update: P-from-Z needs a specialised order"};
      CSG_UPD(0);
      break;
  }
#undef CSG_UPD
  CS_CUDA(cudaGetLastError());
}

// generic block_update (unit entry), dense_ops.cpp:29-42
__global__ void block_update_kernel(int64_t n, int m, int k, const double* __restrict__ y,
                                    const double* __restrict__ x, const double* __restrict__ c,
                                    double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < k; ++j) {
    double o = y[j * n + i];
    for (int q = 0; q < m; ++q) o = __dadd_rn(o, __dmul_rn(c[q + j * m], x[q * n + i]));
    out[j * n + i] = o;
  }
}

// ------------------------------------------------------------------ classical PCG vector steps
// which 0: z = M^-1 r; p = z                         (solver.cpp:228-231)
// which 1: x += step p; r -= step q  (+ fast dots r.r, r.M^-1 r)   (solver.cpp:241-243)
// which 2: p = M^-1 r + beta p                       (solver.cpp:254-259)
// which 3: fast dots r.r and r.M^-1 r only (setup)

template <int WHICH, bool DOTS>
__global__ void __launch_bounds__(kThreads)
    pcg_vec_kernel(int64_t n, double* x, double* r, double* p, const double* __restrict__ q,
                   const double* __restrict__ inv_diag, DevState* st, double* partial,
                   unsigned* ticket, double* result) {
  if (halted(st)) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double d_rr = 0.0, d_rz = 0.0;
  if (i < n) {
    if constexpr (WHICH == 0) {
      const double rv = r[i];
      p[i] = inv_diag ? __dmul_rn(inv_diag[i], rv) : rv;
    } else if constexpr (WHICH == 1) {
      const double step = st->scal[0];
      x[i] = __dadd_rn(x[i], __dmul_rn(step, p[i]));
      const double rv = __dadd_rn(r[i], __dmul_rn(-step, q[i]));
      r[i] = rv;
      if constexpr (DOTS) {
        const double zv = inv_diag ? __dmul_rn(inv_diag[i], rv) : rv;
        d_rr = rv * rv;
        d_rz = rv * zv;
      }
    } else if constexpr (WHICH == 2) {
      const double rv = r[i];
      const double zv = inv_diag ? __dmul_rn(inv_diag[i], rv) : rv;
      p[i] = __dadd_rn(zv, __dmul_rn(st->scal[1], p[i]));
    } else {
      const double rv = r[i];
      const double zv = inv_diag ? __dmul_rn(inv_diag[i], rv) : rv;
      d_rr = rv * rv;
      d_rz = rv * zv;
    }
  }
  if constexpr (DOTS) {
    __shared__ double red[2][kThreads / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      d_rr += __shfl_down_sync(0xffffffffu, d_rr, off);
      d_rz += __shfl_down_sync(0xffffffffu, d_rz, off);
    }
    if (lane == 0) {
      red[0][warp] = d_rr;
      red[1][warp] = d_rz;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) {
        a += red[0][w];
        b += red[1][w];
      }
      partial[2 * blockIdx.x] = a;
      partial[2 * blockIdx.x + 1] = b;
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      finalize_partials(partial, gridDim.x, 2, result);
      if (threadIdx.x == 0) *ticket = 0u;
    }
  }
}

__global__ void scale2_kernel(int64_t n, double* v, double* g, const double* __restrict__ sv,
                              const double* __restrict__ sg, const double* denom, DevState* st) {
  if (halted(st)) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = *denom;
  v[i] = __ddiv_rn(sv[i], d);
  g[i] = __ddiv_rn(sg[i], d);
}

}  // namespace

// ------------------------------------------------------------------ launchers

void launch_precond_apply(int64_t n, const double* inv_diag, const double* in, double* out,
                          DevState* st, int col, int pending, cudaStream_t s) {
  if (n == 0) return;
  precond_kernel<<<grid_for(n), kThreads, 0, s>>>(n, inv_diag, in, out, st, col, pending);
  CS_CUDA(cudaGetLastError());
}

void launch_bj_factor(int64_t nblocks, int bs, double* f, int* bad_block, cudaStream_t s) {
  if (nblocks == 0) return;
  bj_factor_kernel<<<grid_for(nblocks, 128), 128, 0, s>>>(nblocks, bs, f, bad_block);
  CS_CUDA(cudaGetLastError());
}

void launch_bj_apply(int64_t n, int bs, const double* f, const double* in, double* out,
                     DevState* st, int col, int pending, cudaStream_t s) {
  if (n == 0) return;
  const int64_t nb = (n + bs - 1) / bs;
  const unsigned grid = grid_for(nb, 128);
#define CSG_BJ(B)                                                                               \
  case B:                                                                                      \
    bj_apply_kernel<B><<<grid, 128, 0, s>>>(n, f, in, out, st, col, pending);                  \
    break
  switch (bs) {
    CSG_BJ(1); CSG_BJ(2); CSG_BJ(3); CSG_BJ(4); CSG_BJ(5); CSG_BJ(6); CSG_BJ(7); CSG_BJ(8);
    CSG_BJ(9); CSG_BJ(10); CSG_BJ(11); CSG_BJ(12); CSG_BJ(13); CSG_BJ(14); CSG_BJ(15); CSG_BJ(16);
    default: throw LibError{8, 0, "block_jacobi: bs must be in [1, 16]"};
  }
#undef CSG_BJ
  CS_CUDA(cudaGetLastError());
}

void launch_random_vector(int64_t n, int64_t offset, uint64_t seed, double* out, cudaStream_t s) {
  if (n == 0) return;
  random_kernel<<<grid_for(n), kThreads, 0, s>>>(n, offset, seed, out);
  CS_CUDA(cudaGetLastError());
}

void launch_serial_gram(int64_t n, int ku, int kv, const double* u, int64_t ldu, const double* v,
                        int64_t ldv, double* g, DevState* st, cudaStream_t s) {
  const int ne = ku * kv;
  serial_gram_kernel<<<grid_for(static_cast<int64_t>(ne) * 32, 128), 128, 0, s>>>(n, ku, kv, u, ldu,
                                                                                  v, ldv, g, st);
  CS_CUDA(cudaGetLastError());
}

size_t tree_gram_partial_doubles(int64_t, int ku, int kv) {
  return static_cast<size_t>(kTreeBlocks) * ku * kv;
}

void launch_tree_gram(int64_t n, int ku, int kv, const double* u, int64_t ldu, const double* v,
                      int64_t ldv, double* g, double* partial, unsigned* ticket, DevState* st,
                      cudaStream_t s) {
  tree_gram_kernel<<<kTreeBlocks, kThreads, 0, s>>>(n, ku, kv, u, ldu, v, ldv, g, partial, ticket,
                                                    st);
  CS_CUDA(cudaGetLastError());
}

bool pack_supported(int s) {
  switch (s) {
    case 1: case 2: case 3: case 4: case 5: case 6: case 8: case 10: case 12: case 16:
      return true;
    default:
      return false;
  }
}

size_t pack_partial_doubles(int s, int64_t n) {
  return static_cast<size_t>(pack_grid(n)) * (2 * s * s + 2 * s + 1);
}

void launch_pack(int s, int64_t n, int64_t ld, const double* q, const double* z, const double* p,
                 const double* r, double* packed, double* partial, unsigned* ticket, DevState* st,
                 double* flags, cudaStream_t strm, const PzArgs& pz, const XredArgs& xr) {
#define CSG_PACK(SV) \
  pack_launch<SV>(n, ld, q, z, p, r, packed, partial, ticket, st, flags, strm, pz, xr)
  switch (s) {
    case 1: CSG_PACK(1); break;
    case 2: CSG_PACK(2); break;
    case 3: CSG_PACK(3); break;
    case 4: CSG_PACK(4); break;
    case 5: CSG_PACK(5); break;
    case 6: CSG_PACK(6); break;
    case 8: CSG_PACK(8); break;
    case 10: CSG_PACK(10); break;
    case 12: CSG_PACK(12); break;
    case 16: CSG_PACK(16); break;
    default: throw LibError{9, 0, "pack: unsupported s"};
  }
#undef CSG_PACK
}

bool update_gram_supported(int s) {
  switch (s) {
    case 1: case 2: case 3: case 4: case 5: case 6: case 8: case 10: case 12: case 16:
      return true;
    default:
      return false;
  }
}

constexpr int kUpdGramMaxBlocks = 148 * 8;

size_t update_gram_partial_doubles(int s) {
  return static_cast<size_t>(kUpdGramMaxBlocks) * s * s;
}

template <int S>
void update_gram_launch(const UpdateArgs& a, double* partial, unsigned* ticket, double* wout,
                        cudaStream_t st) {
  auto kern = a.pz.zs ? update_gram_kernel<S, true> : update_gram_kernel<S, false>;
  const int per_sm = kernel_setup(reinterpret_cast<const void*>(kern), kThreads, 0);
  const int64_t tiles = (a.n + kUpdRows - 1) / kUpdRows;
  const int grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>({tiles, 148 * static_cast<int64_t>(per_sm), kUpdGramMaxBlocks})));
  kern<<<grid, kThreads, 0, st>>>(a, make_cols<S>(a), partial, ticket, wout);
  CS_CUDA(cudaGetLastError());
}

bool launch_fast_update_gram(const UpdateArgs& a, double* partial, unsigned* ticket, double* wout,
                             cudaStream_t st) {
  if (a.beta == nullptr) return false;
  switch (a.s) {
    case 1: update_gram_launch<1>(a, partial, ticket, wout, st); return true;
    case 2: update_gram_launch<2>(a, partial, ticket, wout, st); return true;
    case 3: update_gram_launch<3>(a, partial, ticket, wout, st); return true;
    case 4: update_gram_launch<4>(a, partial, ticket, wout, st); return true;
    case 5: update_gram_launch<5>(a, partial, ticket, wout, st); return true;
    case 6: update_gram_launch<6>(a, partial, ticket, wout, st); return true;
    case 8: update_gram_launch<8>(a, partial, ticket, wout, st); return true;
    case 10: update_gram_launch<10>(a, partial, ticket, wout, st); return true;
    case 12: update_gram_launch<12>(a, partial, ticket, wout, st); return true;
    case 16: update_gram_launch<16>(a, partial, ticket, wout, st); return true;
    default: return false;
  }
}

void launch_pending_flags(int s, const DevState* st, double* flags, cudaStream_t strm) {
  pending_flags_kernel<<<1, 64, 0, strm>>>(s, st, flags);
  CS_CUDA(cudaGetLastError());
}

void launch_fast_update(const UpdateArgs& a, cudaStream_t s) {
  if (a.beta != nullptr)
    update_dispatch<true, true, true>(a, s);
  else
    update_dispatch<false, true, true>(a, s);
}

bool launch_fast_update_tr(const UpdateArgs& a, cudaStream_t st) {
  if (a.n == 0) return true;
  // one row per thread (a row-pair variant with 16-byte accesses measured 25 %
  // slower at 256^3: profiles/r02h_ab_update_pairs_256.txt)
  const unsigned grid = grid_for(a.n);
#define CSG_TR(SV)                                                                          \
  case SV:                                                                                  \
    if (a.beta) update_tr_kernel<SV, true><<<grid, kThreads, 0, st>>>(a, make_cols<SV>(a)); \
    else update_tr_kernel<SV, false><<<grid, kThreads, 0, st>>>(a, make_cols<SV>(a));       \
    break
  switch (a.s) {
    CSG_TR(1); CSG_TR(2); CSG_TR(3); CSG_TR(4); CSG_TR(5); CSG_TR(6); CSG_TR(8);
    CSG_TR(10); CSG_TR(12); CSG_TR(16);
    default: return false;
  }
#undef CSG_TR
  CS_CUDA(cudaGetLastError());
  return true;
}

void launch_ref_xr_update(const UpdateArgs& a, cudaStream_t s) {
  update_dispatch<false, true, false>(a, s);
}

void launch_ref_block_update(const UpdateArgs& a, cudaStream_t s) {
  update_dispatch<true, false, false>(a, s);
}

void launch_block_update(int64_t n, int m, int k, const double* y, const double* x,
                         const double* c, double* out, cudaStream_t s) {
  if (n == 0) return;
  block_update_kernel<<<grid_for(n), kThreads, 0, s>>>(n, m, k, y, x, c, out);
  CS_CUDA(cudaGetLastError());
}

int pcg_vec_blocks(int64_t n) { return static_cast<int>(grid_for(n)); }

void launch_axpby_pcg(int which, int64_t n, double* x, double* r, double* p, const double* q,
                      const double* inv_diag, DevState* st, double* partial, unsigned* ticket,
                      double* result, int serial, cudaStream_t s) {
  if (n == 0) return;
  const unsigned grid = grid_for(n);
  const bool dots = !serial;
  switch (which) {
    case 0:
      pcg_vec_kernel<0, false><<<grid, kThreads, 0, s>>>(n, x, r, p, q, inv_diag, st, partial,
                                                         ticket, result);
      break;
    case 1:
      if (dots)
        pcg_vec_kernel<1, true><<<grid, kThreads, 0, s>>>(n, x, r, p, q, inv_diag, st, partial,
                                                          ticket, result);
      else
        pcg_vec_kernel<1, false><<<grid, kThreads, 0, s>>>(n, x, r, p, q, inv_diag, st, partial,
                                                           ticket, result);
      break;
    case 2:
      pcg_vec_kernel<2, false><<<grid, kThreads, 0, s>>>(n, x, r, p, q, inv_diag, st, partial,
                                                         ticket, result);
      break;
    case 3:
      pcg_vec_kernel<3, true><<<grid, kThreads, 0, s>>>(n, x, r, p, q, inv_diag, st, partial,
                                                        ticket, result);
      break;
    default: throw LibError{9, 0, "bad pcg step"};
  }
  CS_CUDA(cudaGetLastError());
}

void launch_scale2(int64_t n, double* v, double* g, const double* src_v, const double* src_g,
                   const double* denom, DevState* st, cudaStream_t s) {
  if (n == 0) return;
  scale2_kernel<<<grid_for(n), kThreads, 0, s>>>(n, v, g, src_v, src_g, denom, st);
  CS_CUDA(cudaGetLastError());
}

}  // namespace csg
