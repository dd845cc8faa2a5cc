// common.cuh -- shared device/host definitions of libchebstep_gpu (sm_100a).
//
// Data layout in HBM:
//  * Matrix: SELL-32 (compressed to SELL-32P / SELL-32PU, see SellView). Rows are grouped in slices of 32 consecutive rows; a
//    slice stores its nonzeros column-major by slot (slot k of lane l at
//    vals[slice_ptr[s] + k*32 + l]), padded to the slice's widest row with
//    val = 0, col = -1. Columns are int32 local indices (owned rows
//    0..n_local-1, then ghosts), values FP64: 12 B per nonzero. Within a row
//    the reference's stored column order is kept, so the per-row
//    accumulation order equals csr.cpp:116-121 and results are bitwise equal.
//  * Vectors: FP64, blocks column-major with leading dimension `ld`
//    (>= n_local + n_ghost, multiple of 32); ghost slots trail the owned rows
//    of every SpMV operand so the halo lands in place.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace csg {

constexpr int kSliceRows = 32;
constexpr int kMaxS = 64;  // kSmallDenseMax, block.hpp:35

// Error word: (code << 32) | payload, first writer wins (atomicCAS from 0).
struct DevState {
  int k;             // current outer iteration (1-based once the loop runs)
  int done;          // nonzero: every solve kernel returns immediately
  int converged;
  int outer_iters;
  unsigned long long err;      // final error
  unsigned long long pending;  // fast mode: basis breakdown seen in a speculative MPK
  int n_rel, n_da, n_db;
  int pad_;
  double bnorm;
  double rho;        // classical PCG
  double scal[8];    // small scalars (classical PCG step, beta ...)
};

// Pattern-compressed SELL-32 ("SELL-32P"): slice s owns value slots
// [slice_ptr[s], slice_ptr[s+1]) (32 lanes per slot). meta[s] >= 0: explicit
// int32 columns at cols[meta[s] + 32k + lane]. meta[s] < 0: the slice's rows share
// one sorted relative-offset pattern -- slot k of lane l is column row_l + off_k
// if bit l of mask_k is set (else an empty slot), with {off_k, mask_k} at
// pat[pat_index(meta) + k]. Either way a row's entries are visited in its stored
// (ascending) column order, so sums are bitwise the CSR row-serial sums.
// Uniform-value slices (pat_uniform(meta) = U > 0, "SELL-32PU"): every row of the
// slice that has an entry at offset off_k stores the same FP64 value (bitwise),
// so the slice keeps NO value slots: its U slots carry {off_k, mask_k} in pat and
// the value in pval[pat_index(meta) + k]. Slices with an identical (pattern,
// values) table share one table (global dedupe; the tables come first in
// pat/pval), so a constant-coefficient stencil streams no matrix bytes beyond
// meta: a 27-point operator has at most 27 distinct tables, staged once per
// block in shared memory. Lossless: every product v * x[c] uses the stored v,
// the result is bitwise unchanged.
constexpr int kPatShift = 40;
constexpr int64_t kPatIdxMask = (int64_t{1} << kPatShift) - 1;
constexpr int kUniformMaxSlots = 1 << 20;
__host__ __device__ inline int64_t pat_index(int64_t meta) { return (-meta - 1) & kPatIdxMask; }
__host__ __device__ inline int pat_uniform(int64_t meta) {
  return static_cast<int>((-meta - 1) >> kPatShift);
}
__host__ __device__ inline int64_t make_pat_meta(int64_t idx, int uniform_slots) {
  return -((static_cast<int64_t>(uniform_slots) << kPatShift) | idx) - 1;
}

// Uniform-table slot {offset, lane mask, value} (16 bytes; SELL-32PU tables).
struct __align__(16) SlotRec {
  int off;
  unsigned mask;
  double v;
};

// Constant-diagonal classes ("CDIA"): when every slice of a
// contiguous slice range [s0, s1) is uniform-value and the union of their
// tables has <= 32 relative offsets, each carrying ONE value, the range is a
// constant-coefficient stencil in relative-offset space (the DIA format with
// constant diagonals). Its table {off_j, v_j} (sorted by offset) travels as a
// kernel parameter -- every access is an immediate constant-bank operand -- and
// each row keeps only a 32-bit participation word (bit j: the row has an entry
// at off_j). Rows visit their entries in ascending offset = stored column order.
constexpr int kCdiaMax = 32;
struct CdiaTable {
  int n;
  int off[kCdiaMax];
  double v[kCdiaMax];
  double diag;  // every row of the class holds offset 0 with this value (else 0)
  double inv;   // launch-time: 1.0 / diag for the Jacobi epilogue (else 0)
};
struct CdiaClass {  // host side
  int64_t s0, s1;
  CdiaTable t;
  int64_t zstride;  // P if t is a 3 x 9 box stencil with groups P apart (P % 32 == 0), else 0
  // 3x3x3 box in natural ordering, off[9g+3i+j] = g*P + i*L + j - (P+L+1)
  // (P % 4 == 0, P >= 3L, L >= 3): plane-streaming kernel (sell_box_kernel)
  int64_t boxP = 0, boxL = 0;
  bool geo = false;  // box class with geometric participation (separable fast SpMV)
  // geo and the z face bits are plane-uniform (only the first plane may lack its
  // lower neighbour, only the last its upper one): zl0 / zuN are those two bits
  bool zuni = false, zl0 = false, zuN = false;
};

struct SellView {
  int64_t n_local;
  int64_t nslices;
  const int64_t* __restrict__ slice_ptr;
  const double* __restrict__ vals;
  const int32_t* __restrict__ cols;
  const int64_t* __restrict__ meta;
  const int2* __restrict__ pat;
  const double* __restrict__ pval;      // uniform-slice values (parallel to pat)
  const double* __restrict__ inv_diag;  // nullptr for identity
  int max_width;                        // widest slice (value slots)
  int uniform;                          // nonzero: some slices are uniform-value
  int uniform_all;                      // nonzero: every slice is uniform-value
  int64_t table_entries;                // uniform tables occupy pat/pval[0, table_entries)
  const uint32_t* pbits;                // CDIA participation words (device), or nullptr
  const CdiaClass* cdia;                // CDIA classes (HOST pointer; launchers only)
  int ncdia;
  int64_t xlen;                         // elements of every SpMV operand (owned + ghost, even)
};

__host__ __device__ inline unsigned long long make_err(int code, int payload) {
  return (static_cast<unsigned long long>(static_cast<unsigned>(code)) << 32) |
         static_cast<unsigned>(payload);
}

#define CS_CUDA(call)                                                      \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) throw ::csg::CudaError(e_, #call, __FILE__, __LINE__); \
  } while (0)

struct CudaError {
  cudaError_t err;
  std::string what;
  CudaError(cudaError_t e, const char* call, const char* file, int line)
      : err(e),
        what(std::string(cudaGetErrorString(e)) + " in " + call + " at " + file + ":" +
             std::to_string(line)) {}
};

// Library error carrying a CS_* code (thrown inside, mapped at the C-ABI).
struct LibError {
  int code;
  int payload;
  std::string msg;
};

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Launch setup of a kernel on the CURRENT device (thread-safe, cached per
// (device, kernel, threads, smem)): opts in to `smem` bytes of dynamic shared
// memory when above the 48 KB default (the attribute is per device) and
// returns the resident blocks per SM from the occupancy API (>= 1).
int kernel_setup(const void* func, int threads, int smem);

}  // namespace csg

#ifdef __CUDACC__
namespace csg {

// Deterministic finalisation of per-block partials, executed by ALL threads of
// the last block (ticket pattern). partial[b*ne + e] for b < count. Output e is
// summed in a fixed order that depends only on (count, blockDim): wide outputs
// use one thread per entry (serial over b), narrow outputs a strided per-thread
// chain followed by a fixed warp/block tree. Loads bypass L1 (ld.global.cg).
__device__ __forceinline__ void finalize_partials(const double* partial, unsigned count, int ne,
                                                  double* out) {
  if (ne >= 32) {
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
      double s = 0.0;
      for (unsigned b = 0; b < count; ++b) s += __ldcg(partial + static_cast<size_t>(b) * ne + e);
      out[e] = s;
    }
    return;
  }
  __shared__ double fin_red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int e = 0; e < ne; ++e) {
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < count; b += blockDim.x)
      s += __ldcg(partial + static_cast<size_t>(b) * ne + e);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) fin_red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += fin_red[w];
      out[e] = t;
    }
    __syncthreads();
  }
}

}  // namespace csg
#endif  // __CUDACC__
