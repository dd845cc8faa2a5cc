// sell.cu -- device-side matrix assembly into SELL-32 and the inverse
// conversions used by the bit-exactness checks.
//
//  * Stencil generators write the SELL arrays directly on the device, one
//    thread per row, with the reference's assembly conventions
//    (problems.cpp:13-53): x-fastest rows, neighbours visited in
//    (dz, dy, dx) lexicographic order so columns ascend, diagonal 26 / -1
//    for the 27-point operator; the 7-point operator follows the same
//    conventions. Values are exact small integers, so the device
//    assembly is bitwise the CPU assembly.
//  * A rank owning z-planes [z0, z1) numbers its rows 0..n_local-1 and the
//    ghost plane z0-1 (if any) n_local.., then plane z1 (if any); a row's
//    entries keep ascending GLOBAL column order, so per-row summation order
//    is partition-invariant.
//  * CSR -> SELL conversion for uploaded reference CsrMatrix data.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "kernels.cuh"

namespace csg {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int stencil_row_count(const StencilDesc& d, int64_t ix, int64_t iy,
                                                 int64_t iz) {
  if (d.kind == 0) {  // 27-point
    const int cx = 1 + (ix > 0) + (ix + 1 < d.nx);
    const int cy = 1 + (iy > 0) + (iy + 1 < d.ny);
    const int cz = 1 + (iz > 0) + (iz + 1 < d.nz);
    return cx * cy * cz;
  }
  return 1 + (ix > 0) + (ix + 1 < d.nx) + (iy > 0) + (iy + 1 < d.ny) + (iz > 0) +
         (iz + 1 < d.nz);
}

__global__ void stencil_widths_kernel(StencilDesc d, int64_t n_local, int64_t nslices,
                                      int64_t* widths) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t slice = row >> 5;
  if (slice >= nslices) return;
  int cnt = 0;
  if (row < n_local) {
    const int64_t plane = d.nx * d.ny;
    const int64_t iz = d.z0 + row / plane;
    const int64_t rem = row % plane;
    cnt = stencil_row_count(d, rem % d.nx, rem / d.nx, iz);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cnt = max(cnt, __shfl_xor_sync(0xffffffffu, cnt, off));
  if ((threadIdx.x & 31) == 0) widths[slice] = static_cast<int64_t>(cnt) * kSliceRows;
}

// Local index of global grid point (jx, jy, jz) for a rank owning [z0, z1).
__device__ __forceinline__ int32_t local_col(const StencilDesc& d, int64_t n_local, int64_t jx,
                                             int64_t jy, int64_t jz) {
  const int64_t plane = d.nx * d.ny;
  const int64_t in_plane = jy * d.nx + jx;
  if (jz >= d.z0 && jz < d.z1) return static_cast<int32_t>((jz - d.z0) * plane + in_plane);
  const int64_t lo_cnt = d.z0 > 0 ? plane : 0;
  if (jz < d.z0) return static_cast<int32_t>(n_local + in_plane);
  return static_cast<int32_t>(n_local + lo_cnt + in_plane);
}

__global__ void stencil_fill_kernel(StencilDesc d, int64_t n_local, int64_t nslices,
                                    const int64_t* __restrict__ slice_ptr, double* vals,
                                    int32_t* cols, double* diag_out) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t slice = row >> 5;
  if (slice >= nslices) return;
  const int lane = threadIdx.x & 31;
  const int64_t base = slice_ptr[slice];
  const int width = static_cast<int>((slice_ptr[slice + 1] - base) >> 5);
  double* vp = vals + base + lane;
  int32_t* cp = cols + base + lane;
  int k = 0;
  if (row < n_local) {
    const int64_t plane = d.nx * d.ny;
    const int64_t iz = d.z0 + row / plane;
    const int64_t rem = row % plane;
    const int64_t iy = rem / d.nx, ix = rem % d.nx;
    double dg = 0.0;
    if (d.kind == 0) {
      for (int dz = -1; dz <= 1; ++dz) {
        const int64_t jz = iz + dz;
        if (jz < 0 || jz >= d.nz) continue;
        for (int dy = -1; dy <= 1; ++dy) {
          const int64_t jy = iy + dy;
          if (jy < 0 || jy >= d.ny) continue;
          for (int dx = -1; dx <= 1; ++dx) {
            const int64_t jx = ix + dx;
            if (jx < 0 || jx >= d.nx) continue;
            const bool self = (dx == 0 && dy == 0 && dz == 0);
            cp[k * kSliceRows] = local_col(d, n_local, jx, jy, jz);
            vp[k * kSliceRows] = self ? 26.0 : -1.0;
            ++k;
          }
        }
      }
      dg = 26.0;
    } else {
      const double dv = 2.0 * (d.cx + d.cy + d.cz);
      auto put = [&](int64_t jx, int64_t jy, int64_t jz, double v) {
        cp[k * kSliceRows] = local_col(d, n_local, jx, jy, jz);
        vp[k * kSliceRows] = v;
        ++k;
      };
      if (iz > 0) put(ix, iy, iz - 1, -d.cz);
      if (iy > 0) put(ix, iy - 1, iz, -d.cy);
      if (ix > 0) put(ix - 1, iy, iz, -d.cx);
      put(ix, iy, iz, dv);
      if (ix + 1 < d.nx) put(ix + 1, iy, iz, -d.cx);
      if (iy + 1 < d.ny) put(ix, iy + 1, iz, -d.cy);
      if (iz + 1 < d.nz) put(ix, iy, iz + 1, -d.cz);
      dg = dv;
    }
    diag_out[row] = dg;
  }
  for (; k < width; ++k) {  // padding slots
    cp[k * kSliceRows] = -1;
    vp[k * kSliceRows] = 0.0;
  }
}

__global__ void csr_widths_kernel(int64_t n, const int64_t* __restrict__ rowptr, int64_t nslices,
                                  int64_t* widths, int* bad) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t slice = row >> 5;
  if (slice >= nslices) return;
  int64_t len = 0;
  if (row < n) {
    len = rowptr[row + 1] - rowptr[row];
    if (len < 0 || len > (1 << 24)) {
      atomicExch(bad, 1);
      len = 0;
    }
  }
  int cnt = static_cast<int>(len);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cnt = max(cnt, __shfl_xor_sync(0xffffffffu, cnt, off));
  if ((threadIdx.x & 31) == 0) widths[slice] = static_cast<int64_t>(cnt) * kSliceRows;
}

// Diagonal exactly as CsrMatrix::diagonal (csr.cpp:10-15): std::lower_bound
// over the row's stored columns (libstdc++ halving order), 0 when absent.
__device__ double csr_lower_bound_diag(const int64_t* col, const double* val, int64_t first,
                                       int64_t last, int64_t i) {
  int64_t len = last - first;
  while (len > 0) {
    const int64_t half = len >> 1;
    const int64_t mid = first + half;
    if (col[mid] < i) {
      first = mid + 1;
      len = len - half - 1;
    } else {
      len = half;
    }
  }
  if (first == last || col[first] != i) return 0.0;
  return val[first];
}

// Row block [row_begin, row_begin + n) of an n_global CSR with GLOBAL columns:
// owned columns map to c - row_begin, off-block columns to n + (index in the
// sorted ghost list) (partition.cpp numbering); stored order is kept.
__device__ __forceinline__ int32_t local_col(int64_t c, int64_t row_begin, int64_t n,
                                             const int64_t* __restrict__ ghosts, int64_t n_ghost) {
  if (c >= row_begin && c < row_begin + n) return static_cast<int32_t>(c - row_begin);
  int64_t lo = 0, hi = n_ghost;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ghosts[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return static_cast<int32_t>(n + lo);
}

// Rows [r0, r1) (r0 a multiple of 32) whose column/value entries sit in
// col/val at offset rowptr[row] - nnz_base (one streamed chunk of the upload).
__global__ void csr_fill_kernel(int64_t n, int64_t row_begin, int64_t n_global,
                                const int64_t* __restrict__ ghosts, int64_t n_ghost,
                                const int64_t* __restrict__ rowptr,
                                const int64_t* __restrict__ col_c, const double* __restrict__ val_c,
                                int64_t nnz_base, int64_t r0, int64_t slice_end,
                                const int64_t* __restrict__ slice_ptr,
                                double* vals, int32_t* cols, double* diag_out, int* bad) {
  const int64_t row = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t slice = row >> 5;
  if (slice >= slice_end) return;
  const int64_t* col = col_c - nnz_base;  // indexed by the global entry position
  const double* val = val_c - nnz_base;
  const int lane = threadIdx.x & 31;
  const int64_t base = slice_ptr[slice];
  const int width = static_cast<int>((slice_ptr[slice + 1] - base) >> 5);
  double* vp = vals + base + lane;
  int32_t* cp = cols + base + lane;
  int k = 0;
  if (row < n) {
    const int64_t b = rowptr[row], e = rowptr[row + 1];
    for (int64_t t = b; t < e; ++t, ++k) {
      const int64_t c = col[t];
      if (c < 0 || c >= n_global) {
        atomicExch(bad, 2);
        cp[k * kSliceRows] = -1;
        vp[k * kSliceRows] = 0.0;
        continue;
      }
      cp[k * kSliceRows] = local_col(c, row_begin, n, ghosts, n_ghost);
      vp[k * kSliceRows] = val[t];
    }
    diag_out[row] = csr_lower_bound_diag(col, val, b, e, row_begin + row);
  }
  for (; k < width; ++k) {
    cp[k * kSliceRows] = -1;
    vp[k * kSliceRows] = 0.0;
  }
}

// flag[s] = 1 when slice s (explicit SELL-32) references a ghost column
__global__ void slice_ghost_flag_kernel(int64_t n_local, int64_t nslices,
                                        const int64_t* __restrict__ slice_ptr,
                                        const int32_t* __restrict__ cols, unsigned char* flag) {
  const int64_t slice = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (slice >= nslices) return;
  const int lane = threadIdx.x & 31;
  bool g = false;
  for (int64_t t = slice_ptr[slice] + lane; t < slice_ptr[slice + 1]; t += kSliceRows)
    g |= cols[t] >= n_local;
  g = __any_sync(0xffffffffu, g);
  if (lane == 0) flag[slice] = g ? 1 : 0;
}

// halo send buffer: buf[k] = x[idx[k]]
__global__ void halo_gather_kernel(int64_t count, const int32_t* __restrict__ idx,
                                   const double* __restrict__ x, double* __restrict__ buf) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    buf[k] = x[idx[k]];
}

// slots of slice `slice` (value slots, or the pattern length of a uniform slice)
__device__ __forceinline__ int slot_count(const SellView& a, int64_t slice) {
  const int64_t m = a.meta[slice];
  if (m < 0 && pat_uniform(m) > 0) return pat_uniform(m);
  return static_cast<int>((a.slice_ptr[slice + 1] - a.slice_ptr[slice]) >> 5);
}

// column of slot k of `lane` in slice `slice`, or -1 for an empty slot
__device__ __forceinline__ int32_t slot_col(const SellView& a, int64_t slice, int k, int lane,
                                            int64_t row) {
  const int64_t m = a.meta[slice];
  if (m >= 0) return a.cols[m + k * kSliceRows + lane];
  const int2 e = a.pat[pat_index(m) + k];
  return ((e.y >> lane) & 1) ? static_cast<int32_t>(row + e.x) : -1;
}

__device__ __forceinline__ double slot_val(const SellView& a, int64_t slice, int k, int lane) {
  const int64_t m = a.meta[slice];
  if (m < 0 && pat_uniform(m) > 0) return a.pval[pat_index(m) + k];
  return a.vals[a.slice_ptr[slice] + k * kSliceRows + lane];
}

__global__ void sell_row_len_kernel(SellView a, int64_t* len) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= a.n_local) return;
  const int64_t slice = row >> 5;
  const int lane = threadIdx.x & 31;
  const int width = slot_count(a, slice);
  int cnt = 0;
  for (int k = 0; k < width; ++k)
    if (slot_col(a, slice, k, lane, row) >= 0) ++cnt;
  len[row] = cnt;
}

// rows [r0, r1) (r0 % 32 == 0); entries land at col/val[rowptr[row] - base]
__global__ void sell_to_csr_kernel(SellView a, int64_t row_begin,
                                   const int64_t* __restrict__ ghost_global,
                                   const int64_t* __restrict__ rowptr, int64_t* col,
                                   double* val, int64_t r0, int64_t r1, int64_t base) {
  const int64_t row = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= r1 || row >= a.n_local) return;
  const int64_t slice = row >> 5;
  const int lane = threadIdx.x & 31;
  const int width = slot_count(a, slice);
  int64_t o = rowptr[row] - base;
  for (int k = 0; k < width; ++k) {
    const int32_t c = slot_col(a, slice, k, lane, row);
    if (c < 0) continue;
    col[o] = c < a.n_local ? row_begin + c : ghost_global[c - a.n_local];
    val[o] = slot_val(a, slice, k, lane);
    ++o;
  }
}

// ---------------------------------------------------------------- SELL-32 -> SELL-32P(U)
// A slice is pattern-compressed when every row's columns are strictly ascending
// and the union U of the rows' relative offsets (col - row) is small enough that
// 32U value slots + U pattern entries cost less than 32W values + 32W columns.
// It is uniform-value (no value slots at all) when, in addition, every union
// entry carries one bitwise-identical value across the rows that hold it.
// Uniform slices are deduplicated globally: a 64-bit hash of each slice's
// (offset, mask, value) table is sorted, equal hashes share one table (the
// first slice of the group writes it), and a verify pass compares every
// slice's own table against the shared one exactly (a collision disables the
// dedupe and the conversion is redone). The union is built by a warp-wide
// merge of the 32 sorted offset lists.
constexpr int kSentinel = 0x7fffffff;
constexpr unsigned long long kNoTable = ~0ull;
enum SliceKind : int64_t { kExplicit = 0, kValuePattern = 1, kUniform = 2 };

// Merge cursor over one slice's 32 rows (one lane per row). Rows keep their
// entries in ascending GLOBAL column order (the reference's stored order), so
// the union is merged on the global relative offset (global col - global row);
// the table stores the LOCAL relative offset (local col - local row) that the
// SpMV adds to its row index. On a rank whose lower ghost plane lives after its
// owned rows, the first plane's rows are not ascending in local columns, but
// they still are in global ones, and their local offsets stay constant.
struct PatWalk {
  const int32_t* cols;
  const double* vals;
  ColMap m;
  int64_t base, row, grow;
  int len, idx, width;
  bool sorted;
  __device__ int64_t key(int32_t c) const {
    return (c < m.n_local ? m.row_begin + c : m.ghost[c - m.n_local]) - grow;
  }
  __device__ void init(const int64_t* slice_ptr, const int32_t* c, const double* v, ColMap cm,
                       int64_t slice, int lane) {
    cols = c, vals = v, m = cm;
    row = slice * kSliceRows + lane;
    grow = m.row_begin + row;
    base = slice_ptr[slice] + lane;
    width = static_cast<int>((slice_ptr[slice + 1] - slice_ptr[slice]) >> 5);
    len = 0, idx = 0;
    sorted = true;
    int64_t prev = INT64_MIN;
    for (int k = 0; k < width; ++k) {
      const int32_t col = cols[base + k * kSliceRows];
      if (col < 0) break;  // trailing padding
      const int64_t kk = key(col);
      if (kk <= prev) sorted = false;
      prev = kk;
      ++len;
    }
  }
  // next union entry: global key, local offset, lane mask, the value of the
  // lowest holding lane, whether every holding lane stores that value bitwise
  // (uni) and sits at the same local offset (same); false at the end
  __device__ bool next(int64_t& gk, int& off, unsigned& mask, unsigned long long& vbits,
                       bool& uni, bool& same) {
    const int32_t col = idx < len ? cols[base + idx * kSliceRows] : -1;
    const int64_t cur = idx < len ? key(col) : INT64_MAX;
    int64_t mn = cur;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t t = __shfl_xor_sync(0xffffffffu, mn, o);
      mn = t < mn ? t : mn;
    }
    if (mn == INT64_MAX) return false;
    gk = mn;
    const bool hit = cur == mn;
    mask = __ballot_sync(0xffffffffu, hit);
    const int lead = __ffs(mask) - 1;
    const int mine_off = hit ? static_cast<int>(col - row) : 0;
    off = __shfl_sync(0xffffffffu, mine_off, lead);
    same = __all_sync(0xffffffffu, !hit || mine_off == off);
    const unsigned long long mine =
        hit ? static_cast<unsigned long long>(__double_as_longlong(vals[base + idx * kSliceRows]))
            : 0ull;
    vbits = __shfl_sync(0xffffffffu, mine, lead);
    uni = __all_sync(0xffffffffu, !hit || mine == vbits);
    if (hit) ++idx;
    return true;
  }
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long h, unsigned long long v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h ^= h >> 31;
  h *= 0xbf58476d1ce4e5b9ull;
  return h ^ (h >> 29);
}

__global__ void compress_plan_kernel(int64_t nslices, const int64_t* __restrict__ slice_ptr,
                                     const int32_t* __restrict__ cols,
                                     const double* __restrict__ vals, ColMap cm, int64_t* val_cnt,
                                     int64_t* pat_cnt, int64_t* col_cnt, int64_t* kind,
                                     unsigned long long* hash, int allow, int allow_uniform,
                                     int dedupe) {
  const int lane = threadIdx.x & 31;
  const int64_t slice = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (slice >= nslices) return;
  PatWalk w;
  w.init(slice_ptr, cols, vals, cm, slice, lane);
  const int W = w.width;
  bool ok = __all_sync(0xffffffffu, w.sorted) && W > 0 && allow;
  bool uni = ok && allow_uniform;
  int U = 0;
  unsigned long long h = 0x243f6a8885a308d3ull;
  if (ok) {
    int64_t gk;
    int off;
    unsigned mask;
    unsigned long long vb;
    bool u, same;
    while (w.next(gk, off, mask, vb, u, same)) {
      ++U;
      if (!same) {  // one slot must be one local offset for every row holding it
        ok = uni = false;
        break;
      }
      // a uniform table is walked entry by entry (one masked gather per entry),
      // so it only pays while it is not much longer than the slice's slot count:
      // a reordered operator whose 32 rows share few offsets has U >> W (a
      // shuffled 27-point slice: U ~ 800, W = 27) and stays explicit SELL-32
      uni = uni && u && U <= kUniformMaxSlots && 2 * U <= 3 * W;
      if (uni)
        h = mix64(mix64(mix64(mix64(h, static_cast<unsigned>(off)), mask), vb),
                  static_cast<unsigned long long>(gk));
      if (!uni && 264 * U > 384 * W) {
        ok = false;
        break;
      }
    }
  }
  if (lane == 0) {
    const int64_t k = !ok ? kExplicit : !uni ? kValuePattern : kUniform;
    kind[slice] = k | (static_cast<int64_t>(U) << 8);
    val_cnt[slice] = k == kExplicit ? int64_t{kSliceRows} * W
                     : k == kValuePattern ? int64_t{kSliceRows} * U
                                          : 0;
    pat_cnt[slice] = k == kValuePattern ? U : 0;
    col_cnt[slice] = k == kExplicit ? int64_t{kSliceRows} * W : 0;
    // uniform: table hash (top bit clear); dedupe off: the slice index (unique)
    h = mix64(h, static_cast<unsigned long long>(U)) >> 1;
    hash[slice] = k != kUniform ? kNoTable
                  : dedupe      ? h
                                : static_cast<unsigned long long>(slice);
  }
}

// sorted position i: entries of a new table group (first of equal hashes)
__global__ void table_heads_kernel(int64_t n, const unsigned long long* __restrict__ key,
                                   const int32_t* __restrict__ slc,
                                   const int64_t* __restrict__ kind, int64_t* tab_cnt,
                                   int64_t* headpos) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool head = key[i] != kNoTable && (i == 0 || key[i] != key[i - 1]);
  tab_cnt[i] = head ? (kind[slc[i]] >> 8) : 0;
  headpos[i] = head ? i : -1;
}

// per slice: table offset and the representative (first) slice of its group
__global__ void table_assign_kernel(int64_t n, const unsigned long long* __restrict__ key,
                                    const int32_t* __restrict__ slc,
                                    const int64_t* __restrict__ headpos,
                                    const int64_t* __restrict__ tab_ptr, int64_t* slice_tab,
                                    int32_t* slice_rep) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t s = slc[i];
  if (key[i] == kNoTable) {
    slice_tab[s] = -1;
    slice_rep[s] = -1;
    return;
  }
  const int64_t hp = headpos[i];
  slice_tab[s] = tab_ptr[hp];
  slice_rep[s] = slc[hp];
}

__global__ void compress_fill_kernel(int64_t nslices, const int64_t* __restrict__ slice_ptr,
                                     const int32_t* __restrict__ cols,
                                     const double* __restrict__ vals, ColMap cm,
                                     const int64_t* __restrict__ kind,
                                     const int64_t* __restrict__ slice_tab,
                                     const int32_t* __restrict__ slice_rep,
                                     const int64_t* __restrict__ new_ptr,
                                     const int64_t* __restrict__ pat_ptr, int64_t pat_base,
                                     const int64_t* __restrict__ col_ptr, double* nvals,
                                     int32_t* ncols, int2* pat, double* pval, int64_t* pkey,
                                     int64_t* meta) {
  const int lane = threadIdx.x & 31;
  const int64_t slice = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (slice >= nslices) return;
  const int64_t k = kind[slice] & 0xff;
  const int U = static_cast<int>(kind[slice] >> 8);
  const int64_t base = slice_ptr[slice] + lane;
  const int W = static_cast<int>((slice_ptr[slice + 1] - slice_ptr[slice]) >> 5);
  if (k == kExplicit) {
    const int64_t nb = new_ptr[slice] + lane;
    const int64_t cb = col_ptr[slice] + lane;
    for (int q = 0; q < W; ++q) {
      nvals[nb + q * kSliceRows] = vals[base + q * kSliceRows];
      ncols[cb + q * kSliceRows] = cols[base + q * kSliceRows];
    }
    if (lane == 0) meta[slice] = col_ptr[slice];
    return;
  }
  if (k == kUniform && slice_rep[slice] != slice) {  // shares its group's table
    if (lane == 0) meta[slice] = make_pat_meta(slice_tab[slice], U);
    return;
  }
  PatWalk w;
  w.init(slice_ptr, cols, vals, cm, slice, lane);
  const int64_t pb = k == kUniform ? slice_tab[slice] : pat_base + pat_ptr[slice];
  const int64_t nb = new_ptr[slice] + lane;
  int64_t gk;
  int off;
  unsigned mask;
  unsigned long long vb;
  bool u, same;
  for (int q = 0; q < U && w.next(gk, off, mask, vb, u, same); ++q) {
    if (lane == 0) {
      pat[pb + q] = make_int2(off, static_cast<int>(mask));
      pval[pb + q] = k == kUniform ? __longlong_as_double(static_cast<long long>(vb)) : 0.0;
      pkey[pb + q] = gk;
    }
    if (k == kValuePattern) {
      // w.idx was advanced past this entry on the holding lanes
      const bool hit = (mask >> lane) & 1u;
      nvals[nb + q * kSliceRows] = hit ? vals[base + (w.idx - 1) * kSliceRows] : 0.0;
    }
  }
  if (lane == 0) meta[slice] = make_pat_meta(pb, k == kUniform ? U : 0);
}

// every uniform slice against the table it points at, exactly
__global__ void compress_verify_kernel(int64_t nslices, const int64_t* __restrict__ slice_ptr,
                                       const int32_t* __restrict__ cols,
                                       const double* __restrict__ vals, ColMap cm,
                                       const int64_t* __restrict__ kind,
                                       const int64_t* __restrict__ slice_tab,
                                       const int2* __restrict__ pat,
                                       const double* __restrict__ pval,
                                       const int64_t* __restrict__ pkey, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t slice = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (slice >= nslices || (kind[slice] & 0xff) != kUniform) return;
  const int U = static_cast<int>(kind[slice] >> 8);
  const int64_t pb = slice_tab[slice];
  PatWalk w;
  w.init(slice_ptr, cols, vals, cm, slice, lane);
  int64_t gk;
  int off;
  unsigned mask;
  unsigned long long vb;
  bool u, same;
  bool eq = true;
  int q = 0;
  for (; q < U && w.next(gk, off, mask, vb, u, same); ++q) {
    const int2 e = pat[pb + q];
    eq = eq && e.x == off && static_cast<unsigned>(e.y) == mask && pkey[pb + q] == gk &&
         static_cast<unsigned long long>(__double_as_longlong(pval[pb + q])) == vb;
  }
  if (lane == 0 && (!eq || q != U)) atomicExch(bad, 1);
}

__global__ void inv_diag_kernel(int64_t n, const double* __restrict__ diag, double* inv, int* bad) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = diag[i];
  if (!(d > 0.0)) atomicExch(bad, 1);
  inv[i] = 1.0 / d;  // precond.cpp:22, IEEE division
}

inline unsigned grid_for(int64_t threads) {
  return static_cast<unsigned>((threads + kThreads - 1) / kThreads);
}

}  // namespace

void launch_stencil_widths(const StencilDesc& d, int64_t n_local, int64_t nslices, int64_t* widths,
                           cudaStream_t st) {
  stencil_widths_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(d, n_local, nslices, widths);
  CS_CUDA(cudaGetLastError());
}

void launch_stencil_fill(const StencilDesc& d, int64_t n_local, int64_t nslices,
                         const int64_t* slice_ptr, double* vals, int32_t* cols, double* diag,
                         cudaStream_t st) {
  stencil_fill_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(d, n_local, nslices, slice_ptr,
                                                                   vals, cols, diag);
  CS_CUDA(cudaGetLastError());
}

void scan_slice_ptr(const int64_t* widths, int64_t nslices, int64_t* slice_ptr, void* tmp,
                    size_t* tmp_bytes, cudaStream_t st) {
  // slice_ptr[0] = 0, slice_ptr[i+1] = sum_{j<=i} widths[j]: inclusive scan into +1
  if (tmp == nullptr) {
    CS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, *tmp_bytes, widths, slice_ptr + 1, nslices, st));
    return;
  }
  CS_CUDA(cudaMemsetAsync(slice_ptr, 0, sizeof(int64_t), st));
  CS_CUDA(cub::DeviceScan::InclusiveSum(tmp, *tmp_bytes, widths, slice_ptr + 1, nslices, st));
}

void scan_rowptr(const int64_t* len, int64_t n, int64_t* rowptr, void* tmp, size_t* tmp_bytes,
                 cudaStream_t st) {
  scan_slice_ptr(len, n, rowptr, tmp, tmp_bytes, st);
}

void launch_csr_widths(int64_t n, const int64_t* rowptr, int64_t nslices, int64_t* widths,
                       int* bad, cudaStream_t st) {
  csr_widths_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(n, rowptr, nslices, widths, bad);
  CS_CUDA(cudaGetLastError());
}

void launch_csr_fill(int64_t n, int64_t row_begin, int64_t n_global, const int64_t* ghosts,
                     int64_t n_ghost, const int64_t* rowptr, const int64_t* col, const double* val,
                     int64_t nnz_base, int64_t r0, int64_t r1, const int64_t* slice_ptr,
                     double* vals, int32_t* cols, double* diag, int* bad, cudaStream_t st) {
  const int64_t s0 = r0 / kSliceRows, s1 = (r1 + kSliceRows - 1) / kSliceRows;
  if (s1 <= s0) return;
  csr_fill_kernel<<<grid_for((s1 - s0) * 32), kThreads, 0, st>>>(
      n, row_begin, n_global, ghosts, n_ghost, rowptr, col, val, nnz_base, r0, s1, slice_ptr, vals,
      cols, diag, bad);
  CS_CUDA(cudaGetLastError());
}

void launch_slice_ghost_flag(int64_t n_local, int64_t nslices, const int64_t* slice_ptr,
                             const int32_t* cols, unsigned char* flag, cudaStream_t st) {
  if (nslices == 0) return;
  slice_ghost_flag_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(n_local, nslices,
                                                                       slice_ptr, cols, flag);
  CS_CUDA(cudaGetLastError());
}

void launch_halo_gather(int64_t count, const int32_t* idx, const double* x, double* buf,
                        cudaStream_t st) {
  if (count == 0) return;
  const int64_t blocks = std::min<int64_t>((count + kThreads - 1) / kThreads, 148 * 8);
  halo_gather_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, st>>>(count, idx, x, buf);
  CS_CUDA(cudaGetLastError());
}

void launch_sell_row_len(const SellView& a, int64_t* len, cudaStream_t st) {
  sell_row_len_kernel<<<grid_for(a.n_local), kThreads, 0, st>>>(a, len);
  CS_CUDA(cudaGetLastError());
}

void launch_sell_to_csr(const SellView& a, int64_t row_begin, const int64_t* ghost_global,
                        const int64_t* rowptr, int64_t* col, double* val, int64_t r0, int64_t r1,
                        int64_t base, cudaStream_t st) {
  if (r1 <= r0) return;
  sell_to_csr_kernel<<<grid_for(r1 - r0), kThreads, 0, st>>>(a, row_begin, ghost_global, rowptr,
                                                            col, val, r0, r1, base);
  CS_CUDA(cudaGetLastError());
}

void launch_compress_plan(int64_t nslices, const int64_t* slice_ptr, const int32_t* cols,
                          const double* vals, ColMap cm, int64_t* val_cnt, int64_t* pat_cnt,
                          int64_t* col_cnt, int64_t* kind, unsigned long long* hash, int dedupe,
                          cudaStream_t st) {
  if (nslices == 0) return;
  // CS_SELL_EXPLICIT=1 keeps every slice explicit; CS_SELL_VALUES=1 keeps the value
  // slots (no uniform-value slices) -- format A/B experiments, read per conversion
  const int allow = std::getenv("CS_SELL_EXPLICIT") ? 0 : 1;
  const int allow_uniform = std::getenv("CS_SELL_VALUES") ? 0 : 1;
  compress_plan_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(
      nslices, slice_ptr, cols, vals, cm, val_cnt, pat_cnt, col_cnt, kind, hash, allow,
      allow_uniform, dedupe);
  CS_CUDA(cudaGetLastError());
}

void scan_max_i64(const int64_t* in, int64_t n, int64_t* out, void* tmp, size_t* tmp_bytes,
                  cudaStream_t st) {
  CS_CUDA(cub::DeviceScan::InclusiveScan(tmp, *tmp_bytes, in, out, ::cuda::maximum<>{}, n, st));
}

void sort_tables(const unsigned long long* key_in, unsigned long long* key_out,
                 const int32_t* val_in, int32_t* val_out, int64_t n, void* tmp, size_t* tmp_bytes,
                 cudaStream_t st) {
  CS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, *tmp_bytes, key_in, key_out, val_in, val_out,
                                          static_cast<int>(n), 0, 64, st));
}

void launch_table_heads(int64_t n, const unsigned long long* key, const int32_t* slc,
                        const int64_t* kind, int64_t* tab_cnt, int64_t* headpos, cudaStream_t st) {
  if (n == 0) return;
  table_heads_kernel<<<grid_for(n), kThreads, 0, st>>>(n, key, slc, kind, tab_cnt, headpos);
  CS_CUDA(cudaGetLastError());
}

void launch_table_assign(int64_t n, const unsigned long long* key, const int32_t* slc,
                         const int64_t* headpos, const int64_t* tab_ptr, int64_t* slice_tab,
                         int32_t* slice_rep, cudaStream_t st) {
  if (n == 0) return;
  table_assign_kernel<<<grid_for(n), kThreads, 0, st>>>(n, key, slc, headpos, tab_ptr, slice_tab,
                                                        slice_rep);
  CS_CUDA(cudaGetLastError());
}

void launch_iota_i32(int64_t n, int32_t* out, cudaStream_t st);

void launch_compress_fill(int64_t nslices, const int64_t* slice_ptr, const int32_t* cols,
                          const double* vals, ColMap cm, const int64_t* kind,
                          const int64_t* slice_tab, const int32_t* slice_rep,
                          const int64_t* new_ptr, const int64_t* pat_ptr, int64_t pat_base,
                          const int64_t* col_ptr, double* nvals, int32_t* ncols, int2* pat,
                          double* pval, int64_t* pkey, int64_t* meta, cudaStream_t st) {
  if (nslices == 0) return;
  compress_fill_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(
      nslices, slice_ptr, cols, vals, cm, kind, slice_tab, slice_rep, new_ptr, pat_ptr, pat_base,
      col_ptr, nvals, ncols, pat, pval, pkey, meta);
  CS_CUDA(cudaGetLastError());
}

void launch_compress_verify(int64_t nslices, const int64_t* slice_ptr, const int32_t* cols,
                            const double* vals, ColMap cm, const int64_t* kind,
                            const int64_t* slice_tab, const int2* pat, const double* pval,
                            const int64_t* pkey, int* bad, cudaStream_t st) {
  if (nslices == 0) return;
  compress_verify_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(
      nslices, slice_ptr, cols, vals, cm, kind, slice_tab, pat, pval, pkey, bad);
  CS_CUDA(cudaGetLastError());
}

// CDIA participation words: per slice (one warp), its class by binary search
// over the class starts, then every table entry located in the class table by
// its global key (the class table is in key = stored order); lane l collects
// bit j for each entry it holds.
__global__ void cdia_bits_kernel(int64_t nslices, int64_t n_local, int ncls,
                                 const int64_t* __restrict__ starts,
                                 const int64_t* __restrict__ ckeys, const int32_t* __restrict__ nofs,
                                 const int64_t* __restrict__ meta, const int64_t* __restrict__ pkey,
                                 const int2* __restrict__ pat, uint32_t* bits, int* bad,
                                 int* nodiag) {
  const int lane = threadIdx.x & 31;
  const int64_t slice = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (slice >= nslices) return;
  int lo = 0, hi = ncls - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (starts[mid] <= slice) lo = mid;
    else hi = mid - 1;
  }
  const int64_t* ck = ckeys + lo * kCdiaMax;
  const int cn = nofs[lo];
  const int64_t m = meta[slice];
  const int64_t pi = pat_index(m);
  const int U = pat_uniform(m);
  uint32_t w = 0;
  bool ok = true;
  for (int k = 0; k < U; ++k) {
    const int64_t key = pkey[pi + k];
    int j = 0;
    while (j < cn && ck[j] != key) ++j;
    if (j == cn) {
      ok = false;
      break;
    }
    if ((static_cast<unsigned>(pat[pi + k].y) >> lane) & 1u) w |= 1u << j;
  }
  if (!ok && lane == 0) atomicExch(bad, 1);
  // class-uniform diagonal: every owned row must hold key 0
  int j0 = 0;
  while (j0 < cn && ck[j0] != 0) ++j0;
  const int64_t row = slice * kSliceRows + lane;
  if (row < n_local && (j0 == cn || !((w >> j0) & 1u))) atomicOr(nodiag + lo, 1);
  bits[row] = w;
}

// Is a 3x3x3 box class "geometric" (the separable plane-sum SpMV applies)?
// Every row's 27-bit participation word must be the outer product of its own
// x / y / z face bits (bit 9g+3i+j = z[g] & y[i] & x[j], with x = {b12, 1, b14},
// y = {b10, 1, b16}, z = {b4, 1, b22}), and its x / y face bits must equal those
// of the row one plane below when that row is in the class too.
__global__ void cdia_geo_kernel(const uint32_t* __restrict__ bits, int64_t r0, int64_t r1,
                                int64_t P, int* bad) {
  const int64_t r = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  const uint32_t w = bits[r];
  const uint32_t fx[3] = {(w >> 12) & 1u, 1u, (w >> 14) & 1u};
  const uint32_t fy[3] = {(w >> 10) & 1u, 1u, (w >> 16) & 1u};
  const uint32_t fz[3] = {(w >> 4) & 1u, 1u, (w >> 22) & 1u};
  uint32_t e = 0;
  for (int g = 0; g < 3; ++g)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) e |= (fz[g] & fy[i] & fx[j]) << (9 * g + 3 * i + j);
  bool ok = e == (w & 0x7FFFFFFu);
  constexpr uint32_t kXY = (1u << 10) | (1u << 12) | (1u << 14) | (1u << 16);
  if (r - P >= r0) ok = ok && ((bits[r - P] ^ w) & kXY) == 0u;
  if (!ok) atomicOr(bad, 1);
  // bit 1: the z face bits are not plane-uniform -- every plane but the first has
  // its lower neighbour plane (bit 4), every plane but the last its upper one
  // (bit 22), and the first / last plane share one value each. Without it the
  // separable kernel takes the z bits from plane flags and the x / y bits from
  // one plane per column: no participation-word stream.
  const int64_t m = (r - r0) / P, last = (r1 - r0 - 1) / P;
  bool zok = m == 0 ? (((w ^ bits[r0]) >> 4) & 1u) == 0u : ((w >> 4) & 1u) != 0u;
  if (m == last) zok = zok && (((w ^ bits[r0 + last * P]) >> 22) & 1u) == 0u;
  else zok = zok && ((w >> 22) & 1u) != 0u;
  if (!zok) atomicOr(bad, 2);
}

void launch_cdia_geo_check(const uint32_t* bits, int64_t r0, int64_t r1, int64_t P, int* bad,
                           cudaStream_t st) {
  if (r1 <= r0) return;
  cdia_geo_kernel<<<grid_for(r1 - r0), kThreads, 0, st>>>(bits, r0, r1, P, bad);
  CS_CUDA(cudaGetLastError());
}

void launch_cdia_bits(int64_t nslices, int64_t n_local, int ncls, const int64_t* starts,
                      const int64_t* ckeys, const int32_t* nofs, const int64_t* meta,
                      const int64_t* pkey, const int2* pat, uint32_t* bits, int* bad,
                      int* nodiag, cudaStream_t st) {
  if (nslices == 0) return;
  cdia_bits_kernel<<<grid_for(nslices * 32), kThreads, 0, st>>>(
      nslices, n_local, ncls, starts, ckeys, nofs, meta, pkey, pat, bits, bad, nodiag);
  CS_CUDA(cudaGetLastError());
}

__global__ void iota_i32_kernel(int64_t n, int32_t* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<int32_t>(i);
}

void launch_iota_i32(int64_t n, int32_t* out, cudaStream_t st) {
  if (n == 0) return;
  iota_i32_kernel<<<grid_for(n), kThreads, 0, st>>>(n, out);
  CS_CUDA(cudaGetLastError());
}

void launch_inv_diag(int64_t n, const double* diag, double* inv_diag, int* bad, cudaStream_t st) {
  if (n == 0) return;
  inv_diag_kernel<<<grid_for(n), kThreads, 0, st>>>(n, diag, inv_diag, bad);
  CS_CUDA(cudaGetLastError());
}

}  // namespace csg
