// partition.cpp -- host-side row partitioning and halo maps (no GPU needed).
//
// The reference is a single address space; these are the
// new components the multi-GPU path needs: a contiguous,
// plane-aligned row-block split and, for general CSR blocks, the ghost list
// (sorted unique off-block columns) with columns remapped to the local
// numbering owned 0..n_loc-1, ghosts n_loc.. in ascending global order. The
// order of nonzeros inside each row is untouched, which keeps the per-row
// accumulation order -- and so the SpMV result -- partition-invariant.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "chebstep_gpu.h"

extern "C" int cs_partition_rows(int64_t n_rows, int64_t plane, int nranks, int rank,
                                 int64_t* begin, int64_t* end) {
  if (nranks < 1 || rank < 0 || rank >= nranks || plane < 1 || n_rows < 0 ||
      n_rows % plane != 0)
    return CS_ERR_INVALID_ARGUMENT;
  const int64_t planes = n_rows / plane;
  if (planes < nranks) return CS_ERR_INVALID_ARGUMENT;  // every rank owns >= 1 plane
  const int64_t base = planes / nranks, extra = planes % nranks;
  const int64_t p0 = rank * base + std::min<int64_t>(rank, extra);
  const int64_t p1 = p0 + base + (rank < extra ? 1 : 0);
  *begin = p0 * plane;
  *end = p1 * plane;
  return CS_OK;
}

extern "C" int cs_halo_map_csr(int64_t row_begin, int64_t row_end, const int64_t* rowptr_local,
                               const int64_t* col_global, int64_t* n_ghost, int64_t* ghost_cols,
                               int64_t ghost_cap, int32_t* col_local) {
  if (row_end < row_begin) return CS_ERR_INVALID_ARGUMENT;
  const int64_t n_loc = row_end - row_begin;
  const int64_t nnz = rowptr_local[n_loc] - rowptr_local[0];
  std::vector<int64_t> ghosts;
  for (int64_t k = 0; k < nnz; ++k) {
    const int64_t c = col_global[k];
    if (c < row_begin || c >= row_end) ghosts.push_back(c);
  }
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  *n_ghost = static_cast<int64_t>(ghosts.size());
  if (ghost_cols == nullptr) return CS_OK;
  if (ghost_cap < *n_ghost) return CS_ERR_DIMENSION;
  std::copy(ghosts.begin(), ghosts.end(), ghost_cols);
  if (n_loc + *n_ghost > INT32_MAX) return CS_ERR_DIMENSION;
  if (col_local != nullptr)
    for (int64_t k = 0; k < nnz; ++k) {
      const int64_t c = col_global[k];
      if (c >= row_begin && c < row_end) {
        col_local[k] = static_cast<int32_t>(c - row_begin);
      } else {
        const auto it = std::lower_bound(ghosts.begin(), ghosts.end(), c);
        col_local[k] = static_cast<int32_t>(n_loc + (it - ghosts.begin()));
      }
    }
  return CS_OK;
}
