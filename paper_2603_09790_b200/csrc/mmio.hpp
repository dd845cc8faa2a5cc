// mmio.hpp -- host CSR ingestion (mmio.cpp): Matrix Market I/O and validation.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

namespace csg {

struct HostCsr {
  int64_t n = 0;
  std::vector<int64_t> rowptr, col;
  std::vector<double> val;
};

HostCsr* mm_read(const std::string& path, bool require_spd);
void mm_write(const std::string& path, int64_t n, const int64_t* rp, const int64_t* ci,
              const double* v);
void validate_structure_host(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                             int64_t rowptr_len, int64_t nnz_len);
void validate_symmetric_host(int64_t n, const int64_t* rp, const int64_t* ci, const double* v);
void validate_spd_diagonal_host(int64_t n, const int64_t* rp, const int64_t* ci, const double* v);

}  // namespace csg
