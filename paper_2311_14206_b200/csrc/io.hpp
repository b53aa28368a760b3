// Matrix Market and SKRYRCY1 recycle-space files (host only; io.cpp).
#pragma once

#include "common.hpp"

#include <istream>
#include <ostream>
#include <string>
#include <vector>

namespace sdr {

/// CSR arrays as SparseMatrix holds them (sparse.hpp:79-81).
struct HostCsr {
  i64 rows = 0, cols = 0;
  std::vector<i64> offsets, columns;
  std::vector<double> values;
};

HostCsr mm_read(std::istream& in);
HostCsr mm_read_file(const std::string& path);
void mm_write(std::ostream& out, i64 rows, i64 cols, const i64* offsets, const i64* columns, const double* values);
void mm_write_file(const std::string& path, i64 rows, i64 cols, const i64* offsets, const i64* columns,
                   const double* values);

/// Recycle-space dump: U n x k, SU / SAU s x k, column-major.
struct SpaceFile {
  i64 n = 0, s = 0, k = 0, provenance = 0;
  std::vector<double> U, SU, SAU;
};
void space_write(std::ostream& out, const SpaceFile& f);
SpaceFile space_read(std::istream& in);
void space_write_file(const std::string& path, const SpaceFile& f);
SpaceFile space_read_file(const std::string& path);

}  // namespace sdr
