// Host-side file formats around the hot path:
// Matrix Market ingestion / output (matrix_market.hpp:20-181) producing the
// CSR arrays sdr_csr_create uploads, and the SKRYRCY1 recycle-space dump
// (recycle.hpp:337-385). Same accepted headers, message texts and semantics
// as the reference: symmetric storage mirrored, explicit (summed) zeros
// dropped, duplicates summed, 17-significant-digit output, native-endian
// binary dump with magic / size / provenance header.
#include "io.hpp"

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

namespace sdr {

namespace {

struct LineReader {
  std::istream& in;
  long line = 0;
  /// Next line that is neither blank nor a comment ('%' after line 1).
  bool next(std::string& out) {
    while (std::getline(in, out)) {
      ++line;
      if (!out.empty() && out.back() == '\r') out.pop_back();
      const auto p = out.find_first_not_of(" \t");
      if (p == std::string::npos) continue;
      if (out[p] == '%' && line > 1) continue;
      return true;
    }
    return false;
  }
  [[noreturn]] void fail(const std::string& what) const {
    throw runtime("Matrix Market parse error at line " + std::to_string(line) + ": " + what);
  }
};

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> t;
  std::istringstream ss(s);
  std::string w;
  while (ss >> w) t.push_back(w);
  return t;
}

std::string lower(std::string s) {
  for (auto& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

long long parse_int(const std::string& tok, const LineReader& rd) {
  long long v = 0;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (r.ec != std::errc{} || r.ptr != tok.data() + tok.size()) rd.fail("expected integer, got '" + tok + "'");
  return v;
}

double parse_real(const std::string& tok, const LineReader& rd) {
  double v = 0.0;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (r.ec != std::errc{} || r.ptr != tok.data() + tok.size()) rd.fail("expected real number, got '" + tok + "'");
  return v;
}

struct Entry {
  i64 r, c;
  double v;
};

/// SparseMatrix::from_triplets (sparse.hpp:40-73): row-major order,
/// duplicates summed in input order, zero sums dropped.
HostCsr assemble(i64 rows, i64 cols, std::vector<Entry>& e) {
  std::stable_sort(e.begin(), e.end(), [](const Entry& a, const Entry& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
  HostCsr h;
  h.rows = rows;
  h.cols = cols;
  h.offsets.assign(static_cast<size_t>(rows) + 1, 0);
  h.columns.reserve(e.size());
  h.values.reserve(e.size());
  for (size_t i = 0; i < e.size();) {
    const i64 r = e[i].r, c = e[i].c;
    double v = 0.0;
    for (; i < e.size() && e[i].r == r && e[i].c == c; ++i) v += e[i].v;
    if (v != 0.0) {
      h.columns.push_back(c);
      h.values.push_back(v);
      ++h.offsets[static_cast<size_t>(r) + 1];
    }
  }
  for (i64 r = 0; r < rows; ++r) h.offsets[static_cast<size_t>(r) + 1] += h.offsets[static_cast<size_t>(r)];
  return h;
}

void read_raw(std::istream& in, void* p, size_t bytes, const char* what) {
  in.read(static_cast<char*>(p), static_cast<std::streamsize>(bytes));
  if (static_cast<size_t>(in.gcount()) != bytes)
    throw runtime(std::string("recycle-space load: truncated file while reading ") + what);
}

void write_raw(std::ostream& out, const void* p, size_t bytes) {
  out.write(static_cast<const char*>(p), static_cast<std::streamsize>(bytes));
}

constexpr char kMagic[8] = {'S', 'K', 'R', 'Y', 'R', 'C', 'Y', '1'};

}  // namespace

HostCsr mm_read(std::istream& in) {  // matrix_market.hpp:83-159
  LineReader rd{in};
  std::string line;
  if (!rd.next(line)) rd.fail("empty stream");
  const auto hdr = split_ws(line);
  if (hdr.size() != 5 || lower(hdr[0]) != "%%matrixmarket" || lower(hdr[1]) != "matrix")
    rd.fail("expected header '%%MatrixMarket matrix <format> <field> <symmetry>'");
  const std::string format = lower(hdr[2]), field = lower(hdr[3]), symmetry = lower(hdr[4]);
  if (format != "coordinate" && format != "array") rd.fail("unsupported format '" + format + "'");
  if (field != "real" && field != "integer") rd.fail("unsupported field '" + field + "' (this build reads real data)");
  if (symmetry != "general" && symmetry != "symmetric") rd.fail("unsupported symmetry '" + symmetry + "'");
  const bool sym = symmetry == "symmetric";
  if (!rd.next(line)) rd.fail("missing size line");
  const auto sz = split_ws(line);
  std::vector<Entry> e;
  if (format == "coordinate") {
    if (sz.size() != 3) rd.fail("coordinate size line needs 'rows cols nnz'");
    const long long rows = parse_int(sz[0], rd), cols = parse_int(sz[1], rd), nnz = parse_int(sz[2], rd);
    if (rows < 0 || cols < 0 || nnz < 0) rd.fail("negative size");
    if (sym && rows != cols) rd.fail("symmetric matrix must be square");
    e.reserve(static_cast<size_t>(sym ? 2 * nnz : nnz));
    for (long long q = 0; q < nnz; ++q) {
      if (!rd.next(line))
        rd.fail("unexpected end of data: entry " + std::to_string(q + 1) + " of " + std::to_string(nnz) + " missing");
      const auto t = split_ws(line);
      if (t.size() != 3) rd.fail("coordinate entry needs 'row col value'");
      const long long i = parse_int(t[0], rd), j = parse_int(t[1], rd);
      const double v = parse_real(t[2], rd);
      if (i < 1 || i > rows || j < 1 || j > cols)
        rd.fail("entry (" + std::to_string(i) + ", " + std::to_string(j) + ") outside " + std::to_string(rows) + "x" +
                std::to_string(cols));
      e.push_back({i - 1, j - 1, v});
      if (sym && i != j) e.push_back({j - 1, i - 1, v});
    }
    return assemble(rows, cols, e);
  }
  if (sz.size() != 2) rd.fail("array size line needs 'rows cols'");
  const long long rows = parse_int(sz[0], rd), cols = parse_int(sz[1], rd);
  if (rows < 0 || cols < 0) rd.fail("negative size");
  if (sym && rows != cols) rd.fail("symmetric matrix must be square");
  for (long long j = 0; j < cols; ++j) {  // column-major; symmetric keeps the lower triangle
    for (long long i = sym ? j : 0; i < rows; ++i) {
      if (!rd.next(line)) rd.fail("unexpected end of data in array body");
      const auto t = split_ws(line);
      if (t.size() != 1) rd.fail("array entry needs a single value per line");
      const double v = parse_real(t[0], rd);
      e.push_back({i, j, v});
      if (sym && i != j) e.push_back({j, i, v});
    }
  }
  return assemble(rows, cols, e);
}

HostCsr mm_read_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw runtime("cannot open Matrix Market file '" + path + "'");
  return mm_read(in);
}

void mm_write(std::ostream& out, i64 rows, i64 cols, const i64* offsets, const i64* columns, const double* values) {
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << rows << " " << cols << " " << offsets[rows] << "\n";
  char buf[64];
  for (i64 r = 0; r < rows; ++r)
    for (i64 p = offsets[r]; p < offsets[r + 1]; ++p) {
      std::snprintf(buf, sizeof(buf), "%.16e", values[p]);
      out << (r + 1) << " " << (columns[p] + 1) << " " << buf << "\n";
    }
}

void mm_write_file(const std::string& path, i64 rows, i64 cols, const i64* offsets, const i64* columns,
                   const double* values) {
  std::ofstream out(path);
  if (!out) throw runtime("cannot open '" + path + "' for writing");
  mm_write(out, rows, cols, offsets, columns, values);
  if (!out) throw runtime("write to '" + path + "' failed");
}

void space_write(std::ostream& out, const SpaceFile& f) {  // recycle.hpp:339-353
  write_raw(out, kMagic, sizeof(kMagic));
  write_raw(out, &f.n, sizeof(f.n));
  write_raw(out, &f.s, sizeof(f.s));
  write_raw(out, &f.k, sizeof(f.k));
  write_raw(out, &f.provenance, sizeof(f.provenance));
  write_raw(out, f.U.data(), sizeof(double) * f.U.size());
  write_raw(out, f.SU.data(), sizeof(double) * f.SU.size());
  write_raw(out, f.SAU.data(), sizeof(double) * f.SAU.size());
}

SpaceFile space_read(std::istream& in) {  // recycle.hpp:355-378
  char magic[8];
  read_raw(in, magic, sizeof(magic), "magic");
  if (!std::equal(magic, magic + 8, kMagic)) throw runtime("recycle-space load: bad magic (not a recycle-space dump)");
  SpaceFile f;
  read_raw(in, &f.n, sizeof(f.n), "dimensions");
  read_raw(in, &f.s, sizeof(f.s), "dimensions");
  read_raw(in, &f.k, sizeof(f.k), "dimensions");
  read_raw(in, &f.provenance, sizeof(f.provenance), "provenance");
  if (f.n < 0 || f.s < 0 || f.k < 0 || f.provenance < 0 || f.provenance > 4)
    throw runtime("recycle-space load: corrupt header");
  // read in bounded pieces so a corrupt size fails as truncation, not as a huge allocation
  auto block = [&](std::vector<double>& v, i64 count, const char* what) {
    v.clear();
    constexpr i64 kPiece = i64{1} << 20;
    for (i64 done = 0; done < count;) {
      const i64 take = std::min(kPiece, count - done);
      v.resize(static_cast<size_t>(done + take));
      read_raw(in, v.data() + done, sizeof(double) * static_cast<size_t>(take), what);
      done += take;
    }
  };
  block(f.U, f.n * f.k, "U");
  block(f.SU, f.s * f.k, "SU");
  block(f.SAU, f.s * f.k, "SAU");
  return f;
}

void space_write_file(const std::string& path, const SpaceFile& f) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw runtime("cannot open '" + path + "' for writing");
  space_write(out, f);
  if (!out) throw runtime("write to '" + path + "' failed");
}

SpaceFile space_read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw runtime("cannot open recycle-space file '" + path + "'");
  return space_read(in);
}

}  // namespace sdr
