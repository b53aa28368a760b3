// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A single-threaded CPU restatement of the reference GMRES-SDR library
// (`skrylov`, /root/reference/proj/include/skrylov) used as the parity
// checker for the B200 product in paper_2311_14206_b200/. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load it; the product never links, imports or calls anything here.
//
// Why a restatement: the reference is header-only C++20 on Eigen3 + FFTW3 +
// LAPACKE, none of which exist in this image, so it cannot be
// compiled. Every function below cites the reference file:line it follows.
// Substitutions (numerically equivalent maps, different rounding):
//   * Eigen dense algebra            -> plain loops (same summation order as
//                                       Eigen's scalar path is NOT guaranteed)
//   * FFTW REDFT10 (sketch.hpp:55-61) -> radix-2 FFT DCT-II (n a power of two)
//                                       or the reference's own direct formula
//                                       (sketch.hpp:65-79) with exact integer
//                                       phase reduction
//   * Eigen::JacobiSVD (recycle.hpp:100) -> LAPACK dgesvd (same singular
//                                       values / subspaces; signs of singular
//                                       vectors cancel in the pencil)
//   * LAPACKE dgees/dtrsen (detail/lapack.hpp:25-60) -> the same LAPACK
//                                       routines from scipy's bundled OpenBLAS
// Parity pins: the reference's own known-answer tests (mt19937_64 10000th
// output, convdiff stencil coefficients, A=2.5I breakdown, identity-sketch
// collapse to dense GMRES, exact counter arithmetic, ...) are re-run against
// this file in tests/test_oracle_*.py.
//
// New (not in the reference, parity unpinned, defined identically on the
// GPU): the sparse-sign sketch (SparseSign) and the 3D /
// per-direction convection-diffusion generators used by BASELINE configs.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <thread>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <mutex>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

extern "C" {
void scipy_dgees_(const char* jobvs, const char* sort, void* select, const int* n, double* a,
                  const int* lda, int* sdim, double* wr, double* wi, double* vs, const int* ldvs,
                  double* work, const int* lwork, int* bwork, int* info, size_t, size_t);
void scipy_dtrsen_(const char* job, const char* compq, const int* select, const int* n, double* t,
                   const int* ldt, double* q, const int* ldq, double* wr, double* wi, int* m,
                   double* s, double* sep, double* work, const int* lwork, int* iwork,
                   const int* liwork, int* info, size_t, size_t);
void scipy_dgesvd_(const char* jobu, const char* jobvt, const int* m, const int* n, double* a,
                   const int* lda, double* s, double* u, const int* ldu, double* vt,
                   const int* ldvt, double* work, const int* lwork, int* info, size_t, size_t);
}

namespace oracle {

using Index = std::int64_t;
using Vec = std::vector<double>;

// ---------------------------------------------------------------- dense ---

/// Column-major dense matrix (stands in for Eigen::MatrixXd).
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + j * rows)]; }
  double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + j * rows)]; }
  double* col(Index j) { return a.data() + j * rows; }
  const double* col(Index j) const { return a.data() + j * rows; }
  void resize_cols(Index c) {
    a.resize(static_cast<size_t>(rows * c), 0.0);
    cols = c;
  }
};

/// Host threads for the long loops (bench.py's all-cores CPU baseline):
/// ORC_THREADS, default 1 — the reference is single-threaded, and with one
/// thread every result is the plain sequential loop's (the parity tests).
inline int threads() {
  const char* e = std::getenv("ORC_THREADS");  // read per call: the bench switches it between samples
  const int v = e ? std::atoi(e) : 1;
  return v > 1 ? v : 1;
}

/// f(begin, end, thread) over [0, n) split into threads() contiguous ranges
/// (plain std::thread: no OpenMP runtime next to the host process's own).
template <class F>
inline void parallel_ranges(Index n, F&& f) {
  const int nt = threads();
  if (nt == 1 || n < 100000) {
    f(Index{0}, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt, t); });
  f(Index{0}, n / nt, 0);
  for (auto& x : th) x.join();
}

inline double dot(const double* x, const double* y, Index n) {
  if (threads() > 1 && n >= 100000) {  // per-range sums added in range order
    std::vector<double> part(static_cast<size_t>(threads()), 0.0);
    parallel_ranges(n, [&](Index b, Index e, int t) {
      double s = 0.0;
      for (Index i = b; i < e; ++i) s += x[i] * y[i];
      part[static_cast<size_t>(t)] = s;
    });
    double s = 0.0;
    for (double v : part) s += v;
    return s;
  }
  double s = 0.0;
  for (Index i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
inline double norm(const double* x, Index n) { return std::sqrt(dot(x, x, n)); }
inline double norm(const Vec& x) { return norm(x.data(), static_cast<Index>(x.size())); }

// ------------------------------------------------------------------ rng ---
// rng.hpp:25-96

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t next_u64() { return engine_(); }
  double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }  // rng.hpp:32
  std::uint64_t uniform_below(std::uint64_t bound) {                              // rng.hpp:35-42
    if (bound == 0) throw std::invalid_argument("Rng::uniform_below: bound must be positive");
    const std::uint64_t threshold = (-bound) % bound;
    for (;;) {
      const std::uint64_t r = engine_();
      if (r >= threshold) return r % bound;
    }
  }
  double gaussian() {  // rng.hpp:45-60
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = 0.0;
    do {
      u1 = uniform();
    } while (u1 <= 0.0);
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    spare_ = radius * std::sin(angle);
    have_spare_ = true;
    return radius * std::cos(angle);
  }
  double sign() { return (engine_() & 1u) ? 1.0 : -1.0; }  // rng.hpp:63
  std::vector<Index> sample_without_replacement(Index n, Index k) {  // rng.hpp:66-78
    if (k < 0 || n < 0 || k > n)
      throw std::invalid_argument("Rng::sample_without_replacement: need 0 <= k <= n");
    std::vector<Index> idx(static_cast<size_t>(n));
    std::iota(idx.begin(), idx.end(), Index{0});
    for (Index i = 0; i < k; ++i) {
      const auto j = i + static_cast<Index>(uniform_below(static_cast<std::uint64_t>(n - i)));
      std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(j)]);
    }
    idx.resize(static_cast<size_t>(k));
    std::sort(idx.begin(), idx.end());
    return idx;
  }

 private:
  std::mt19937_64 engine_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

inline Vec gaussian_vector(Index n, std::uint64_t seed) {  // rng.hpp:87-96
  Rng rng(seed);
  Vec v(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) v[static_cast<size_t>(i)] = rng.gaussian();
  return v;
}

// --------------------------------------------------------------- sparse ---
// sparse.hpp:15-150

struct Triplet {
  Index row = 0, col = 0;
  double value = 0.0;
};

class SparseMatrix {
 public:
  SparseMatrix() = default;
  SparseMatrix(Index rows, Index cols, std::vector<Index> offsets, std::vector<Index> columns,
               Vec values)
      : rows_(rows), cols_(cols), offsets_(std::move(offsets)), columns_(std::move(columns)),
        values_(std::move(values)) {
    validate();
  }

  static SparseMatrix from_triplets(Index rows, Index cols, std::vector<Triplet> t) {  // :40-73
    for (const auto& e : t)
      if (e.row < 0 || e.row >= rows || e.col < 0 || e.col >= cols)
        throw std::invalid_argument("SparseMatrix::from_triplets: entry (" + std::to_string(e.row) +
                                    ", " + std::to_string(e.col) + ") outside " +
                                    std::to_string(rows) + "x" + std::to_string(cols));
    std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
      return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    std::vector<Index> offsets(static_cast<size_t>(rows) + 1, 0), columns;
    Vec values;
    columns.reserve(t.size());
    values.reserve(t.size());
    size_t i = 0;
    while (i < t.size()) {
      const Index r = t[i].row, c = t[i].col;
      double v = 0.0;
      while (i < t.size() && t[i].row == r && t[i].col == c) v += t[i++].value;
      if (v != 0.0) {
        columns.push_back(c);
        values.push_back(v);
        ++offsets[static_cast<size_t>(r) + 1];
      }
    }
    for (size_t r = 0; r < static_cast<size_t>(rows); ++r) offsets[r + 1] += offsets[r];
    return SparseMatrix(rows, cols, std::move(offsets), std::move(columns), std::move(values));
  }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index nonzeros() const { return static_cast<Index>(values_.size()); }
  const std::vector<Index>& offsets() const { return offsets_; }
  const std::vector<Index>& columns() const { return columns_; }
  const Vec& values() const { return values_; }

  void apply(const double* x, Index xlen, double* y) const {  // :84-98
    if (xlen != cols_)
      throw std::invalid_argument("SparseMatrix::apply: matrix has " + std::to_string(cols_) +
                                  " columns but vector has " + std::to_string(xlen) + " entries");
    parallel_ranges(rows_, [&](Index rb, Index re, int) {  // rows are independent: same sums, any thread count
      for (Index r = rb; r < re; ++r) {
        double acc = 0.0;
        for (Index p = offsets_[static_cast<size_t>(r)]; p < offsets_[static_cast<size_t>(r) + 1]; ++p)
          acc += values_[static_cast<size_t>(p)] * x[columns_[static_cast<size_t>(p)]];
        y[r] = acc;
      }
    });
  }

 private:
  void validate() const {  // :117-143
    if (rows_ < 0 || cols_ < 0) throw std::invalid_argument("SparseMatrix: negative dimensions");
    if (offsets_.size() != static_cast<size_t>(rows_) + 1)
      throw std::invalid_argument("SparseMatrix: offsets size " + std::to_string(offsets_.size()) +
                                  " does not match rows + 1 = " + std::to_string(rows_ + 1));
    if (offsets_.front() != 0) throw std::invalid_argument("SparseMatrix: offsets must start at 0");
    if (offsets_.back() != static_cast<Index>(values_.size()) || columns_.size() != values_.size())
      throw std::invalid_argument("SparseMatrix: offsets/columns/values sizes inconsistent");
    for (size_t r = 0; r < static_cast<size_t>(rows_); ++r) {
      if (offsets_[r + 1] < offsets_[r])
        throw std::invalid_argument("SparseMatrix: offsets decrease at row " + std::to_string(r));
      for (Index p = offsets_[r]; p < offsets_[r + 1]; ++p) {
        const auto c = columns_[static_cast<size_t>(p)];
        if (c < 0 || c >= cols_)
          throw std::invalid_argument("SparseMatrix: column index " + std::to_string(c) +
                                      " out of range in row " + std::to_string(r));
        if (p > offsets_[r] && columns_[static_cast<size_t>(p) - 1] >= c)
          throw std::invalid_argument(
              "SparseMatrix: column indices not strictly increasing in row " + std::to_string(r));
        if (!std::isfinite(values_[static_cast<size_t>(p)]))
          throw std::invalid_argument("SparseMatrix: non-finite value in row " + std::to_string(r));
      }
    }
  }
  Index rows_ = 0, cols_ = 0;
  std::vector<Index> offsets_{0}, columns_;
  Vec values_;
};

/// operator_ref.hpp:20-56 — type-erased y = A x with a dimension check.
class OperatorRef {
 public:
  using Apply = std::function<void(const double*, double*)>;
  OperatorRef(Index rows, Index cols, Apply fn) : rows_(rows), cols_(cols), fn_(std::move(fn)) {}
  explicit OperatorRef(const SparseMatrix& A)
      : rows_(A.rows()), cols_(A.cols()),
        fn_([&A](const double* x, double* y) { A.apply(x, A.cols(), y); }) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  void apply(const Vec& x, Vec& y) const {
    if (static_cast<Index>(x.size()) != cols_)
      throw std::invalid_argument("OperatorRef::apply: operator has " + std::to_string(cols_) +
                                  " columns but vector has " + std::to_string(x.size()) +
                                  " entries");
    y.assign(static_cast<size_t>(rows_), 0.0);
    fn_(x.data(), y.data());
  }
  void apply_raw(const double* x, double* y) const { fn_(x, y); }

 private:
  Index rows_ = 0, cols_ = 0;
  Apply fn_;
};

// ------------------------------------------------------------- problems ---
// problems.hpp:38-88 (reference generators) + new BASELINE generators

inline SparseMatrix gen_neumann(Index g, double shift) {  // problems.hpp:38-62
  if (g < 2) throw std::invalid_argument("gen_neumann: grid_side must be at least 2");
  const Index n = g * g;
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(5 * n));
  auto reflect = [g](Index i) {
    if (i < 0) return -i;
    if (i >= g) return 2 * g - 2 - i;
    return i;
  };
  for (Index r = 0; r < g; ++r)
    for (Index c = 0; c < g; ++c) {
      const Index p = r * g + c;
      t.push_back({p, p, 4.0 + shift});
      const Index nbr[4][2] = {{r - 1, c}, {r + 1, c}, {r, c - 1}, {r, c + 1}};
      for (const auto& d : nbr) t.push_back({p, reflect(d[0]) * g + reflect(d[1]), -1.0});
    }
  return SparseMatrix::from_triplets(n, n, std::move(t));
}

inline SparseMatrix gen_convdiff(Index n, double alpha) {  // problems.hpp:70-88
  if (n < 1) throw std::invalid_argument("gen_convdiff: n must be positive");
  const double h2 = static_cast<double>((n + 1) * (n + 1));
  const double cv = alpha * static_cast<double>(n + 1) / 2.0;
  const Index N = n * n;
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(5 * N));
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      const Index p = i * n + j;
      t.push_back({p, p, -4.0 * h2});
      if (i > 0) t.push_back({p, p - n, h2 - cv});
      if (i + 1 < n) t.push_back({p, p + n, h2 + cv});
      if (j > 0) t.push_back({p, p - 1, h2 - cv});
      if (j + 1 < n) t.push_back({p, p + 1, h2 + cv});
    }
  return SparseMatrix::from_triplets(N, N, std::move(t));
}

/// NEW (BASELINE C1/C3): -Δu + β·∇u on an n×n interior grid, h = 1/(n+1),
/// central differences, Dirichlet, lexicographic p = iy·n + ix (x fastest).
/// β_x couples p±1, β_y couples p±n. With β_x == β_y == β this equals
/// −gen_convdiff(n, −β) bit for bit. Optional
/// diagonal shift and per-row relative diagonal perturbation (C3).
inline SparseMatrix gen_convdiff2d(Index n, double bx, double by, double shift = 0.0,
                                   const Vec* diag_rel = nullptr) {
  const double h2 = static_cast<double>((n + 1) * (n + 1));
  const double cx = bx * static_cast<double>(n + 1) / 2.0;
  const double cy = by * static_cast<double>(n + 1) / 2.0;
  const Index N = n * n;
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(5 * N));
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      const Index p = i * n + j;
      double d = 4.0 * h2 + shift;
      if (diag_rel) d = d + d * (*diag_rel)[static_cast<size_t>(p)];
      t.push_back({p, p, d});
      if (i > 0) t.push_back({p, p - n, -h2 - cy});
      if (i + 1 < n) t.push_back({p, p + n, -h2 + cy});
      if (j > 0) t.push_back({p, p - 1, -h2 - cx});
      if (j + 1 < n) t.push_back({p, p + 1, -h2 + cx});
    }
  return SparseMatrix::from_triplets(N, N, std::move(t));
}

/// NEW (BASELINE C2/C5): 7-point −Δu + β·∇u on an n³ interior grid,
/// h = 1/(n+1), Dirichlet, p = iz·n² + iy·n + ix (x fastest).
/// 3D analogue of gen_convdiff (BASELINE C2/C5: 7-point -Δu + β·∇u, h = 1/(n+1),
/// lexicographic order x fastest). No reference code (unpinned);
/// entries as from_triplets would produce them (:40-73: rows in order,
/// increasing columns, exact zeros dropped), written row by row so C5
/// (N = 2^27, 0.94 G entries) needs no 22 GB triplet sort.
inline SparseMatrix gen_convdiff3d(Index n, double bx, double by, double bz) {
  const double h2 = static_cast<double>((n + 1) * (n + 1));
  const double c[3] = {bx * static_cast<double>(n + 1) / 2.0, by * static_cast<double>(n + 1) / 2.0,
                       bz * static_cast<double>(n + 1) / 2.0};
  const Index N = n * n * n;
  const Index stride[3] = {1, n, n * n};
  std::vector<Index> offsets(static_cast<size_t>(N) + 1, 0), columns;
  Vec values;
  columns.reserve(static_cast<size_t>(7 * N));
  values.reserve(static_cast<size_t>(7 * N));
  auto put = [&](Index col, double v) {
    if (v != 0.0) {
      columns.push_back(col);
      values.push_back(v);
    }
  };
  for (Index z = 0; z < n; ++z)
    for (Index y = 0; y < n; ++y)
      for (Index x = 0; x < n; ++x) {
        const Index p = z * n * n + y * n + x;
        const Index coord[3] = {x, y, z};
        for (int d = 2; d >= 0; --d)  // columns below p, increasing
          if (coord[d] > 0) put(p - stride[d], -h2 - c[d]);
        put(p, 6.0 * h2);
        for (int d = 0; d < 3; ++d)  // columns above p, increasing
          if (coord[d] + 1 < n) put(p + stride[d], -h2 + c[d]);
        offsets[static_cast<size_t>(p) + 1] = static_cast<Index>(columns.size());
      }
  return SparseMatrix(N, N, std::move(offsets), std::move(columns), std::move(values));
}

// --------------------------------------------------------------- sketch ---
// sketch.hpp:55-162 plus the new sparse-sign map

namespace detail {

/// Per-length DCT-II plan, cached like the reference's FFTW plan cache
/// (DctPlanCache, sketch.hpp:27-50: one plan per n behind a mutex): the
/// bit reversal and per-stage twiddles of an h = n/2 point complex FFT, the
/// real-FFT untangling twiddles e^{-2πik/n} and the DCT phase e^{-iπk/2n}.
struct DctPlan {
  Index n = 0, h = 0;
  std::vector<std::uint32_t> rev;
  std::vector<std::complex<double>> tw;     // stage len: tw[len/2 - 1 + k] = e^{-2πik/len}
  std::vector<std::complex<double>> post;   // e^{-2πik/n}, k < h
  std::vector<std::complex<double>> shift;  // e^{-iπk/2n}, k < n
};

inline const DctPlan& dct_plan(Index n) {
  static std::mutex mu;
  static std::map<Index, std::unique_ptr<DctPlan>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto& slot = cache[n];
  if (slot) return *slot;
  auto p = std::make_unique<DctPlan>();
  const double pi = 3.14159265358979323846;
  p->n = n;
  p->h = n / 2;
  const Index h = p->h;
  int bits = 0;
  while ((Index{1} << bits) < h) ++bits;
  p->rev.resize(static_cast<size_t>(h));
  for (Index i = 0; i < h; ++i) {
    std::uint32_t r = 0;
    for (int b = 0; b < bits; ++b) r |= ((static_cast<std::uint32_t>(i) >> b) & 1u) << (bits - 1 - b);
    p->rev[static_cast<size_t>(i)] = r;
  }
  p->tw.resize(static_cast<size_t>(std::max<Index>(h, 1)));
  for (Index len = 2; len <= h; len <<= 1)
    for (Index k = 0; k < len / 2; ++k) {
      const double ang = -2.0 * pi * static_cast<double>(k) / static_cast<double>(len);
      p->tw[static_cast<size_t>(len / 2 - 1 + k)] = {std::cos(ang), std::sin(ang)};
    }
  p->post.resize(static_cast<size_t>(h));
  for (Index k = 0; k < h; ++k) {
    const double ang = -2.0 * pi * static_cast<double>(k) / static_cast<double>(n);
    p->post[static_cast<size_t>(k)] = {std::cos(ang), std::sin(ang)};
  }
  p->shift.resize(static_cast<size_t>(n));
  for (Index k = 0; k < n; ++k) {
    const double ang = -pi * static_cast<double>(k) / (2.0 * static_cast<double>(n));
    p->shift[static_cast<size_t>(k)] = {std::cos(ang), std::sin(ang)};
  }
  slot = std::move(p);
  return *slot;
}

/// Orthonormal DCT-II of length n (power of two, n >= 2): Makhoul's
/// reordering v = (x_0, x_2, ..., x_3, x_1), V = FFT_n(v) computed as a
/// real FFT (one n/2-point complex FFT plus untangling), X_k = Re(e^{-iπk/2n}
/// V_k) with the orthonormal scaling. Same map as sketch.hpp:55-61 (FFTW
/// REDFT10 + orthonormal scaling).
inline void dct2_orthonormal_pow2(const double* in, double* out, Index n) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  const DctPlan& p = dct_plan(n);
  const Index h = p.h;
  // z_m = v_{2m} + i v_{2m+1}; v_j = x_{2j} (j < n/2), v_{n-1-j} = x_{2j+1}
  auto v = [&](Index j) { return j < h ? in[2 * j] : in[2 * (n - 1 - j) + 1]; };
  std::vector<std::complex<double>> z(static_cast<size_t>(h));
  for (Index m = 0; m < h; ++m) z[p.rev[static_cast<size_t>(m)]] = {v(2 * m), v(2 * m + 1)};
  for (Index len = 2; len <= h; len <<= 1) {
    const std::complex<double>* w = p.tw.data() + (len / 2 - 1);
    for (Index i = 0; i < h; i += len)
      for (Index k = 0; k < len / 2; ++k) {
        const std::complex<double> a = z[static_cast<size_t>(i + k)], b = z[static_cast<size_t>(i + k + len / 2)] * w[k];
        z[static_cast<size_t>(i + k)] = a + b;
        z[static_cast<size_t>(i + k + len / 2)] = a - b;
      }
  }
  const double s0 = 1.0 / std::sqrt(static_cast<double>(n));
  const double s = std::sqrt(2.0 / static_cast<double>(n));
  auto V = [&](Index k) -> std::complex<double> {  // FFT_n(v)_k for 0 <= k <= h
    if (k == h) return {z[0].real() - z[0].imag(), 0.0};
    const std::complex<double> a = z[static_cast<size_t>(k)], b = std::conj(z[static_cast<size_t>((h - k) % h)]);
    const std::complex<double> even = 0.5 * (a + b), odd = std::complex<double>(0.0, -0.5) * (a - b);
    return even + p.post[static_cast<size_t>(k)] * odd;
  };
  for (Index k = 0; k <= h; ++k) {
    const std::complex<double> vk = V(k);
    out[k] = (p.shift[static_cast<size_t>(k)] * vk).real() * (k == 0 ? s0 : s);
    if (k > 0 && k < h)  // V_{n-k} = conj(V_k) (real input)
      out[n - k] = (p.shift[static_cast<size_t>(n - k)] * std::conj(vk)).real() * s;
  }
}

/// sketch.hpp:65-79 — selected rows evaluated term by term, with the phase
/// k(2j+1) reduced exactly modulo 4n before the cosine (the reference forms
/// θ·k·(2j+1) in floating point; this is the same map, tighter rounding).
inline void dct2_selected_direct(const double* x, Index n, const std::vector<Index>& rows, double* out) {
  const std::uint64_t four_n = 4u * static_cast<std::uint64_t>(n);
  for (size_t q = 0; q < rows.size(); ++q) {
    const std::uint64_t k = static_cast<std::uint64_t>(rows[q]);
    double acc = 0.0;
    for (Index j = 0; j < n; ++j) {
      const std::uint64_t ph = (k * (2u * static_cast<std::uint64_t>(j) + 1u)) % four_n;
      acc += x[j] * std::cos(3.14159265358979323846 * static_cast<double>(ph) / (2.0 * static_cast<double>(n)));
    }
    const double alpha = rows[q] == 0 ? std::sqrt(1.0 / static_cast<double>(n)) : std::sqrt(2.0 / static_cast<double>(n));
    out[q] = alpha * acc;
  }
}

/// splitmix64 finalizer (Steele, Lea, Flood 2014) — the counter hash of the
/// sparse-sign map. MUST match paper_2311_14206_b200/csrc/sketch_common.hpp.
inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/// min ||A y - b|| by Householder QR with column pivoting, the basic
/// solution for a rank-deficient A (the fallback of baseline.hpp:175-177,
/// Eigen's colPivHouseholderQr: rank threshold eps * min(rows, cols) * |r_max|).
inline Vec least_squares(Mat A, Vec b) {
  const Index m = A.rows, n = A.cols;
  std::vector<Index> perm(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) perm[static_cast<size_t>(j)] = j;
  std::vector<double> cn(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) cn[static_cast<size_t>(j)] = dot(A.col(j), A.col(j), m);
  const Index kmax = std::min(m, n);
  double rmax = 0.0;
  Index rank = 0;
  for (Index k = 0; k < kmax; ++k) {
    Index piv = k;  // the column of largest remaining norm
    for (Index j = k + 1; j < n; ++j)
      if (cn[static_cast<size_t>(j)] > cn[static_cast<size_t>(piv)]) piv = j;
    if (piv != k) {
      for (Index i = 0; i < m; ++i) std::swap(A(i, k), A(i, piv));
      std::swap(cn[static_cast<size_t>(k)], cn[static_cast<size_t>(piv)]);
      std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(piv)]);
    }
    double nrm = 0.0;
    for (Index i = k; i < m; ++i) nrm += A(i, k) * A(i, k);
    nrm = std::sqrt(nrm);
    if (nrm > 0.0) {
      const double alpha = A(k, k) > 0.0 ? -nrm : nrm;
      std::vector<double> v(static_cast<size_t>(m - k));
      for (Index i = k; i < m; ++i) v[static_cast<size_t>(i - k)] = A(i, k);
      v[0] -= alpha;
      const double vn2 = dot(v.data(), v.data(), m - k);
      if (vn2 > 0.0) {
        for (Index j = k; j < n; ++j) {
          double d = 0.0;
          for (Index i = k; i < m; ++i) d += v[static_cast<size_t>(i - k)] * A(i, j);
          d *= 2.0 / vn2;
          for (Index i = k; i < m; ++i) A(i, j) -= d * v[static_cast<size_t>(i - k)];
        }
        double d = 0.0;
        for (Index i = k; i < m; ++i) d += v[static_cast<size_t>(i - k)] * b[static_cast<size_t>(i)];
        d *= 2.0 / vn2;
        for (Index i = k; i < m; ++i) b[static_cast<size_t>(i)] -= d * v[static_cast<size_t>(i - k)];
      }
    }
    rmax = std::max(rmax, std::abs(A(k, k)));
    for (Index j = k + 1; j < n; ++j) {  // downdate the remaining column norms
      double s = 0.0;
      for (Index i = k + 1; i < m; ++i) s += A(i, j) * A(i, j);
      cn[static_cast<size_t>(j)] = s;
    }
  }
  const double thr = std::numeric_limits<double>::epsilon() * static_cast<double>(kmax) * rmax;
  for (Index k = 0; k < kmax; ++k)
    if (std::abs(A(k, k)) > thr) rank = k + 1;
    else break;
  Vec z(static_cast<size_t>(n), 0.0);
  for (Index i = rank - 1; i >= 0; --i) {
    double acc = b[static_cast<size_t>(i)];
    for (Index j = i + 1; j < rank; ++j) acc -= A(i, j) * z[static_cast<size_t>(j)];
    z[static_cast<size_t>(i)] = acc / A(i, i);
  }
  Vec y(static_cast<size_t>(n), 0.0);
  for (Index j = 0; j < n; ++j) y[static_cast<size_t>(perm[static_cast<size_t>(j)])] = z[static_cast<size_t>(j)];
  return y;
}

}  // namespace detail

enum class SketchKind { subsampled_dct = 0, identity = 1, sparse_sign = 2 };
enum class SketchBackend { automatic, fft, direct };

class SketchOperator {
 public:
  /// sketch.hpp:105-122: n signs drawn first, then s rows.
  static SketchOperator subsampled_dct(Index n, Index s, std::uint64_t seed,
                                       SketchBackend backend = SketchBackend::automatic) {
    if (n < 2 || s < 1 || s >= n)
      throw std::invalid_argument("SketchOperator: need 1 <= s < n, got s = " + std::to_string(s) +
                                  ", n = " + std::to_string(n));
    SketchOperator S;
    S.kind_ = SketchKind::subsampled_dct;
    S.n_ = n;
    S.s_ = s;
    S.seed_ = seed;
    S.backend_ = backend;
    Rng rng(seed);
    S.signs_.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) S.signs_[static_cast<size_t>(i)] = rng.sign();
    S.rows_ = rng.sample_without_replacement(n, s);
    S.scale_ = std::sqrt(static_cast<double>(n) / static_cast<double>(s));
    return S;
  }

  static SketchOperator identity(Index n) {  // sketch.hpp:125-132
    if (n < 1) throw std::invalid_argument("SketchOperator::identity: n must be positive");
    SketchOperator S;
    S.kind_ = SketchKind::identity;
    S.n_ = n;
    S.s_ = n;
    return S;
  }

  /// NEW — sparse sign embedding, block (Kane–Nelson) construction. Rows are
  /// split into ζ contiguous blocks [⌊l·s/ζ⌋, ⌊(l+1)·s/ζ⌋); column j holds
  /// exactly one nonzero ±1/√ζ in each block (so ζ distinct rows). With
  /// key = Rng(seed).next_u64(), nc = ⌈ζ/4⌉ and, for the chunk c = ⌊l/4⌋,
  /// h = mix64(key + (j·nc + c + 1)·φ64), entry l takes the 16-bit field
  /// f = h >> 16·(l mod 4):
  ///   row = block_begin + (((f >> 1) & 0x7FFF) · block_size) >> 15,  sign = f & 1 ? +1 : −1.
  static SketchOperator sparse_sign(Index n, Index s, std::uint64_t seed, Index zeta) {
    if (n < 1 || s < 1 || zeta < 1 || zeta > s)
      throw std::invalid_argument("SketchOperator::sparse_sign: need n >= 1 and 1 <= zeta <= s, got n = " +
                                  std::to_string(n) + ", s = " + std::to_string(s) +
                                  ", zeta = " + std::to_string(zeta));
    SketchOperator S;
    S.kind_ = SketchKind::sparse_sign;
    S.n_ = n;
    S.s_ = s;
    S.seed_ = seed;
    S.zeta_ = zeta;
    Rng rng(seed);
    S.key_ = rng.next_u64();
    return S;
  }

  Index input_dim() const { return n_; }
  Index sketch_dim() const { return s_; }
  SketchKind kind() const { return kind_; }
  std::uint64_t seed() const { return seed_; }
  const std::vector<Index>& rows() const { return rows_; }
  const Vec& signs() const { return signs_; }
  Index zeta() const { return zeta_; }
  std::uint64_t key() const { return key_; }

  /// (row, sign) of entry l of column j of the sparse-sign map.
  void sparse_entry(Index j, Index l, Index* row, double* sign) const {
    const std::uint64_t nc = static_cast<std::uint64_t>((zeta_ + 3) / 4);
    const std::uint64_t h = detail::mix64(
        key_ + (static_cast<std::uint64_t>(j) * nc + static_cast<std::uint64_t>(l / 4) + 1u) * 0x9E3779B97F4A7C15ull);
    const std::uint32_t f = static_cast<std::uint32_t>(h >> (16 * (l % 4))) & 0xFFFFu;
    const Index b0 = (l * s_) / zeta_, b1 = ((l + 1) * s_) / zeta_;
    const std::uint64_t bs = static_cast<std::uint64_t>(b1 - b0);
    *row = b0 + static_cast<Index>((static_cast<std::uint64_t>((f >> 1) & 0x7FFFu) * bs) >> 15);
    *sign = (f & 1u) ? 1.0 : -1.0;
  }

  void apply(const double* x, Index xlen, double* out) const {  // sketch.hpp:139-162
    if (xlen != n_)
      throw std::invalid_argument("SketchOperator::apply: operator takes length " +
                                  std::to_string(n_) + " but vector has length " +
                                  std::to_string(xlen));
    if (kind_ == SketchKind::identity) {
      std::copy(x, x + n_, out);
      return;
    }
    if (kind_ == SketchKind::sparse_sign) {
      std::fill(out, out + s_, 0.0);
      const double inv = 1.0 / std::sqrt(static_cast<double>(zeta_));
      // sparse_entry's map with each chunk hash evaluated once (four entries
      // per hash) and the sign applied by flipping the sign bit (no
      // data-dependent branch). Columns go in chunks, within a chunk block
      // by block: a row belongs to one block, so every out[r] receives its
      // terms in increasing j — the same additions in the same order as the
      // plain entry loop (bitwise the same result).
      const std::uint64_t nc = static_cast<std::uint64_t>((zeta_ + 3) / 4);
      std::vector<Index> b0(static_cast<size_t>(zeta_)), bs(static_cast<size_t>(zeta_));
      for (Index l = 0; l < zeta_; ++l) {
        b0[static_cast<size_t>(l)] = (l * s_) / zeta_;
        bs[static_cast<size_t>(l)] = ((l + 1) * s_) / zeta_ - b0[static_cast<size_t>(l)];
      }
      constexpr Index kChunk = 2048;
      if (threads() > 1 && n_ > 100000) {
        // several host threads (bench baseline only): contiguous column
        // ranges into per-thread rows, added in thread order
        const int nt = threads();
        std::vector<Vec> part(static_cast<size_t>(nt), Vec(static_cast<size_t>(s_), 0.0));
        parallel_ranges(n_, [&](Index jb, Index je, int tid) {
          Vec& o = part[static_cast<size_t>(tid)];
          for (Index j = jb; j < je; ++j) {
            const double xv = x[j] * inv;
            for (std::uint64_t c = 0; c < nc; ++c) {
              const std::uint64_t h =
                  detail::mix64(key_ + (static_cast<std::uint64_t>(j) * nc + c + 1u) * 0x9E3779B97F4A7C15ull);
              for (Index e = 0; e < 4; ++e) {
                const Index l = static_cast<Index>(4 * c) + e;
                if (l >= zeta_) break;
                const std::uint32_t f = static_cast<std::uint32_t>(h >> (16 * e)) & 0xFFFFu;
                const Index r = b0[static_cast<size_t>(l)] +
                                static_cast<Index>((static_cast<std::uint64_t>((f >> 1) & 0x7FFFu) *
                                                    static_cast<std::uint64_t>(bs[static_cast<size_t>(l)])) >> 15);
                std::uint64_t bits;
                std::memcpy(&bits, &xv, sizeof(bits));
                bits ^= static_cast<std::uint64_t>(~f & 1u) << 63;
                double term;
                std::memcpy(&term, &bits, sizeof(term));
                o[static_cast<size_t>(r)] += term;
              }
            }
          }
        });
        for (int t = 0; t < nt; ++t)
          for (Index r = 0; r < s_; ++r) out[r] += part[static_cast<size_t>(t)][static_cast<size_t>(r)];
        return;
      }
      std::vector<std::uint64_t> hc(static_cast<size_t>(kChunk * nc));
      std::vector<std::uint64_t> xb(static_cast<size_t>(kChunk));
      for (Index j0 = 0; j0 < n_; j0 += kChunk) {
        const Index len = std::min(kChunk, n_ - j0);
        for (Index q = 0; q < len; ++q) {
          const std::uint64_t j = static_cast<std::uint64_t>(j0 + q);
          const double v = x[j0 + q] * inv;
          std::memcpy(&xb[static_cast<size_t>(q)], &v, sizeof(v));
          for (std::uint64_t c = 0; c < nc; ++c)
            hc[static_cast<size_t>(c * kChunk + q)] = detail::mix64(key_ + (j * nc + c + 1u) * 0x9E3779B97F4A7C15ull);
        }
        for (Index l = 0; l < zeta_; ++l) {
          const std::uint64_t* hl = hc.data() + (l / 4) * kChunk;
          const int sh = static_cast<int>(16 * (l % 4));
          const Index base = b0[static_cast<size_t>(l)];
          const std::uint64_t bsz = static_cast<std::uint64_t>(bs[static_cast<size_t>(l)]);
          for (Index q = 0; q < len; ++q) {
            const std::uint32_t f = static_cast<std::uint32_t>(hl[q] >> sh) & 0xFFFFu;
            const Index r = base + static_cast<Index>((static_cast<std::uint64_t>((f >> 1) & 0x7FFFu) * bsz) >> 15);
            const std::uint64_t bits = xb[static_cast<size_t>(q)] ^ (static_cast<std::uint64_t>(~f & 1u) << 63);
            double term;
            std::memcpy(&term, &bits, sizeof(term));
            out[r] += term;
          }
        }
      }
      return;
    }
    Vec flipped(static_cast<size_t>(n_));
    for (Index i = 0; i < n_; ++i) flipped[static_cast<size_t>(i)] = signs_[static_cast<size_t>(i)] * x[i];
    const bool pow2 = (n_ & (n_ - 1)) == 0;
    if (backend_ != SketchBackend::direct && pow2) {
      Vec transformed(static_cast<size_t>(n_));
      detail::dct2_orthonormal_pow2(flipped.data(), transformed.data(), n_);
      for (Index q = 0; q < s_; ++q) out[q] = scale_ * transformed[static_cast<size_t>(rows_[static_cast<size_t>(q)])];
    } else {
      detail::dct2_selected_direct(flipped.data(), n_, rows_, out);
      for (Index q = 0; q < s_; ++q) out[q] *= scale_;
    }
  }
  Vec apply(const Vec& x) const {
    Vec out(static_cast<size_t>(s_));
    apply(x.data(), static_cast<Index>(x.size()), out.data());
    return out;
  }

 private:
  SketchKind kind_ = SketchKind::identity;
  Index n_ = 0, s_ = 0, zeta_ = 0;
  std::uint64_t seed_ = 0, key_ = 0;
  Vec signs_;
  std::vector<Index> rows_;
  double scale_ = 1.0;
  SketchBackend backend_ = SketchBackend::automatic;
};

// ------------------------------------------------------------- counters ---

struct Counters {  // counters.hpp:12-24
  std::int64_t matvecs = 0, inner_products = 0, sketch_applies = 0;
  Counters& operator+=(const Counters& o) {
    matvecs += o.matvecs;
    inner_products += o.inner_products;
    sketch_applies += o.sketch_applies;
    return *this;
  }
};

// -------------------------------------------------------------- arnoldi ---
// arnoldi.hpp:26-119

struct KrylovState {
  Mat V, H, SV, SAV;
  Index j = 0, t = 0, m_max = 0;
  double r0_norm = 0.0;
  bool breakdown = false;
  Index basis_cols() const { return breakdown ? j : j + 1; }
};

struct StepResult {
  double h_subdiag = 0.0;
  bool breakdown = false;
};

inline KrylovState init_krylov(const Vec& r0, const SketchOperator& S, Index t, Index m_max,
                               Counters* counters = nullptr) {  // arnoldi.hpp:47-72
  if (t < 1) throw std::invalid_argument("init_krylov: truncation window must be at least 1");
  if (m_max < 1) throw std::invalid_argument("init_krylov: m_max must be at least 1");
  if (static_cast<Index>(r0.size()) != S.input_dim())
    throw std::invalid_argument("init_krylov: residual length " + std::to_string(r0.size()) +
                                " does not match sketch input " + std::to_string(S.input_dim()));
  KrylovState st;
  st.t = t;
  st.m_max = m_max;
  st.r0_norm = norm(r0);
  if (counters) ++counters->inner_products;
  if (st.r0_norm == 0.0) throw std::domain_error("init_krylov: zero initial residual (already converged)");
  const Index n = static_cast<Index>(r0.size()), s = S.sketch_dim();
  st.V = Mat(n, m_max + 1);
  st.H = Mat(m_max + 1, m_max);
  st.SV = Mat(s, m_max + 1);
  st.SAV = Mat(s, m_max);
  for (Index i = 0; i < n; ++i) st.V(i, 0) = r0[static_cast<size_t>(i)] / st.r0_norm;
  Vec sr0 = S.apply(r0);
  if (counters) ++counters->sketch_applies;
  for (Index i = 0; i < s; ++i) st.SV(i, 0) = sr0[static_cast<size_t>(i)] / st.r0_norm;
  return st;
}

inline StepResult arnoldi_step(KrylovState& st, const OperatorRef& A, const SketchOperator& S,
                               Counters* counters = nullptr, double breakdown_tol = 1e-14) {
  if (st.breakdown) throw std::logic_error("arnoldi_step: basis already broke down");
  if (st.j >= st.m_max) throw std::logic_error("arnoldi_step: step capacity exhausted");
  const Index j = st.j, n = st.V.rows, s = st.SV.rows;
  Vec w(static_cast<size_t>(n));
  A.apply_raw(st.V.col(j), w.data());  // arnoldi.hpp:87
  if (counters) ++counters->matvecs;
  const double norm_before = norm(w);
  if (counters) ++counters->inner_products;
  const Index i0 = std::max<Index>(0, j - st.t + 1);
  for (Index i = i0; i <= j; ++i) {  // MGS window, arnoldi.hpp:91-97
    const double h = dot(st.V.col(i), w.data(), n);
    if (counters) ++counters->inner_products;
    st.H(i, j) = h;
    const double* vi = st.V.col(i);
    parallel_ranges(n, [&](Index rb, Index re, int) {
      for (Index r = rb; r < re; ++r) w[static_cast<size_t>(r)] -= h * vi[r];
    });
  }
  const double h_next = norm(w);
  if (counters) ++counters->inner_products;
  StepResult res;
  auto fill_sav = [&](Index ncols) {  // arnoldi.hpp:115
    for (Index r = 0; r < s; ++r) {
      double acc = 0.0;
      for (Index q = 0; q < ncols; ++q) acc += st.SV(r, i0 + q) * st.H(i0 + q, j);
      st.SAV(r, j) = acc;
    }
  };
  if (h_next <= breakdown_tol * norm_before) {  // arnoldi.hpp:101-108
    st.H(j + 1, j) = 0.0;
    fill_sav(j - i0 + 1);
    st.breakdown = true;
    st.j = j + 1;
    res.breakdown = true;
    return res;
  }
  st.H(j + 1, j) = h_next;
  parallel_ranges(n, [&](Index rb, Index re, int) {
    for (Index r = rb; r < re; ++r) st.V(r, j + 1) = w[static_cast<size_t>(r)] / h_next;
  });
  Vec sv(static_cast<size_t>(s));
  S.apply(st.V.col(j + 1), n, sv.data());
  if (counters) ++counters->sketch_applies;
  for (Index r = 0; r < s; ++r) st.SV(r, j + 1) = sv[static_cast<size_t>(r)];
  fill_sav(j - i0 + 2);
  st.j = j + 1;
  res.h_subdiag = h_next;
  return res;
}

// -------------------------------------------------------- incremental QR ---
// incremental_qr.hpp:26-162

class IncrementalQR {
 public:
  IncrementalQR(Index rows, Index capacity, double rank_tol = 1e-12) : rank_tol_(rank_tol) {
    if (rows < 1) throw std::invalid_argument("IncrementalQR: rows must be positive");
    if (capacity < 1) capacity = 1;
    m_ = Mat(rows, capacity);
    q_ = Mat(rows, capacity);
    r_ = Mat(capacity, capacity);
  }
  Index rows() const { return m_.rows; }
  Index cols() const { return p_; }
  struct AppendInfo {
    Index column = 0;
    bool rank_deficient = false;
  };
  AppendInfo append(const double* col, Index len) {  // :46-79
    if (len != m_.rows)
      throw std::invalid_argument("IncrementalQR::append: column length " + std::to_string(len) +
                                  " does not match " + std::to_string(m_.rows) + " rows");
    if (p_ == m_.cols) grow();
    const Index p = p_, s = m_.rows;
    std::copy(col, col + s, m_.col(p));
    Vec w(col, col + s), coeffs(static_cast<size_t>(p), 0.0), c(static_cast<size_t>(p));
    for (int pass = 0; pass < 2; ++pass) {
      if (p > 0) {
        for (Index q = 0; q < p; ++q) c[static_cast<size_t>(q)] = dot(q_.col(q), w.data(), s);
        for (Index q = 0; q < p; ++q) {
          const double* qc = q_.col(q);
          for (Index r = 0; r < s; ++r) w[static_cast<size_t>(r)] -= qc[r] * c[static_cast<size_t>(q)];
        }
        for (Index q = 0; q < p; ++q) coeffs[static_cast<size_t>(q)] += c[static_cast<size_t>(q)];
      }
    }
    const double rho = norm(w);
    AppendInfo info;
    info.column = p;
    for (Index q = 0; q < p; ++q) r_(q, p) = coeffs[static_cast<size_t>(q)];
    if (rho <= rank_tol_ * norm(col, s)) {
      info.rank_deficient = true;
      std::fill(q_.col(p), q_.col(p) + s, 0.0);
      r_(p, p) = 0.0;
      state_.push_back(2);
    } else {
      for (Index r = 0; r < s; ++r) q_(r, p) = w[static_cast<size_t>(r)] / rho;
      r_(p, p) = rho;
      state_.push_back(0);
    }
    ++p_;
    return info;
  }
  void exclude(Index column) {
    check(column);
    state_[static_cast<size_t>(column)] = 1;
  }
  bool is_excluded(Index column) const {
    check(column);
    return state_[static_cast<size_t>(column)] == 1;
  }
  struct Solution {
    Vec y;
    double residual_norm = 0.0;
  };
  Solution solve(const Vec& rhs) const {  // :107-135
    if (static_cast<Index>(rhs.size()) != m_.rows)
      throw std::invalid_argument("IncrementalQR::solve: rhs length " + std::to_string(rhs.size()) +
                                  " does not match " + std::to_string(m_.rows) + " rows");
    for (Index i = 0; i < p_; ++i)
      if (state_[static_cast<size_t>(i)] == 2)
        throw std::runtime_error("IncrementalQR::solve: column " + std::to_string(i) +
                                 " is rank-deficient and unresolved; exclude it or rebuild");
    std::vector<Index> used;
    for (Index i = 0; i < p_; ++i)
      if (state_[static_cast<size_t>(i)] == 0) used.push_back(i);
    Solution sol;
    sol.y.assign(static_cast<size_t>(p_), 0.0);
    const Index s = m_.rows;
    if (!used.empty()) {
      Vec c(used.size());
      for (size_t q = 0; q < used.size(); ++q) c[q] = dot(q_.col(used[q]), rhs.data(), s);
      for (size_t q = used.size(); q-- > 0;) {
        double acc = c[q];
        for (size_t q2 = q + 1; q2 < used.size(); ++q2)
          acc -= r_(used[q], used[q2]) * sol.y[static_cast<size_t>(used[q2])];
        sol.y[static_cast<size_t>(used[q])] = acc / r_(used[q], used[q]);
      }
    }
    Vec res(rhs);
    for (Index q = 0; q < p_; ++q) {
      const double yq = sol.y[static_cast<size_t>(q)];
      const double* mc = m_.col(q);
      for (Index r = 0; r < s; ++r) res[static_cast<size_t>(r)] -= mc[r] * yq;
    }
    sol.residual_norm = norm(res);
    return sol;
  }
  const Mat& raw() const { return m_; }
  const Mat& q() const { return q_; }
  const Mat& r() const { return r_; }

 private:
  void check(Index column) const {
    if (column < 0 || column >= p_) throw std::invalid_argument("IncrementalQR: no column " + std::to_string(column));
  }
  void grow() {  // :149-156
    const Index cap = 2 * m_.cols;
    m_.resize_cols(cap);
    q_.resize_cols(cap);
    Mat r2(cap, cap);
    for (Index j = 0; j < p_; ++j)
      for (Index i = 0; i < p_; ++i) r2(i, j) = r_(i, j);
    r_ = std::move(r2);
  }
  Mat m_, q_, r_;
  std::vector<int> state_;  // 0 ok, 1 excluded, 2 unresolved
  double rank_tol_ = 1e-12;
  Index p_ = 0;
};

// -------------------------------------------------------------- recycle ---
// recycle.hpp:31-318, detail/lapack.hpp:25-60

struct RecycleSpace {
  enum class Provenance { empty = 0, fresh, reused, exact_resketch, inexact_carryover };
  Mat U, SU, SAU;
  Provenance provenance = Provenance::empty;
  Index dim() const { return U.cols; }
  bool empty() const { return U.cols == 0; }
  void drop_columns(const std::vector<Index>& cols) {  // recycle.hpp:48-71
    if (cols.empty()) return;
    std::vector<bool> drop(static_cast<size_t>(dim()), false);
    for (const auto c : cols) {
      if (c < 0 || c >= dim()) throw std::invalid_argument("RecycleSpace::drop_columns: no column " + std::to_string(c));
      drop[static_cast<size_t>(c)] = true;
    }
    Index keep = 0;
    for (Index c = 0; c < dim(); ++c)
      if (!drop[static_cast<size_t>(c)]) ++keep;
    Mat u(U.rows, keep), su(SU.rows, keep), sau(SAU.rows, keep);
    Index q = 0;
    for (Index c = 0; c < dim(); ++c) {
      if (drop[static_cast<size_t>(c)]) continue;
      std::copy(U.col(c), U.col(c) + U.rows, u.col(q));
      std::copy(SU.col(c), SU.col(c) + SU.rows, su.col(q));
      std::copy(SAU.col(c), SAU.col(c) + SAU.rows, sau.col(q));
      ++q;
    }
    U = std::move(u);
    SU = std::move(su);
    SAU = std::move(sau);
  }
};

struct HarmonicPencil {
  Mat u, v, m_mat;
  Vec sigma;
  Index rank() const { return static_cast<Index>(sigma.size()); }
};

inline HarmonicPencil truncated_svd(const Mat& SAW, double rank_tol = 1e-12) {  // recycle.hpp:98-110
  if (!(rank_tol >= 0.0)) throw std::invalid_argument("truncated_svd: rank_tol must be >= 0");
  const int m = static_cast<int>(SAW.rows), n = static_cast<int>(SAW.cols);
  const int mn = std::min(m, n);
  Mat a = SAW, u(m, mn), vt(mn, n);
  Vec sv(static_cast<size_t>(mn));
  int info = 0, lwork = -1;
  double wq = 0.0;
  const int ldu = std::max(1, m), ldvt = std::max(1, mn), lda = std::max(1, m);
  if (mn > 0) {
    scipy_dgesvd_("S", "S", &m, &n, a.a.data(), &lda, sv.data(), u.a.data(), &ldu, vt.a.data(), &ldvt, &wq, &lwork, &info, 1, 1);
    lwork = static_cast<int>(wq) + 1;
    Vec work(static_cast<size_t>(lwork));
    scipy_dgesvd_("S", "S", &m, &n, a.a.data(), &lda, sv.data(), u.a.data(), &ldu, vt.a.data(), &ldvt, work.data(), &lwork, &info, 1, 1);
    if (info != 0) throw std::runtime_error("truncated_svd: dgesvd failed with info = " + std::to_string(info));
  }
  Index l = 0;
  const double cutoff = mn > 0 ? rank_tol * sv[0] : 0.0;
  while (l < mn && sv[static_cast<size_t>(l)] > cutoff && sv[static_cast<size_t>(l)] > 0.0) ++l;
  HarmonicPencil p;
  p.u = Mat(m, l);
  p.v = Mat(n, l);
  p.sigma.assign(sv.begin(), sv.begin() + l);
  for (Index c = 0; c < l; ++c) {
    for (Index r = 0; r < m; ++r) p.u(r, c) = u(r, c);
    for (Index r = 0; r < n; ++r) p.v(r, c) = vt(c, r);
  }
  return p;
}

inline void fill_pencil(HarmonicPencil& p, const Mat& SW) {  // recycle.hpp:114-118
  if (SW.rows != p.u.rows || SW.cols != p.v.rows)
    throw std::invalid_argument("fill_pencil: SW dimensions do not match the decomposition");
  const Index l = p.rank(), s = SW.rows, q = SW.cols;
  Mat swv(s, l);
  for (Index c = 0; c < l; ++c)
    for (Index k = 0; k < q; ++k) {
      const double vk = p.v(k, c);
      for (Index r = 0; r < s; ++r) swv(r, c) += SW(r, k) * vk;
    }
  p.m_mat = Mat(l, l);
  for (Index c = 0; c < l; ++c)
    for (Index r = 0; r < l; ++r) p.m_mat(r, c) = dot(p.u.col(r), swv.col(c), s);
}

struct HarmonicPairs {
  Mat coeffs;
  std::vector<std::complex<double>> mu;
  Index k_requested = 0, k_effective = 0;
  bool pair_extended = false, rank_limited = false;
};

inline HarmonicPairs harmonic_pairs(const HarmonicPencil& p, Index k) {  // recycle.hpp:149-218
  if (k < 0) throw std::invalid_argument("harmonic_pairs: k must be nonnegative");
  if (p.m_mat.rows != p.rank() || p.m_mat.cols != p.rank())
    throw std::invalid_argument("harmonic_pairs: pencil is incomplete (m_mat not filled)");
  const Index l = p.rank();
  HarmonicPairs hp;
  hp.k_requested = k;
  if (k > l) {
    k = l;
    hp.rank_limited = true;
  }
  if (k == 0 || l == 0) {
    hp.coeffs = Mat(p.v.rows, 0);
    return hp;
  }
  Mat c(l, l);
  for (Index j = 0; j < l; ++j)
    for (Index i = 0; i < l; ++i) c(i, j) = (1.0 / p.sigma[static_cast<size_t>(i)]) * p.m_mat(i, j);
  // real_schur (detail/lapack.hpp:25-42)
  const int n = static_cast<int>(l);
  Mat q(l, l);
  Vec wr(static_cast<size_t>(l)), wi(static_cast<size_t>(l));
  int sdim = 0, info = 0;
  int lwork = 80 * n + 64;
  Vec work(static_cast<size_t>(lwork));
  scipy_dgees_("V", "N", nullptr, &n, c.a.data(), &n, &sdim, wr.data(), wi.data(), q.a.data(), &n,
               work.data(), &lwork, nullptr, &info, 1, 1);
  if (info != 0) throw std::runtime_error("real_schur: dgees failed with info = " + std::to_string(info));
  std::vector<Index> order(static_cast<size_t>(l));
  std::iota(order.begin(), order.end(), Index{0});
  auto absmu = [&](Index i) { return std::hypot(wr[static_cast<size_t>(i)], wi[static_cast<size_t>(i)]); };
  std::sort(order.begin(), order.end(), [&](Index a, Index b) {
    const double ma = absmu(a), mb = absmu(b);
    if (ma != mb) return ma > mb;
    if (wr[static_cast<size_t>(a)] != wr[static_cast<size_t>(b)]) return wr[static_cast<size_t>(a)] > wr[static_cast<size_t>(b)];
    return a < b;
  });
  std::vector<int> sel(static_cast<size_t>(l), 0);
  for (Index i = 0; i < k; ++i) sel[static_cast<size_t>(order[static_cast<size_t>(i)])] = 1;
  for (Index i = 0; i + 1 < l;) {
    if (wi[static_cast<size_t>(i)] != 0.0) {
      if (sel[static_cast<size_t>(i)] != sel[static_cast<size_t>(i) + 1]) {
        sel[static_cast<size_t>(i)] = sel[static_cast<size_t>(i) + 1] = 1;
        hp.pair_extended = true;
      }
      i += 2;
    } else {
      ++i;
    }
  }
  Index k_eff = 0;
  for (int s : sel) k_eff += s;
  // reorder_schur (detail/lapack.hpp:45-60)
  int mm = 0, liwork = std::max(1, n * n), lw2 = std::max(1, n * n);
  double scond = 0.0, sep = 0.0;
  Vec w2(static_cast<size_t>(lw2));
  std::vector<int> iw(static_cast<size_t>(liwork));
  scipy_dtrsen_("N", "V", sel.data(), &n, c.a.data(), &n, q.a.data(), &n, wr.data(), wi.data(), &mm,
                &scond, &sep, w2.data(), &lw2, iw.data(), &liwork, &info, 1, 1);
  if (info != 0) throw std::runtime_error("reorder_schur: dtrsen failed with info = " + std::to_string(info));
  hp.k_effective = k_eff;
  hp.coeffs = Mat(p.v.rows, k_eff);
  for (Index cc = 0; cc < k_eff; ++cc)
    for (Index kk = 0; kk < l; ++kk) {
      const double qv = q(kk, cc);
      for (Index r = 0; r < p.v.rows; ++r) hp.coeffs(r, cc) += p.v(r, kk) * qv;
    }
  for (Index i = 0; i < k_eff; ++i) hp.mu.emplace_back(wr[static_cast<size_t>(i)], wi[static_cast<size_t>(i)]);
  return hp;
}

inline RecycleSpace update_recycle(const KrylovState& st, const RecycleSpace& cur, Index k,
                                   double rank_tol = 1e-12, Counters* counters = nullptr,
                                   std::vector<std::string>* notes = nullptr) {  // recycle.hpp:226-289
  const Index j = st.j;
  if (j < 1) throw std::invalid_argument("update_recycle: no Arnoldi steps taken");
  const Index kh = cur.dim(), s = st.SV.rows, n = st.V.rows;
  Mat SAW(s, kh + j), SW(s, kh + j);
  for (Index c = 0; c < kh; ++c)
    for (Index r = 0; r < s; ++r) {
      SAW(r, c) = cur.SAU(r, c);
      SW(r, c) = cur.SU(r, c);
    }
  for (Index c = 0; c < j; ++c)
    for (Index r = 0; r < s; ++r) {
      SAW(r, kh + c) = st.SAV(r, c);
      SW(r, kh + c) = st.SV(r, c);
    }
  HarmonicPencil pencil = truncated_svd(SAW, rank_tol);
  fill_pencil(pencil, SW);
  HarmonicPairs hp = harmonic_pairs(pencil, k);
  if (notes) {
    if (hp.rank_limited)
      notes->push_back("deflation space limited to pencil rank " + std::to_string(pencil.rank()) +
                       " (requested " + std::to_string(hp.k_requested) + ")");
    if (hp.pair_extended) notes->push_back("deflation space grew by one to keep a conjugate pair together");
  }
  RecycleSpace next;
  next.provenance = cur.empty() ? RecycleSpace::Provenance::fresh : cur.provenance;
  const Index ke = hp.k_effective;
  if (ke == 0) return next;
  next.U = Mat(n, ke);
  next.SU = Mat(s, ke);
  next.SAU = Mat(s, ke);
  for (Index q = 0; q < ke; ++q) {
    for (Index i = 0; i < j; ++i) {
      const double cf = hp.coeffs(kh + i, q);
      const double* vi = st.V.col(i);
      for (Index r = 0; r < n; ++r) next.U(r, q) += vi[r] * cf;
      for (Index r = 0; r < s; ++r) {
        next.SU(r, q) += st.SV(r, i) * cf;
        next.SAU(r, q) += st.SAV(r, i) * cf;
      }
    }
    for (Index i = 0; i < kh; ++i) {
      const double cf = hp.coeffs(i, q);
      for (Index r = 0; r < n; ++r) next.U(r, q) += cur.U(r, i) * cf;
      for (Index r = 0; r < s; ++r) {
        next.SU(r, q) += cur.SU(r, i) * cf;
        next.SAU(r, q) += cur.SAU(r, i) * cf;
      }
    }
  }
  std::vector<Index> bad;
  for (Index q = 0; q < ke; ++q) {
    const double nrm = norm(next.U.col(q), n);
    if (counters) ++counters->inner_products;
    if (nrm == 0.0 || !std::isfinite(nrm)) {
      bad.push_back(q);
      continue;
    }
    for (Index r = 0; r < n; ++r) next.U(r, q) /= nrm;
    for (Index r = 0; r < s; ++r) {
      next.SU(r, q) /= nrm;
      next.SAU(r, q) /= nrm;
    }
  }
  if (!bad.empty()) {
    next.drop_columns(bad);
    if (notes) notes->push_back("dropped " + std::to_string(bad.size()) + " degenerate deflation columns after the harmonic update");
  }
  if (next.empty()) next.provenance = RecycleSpace::Provenance::empty;
  return next;
}

enum class RefreshMode { exact, inexact };

inline void refresh_for_new_matrix(RecycleSpace& space, const OperatorRef& A, const SketchOperator& S,
                                   RefreshMode mode, Counters* counters = nullptr) {  // recycle.hpp:297-318
  if (space.empty()) return;
  if (space.U.rows != A.cols())
    throw std::invalid_argument("refresh_for_new_matrix: space has " + std::to_string(space.U.rows) +
                                " rows but the operator takes " + std::to_string(A.cols()));
  if (mode == RefreshMode::inexact) {
    space.provenance = RecycleSpace::Provenance::inexact_carryover;
    return;
  }
  Vec au(static_cast<size_t>(A.rows())), sau(static_cast<size_t>(S.sketch_dim()));
  for (Index q = 0; q < space.dim(); ++q) {
    A.apply_raw(space.U.col(q), au.data());
    if (counters) ++counters->matvecs;
    S.apply(au.data(), static_cast<Index>(au.size()), sau.data());
    if (counters) ++counters->sketch_applies;
    for (Index r = 0; r < S.sketch_dim(); ++r) space.SAU(r, q) = sau[static_cast<size_t>(r)];
  }
  space.provenance = RecycleSpace::Provenance::exact_resketch;
}

// --------------------------------------------------------------- report ---
// report.hpp:16-63

enum class SolveStatus { converged = 0, max_restarts = 1, breakdown = 2, diverged = 3 };
struct ResidualSample {
  std::int64_t iteration = 0;
  double value = 0.0;
};
struct CycleStats {
  Index steps = 0;
  double entry_residual = 0, sketched_entry = 0, exit_sres = 0, exit_residual = 0, safety_after = 0,
         basis_cond = 0;
  Index deflation_rank = 0;
};
struct SolveReport {
  SolveStatus status = SolveStatus::max_restarts;
  std::int64_t iterations = 0;
  int cycles = 0;
  double rhs_norm = 0.0;
  double final_relative_residual = std::numeric_limits<double>::quiet_NaN();
  Counters counters;
  std::vector<ResidualSample> sketched_residuals, true_residuals;
  std::vector<CycleStats> cycle_stats;
  std::vector<std::string> notes;
  std::string error;
  double seconds = 0.0;
};

// --------------------------------------------------------------- solver ---
// solver.hpp:33-459

enum class SequenceVariant { reuse = 0, exact = 1, inexact = 2 };

struct SolverConfig {  // solver.hpp:48-79
  Index m = 100, t = 2, k = 20, s = 0;
  double tol = 1e-6, safety_init = 1.4;
  int max_restarts = 10;
  SequenceVariant variant = SequenceVariant::reuse;
  std::uint64_t sketch_seed = 0x5eedULL;
  double rank_tol = 1e-12, breakdown_tol = 1e-14;
  void validate() const {
    if (m < 1) throw std::invalid_argument("SolverConfig: m must be at least 1");
    if (t < 1) throw std::invalid_argument("SolverConfig: t must be at least 1");
    if (k < 0 || k >= m)
      throw std::invalid_argument("SolverConfig: need 0 <= k < m, got k = " + std::to_string(k) +
                                  ", m = " + std::to_string(m));
    if (s < 2 * (m + k))
      throw std::invalid_argument("SolverConfig: sketch size s = " + std::to_string(s) +
                                  " is below 2 (m + k) = " + std::to_string(2 * (m + k)));
    if (!(tol > 0.0 && tol < 1.0)) throw std::invalid_argument("SolverConfig: tol must lie in (0, 1)");
    if (!(safety_init >= 1.0)) throw std::invalid_argument("SolverConfig: safety_init must be at least 1");
    if (max_restarts < 1) throw std::invalid_argument("SolverConfig: max_restarts must be at least 1");
    if (!(rank_tol >= 0.0)) throw std::invalid_argument("SolverConfig: rank_tol must be >= 0");
    if (!(breakdown_tol >= 0.0)) throw std::invalid_argument("SolverConfig: breakdown_tol must be >= 0");
  }
};

struct CycleResult {
  Vec correction, residual;
  double residual_norm = 0, sres = 0, entry_norm = 0, sketched_entry = 0;
  Index steps = 0;
  bool converged = false, breakdown = false;
  double safety = 1.0;
};

inline double matrix_cond_2(const Mat& Min) {
  const int m = static_cast<int>(Min.rows), n = static_cast<int>(Min.cols);
  const int mn = std::min(m, n);
  Mat a = Min;
  Vec sv(static_cast<size_t>(mn));
  int info = 0, lwork = -1, one = 1;
  double wq = 0.0, du = 0.0;
  scipy_dgesvd_("N", "N", &m, &n, a.a.data(), &m, sv.data(), &du, &one, &du, &one, &wq, &lwork, &info, 1, 1);
  lwork = static_cast<int>(wq) + 1;
  Vec work(static_cast<size_t>(lwork));
  scipy_dgesvd_("N", "N", &m, &n, a.a.data(), &m, sv.data(), &du, &one, &du, &one, work.data(), &lwork, &info, 1, 1);
  if (info != 0) throw std::runtime_error("basis_cond: dgesvd failed");
  return sv[static_cast<size_t>(mn - 1)] > 0.0 ? sv[0] / sv[static_cast<size_t>(mn - 1)]
                                               : std::numeric_limits<double>::infinity();
}

inline CycleResult solve_cycle(const OperatorRef& A, const Vec& r0, RecycleSpace& space,
                               const SketchOperator& S, const SolverConfig& cfg, double tol_abs,
                               double safety_in, Counters& counters, SolveReport* report,
                               int cycle_index, std::int64_t iteration_base) {  // solver.hpp:128-254
  CycleResult out;
  out.safety = std::max(1.0, safety_in);
  KrylovState st = init_krylov(r0, S, cfg.t, cfg.m, &counters);
  out.entry_norm = st.r0_norm;
  const Index s = S.sketch_dim(), n = static_cast<Index>(r0.size());
  Vec sr0(static_cast<size_t>(s));
  for (Index r = 0; r < s; ++r) sr0[static_cast<size_t>(r)] = st.SV(r, 0) * st.r0_norm;
  out.sketched_entry = norm(sr0);

  IncrementalQR qr(s, space.dim() + cfg.m, cfg.rank_tol);
  for (;;) {  // solver.hpp:144-159
    std::vector<Index> bad;
    for (Index q = 0; q < space.dim(); ++q)
      if (qr.append(space.SAU.col(q), s).rank_deficient) bad.push_back(q);
    if (bad.empty()) break;
    space.drop_columns(bad);
    if (report)
      report->notes.push_back("cycle " + std::to_string(cycle_index) + ": dropped " + std::to_string(bad.size()) +
                              " deflation columns with rank-deficient sketched images");
    qr = IncrementalQR(s, space.dim() + cfg.m, cfg.rank_tol);
    if (space.empty()) break;
  }
  const Index k_hat = space.dim();
  Vec y;
  double sres = out.sketched_entry;
  bool done = false;
  while (!done && st.j < cfg.m && !st.breakdown) {  // solver.hpp:165-216
    arnoldi_step(st, A, S, &counters, cfg.breakdown_tol);
    const Index j = st.j;
    const auto info = qr.append(st.SAV.col(j - 1), s);
    if (info.rank_deficient) {
      qr.exclude(info.column);
      if (report)
        report->notes.push_back("cycle " + std::to_string(cycle_index) + ", step " + std::to_string(j) +
                                ": sketched basis column rank-deficient; excluded from the least-squares problem");
    }
    const auto sol = qr.solve(sr0);
    y = sol.y;
    sres = sol.residual_norm;
    const std::int64_t global_iter = iteration_base + j;
    if (report) report->sketched_residuals.push_back({global_iter, sres});
    const bool last = j == cfg.m || st.breakdown;
    if (sres < tol_abs / out.safety || last) {
      out.correction.assign(static_cast<size_t>(n), 0.0);
      for (Index i = 0; i < j; ++i) {
        const double yi = y[static_cast<size_t>(k_hat + i)];
        const double* vi = st.V.col(i);
        for (Index r = 0; r < n; ++r) out.correction[static_cast<size_t>(r)] += vi[r] * yi;
      }
      for (Index q = 0; q < k_hat; ++q) {
        const double yq = y[static_cast<size_t>(q)];
        const double* uq = space.U.col(q);
        for (Index r = 0; r < n; ++r) out.correction[static_cast<size_t>(r)] += uq[r] * yq;
      }
      Vec a_corr;
      A.apply(out.correction, a_corr);
      ++counters.matvecs;
      out.residual.resize(static_cast<size_t>(n));
      for (Index r = 0; r < n; ++r)
        out.residual[static_cast<size_t>(r)] = r0[static_cast<size_t>(r)] - a_corr[static_cast<size_t>(r)];
      out.residual_norm = norm(out.residual);
      ++counters.inner_products;
      if (report) report->true_residuals.push_back({global_iter, out.residual_norm});
      if (out.residual_norm < tol_abs) {
        out.converged = true;
        done = true;
      } else {
        if (sres > 0.0) out.safety = std::max(out.safety, out.residual_norm / sres);
        if (last) done = true;
      }
    }
  }
  out.steps = st.j;
  out.sres = sres;
  out.breakdown = st.breakdown;
  if (report) {
    CycleStats cs;
    cs.steps = st.j;
    cs.entry_residual = out.entry_norm;
    cs.sketched_entry = out.sketched_entry;
    cs.exit_sres = sres;
    cs.exit_residual = out.residual_norm;
    cs.safety_after = out.safety;
    if (st.j >= 1 && !st.breakdown) {
      Mat svb(s, st.j + 1);
      std::copy(st.SV.a.begin(), st.SV.a.begin() + s * (st.j + 1), svb.a.begin());
      cs.basis_cond = matrix_cond_2(svb);
    }
    report->cycle_stats.push_back(cs);
  }
  if (cfg.k > 0 && st.j >= 1) {  // solver.hpp:242-252
    std::vector<std::string> notes;
    space = update_recycle(st, space, cfg.k, cfg.rank_tol, &counters, &notes);
    if (report && !report->cycle_stats.empty()) report->cycle_stats.back().deflation_rank = space.dim();
    if (report)
      for (auto& nn : notes) report->notes.push_back("cycle " + std::to_string(cycle_index) + ": " + nn);
  } else if (cfg.k == 0) {
    space = RecycleSpace{};
  }
  return out;
}

struct SolveResult {
  Vec x;
  SolveReport report;
  RecycleSpace space;
};

inline SolveResult solve(const OperatorRef& A, const Vec& b, const SolverConfig& cfg, RecycleSpace space = {},
                         const SketchOperator* sketch = nullptr, const Vec* x0 = nullptr) {  // solver.hpp:269-365
  cfg.validate();
  if (A.rows() != A.cols())
    throw std::invalid_argument("solve: operator must be square, got " + std::to_string(A.rows()) + " x " +
                                std::to_string(A.cols()));
  if (static_cast<Index>(b.size()) != A.rows())
    throw std::invalid_argument("solve: rhs length " + std::to_string(b.size()) +
                                " does not match operator size " + std::to_string(A.rows()));
  if (x0 && x0->size() != b.size())
    throw std::invalid_argument("solve: x0 length " + std::to_string(x0->size()) +
                                " does not match rhs length " + std::to_string(b.size()));
  std::optional<SketchOperator> own;
  if (!sketch) {
    own = SketchOperator::subsampled_dct(A.rows(), cfg.s, cfg.sketch_seed);
    sketch = &*own;
  }
  if (sketch->input_dim() != A.rows())
    throw std::invalid_argument("solve: sketch takes length " + std::to_string(sketch->input_dim()) +
                                " but the operator is " + std::to_string(A.rows()) + " x " + std::to_string(A.cols()));
  if (sketch->sketch_dim() < 2 * (cfg.m + cfg.k))
    throw std::invalid_argument("solve: sketch size " + std::to_string(sketch->sketch_dim()) +
                                " is below 2 (m + k) = " + std::to_string(2 * (cfg.m + cfg.k)));
  if (!space.empty() && space.U.rows != A.rows())
    throw std::invalid_argument("solve: recycle space has " + std::to_string(space.U.rows) +
                                " rows but the operator is " + std::to_string(A.rows()) + " x " + std::to_string(A.cols()));
  const auto t0 = std::chrono::steady_clock::now();
  SolveResult result;
  SolveReport& rep = result.report;
  rep.rhs_norm = norm(b);
  ++rep.counters.inner_products;
  const double tol_abs = cfg.tol * rep.rhs_norm;
  const Index n = static_cast<Index>(b.size());
  result.x = x0 ? *x0 : Vec(static_cast<size_t>(n), 0.0);
  Vec r;
  bool x0_nonzero = false;
  if (x0)
    for (double v : *x0)
      if (v != 0.0) x0_nonzero = true;
  if (x0_nonzero) {
    Vec ax;
    A.apply(*x0, ax);
    ++rep.counters.matvecs;
    r.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) r[static_cast<size_t>(i)] = b[static_cast<size_t>(i)] - ax[static_cast<size_t>(i)];
  } else {
    r = b;
  }
  double safety = cfg.safety_init, res_norm = std::numeric_limits<double>::quiet_NaN();
  bool have = false;
  for (int cycle = 1; cycle <= cfg.max_restarts; ++cycle) {
    CycleResult cr;
    try {
      cr = solve_cycle(A, r, space, *sketch, cfg, tol_abs, safety, rep.counters, &rep, cycle, rep.iterations);
    } catch (const std::domain_error&) {
      rep.status = SolveStatus::converged;
      res_norm = 0.0;
      have = true;
      break;
    }
    rep.cycles = cycle;
    rep.iterations += cr.steps;
    safety = cr.safety;
    for (Index i = 0; i < n && !cr.correction.empty(); ++i)
      result.x[static_cast<size_t>(i)] += cr.correction[static_cast<size_t>(i)];
    r = cr.residual;
    res_norm = cr.residual_norm;
    have = true;
    if (cr.converged) {
      rep.status = SolveStatus::converged;
      break;
    }
    if (cr.breakdown) {
      rep.status = SolveStatus::breakdown;
      rep.notes.push_back("cycle " + std::to_string(cycle) + ": basis exhausted before reaching the target");
      break;
    }
    if (cr.steps == cfg.m && cr.sres > 0.99 * cr.sketched_entry) {
      rep.status = SolveStatus::diverged;
      rep.notes.push_back("cycle " + std::to_string(cycle) + ": sketched residual improved by less than 1% over a full cycle");
      break;
    }
    if (cycle == cfg.max_restarts) rep.status = SolveStatus::max_restarts;
  }
  if (have) rep.final_relative_residual = rep.rhs_norm > 0.0 ? res_norm / rep.rhs_norm : res_norm;
  result.space = std::move(space);
  rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

struct ProblemInstance {
  std::shared_ptr<const SparseMatrix> matrix;
  Vec rhs, x0;
  double target_tol = 0.0;
};
struct ProblemSequence {
  std::vector<ProblemInstance> problems;
  bool shared_matrix = false;
};
struct SequenceResult {
  std::vector<SolveReport> reports;
  std::vector<Vec> solutions;
  RecycleSpace space;
};

inline SequenceResult solve_sequence(const ProblemSequence& seq, const SolverConfig& cfg,
                                     const SketchOperator* sketch = nullptr, RecycleSpace initial = {}) {
  // solver.hpp:385-459
  cfg.validate();
  if (seq.problems.empty()) return {};
  const Index n = seq.problems.front().matrix->rows();
  std::optional<SketchOperator> own;
  if (!sketch) {
    own = SketchOperator::subsampled_dct(n, cfg.s, cfg.sketch_seed);
    sketch = &*own;
  }
  SequenceResult result;
  result.space = std::move(initial);
  const SparseMatrix* prev = nullptr;
  for (size_t i = 0; i < seq.problems.size(); ++i) {
    const ProblemInstance& prob = seq.problems[i];
    SolverConfig local = cfg;
    if (prob.target_tol > 0.0) local.tol = prob.target_tol;
    Counters pre;
    try {
      if (!prob.matrix) throw std::invalid_argument("solve_sequence: problem " + std::to_string(i) + " has no matrix");
      if (prob.matrix->rows() != n || prob.matrix->cols() != n)
        throw std::invalid_argument("solve_sequence: problem " + std::to_string(i) + " is " +
                                    std::to_string(prob.matrix->rows()) + " x " + std::to_string(prob.matrix->cols()) +
                                    " but the sequence runs at size " + std::to_string(n));
      const bool changed = prev != nullptr && prev != prob.matrix.get() && !seq.shared_matrix;
      std::string note;
      OperatorRef op(*prob.matrix);
      if (changed && !result.space.empty()) {
        switch (local.variant) {
          case SequenceVariant::exact: refresh_for_new_matrix(result.space, op, *sketch, RefreshMode::exact, &pre); break;
          case SequenceVariant::inexact: refresh_for_new_matrix(result.space, op, *sketch, RefreshMode::inexact, &pre); break;
          case SequenceVariant::reuse:
            refresh_for_new_matrix(result.space, op, *sketch, RefreshMode::inexact, &pre);
            note = "matrix changed under variant=reuse; sketched image carried unrefreshed";
            break;
        }
      } else if (prev != nullptr && !result.space.empty()) {
        result.space.provenance = RecycleSpace::Provenance::reused;
      }
      SolveResult sr = solve(op, prob.rhs, local, std::move(result.space), sketch, prob.x0.empty() ? nullptr : &prob.x0);
      result.space = std::move(sr.space);
      sr.report.counters += pre;
      if (!note.empty()) sr.report.notes.push_back(note);
      result.reports.push_back(std::move(sr.report));
      result.solutions.push_back(std::move(sr.x));
    } catch (const std::exception& e) {
      SolveReport rep;
      rep.error = e.what();
      rep.counters = pre;
      rep.notes.push_back("system " + std::to_string(i) + " aborted: " + e.what());
      result.reports.push_back(std::move(rep));
      result.solutions.emplace_back();
    }
    prev = prob.matrix.get();
  }
  return result;
}

// ------------------------------------------------------------- baseline ---
// Classical restarted GMRES, the reference's comparison point
// (baseline.hpp:51-216): full modified Gram-Schmidt against the whole basis,
// Givens rotations on the Hessenberg column, one verification product per
// cycle. Statuses / counters / notes as the reference.

struct BaselineConfig {
  Index m = 100;
  double tol = 1e-6;
  int max_restarts = 10;
  double breakdown_tol = 1e-14;
};

inline SolveResult baseline_gmres(const OperatorRef& A, const Vec& b, const BaselineConfig& cfg,
                                  const Vec* x0 = nullptr) {
  if (cfg.m < 1) throw std::invalid_argument("BaselineConfig: m must be at least 1");
  if (!(cfg.tol > 0.0 && cfg.tol < 1.0)) throw std::invalid_argument("BaselineConfig: tol must lie in (0, 1)");
  if (cfg.max_restarts < 1) throw std::invalid_argument("BaselineConfig: max_restarts must be at least 1");
  if (!(cfg.breakdown_tol >= 0.0)) throw std::invalid_argument("BaselineConfig: breakdown_tol must be >= 0");
  const Index n = static_cast<Index>(b.size());
  if (A.rows() != A.cols())
    throw std::invalid_argument("baseline_gmres: operator must be square, got " + std::to_string(A.rows()) + " x " +
                                std::to_string(A.cols()));
  if (n != A.rows())
    throw std::invalid_argument("baseline_gmres: rhs length " + std::to_string(n) + " does not match operator size " +
                                std::to_string(A.rows()));
  if (x0 && static_cast<Index>(x0->size()) != n)
    throw std::invalid_argument("baseline_gmres: x0 length " + std::to_string(x0->size()) +
                                " does not match rhs length " + std::to_string(n));
  const auto t0 = std::chrono::steady_clock::now();
  SolveResult out;
  SolveReport& rep = out.report;
  rep.rhs_norm = norm(b.data(), n);
  ++rep.counters.inner_products;
  const double tol_abs = cfg.tol * rep.rhs_norm;
  out.x = x0 ? *x0 : Vec(static_cast<size_t>(n), 0.0);
  Vec r = b;
  bool x0_nonzero = false;
  if (x0)
    for (double v : *x0) x0_nonzero = x0_nonzero || v != 0.0;
  if (x0_nonzero) {
    Vec ax(static_cast<size_t>(n));
    A.apply_raw(x0->data(), ax.data());
    ++rep.counters.matvecs;
    for (Index i = 0; i < n; ++i) r[static_cast<size_t>(i)] -= ax[static_cast<size_t>(i)];
  }
  const Index m = cfg.m;
  std::vector<Vec> V(static_cast<size_t>(m + 1), Vec(static_cast<size_t>(n)));
  Mat H(m + 1, m), R(m + 1, m);
  Vec g(static_cast<size_t>(m + 1)), cs(static_cast<size_t>(m)), sn(static_cast<size_t>(m)), w(static_cast<size_t>(n));
  double res_norm = std::numeric_limits<double>::quiet_NaN();
  bool have = false;
  for (int cycle = 1; cycle <= cfg.max_restarts; ++cycle) {
    const double beta = norm(r.data(), n);
    ++rep.counters.inner_products;
    if (beta == 0.0) {
      rep.status = SolveStatus::converged;
      res_norm = 0.0;
      have = true;
      break;
    }
    rep.cycles = cycle;
    for (Index i = 0; i < n; ++i) V[0][static_cast<size_t>(i)] = r[static_cast<size_t>(i)] / beta;
    H = Mat(m + 1, m);
    R = Mat(m + 1, m);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    Index p = 0;
    bool breakdown = false;
    double est = beta;
    while (p < m) {
      const Index q = p;
      A.apply_raw(V[static_cast<size_t>(q)].data(), w.data());
      ++rep.counters.matvecs;
      for (Index i = 0; i <= q; ++i) {  // modified Gram-Schmidt over the whole basis
        const double h = dot(V[static_cast<size_t>(i)].data(), w.data(), n);
        ++rep.counters.inner_products;
        H(i, q) = h;
        for (Index e = 0; e < n; ++e) w[static_cast<size_t>(e)] -= h * V[static_cast<size_t>(i)][static_cast<size_t>(e)];
      }
      const double h_next = norm(w.data(), n);
      ++rep.counters.inner_products;
      H(q + 1, q) = h_next;
      double cn = 0.0;
      for (Index i = 0; i <= q + 1; ++i) cn += H(i, q) * H(i, q);
      cn = std::sqrt(cn);
      if (h_next <= cfg.breakdown_tol * cn) {
        H(q + 1, q) = 0.0;
        breakdown = true;
      } else {
        for (Index e = 0; e < n; ++e) V[static_cast<size_t>(q + 1)][static_cast<size_t>(e)] = w[static_cast<size_t>(e)] / h_next;
      }
      for (Index i = 0; i <= q + 1; ++i) R(i, q) = H(i, q);
      for (Index i = 0; i < q; ++i) {  // earlier rotations
        const double a = R(i, q), bb = R(i + 1, q);
        R(i, q) = cs[static_cast<size_t>(i)] * a + sn[static_cast<size_t>(i)] * bb;
        R(i + 1, q) = -sn[static_cast<size_t>(i)] * a + cs[static_cast<size_t>(i)] * bb;
      }
      const double a = R(q, q), bb = R(q + 1, q), rr = std::hypot(a, bb);
      const double c = rr > 0.0 ? a / rr : 1.0, sg = rr > 0.0 ? bb / rr : 0.0;
      cs[static_cast<size_t>(q)] = c;
      sn[static_cast<size_t>(q)] = sg;
      R(q, q) = rr;
      R(q + 1, q) = 0.0;
      const double ga = g[static_cast<size_t>(q)];
      g[static_cast<size_t>(q)] = c * ga;
      g[static_cast<size_t>(q + 1)] = -sg * ga;
      est = std::abs(g[static_cast<size_t>(q + 1)]);
      ++p;
      rep.sketched_residuals.push_back({rep.iterations + p, est});
      if (est < tol_abs || breakdown) break;
    }
    // cycle iterate: R y = g (dense least squares on H if a pivot vanished)
    Vec y(static_cast<size_t>(p), 0.0);
    bool diag_ok = true;
    for (Index i = 0; i < p; ++i) diag_ok = diag_ok && R(i, i) != 0.0;
    if (diag_ok) {
      for (Index i = p - 1; i >= 0; --i) {
        double acc = g[static_cast<size_t>(i)];
        for (Index k2 = i + 1; k2 < p; ++k2) acc -= R(i, k2) * y[static_cast<size_t>(k2)];
        y[static_cast<size_t>(i)] = acc / R(i, i);
      }
    } else {
      Mat Hp(p + 1, p);
      for (Index jj = 0; jj < p; ++jj)
        for (Index i = 0; i <= p; ++i) Hp(i, jj) = H(i, jj);
      Vec rhs(static_cast<size_t>(p + 1), 0.0);
      rhs[0] = beta;
      y = detail::least_squares(Hp, rhs);
    }
    Vec corr(static_cast<size_t>(n), 0.0);
    for (Index jj = 0; jj < p; ++jj)
      for (Index e = 0; e < n; ++e)
        corr[static_cast<size_t>(e)] += V[static_cast<size_t>(jj)][static_cast<size_t>(e)] * y[static_cast<size_t>(jj)];
    for (Index e = 0; e < n; ++e) out.x[static_cast<size_t>(e)] += corr[static_cast<size_t>(e)];
    Vec acorr(static_cast<size_t>(n));
    A.apply_raw(corr.data(), acorr.data());
    ++rep.counters.matvecs;
    for (Index e = 0; e < n; ++e) r[static_cast<size_t>(e)] -= acorr[static_cast<size_t>(e)];
    res_norm = norm(r.data(), n);
    ++rep.counters.inner_products;
    have = true;
    rep.iterations += p;
    rep.true_residuals.push_back({rep.iterations, res_norm});
    CycleStats st;
    st.steps = p;
    st.entry_residual = beta;
    st.sketched_entry = beta;
    st.exit_sres = est;
    st.exit_residual = res_norm;
    st.safety_after = 1.0;
    rep.cycle_stats.push_back(st);
    if (res_norm < tol_abs) {
      rep.status = SolveStatus::converged;
      break;
    }
    if (breakdown) {
      rep.status = SolveStatus::breakdown;
      rep.notes.push_back("cycle " + std::to_string(cycle) + ": basis exhausted before reaching the target");
      break;
    }
    if (p == m && est > 0.99 * beta) {
      rep.status = SolveStatus::diverged;
      rep.notes.push_back("cycle " + std::to_string(cycle) +
                          ": residual estimate improved by less than 1% over a full cycle");
      break;
    }
    if (cycle == cfg.max_restarts) rep.status = SolveStatus::max_restarts;
  }
  if (have) rep.final_relative_residual = rep.rhs_norm > 0.0 ? res_norm / rep.rhs_norm : res_norm;
  rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

}  // namespace oracle
