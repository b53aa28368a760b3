// Host-side small dense algebra of the hot path: the incremental sketched
// least-squares QR (incremental_qr.hpp:26-162) and the harmonic-Ritz pencil
// selection (recycle.hpp:98-218, detail/lapack.hpp:25-60). These operate on
// s x (k+m) sketches (s <= a few hundred) and stay on the host, as in the
// reference; the BLAS-2 kernels go through OpenBLAS (CPU-dispatched) so the
// per-step host work hides under the device step.
#pragma once

#include "common.hpp"

#include <complex>
#include <vector>

extern "C" {
void scipy_dgemv_(const char* trans, const int* m, const int* n, const double* alpha, const double* a, const int* lda,
                  const double* x, const int* incx, const double* beta, double* y, const int* incy, size_t);
void scipy_dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k, const double* alpha,
                  const double* a, const int* lda, const double* b, const int* ldb, const double* beta, double* c,
                  const int* ldc, size_t, size_t);
double scipy_ddot_(const int* n, const double* x, const int* incx, const double* y, const int* incy);
double scipy_dnrm2_(const int* n, const double* x, const int* incx);
void scipy_dgees_(const char* jobvs, const char* sort, void* select, const int* n, double* a, const int* lda, int* sdim,
                  double* wr, double* wi, double* vs, const int* ldvs, double* work, const int* lwork, int* bwork,
                  int* info, size_t, size_t);
void scipy_dtrsen_(const char* job, const char* compq, const int* select, const int* n, double* t, const int* ldt,
                   double* q, const int* ldq, double* wr, double* wi, int* m, double* s, double* sep, double* work,
                   const int* lwork, int* iwork, const int* liwork, int* info, size_t, size_t);
void scipy_dgesvd_(const char* jobu, const char* jobvt, const int* m, const int* n, double* a, const int* lda, double* s,
                   double* u, const int* ldu, double* vt, const int* ldvt, double* work, const int* lwork, int* info,
                   size_t, size_t);
void scipy_dgesdd_(const char* jobz, const int* m, const int* n, double* a, const int* lda, double* s, double* u,
                   const int* ldu, double* vt, const int* ldvt, double* work, const int* lwork, int* iwork, int* info,
                   size_t);
void scipy_dtrcon_(const char* norm, const char* uplo, const char* diag, const int* n, const double* a, const int* lda,
                   double* rcond, double* work, int* iwork, int* info, size_t, size_t, size_t);
void scipy_dtrsm_(const char* side, const char* uplo, const char* transa, const char* diag, const int* m, const int* n,
                  const double* alpha, const double* a, const int* lda, double* b, const int* ldb, size_t, size_t, size_t,
                  size_t);
void scipy_openblas_set_num_threads(int);
}

namespace sdr {

/// Column-major host matrix.
struct HMat {
  i64 rows = 0, cols = 0;
  std::vector<double> a;
  HMat() = default;
  HMat(i64 r, i64 c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(i64 i, i64 j) { return a[static_cast<size_t>(i + j * rows)]; }
  double operator()(i64 i, i64 j) const { return a[static_cast<size_t>(i + j * rows)]; }
  double* col(i64 j) { return a.data() + j * rows; }
  const double* col(i64 j) const { return a.data() + j * rows; }
};

double hdot(const double* x, const double* y, i64 n);
double hnorm(const double* x, i64 n);
/// y = beta*y + alpha*op(A) x, A rows x cols column-major with leading dim lda.
void hgemv(bool trans, i64 rows, i64 cols, double alpha, const double* A, i64 lda, const double* x, double beta, double* y);

/// IncrementalQR with the reference's semantics: two-pass classical
/// Gram–Schmidt append, relative rank test rho <= rank_tol * ||col|| ->
/// rank-deficient sentinel, exclusion, and a least-squares solve whose
/// residual is evaluated against the raw appended columns.
class HostQR {
 public:
  HostQR(i64 rows, i64 capacity, double rank_tol);
  i64 rows() const { return rows_; }
  i64 cols() const { return p_; }
  struct AppendInfo {
    i64 column = 0;
    bool rank_deficient = false;
  };
  AppendInfo append(const double* col, i64 len);
  void exclude(i64 column);
  /// Solve min ||rhs - M y||; y has cols() entries. Q^T rhs per column is
  /// cached while rhs stays the same buffer contents (set via set_rhs).
  double solve(const double* rhs, i64 len, double* y);
  void set_rhs(const double* rhs, i64 len);
  double solve_cached(double* y);
  void factors(double* Q, double* R) const;
  /// No column rank-deficient or excluded: M = Q R holds for all columns.
  bool clean() const;

 private:
  void grow();
  void check(i64 column) const;
  i64 rows_, cap_, p_ = 0;
  double rank_tol_;
  std::vector<double> m_, q_, r_;  // rows x cap, rows x cap, cap x cap
  std::vector<int> state_;         // 0 ok, 1 excluded, 2 unresolved
  std::vector<double> rhs_, qtb_;
  std::vector<char> qtb_valid_;
  std::vector<double> ws_, wc_, wcoef_;  // append / solve scratch
};

/// truncated_svd + fill_pencil + harmonic_pairs. coeffs: p x k_eff.
struct Harmonic {
  i64 rank = 0, k_requested = 0, k_eff = 0;
  bool pair_extended = false, rank_limited = false;
  HMat coeffs;
  std::vector<std::complex<double>> mu;
  double svd_ms = 0.0, schur_ms = 0.0, rest_ms = 0.0;  // host cost breakdown
};
/// With Q (s x p, orthonormal) and R (p x p) such that SAW = Q R (the cycle's
/// least-squares factorization), the SVD is taken of R: SAW = (Q U_R) S V^T.
Harmonic harmonic_extract(const HMat& SAW, const HMat& SW, i64 k, double rank_tol, const HMat* Q = nullptr,
                          const HMat* R = nullptr);

/// sigma_max / sigma_min of a small dense block (basis_cond, solver.hpp:230-236).
double cond2(const HMat& A);

void init_host_blas();

}  // namespace sdr
