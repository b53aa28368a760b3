#include "host_linalg.hpp"

#include <chrono>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

namespace sdr {

void init_host_blas() {
  static bool done = false;
  if (!done) {
    scipy_openblas_set_num_threads(1);  // deterministic, no oversubscription
    done = true;
  }
}

double hdot(const double* x, const double* y, i64 n) {
  const int nn = static_cast<int>(n), one = 1;
  return n > 0 ? scipy_ddot_(&nn, x, &one, y, &one) : 0.0;
}

double hnorm(const double* x, i64 n) { return std::sqrt(hdot(x, x, n)); }

void hgemv(bool trans, i64 rows, i64 cols, double alpha, const double* A, i64 lda, const double* x, double beta,
           double* y) {
  if (rows == 0 || cols == 0) {
    const i64 ny = trans ? cols : rows;
    for (i64 i = 0; i < ny; ++i) y[i] = beta == 0.0 ? 0.0 : beta * y[i];
    return;
  }
  const int m = static_cast<int>(rows), n = static_cast<int>(cols), ld = static_cast<int>(lda), one = 1;
  scipy_dgemv_(trans ? "T" : "N", &m, &n, &alpha, A, &ld, x, &one, &beta, y, &one, 1);
}

HostQR::HostQR(i64 rows, i64 capacity, double rank_tol) : rows_(rows), cap_(std::max<i64>(capacity, 1)), rank_tol_(rank_tol) {
  if (rows < 1) throw invalid("IncrementalQR: rows must be positive");
  m_.assign(static_cast<size_t>(rows_ * cap_), 0.0);
  q_.assign(static_cast<size_t>(rows_ * cap_), 0.0);
  r_.assign(static_cast<size_t>(cap_ * cap_), 0.0);
}

void HostQR::grow() {  // incremental_qr.hpp:149-156
  const i64 cap = 2 * cap_;
  m_.resize(static_cast<size_t>(rows_ * cap), 0.0);
  q_.resize(static_cast<size_t>(rows_ * cap), 0.0);
  std::vector<double> r2(static_cast<size_t>(cap * cap), 0.0);
  for (i64 j = 0; j < p_; ++j)
    for (i64 i = 0; i < p_; ++i) r2[static_cast<size_t>(i + j * cap)] = r_[static_cast<size_t>(i + j * cap_)];
  r_.swap(r2);
  cap_ = cap;
}

HostQR::AppendInfo HostQR::append(const double* col, i64 len) {  // incremental_qr.hpp:46-79
  if (len != rows_)
    throw invalid("IncrementalQR::append: column length " + std::to_string(len) + " does not match " +
                  std::to_string(rows_) + " rows");
  if (p_ == cap_) grow();
  const i64 p = p_, s = rows_;
  std::copy(col, col + s, m_.data() + p * s);
  // scratch reused across appends (one column per Arnoldi step on the host)
  std::vector<double>& w = ws_;
  std::vector<double>& c = wc_;
  std::vector<double>& coeffs = wcoef_;
  w.assign(col, col + s);
  c.resize(static_cast<size_t>(p));
  coeffs.assign(static_cast<size_t>(p), 0.0);
  for (int pass = 0; pass < 2; ++pass) {
    if (p > 0) {
      hgemv(true, s, p, 1.0, q_.data(), s, w.data(), 0.0, c.data());
      hgemv(false, s, p, -1.0, q_.data(), s, c.data(), 1.0, w.data());
      for (i64 q = 0; q < p; ++q) coeffs[static_cast<size_t>(q)] += c[static_cast<size_t>(q)];
    }
  }
  const double rho = hnorm(w.data(), s);
  AppendInfo info;
  info.column = p;
  for (i64 q = 0; q < p; ++q) r_[static_cast<size_t>(q + p * cap_)] = coeffs[static_cast<size_t>(q)];
  double* qc = q_.data() + p * s;
  if (rho <= rank_tol_ * hnorm(col, s)) {
    info.rank_deficient = true;
    std::fill(qc, qc + s, 0.0);
    r_[static_cast<size_t>(p + p * cap_)] = 0.0;
    state_.push_back(2);
  } else {
    for (i64 r = 0; r < s; ++r) qc[r] = w[static_cast<size_t>(r)] / rho;
    r_[static_cast<size_t>(p + p * cap_)] = rho;
    state_.push_back(0);
  }
  ++p_;
  qtb_valid_.push_back(0);
  qtb_.push_back(0.0);
  return info;
}

void HostQR::check(i64 column) const {
  if (column < 0 || column >= p_) throw invalid("IncrementalQR: no column " + std::to_string(column));
}

void HostQR::exclude(i64 column) {
  check(column);
  state_[static_cast<size_t>(column)] = 1;
}

void HostQR::set_rhs(const double* rhs, i64 len) {
  if (len != rows_)
    throw invalid("IncrementalQR::solve: rhs length " + std::to_string(len) + " does not match " +
                  std::to_string(rows_) + " rows");
  rhs_.assign(rhs, rhs + len);
  std::fill(qtb_valid_.begin(), qtb_valid_.end(), 0);
}

double HostQR::solve(const double* rhs, i64 len, double* y) {
  set_rhs(rhs, len);
  return solve_cached(y);
}

double HostQR::solve_cached(double* y) {  // incremental_qr.hpp:107-135
  for (i64 i = 0; i < p_; ++i)
    if (state_[static_cast<size_t>(i)] == 2)
      throw runtime("IncrementalQR::solve: column " + std::to_string(i) +
                    " is rank-deficient and unresolved; exclude it or rebuild");
  const i64 s = rows_;
  std::vector<i64> used;
  used.reserve(static_cast<size_t>(p_));
  for (i64 i = 0; i < p_; ++i)
    if (state_[static_cast<size_t>(i)] == 0) used.push_back(i);
  std::fill(y, y + p_, 0.0);
  for (size_t q = 0; q < used.size(); ++q) {
    const i64 c = used[q];
    if (!qtb_valid_[static_cast<size_t>(c)]) {
      qtb_[static_cast<size_t>(c)] = hdot(q_.data() + c * s, rhs_.data(), s);
      qtb_valid_[static_cast<size_t>(c)] = 1;
    }
  }
  // back substitution by columns (contiguous reads of R)
  std::vector<double>& acc = wc_;
  acc.resize(used.size());
  for (size_t q = 0; q < used.size(); ++q) acc[q] = qtb_[static_cast<size_t>(used[q])];
  for (size_t q = used.size(); q-- > 0;) {
    const i64 uq = used[q];
    const double yq = acc[q] / r_[static_cast<size_t>(uq + uq * cap_)];
    y[uq] = yq;
    const double* rcol = r_.data() + uq * cap_;
    for (size_t q2 = 0; q2 < q; ++q2) acc[q2] -= rcol[used[q2]] * yq;
  }
  std::vector<double>& res = ws_;
  res.assign(rhs_.begin(), rhs_.end());
  hgemv(false, s, p_, -1.0, m_.data(), s, y, 1.0, res.data());
  return hnorm(res.data(), s);
}

bool HostQR::clean() const {
  for (int st : state_)
    if (st != 0) return false;
  return true;
}

void HostQR::factors(double* Q, double* R) const {
  if (Q) std::copy(q_.begin(), q_.begin() + rows_ * p_, Q);
  if (R)
    for (i64 j = 0; j < p_; ++j)
      for (i64 i = 0; i < p_; ++i) R[i + j * p_] = r_[static_cast<size_t>(i + j * cap_)];
}

// ------------------------------------------------------------------ harmonic

namespace {

void thin_svd(const HMat& A, std::vector<double>& sv, HMat* U, HMat* V) {
  const int m = static_cast<int>(A.rows), n = static_cast<int>(A.cols), mn = std::min(m, n);
  sv.assign(static_cast<size_t>(mn), 0.0);
  if (mn == 0) {
    if (U) *U = HMat(m, 0);
    if (V) *V = HMat(n, 0);
    return;
  }
  HMat a = A, u(m, mn), vt(mn, n);
  const bool vec = U || V;
  // divide-and-conquer SVD (the reference uses Eigen::JacobiSVD; singular
  // values and subspaces agree to rounding, singular-vector signs cancel in
  // the pencil C = diag(1/sigma) u^T SW v)
  const char* job = vec ? "S" : "N";
  int info = 0, lwork = -1, lda = std::max(1, m), ldu = vec ? std::max(1, m) : 1, ldvt = vec ? std::max(1, mn) : 1;
  std::vector<int> iwork(static_cast<size_t>(8 * mn));
  double wq = 0.0;
  scipy_dgesdd_(job, &m, &n, a.a.data(), &lda, sv.data(), u.a.data(), &ldu, vt.a.data(), &ldvt, &wq, &lwork,
                iwork.data(), &info, 1);
  lwork = static_cast<int>(wq) + 1;
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dgesdd_(job, &m, &n, a.a.data(), &lda, sv.data(), u.a.data(), &ldu, vt.a.data(), &ldvt, work.data(), &lwork,
                iwork.data(), &info, 1);
  if (info != 0) throw runtime("truncated_svd: dgesdd failed with info = " + std::to_string(info));
  if (U) *U = u;
  if (V) {
    *V = HMat(n, mn);
    for (i64 c = 0; c < mn; ++c)
      for (i64 r = 0; r < n; ++r) (*V)(r, c) = vt(c, r);
  }
}

}  // namespace

double cond2(const HMat& A) {
  std::vector<double> sv;
  thin_svd(A, sv, nullptr, nullptr);
  if (sv.empty()) return 1.0;
  return sv.back() > 0.0 ? sv.front() / sv.back() : std::numeric_limits<double>::infinity();
}

Harmonic harmonic_extract(const HMat& SAW, const HMat& SW, i64 k, double rank_tol, const HMat* Qf, const HMat* Rf) {
  if (!(rank_tol >= 0.0)) throw invalid("truncated_svd: rank_tol must be >= 0");
  if (k < 0) throw invalid("harmonic_pairs: k must be nonnegative");
  if (SW.rows != SAW.rows || SW.cols != SAW.cols) throw invalid("fill_pencil: SW dimensions do not match the decomposition");
  std::vector<double> sv;
  HMat U, V;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const bool have_qr =
      Qf && Rf && Qf->rows == SAW.rows && Qf->cols == SAW.cols && Rf->rows == SAW.cols && Rf->cols == SAW.cols;
  // Fast path. With SAW = Q R and R well conditioned, every singular value
  // of SAW lies far above rank_tol·sigma_1, so the truncated SVD keeps all p
  // directions (l = p) and the pencil C = Sigma^{-1} U^T SW V is the
  // orthogonal similarity V^T M V of M = R^{-1} Q^T SW. The Schur form of M
  // then carries the same eigenvalues, and its reordered leading Schur
  // vectors span V times C's (the coefficients below, since V is implicit).
  // The 1-norm estimate of cond(R) is within a factor ~p of the 2-norm one,
  // so rcond > 1e-7 keeps the decision exact for rank_tol <= 1e-10.
  bool fast = false;
  HMat Mf;
  if (have_qr && rank_tol <= 1e-10 && SAW.cols > 0) {
    const int pp = static_cast<int>(SAW.cols);
    double rcond = 0.0;
    int info = 0;
    std::vector<double> wk(static_cast<size_t>(3 * pp));
    std::vector<int> iwk(static_cast<size_t>(pp));
    scipy_dtrcon_("1", "U", "N", &pp, Rf->a.data(), &pp, &rcond, wk.data(), iwk.data(), &info, 1, 1, 1);
    if (info == 0 && rcond > 1e-7) {
      const int ss = static_cast<int>(SAW.rows);
      const double one = 1.0, zero = 0.0;
      Mf = HMat(pp, pp);
      scipy_dgemm_("T", "N", &pp, &pp, &ss, &one, Qf->a.data(), &ss, SW.a.data(), &ss, &zero, Mf.a.data(), &pp, 1, 1);
      scipy_dtrsm_("L", "U", "N", "N", &pp, &pp, &one, Rf->a.data(), &pp, Mf.a.data(), &pp, 1, 1, 1, 1);
      fast = true;
    }
  }
  if (fast) {
    // l = p; V = I
  } else if (have_qr) {
    // SAW = Q R: singular values / right vectors of R, left vectors Q U_R
    HMat UR;
    thin_svd(*Rf, sv, &UR, &V);
    U = HMat(SAW.rows, UR.cols);
    const int m = static_cast<int>(SAW.rows), n = static_cast<int>(UR.cols), kk = static_cast<int>(Qf->cols);
    const double one = 1.0, zero = 0.0;
    if (m > 0 && n > 0 && kk > 0)
      scipy_dgemm_("N", "N", &m, &n, &kk, &one, Qf->a.data(), &m, UR.a.data(), &kk, &zero, U.a.data(), &m, 1, 1);
  } else {
    thin_svd(SAW, sv, &U, &V);
  }
  const auto t1 = clk::now();
  i64 l = 0;  // recycle.hpp:102-104
  const double cutoff = sv.empty() ? 0.0 : rank_tol * sv[0];
  if (fast)
    l = SAW.cols;
  else
    while (l < static_cast<i64>(sv.size()) && sv[static_cast<size_t>(l)] > cutoff && sv[static_cast<size_t>(l)] > 0.0) ++l;
  const i64 s = SAW.rows, p = SAW.cols;
  Harmonic out;
  out.rank = l;
  out.k_requested = k;
  if (k > l) {
    k = l;
    out.rank_limited = true;
  }
  if (k == 0 || l == 0) {
    out.coeffs = HMat(p, 0);
    return out;
  }
  // m = u^T SW v (recycle.hpp:114-118), C = diag(1/sigma) m
  HMat C(l, l);
  if (fast) {
    C = std::move(Mf);
  } else {
    HMat swv(s, l);
    for (i64 c = 0; c < l; ++c) hgemv(false, s, p, 1.0, SW.a.data(), s, V.col(c), 0.0, swv.col(c));
    for (i64 c = 0; c < l; ++c) {
      hgemv(true, s, l, 1.0, U.a.data(), s, swv.col(c), 0.0, C.col(c));
      for (i64 r = 0; r < l; ++r) C(r, c) = (1.0 / sv[static_cast<size_t>(r)]) * C(r, c);
    }
  }
  // real Schur (dgees), ordering, conjugate-pair closure, dtrsen (recycle.hpp:167-205)
  const int n = static_cast<int>(l);
  HMat Q(l, l);
  std::vector<double> wr(static_cast<size_t>(l)), wi(static_cast<size_t>(l));
  int sdim = 0, info = 0, lwork = 80 * n + 64;
  std::vector<double> work(static_cast<size_t>(lwork));
  const auto t2 = clk::now();
  scipy_dgees_("V", "N", nullptr, &n, C.a.data(), &n, &sdim, wr.data(), wi.data(), Q.a.data(), &n, work.data(), &lwork,
               nullptr, &info, 1, 1);
  const auto t3 = clk::now();
  if (info != 0) throw runtime("real_schur: dgees failed with info = " + std::to_string(info));
  std::vector<i64> order(static_cast<size_t>(l));
  std::iota(order.begin(), order.end(), i64{0});
  auto mag = [&](i64 i) { return std::hypot(wr[static_cast<size_t>(i)], wi[static_cast<size_t>(i)]); };
  std::sort(order.begin(), order.end(), [&](i64 a, i64 b) {
    const double ma = mag(a), mb = mag(b);
    if (ma != mb) return ma > mb;
    if (wr[static_cast<size_t>(a)] != wr[static_cast<size_t>(b)]) return wr[static_cast<size_t>(a)] > wr[static_cast<size_t>(b)];
    return a < b;
  });
  std::vector<int> sel(static_cast<size_t>(l), 0);
  for (i64 i = 0; i < k; ++i) sel[static_cast<size_t>(order[static_cast<size_t>(i)])] = 1;
  for (i64 i = 0; i + 1 < l;) {
    if (wi[static_cast<size_t>(i)] != 0.0) {
      if (sel[static_cast<size_t>(i)] != sel[static_cast<size_t>(i) + 1]) {
        sel[static_cast<size_t>(i)] = sel[static_cast<size_t>(i) + 1] = 1;
        out.pair_extended = true;
      }
      i += 2;
    } else {
      ++i;
    }
  }
  i64 ke = 0;
  for (int v : sel) ke += v;
  int mm = 0, nn2 = std::max(1, n * n);
  double scond = 0.0, sep = 0.0;
  std::vector<double> w2(static_cast<size_t>(nn2));
  std::vector<int> iw(static_cast<size_t>(nn2));
  scipy_dtrsen_("N", "V", sel.data(), &n, C.a.data(), &n, Q.a.data(), &n, wr.data(), wi.data(), &mm, &scond, &sep,
                w2.data(), &nn2, iw.data(), &nn2, &info, 1, 1);
  if (info != 0) throw runtime("reorder_schur: dtrsen failed with info = " + std::to_string(info));
  out.k_eff = ke;
  out.coeffs = HMat(p, ke);
  if (fast)
    for (i64 c = 0; c < ke; ++c) std::copy(Q.col(c), Q.col(c) + p, out.coeffs.col(c));
  else
    for (i64 c = 0; c < ke; ++c) hgemv(false, p, l, 1.0, V.a.data(), p, Q.col(c), 0.0, out.coeffs.col(c));
  for (i64 i = 0; i < ke; ++i) out.mu.emplace_back(wr[static_cast<size_t>(i)], wi[static_cast<size_t>(i)]);
  const auto t4 = clk::now();
  auto ms = [](clk::duration d) { return std::chrono::duration<double, std::milli>(d).count(); };
  out.svd_ms = ms(t1 - t0);
  out.schur_ms = ms(t3 - t2);
  out.rest_ms = ms(t2 - t1) + ms(t4 - t3);
  return out;
}

}  // namespace sdr
