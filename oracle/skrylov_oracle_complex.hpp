// ORACLE — TEST INFRASTRUCTURE ONLY. Complex-fp64 GMRES-SDR on the CPU.
//
// The reference's scalars are real; complex is "a compile-level variant, not
// required for acceptance", so there is no reference code for
// it: PARITY UNPINNED against the reference. This is the reference algorithm
// (the files cited per function) with the scalar type made complex:
// conjugated inner products, complex least squares, and the harmonic-Ritz
// pencil through complex Schur (zgees / ztrsen) — with complex Schur vectors
// there are no conjugate pairs to keep together (recycle.hpp:184-197 is a
// real-arithmetic rule). The sketch S is real: S z = S Re z + i S Im z
// (C4 "SRDCT (Re/Im)"). Pinned by its own closed forms:
// identity-sketch collapse to dense complex GMRES (tests/test_oracle.py).
#pragma once

#include "skrylov_oracle.hpp"

#include <complex>

extern "C" {
void scipy_zgesvd_(const char* jobu, const char* jobvt, const int* m, const int* n, std::complex<double>* a,
                   const int* lda, double* s, std::complex<double>* u, const int* ldu, std::complex<double>* vt,
                   const int* ldvt, std::complex<double>* work, const int* lwork, double* rwork, int* info, size_t,
                   size_t);
void scipy_zgees_(const char* jobvs, const char* sort, void* select, const int* n, std::complex<double>* a,
                  const int* lda, int* sdim, std::complex<double>* w, std::complex<double>* vs, const int* ldvs,
                  std::complex<double>* work, const int* lwork, double* rwork, int* bwork, int* info, size_t, size_t);
void scipy_ztrsen_(const char* job, const char* compq, const int* select, const int* n, std::complex<double>* t,
                   const int* ldt, std::complex<double>* q, const int* ldq, std::complex<double>* w, int* m, double* s,
                   double* sep, std::complex<double>* work, const int* lwork, int* info, size_t, size_t);
}

namespace oracle {
namespace cplx {

using Z = std::complex<double>;
using ZVec = std::vector<Z>;

struct ZMat {
  Index rows = 0, cols = 0;
  ZVec a;
  ZMat() = default;
  ZMat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), Z(0.0, 0.0)) {}
  Z& operator()(Index i, Index j) { return a[static_cast<size_t>(j * rows + i)]; }
  const Z& operator()(Index i, Index j) const { return a[static_cast<size_t>(j * rows + i)]; }
  Z* col(Index j) { return a.data() + j * rows; }
  const Z* col(Index j) const { return a.data() + j * rows; }
};

/// x^H y (conjugate-linear in x: the complex Euclidean inner product).
inline Z dotc(const Z* x, const Z* y, Index n) {
  Z acc(0.0, 0.0);
  for (Index i = 0; i < n; ++i) acc += std::conj(x[i]) * y[i];
  return acc;
}
inline double znorm(const Z* x, Index n) {
  double acc = 0.0;
  for (Index i = 0; i < n; ++i) acc += std::norm(x[i]);
  return std::sqrt(acc);
}

/// Complex CSR (sparse.hpp:27-150 with complex values; columns strictly
/// increasing per row), y = A x in CSR order.
struct ZCsr {
  Index n = 0;
  std::vector<Index> off, col;
  ZVec val;
  void apply(const Z* x, Z* y) const {
    for (Index r = 0; r < n; ++r) {
      Z acc(0.0, 0.0);
      for (Index p = off[static_cast<size_t>(r)]; p < off[static_cast<size_t>(r) + 1]; ++p)
        acc += val[static_cast<size_t>(p)] * x[col[static_cast<size_t>(p)]];
      y[r] = acc;
    }
  }
};

/// S z = S Re z + i S Im z for the real sketch S.
inline void sketch_apply(const SketchOperator& S, const Z* z, Index n, Z* out) {
  Vec re(static_cast<size_t>(n)), im(static_cast<size_t>(n)), sr(static_cast<size_t>(S.sketch_dim())),
      si(static_cast<size_t>(S.sketch_dim()));
  for (Index i = 0; i < n; ++i) {
    re[static_cast<size_t>(i)] = z[i].real();
    im[static_cast<size_t>(i)] = z[i].imag();
  }
  S.apply(re.data(), n, sr.data());
  S.apply(im.data(), n, si.data());
  for (Index r = 0; r < S.sketch_dim(); ++r) out[r] = Z(sr[static_cast<size_t>(r)], si[static_cast<size_t>(r)]);
}

// ------------------------------------------------------------ arnoldi ---
struct KrylovState {  // arnoldi.hpp:26-38
  ZMat V, H, SV, SAV;
  Index j = 0, t = 0, m_max = 0;
  double r0_norm = 0.0;
  bool breakdown = false;
};

inline KrylovState init_krylov(const ZVec& r0, const SketchOperator& S, Index t, Index m_max,
                               Counters* counters) {  // arnoldi.hpp:47-72
  KrylovState st;
  st.t = t;
  st.m_max = m_max;
  const Index n = static_cast<Index>(r0.size()), s = S.sketch_dim();
  st.r0_norm = znorm(r0.data(), n);
  if (counters) ++counters->inner_products;
  if (st.r0_norm == 0.0) throw std::domain_error("init_krylov: zero initial residual (already converged)");
  st.V = ZMat(n, m_max + 1);
  st.H = ZMat(m_max + 1, m_max);
  st.SV = ZMat(s, m_max + 1);
  st.SAV = ZMat(s, m_max);
  for (Index i = 0; i < n; ++i) st.V(i, 0) = r0[static_cast<size_t>(i)] / st.r0_norm;
  ZVec sr0(static_cast<size_t>(s));
  sketch_apply(S, r0.data(), n, sr0.data());
  if (counters) ++counters->sketch_applies;
  for (Index i = 0; i < s; ++i) st.SV(i, 0) = sr0[static_cast<size_t>(i)] / st.r0_norm;
  return st;
}

inline bool arnoldi_step(KrylovState& st, const ZCsr& A, const SketchOperator& S, Counters* counters,
                         double breakdown_tol) {  // arnoldi.hpp:82-119
  const Index j = st.j, n = st.V.rows, s = st.SV.rows;
  ZVec w(static_cast<size_t>(n));
  A.apply(st.V.col(j), w.data());
  if (counters) ++counters->matvecs;
  const double norm_before = znorm(w.data(), n);
  if (counters) ++counters->inner_products;
  const Index i0 = std::max<Index>(0, j - st.t + 1);
  for (Index i = i0; i <= j; ++i) {  // MGS window, arnoldi.hpp:91-97 (h = v_i^H w)
    const Z h = dotc(st.V.col(i), w.data(), n);
    if (counters) ++counters->inner_products;
    st.H(i, j) = h;
    const Z* vi = st.V.col(i);
    for (Index r = 0; r < n; ++r) w[static_cast<size_t>(r)] -= h * vi[r];
  }
  const double h_next = znorm(w.data(), n);
  if (counters) ++counters->inner_products;
  auto fill_sav = [&](Index ncols) {  // arnoldi.hpp:115
    for (Index r = 0; r < s; ++r) {
      Z acc(0.0, 0.0);
      for (Index q = 0; q < ncols; ++q) acc += st.SV(r, i0 + q) * st.H(i0 + q, j);
      st.SAV(r, j) = acc;
    }
  };
  if (h_next <= breakdown_tol * norm_before) {  // arnoldi.hpp:101-108
    st.H(j + 1, j) = 0.0;
    fill_sav(j - i0 + 1);
    st.breakdown = true;
    st.j = j + 1;
    return true;
  }
  st.H(j + 1, j) = h_next;
  for (Index r = 0; r < n; ++r) st.V(r, j + 1) = w[static_cast<size_t>(r)] / h_next;
  ZVec sv(static_cast<size_t>(s));
  sketch_apply(S, st.V.col(j + 1), n, sv.data());
  if (counters) ++counters->sketch_applies;
  for (Index r = 0; r < s; ++r) st.SV(r, j + 1) = sv[static_cast<size_t>(r)];
  fill_sav(j - i0 + 2);
  st.j = j + 1;
  return false;
}

// -------------------------------------------------------- incremental QR ---
class IncrementalQR {  // incremental_qr.hpp:26-162, complex (Q^H projections)
 public:
  IncrementalQR(Index rows, Index capacity, double rank_tol) : s_(rows), rank_tol_(rank_tol) {
    cap_ = std::max<Index>(capacity, 1);
    m_ = ZMat(rows, cap_);
    q_ = ZMat(rows, cap_);
    r_ = ZMat(cap_, cap_);
  }
  Index cols() const { return p_; }
  struct AppendInfo {
    Index column = 0;
    bool rank_deficient = false;
  };
  AppendInfo append(const Z* col) {  // :46-79, two projection passes
    if (p_ == cap_) grow();
    const Index p = p_, s = s_;
    std::copy(col, col + s, m_.col(p));
    ZVec w(col, col + s), coeffs(static_cast<size_t>(p), Z(0.0, 0.0)), c(static_cast<size_t>(p));
    for (int pass = 0; pass < 2; ++pass) {
      for (Index q = 0; q < p; ++q) c[static_cast<size_t>(q)] = dotc(q_.col(q), w.data(), s);
      for (Index q = 0; q < p; ++q) {
        const Z* qc = q_.col(q);
        for (Index r = 0; r < s; ++r) w[static_cast<size_t>(r)] -= qc[r] * c[static_cast<size_t>(q)];
      }
      for (Index q = 0; q < p; ++q) coeffs[static_cast<size_t>(q)] += c[static_cast<size_t>(q)];
    }
    const double rho = znorm(w.data(), s);
    AppendInfo info;
    info.column = p;
    for (Index q = 0; q < p; ++q) r_(q, p) = coeffs[static_cast<size_t>(q)];
    if (rho <= rank_tol_ * znorm(col, s)) {
      info.rank_deficient = true;
      std::fill(q_.col(p), q_.col(p) + s, Z(0.0, 0.0));
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
  void exclude(Index column) { state_[static_cast<size_t>(column)] = 1; }
  /// :107-135: y over the used columns by back substitution; the residual
  /// against the raw columns.
  double solve(const ZVec& rhs, ZVec& y) const {
    for (Index i = 0; i < p_; ++i)
      if (state_[static_cast<size_t>(i)] == 2)
        throw std::runtime_error("IncrementalQR::solve: column " + std::to_string(i) +
                                 " is rank-deficient and unresolved; exclude it or rebuild");
    std::vector<Index> used;
    for (Index i = 0; i < p_; ++i)
      if (state_[static_cast<size_t>(i)] == 0) used.push_back(i);
    y.assign(static_cast<size_t>(p_), Z(0.0, 0.0));
    ZVec c(used.size());
    for (size_t q = 0; q < used.size(); ++q) c[q] = dotc(q_.col(used[q]), rhs.data(), s_);
    for (size_t q = used.size(); q-- > 0;) {
      Z acc = c[q];
      for (size_t q2 = q + 1; q2 < used.size(); ++q2) acc -= r_(used[q], used[q2]) * y[static_cast<size_t>(used[q2])];
      y[static_cast<size_t>(used[q])] = acc / r_(used[q], used[q]);
    }
    ZVec res(rhs);
    for (Index q = 0; q < p_; ++q)
      for (Index r = 0; r < s_; ++r) res[static_cast<size_t>(r)] -= m_(r, q) * y[static_cast<size_t>(q)];
    return znorm(res.data(), s_);
  }

 private:
  void grow() {
    const Index cap = 2 * cap_;
    ZMat m2(s_, cap), q2(s_, cap), r2(cap, cap);
    for (Index j = 0; j < p_; ++j) {
      std::copy(m_.col(j), m_.col(j) + s_, m2.col(j));
      std::copy(q_.col(j), q_.col(j) + s_, q2.col(j));
      for (Index i = 0; i < p_; ++i) r2(i, j) = r_(i, j);
    }
    m_ = std::move(m2);
    q_ = std::move(q2);
    r_ = std::move(r2);
    cap_ = cap;
  }
  Index s_ = 0, cap_ = 0, p_ = 0;
  double rank_tol_;
  ZMat m_, q_, r_;
  std::vector<int> state_;
};

// ------------------------------------------------------------- recycle ---
struct RecycleSpace {  // recycle.hpp:31-72
  ZMat U, SU, SAU;
  Index dim() const { return U.cols; }
  bool empty() const { return U.cols == 0; }
  void drop_columns(const std::vector<Index>& cols) {
    std::vector<bool> drop(static_cast<size_t>(dim()), false);
    for (Index c : cols) drop[static_cast<size_t>(c)] = true;
    Index keep = 0;
    for (Index c = 0; c < dim(); ++c) keep += drop[static_cast<size_t>(c)] ? 0 : 1;
    ZMat u(U.rows, keep), su(SU.rows, keep), sau(SAU.rows, keep);
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

struct Harmonic {
  ZMat coeffs;  // (kh + j) x k_eff
  Index rank = 0, k_eff = 0;
  bool rank_limited = false;
};

/// recycle.hpp:98-218 in complex arithmetic: truncated SVD of SAW
/// (zgesvd, rank = #{σ_i > rank_tol σ_1, σ_i > 0}), m = U^H SW V, C =
/// Σ^-1 m, complex Schur C = Q T Q^H (zgees), Ritz values ordered by |μ|
/// descending, then Re μ descending, then Schur position; the first k moved
/// to the top (ztrsen); coefficients V Q(:, 0:k).
inline Harmonic harmonic(const ZMat& SAW, const ZMat& SW, Index k, double rank_tol) {
  const int m = static_cast<int>(SAW.rows), n = static_cast<int>(SAW.cols);
  const int mn = std::min(m, n);
  ZMat a = SAW, u(m, mn), vt(mn, n);
  Vec sv(static_cast<size_t>(mn)), rwork(static_cast<size_t>(5 * std::max(mn, 1)));
  int info = 0, lwork = -1;
  Z wq;
  const int ldu = std::max(1, m), ldvt = std::max(1, mn), lda = std::max(1, m);
  scipy_zgesvd_("S", "S", &m, &n, a.a.data(), &lda, sv.data(), u.a.data(), &ldu, vt.a.data(), &ldvt, &wq, &lwork,
                rwork.data(), &info, 1, 1);
  lwork = static_cast<int>(wq.real()) + 1;
  ZVec work(static_cast<size_t>(lwork));
  scipy_zgesvd_("S", "S", &m, &n, a.a.data(), &lda, sv.data(), u.a.data(), &ldu, vt.a.data(), &ldvt, work.data(), &lwork,
                rwork.data(), &info, 1, 1);
  if (info != 0) throw std::runtime_error("truncated_svd: zgesvd failed with info = " + std::to_string(info));
  Index l = 0;
  const double cutoff = mn > 0 ? rank_tol * sv[0] : 0.0;
  while (l < mn && sv[static_cast<size_t>(l)] > cutoff && sv[static_cast<size_t>(l)] > 0.0) ++l;
  Harmonic hp;
  hp.rank = l;
  if (k > l) {
    k = l;
    hp.rank_limited = true;
  }
  if (k == 0) {
    hp.coeffs = ZMat(n, 0);
    return hp;
  }
  // V = vt^H (n x l); SWV = SW V; M = U^H SWV; C = Σ^-1 M
  ZMat V(n, l);
  for (Index c = 0; c < l; ++c)
    for (Index r = 0; r < n; ++r) V(r, c) = std::conj(vt(c, r));
  const Index s = SW.rows;
  ZMat swv(s, l);
  for (Index c = 0; c < l; ++c)
    for (Index q = 0; q < n; ++q) {
      const Z vq = V(q, c);
      for (Index r = 0; r < s; ++r) swv(r, c) += SW(r, q) * vq;
    }
  ZMat C(l, l);
  for (Index c = 0; c < l; ++c)
    for (Index r = 0; r < l; ++r) C(r, c) = dotc(u.col(r), swv.col(c), s) / sv[static_cast<size_t>(r)];
  const int nl = static_cast<int>(l);
  ZMat Q(l, l);
  ZVec w(static_cast<size_t>(l));
  Vec rw(static_cast<size_t>(l));
  int sdim = 0;
  int lw = std::max(1, 64 * nl);
  ZVec wk(static_cast<size_t>(lw));
  scipy_zgees_("V", "N", nullptr, &nl, C.a.data(), &nl, &sdim, w.data(), Q.a.data(), &nl, wk.data(), &lw, rw.data(),
               nullptr, &info, 1, 1);
  if (info != 0) throw std::runtime_error("complex_schur: zgees failed with info = " + std::to_string(info));
  std::vector<Index> order(static_cast<size_t>(l));
  std::iota(order.begin(), order.end(), Index{0});
  std::sort(order.begin(), order.end(), [&](Index x, Index y) {
    const double mx = std::abs(w[static_cast<size_t>(x)]), my = std::abs(w[static_cast<size_t>(y)]);
    if (mx != my) return mx > my;
    if (w[static_cast<size_t>(x)].real() != w[static_cast<size_t>(y)].real())
      return w[static_cast<size_t>(x)].real() > w[static_cast<size_t>(y)].real();
    return x < y;
  });
  std::vector<int> sel(static_cast<size_t>(l), 0);
  for (Index i = 0; i < k; ++i) sel[static_cast<size_t>(order[static_cast<size_t>(i)])] = 1;
  int mm = 0;
  double scond = 0.0, sep = 0.0;
  int lw2 = std::max(1, nl * nl);
  ZVec wk2(static_cast<size_t>(lw2));
  scipy_ztrsen_("N", "V", sel.data(), &nl, C.a.data(), &nl, Q.a.data(), &nl, w.data(), &mm, &scond, &sep, wk2.data(),
                &lw2, &info, 1, 1);
  if (info != 0) throw std::runtime_error("reorder_schur: ztrsen failed with info = " + std::to_string(info));
  hp.k_eff = k;
  hp.coeffs = ZMat(n, k);
  for (Index c = 0; c < k; ++c)
    for (Index q = 0; q < l; ++q) {
      const Z qv = Q(q, c);
      for (Index r = 0; r < n; ++r) hp.coeffs(r, c) += V(r, q) * qv;
    }
  return hp;
}

inline void update_recycle(const KrylovState& st, RecycleSpace& space, Index k, double rank_tol, Counters& counters,
                           std::vector<std::string>* notes) {  // recycle.hpp:226-289
  const Index j = st.j, kh = space.dim(), s = st.SV.rows, n = st.V.rows;
  ZMat SAW(s, kh + j), SW(s, kh + j);
  for (Index c = 0; c < kh; ++c)
    for (Index r = 0; r < s; ++r) {
      SAW(r, c) = space.SAU(r, c);
      SW(r, c) = space.SU(r, c);
    }
  for (Index c = 0; c < j; ++c)
    for (Index r = 0; r < s; ++r) {
      SAW(r, kh + c) = st.SAV(r, c);
      SW(r, kh + c) = st.SV(r, c);
    }
  Harmonic hp = harmonic(SAW, SW, k, rank_tol);
  if (notes && hp.rank_limited)
    notes->push_back("deflation space limited to pencil rank " + std::to_string(hp.rank) + " (requested " +
                     std::to_string(k) + ")");
  RecycleSpace next;
  const Index ke = hp.k_eff;
  if (ke == 0) {
    space = next;
    return;
  }
  next.U = ZMat(n, ke);
  next.SU = ZMat(s, ke);
  next.SAU = ZMat(s, ke);
  for (Index q = 0; q < ke; ++q) {
    for (Index i = 0; i < j; ++i) {
      const Z cf = hp.coeffs(kh + i, q);
      for (Index r = 0; r < n; ++r) next.U(r, q) += st.V(r, i) * cf;
      for (Index r = 0; r < s; ++r) {
        next.SU(r, q) += st.SV(r, i) * cf;
        next.SAU(r, q) += st.SAV(r, i) * cf;
      }
    }
    for (Index i = 0; i < kh; ++i) {
      const Z cf = hp.coeffs(i, q);
      for (Index r = 0; r < n; ++r) next.U(r, q) += space.U(r, i) * cf;
      for (Index r = 0; r < s; ++r) {
        next.SU(r, q) += space.SU(r, i) * cf;
        next.SAU(r, q) += space.SAU(r, i) * cf;
      }
    }
  }
  std::vector<Index> bad;
  for (Index q = 0; q < ke; ++q) {  // recycle.hpp:269-286
    const double nrm = znorm(next.U.col(q), n);
    ++counters.inner_products;
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
  space = std::move(next);
}

/// refresh_for_new_matrix, exact (recycle.hpp:297-318): SAU(:, q) = S A u_q.
inline void refresh_exact(RecycleSpace& space, const ZCsr& A, const SketchOperator& S, Counters& counters) {
  const Index n = A.n, s = S.sketch_dim();
  ZVec au(static_cast<size_t>(n));
  for (Index q = 0; q < space.dim(); ++q) {
    A.apply(space.U.col(q), au.data());
    ++counters.matvecs;
    sketch_apply(S, au.data(), n, space.SAU.col(q));
    ++counters.sketch_applies;
  }
  (void)s;
}

// ------------------------------------------------------------- solver ---
struct SolveResult {
  ZVec x;
  SolveReport report;
};

/// solve (solver.hpp:269-365) with solve_cycle (:128-254) inlined: relative
/// tolerance, sketched-residual trigger with the safety ratchet, recursive
/// residual restarts, statuses and counters as in the real oracle.
inline SolveResult solve(const ZCsr& A, const ZVec& b, const SolverConfig& cfg, RecycleSpace& space,
                         const SketchOperator& S) {
  cfg.validate();
  const Index n = A.n, s = S.sketch_dim();
  if (static_cast<Index>(b.size()) != n) throw std::invalid_argument("solve: rhs length does not match operator size");
  if (S.input_dim() != n) throw std::invalid_argument("solve: sketch input size does not match the operator");
  if (s < 2 * (cfg.m + cfg.k))
    throw std::invalid_argument("solve: sketch size " + std::to_string(s) + " is below 2 (m + k) = " +
                                std::to_string(2 * (cfg.m + cfg.k)));
  const auto t0 = std::chrono::steady_clock::now();
  SolveResult res;
  SolveReport& rep = res.report;
  rep.rhs_norm = znorm(b.data(), n);
  ++rep.counters.inner_products;
  const double tol_abs = cfg.tol * rep.rhs_norm;
  res.x.assign(static_cast<size_t>(n), Z(0.0, 0.0));
  ZVec r = b;
  double safety = cfg.safety_init, res_norm = std::numeric_limits<double>::quiet_NaN();
  bool have = false;
  for (int cycle = 1; cycle <= cfg.max_restarts; ++cycle) {
    safety = std::max(1.0, safety);
    KrylovState st;
    try {
      st = init_krylov(r, S, cfg.t, cfg.m, &rep.counters);
    } catch (const std::domain_error&) {
      rep.status = SolveStatus::converged;
      res_norm = 0.0;
      have = true;
      break;
    }
    ZVec sr0(static_cast<size_t>(s));
    for (Index q = 0; q < s; ++q) sr0[static_cast<size_t>(q)] = st.SV(q, 0) * st.r0_norm;
    const double sketched_entry = znorm(sr0.data(), s);
    IncrementalQR qr(s, space.dim() + cfg.m, cfg.rank_tol);
    for (;;) {  // solver.hpp:144-159
      std::vector<Index> bad;
      for (Index q = 0; q < space.dim(); ++q)
        if (qr.append(space.SAU.col(q)).rank_deficient) bad.push_back(q);
      if (bad.empty()) break;
      space.drop_columns(bad);
      rep.notes.push_back("cycle " + std::to_string(cycle) + ": dropped " + std::to_string(bad.size()) +
                          " deflation columns with rank-deficient sketched images");
      qr = IncrementalQR(s, space.dim() + cfg.m, cfg.rank_tol);
      if (space.empty()) break;
    }
    const Index k_hat = space.dim();
    ZVec y;
    double sres = sketched_entry, residual_norm = 0.0;
    bool done = false, converged = false;
    ZVec corr, resid;
    while (!done && st.j < cfg.m && !st.breakdown) {
      arnoldi_step(st, A, S, &rep.counters, cfg.breakdown_tol);
      const Index j = st.j;
      const auto info = qr.append(st.SAV.col(j - 1));
      if (info.rank_deficient) {
        qr.exclude(info.column);
        rep.notes.push_back("cycle " + std::to_string(cycle) + ", step " + std::to_string(j) +
                            ": sketched basis column rank-deficient; excluded from the least-squares problem");
      }
      sres = qr.solve(sr0, y);
      const std::int64_t gi = rep.iterations + j;
      rep.sketched_residuals.push_back({gi, sres});
      const bool last = j == cfg.m || st.breakdown;
      if (sres < tol_abs / safety || last) {
        corr.assign(static_cast<size_t>(n), Z(0.0, 0.0));
        for (Index i = 0; i < j; ++i) {
          const Z yi = y[static_cast<size_t>(k_hat + i)];
          for (Index q = 0; q < n; ++q) corr[static_cast<size_t>(q)] += st.V(q, i) * yi;
        }
        for (Index p = 0; p < k_hat; ++p) {
          const Z yp = y[static_cast<size_t>(p)];
          for (Index q = 0; q < n; ++q) corr[static_cast<size_t>(q)] += space.U(q, p) * yp;
        }
        ZVec ac(static_cast<size_t>(n));
        A.apply(corr.data(), ac.data());
        ++rep.counters.matvecs;
        resid.resize(static_cast<size_t>(n));
        for (Index q = 0; q < n; ++q) resid[static_cast<size_t>(q)] = r[static_cast<size_t>(q)] - ac[static_cast<size_t>(q)];
        residual_norm = znorm(resid.data(), n);
        ++rep.counters.inner_products;
        rep.true_residuals.push_back({gi, residual_norm});
        if (residual_norm < tol_abs) {
          converged = done = true;
        } else {
          if (sres > 0.0) safety = std::max(safety, residual_norm / sres);
          if (last) done = true;
        }
      }
    }
    rep.cycles = cycle;
    rep.iterations += st.j;
    CycleStats cs;
    cs.steps = st.j;
    cs.entry_residual = st.r0_norm;
    cs.sketched_entry = sketched_entry;
    cs.exit_sres = sres;
    cs.exit_residual = residual_norm;
    cs.safety_after = safety;
    if (!corr.empty()) {
      for (Index q = 0; q < n; ++q) res.x[static_cast<size_t>(q)] += corr[static_cast<size_t>(q)];
      r = resid;
    }
    res_norm = residual_norm;
    have = true;
    if (cfg.k > 0 && st.j >= 1) {
      std::vector<std::string> notes;
      update_recycle(st, space, cfg.k, cfg.rank_tol, rep.counters, &notes);
      cs.deflation_rank = space.dim();
      for (auto& nn : notes) rep.notes.push_back("cycle " + std::to_string(cycle) + ": " + nn);
    } else if (cfg.k == 0) {
      space = RecycleSpace{};
    }
    rep.cycle_stats.push_back(cs);
    if (converged) {
      rep.status = SolveStatus::converged;
      break;
    }
    if (st.breakdown) {
      rep.status = SolveStatus::breakdown;
      rep.notes.push_back("cycle " + std::to_string(cycle) + ": basis exhausted before reaching the target");
      break;
    }
    if (st.j == cfg.m && sres > 0.99 * sketched_entry) {
      rep.status = SolveStatus::diverged;
      rep.notes.push_back("cycle " + std::to_string(cycle) + ": sketched residual improved by less than 1% over a full cycle");
      break;
    }
    if (cycle == cfg.max_restarts) rep.status = SolveStatus::max_restarts;
  }
  if (have) rep.final_relative_residual = rep.rhs_norm > 0.0 ? res_norm / rep.rhs_norm : res_norm;
  rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

}  // namespace cplx
}  // namespace oracle
