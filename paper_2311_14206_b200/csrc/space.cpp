// Recycle-space bookkeeping (recycle.hpp:31-72, 297-318), solver config
// validation (solver.hpp:61-78) and sketch construction (sketch.hpp:105-132).
#include <cstdlib>
#include "solver.hpp"

#include <algorithm>
#include <cmath>
#include <memory>

namespace sdr {

void Config::validate() const {  // solver.hpp:61-78
  if (m < 1) throw invalid("SolverConfig: m must be at least 1");
  if (t < 1) throw invalid("SolverConfig: t must be at least 1");
  if (k < 0 || k >= m)
    throw invalid("SolverConfig: need 0 <= k < m, got k = " + std::to_string(k) + ", m = " + std::to_string(m));
  if (s < 2 * (m + k))
    throw invalid("SolverConfig: sketch size s = " + std::to_string(s) + " is below 2 (m + k) = " +
                  std::to_string(2 * (m + k)));
  if (!(tol > 0.0 && tol < 1.0)) throw invalid("SolverConfig: tol must lie in (0, 1)");
  if (!(safety_init >= 1.0)) throw invalid("SolverConfig: safety_init must be at least 1");
  if (max_restarts < 1) throw invalid("SolverConfig: max_restarts must be at least 1");
  if (!(rank_tol >= 0.0)) throw invalid("SolverConfig: rank_tol must be >= 0");
  if (!(breakdown_tol >= 0.0)) throw invalid("SolverConfig: breakdown_tol must be >= 0");
}

void Recycle::drop_columns(const std::vector<i64>& cols) {  // recycle.hpp:48-71
  if (cols.empty()) return;
  std::vector<bool> drop(static_cast<size_t>(dim()), false);
  for (i64 cc : cols) {
    if (cc < 0 || cc >= dim()) throw invalid("RecycleSpace::drop_columns: no column " + std::to_string(cc));
    drop[static_cast<size_t>(cc)] = true;
  }
  std::vector<int> ns;
  std::vector<double> nu;
  i64 keep = 0;
  for (i64 q = 0; q < dim(); ++q)
    if (!drop[static_cast<size_t>(q)]) ++keep;
  HMat su(s, keep), sau(s, keep);
  i64 o = 0;
  for (i64 q = 0; q < dim(); ++q) {
    if (drop[static_cast<size_t>(q)]) continue;
    ns.push_back(slot[static_cast<size_t>(q)]);
    nu.push_back(uscale[static_cast<size_t>(q)]);
    std::copy(SU.col(q), SU.col(q) + s, su.col(o));
    std::copy(SAU.col(q), SAU.col(q) + s, sau.col(o));
    ++o;
  }
  slot.swap(ns);
  uscale.swap(nu);
  SU = std::move(su);
  SAU = std::move(sau);
}

void Recycle::ensure(i64 nloc_, i64 capacity) {
  if (nloc != nloc_ && !empty()) throw invalid("solve: recycle space has " + std::to_string(nloc) + " local rows but the operator block has " + std::to_string(nloc_));
  const i64 ld_new = round_up(std::max<i64>(nloc_, 1), 32);
  if (nloc == nloc_ && ld == ld_new && capacity <= cap) return;
  const i64 cap_new = std::max(capacity, cap);
  DeviceBuffer<double> nb[2];
  nb[0].resize(ld_new * cap_new);
  nb[1].resize(ld_new * cap_new);
  for (i64 q = 0; q < dim(); ++q)
    SDR_CUDA(cudaMemcpy(nb[0].get() + q * ld_new, col(q), sizeof(double) * static_cast<size_t>(nloc_), cudaMemcpyDeviceToDevice));
  for (i64 q = 0; q < dim(); ++q) slot[static_cast<size_t>(q)] = static_cast<int>(q);
  buf[0] = std::move(nb[0]);
  buf[1] = std::move(nb[1]);
  cur = 0;
  nloc = nloc_;
  ld = ld_new;
  cap = cap_new;
}

SketchDev* create_sketch(Context& c, int kind, i64 n, i64 s, std::uint64_t seed, i64 zeta) {
  auto S = std::make_unique<SketchDev>();
  S->kind = kind;
  S->n = n;
  S->s = s;
  S->seed = seed;
  S->zeta = zeta;
  if (kind == kIdentity) {
    if (n < 1) throw invalid("SketchOperator::identity: n must be positive");
    S->s = n;
    return S.release();
  }
  if (kind == kSparseSign) {
    if (n < 1 || s < 1 || zeta < 1 || zeta > s)
      throw invalid("SketchOperator::sparse_sign: need n >= 1 and 1 <= zeta <= s, got n = " + std::to_string(n) +
                    ", s = " + std::to_string(s) + ", zeta = " + std::to_string(zeta));
    if (s > 880) throw invalid("SketchOperator::sparse_sign: device kernel supports s <= 880");
    std::mt19937_64 eng(seed);
    S->key = eng();
    return S.release();
  }
  if (n < 2 || s < 1 || s >= n)
    throw invalid("SketchOperator: need 1 <= s < n, got s = " + std::to_string(s) + ", n = " + std::to_string(n));
  if (s > 4096) throw invalid("SketchOperator: device SRDCT supports s <= 4096");
  if (n >= (int64_t{1} << 31)) throw invalid("SketchOperator: device SRDCT supports n < 2^31");
  SrdctHost h = make_srdct_host(n, s, seed);
  S->scale = std::sqrt(static_cast<double>(n) / static_cast<double>(s));
  std::vector<double> rs(static_cast<size_t>(s));
  for (i64 q = 0; q < s; ++q) {
    const double alpha = h.rows[static_cast<size_t>(q)] == 0 ? std::sqrt(1.0 / static_cast<double>(n))
                                                             : std::sqrt(2.0 / static_cast<double>(n));
    rs[static_cast<size_t>(q)] = alpha * S->scale;
  }
  S->sign_bits.resize(static_cast<i64>(h.sign_bits.size()));
  S->rows.resize(s);
  S->row_scale.resize(s);
  SDR_CUDA(cudaMemcpy(S->sign_bits.get(), h.sign_bits.data(), sizeof(uint32_t) * h.sign_bits.size(), cudaMemcpyHostToDevice));
  SDR_CUDA(cudaMemcpy(S->rows.get(), h.rows.data(), sizeof(int64_t) * h.rows.size(), cudaMemcpyHostToDevice));
  SDR_CUDA(cudaMemcpy(S->row_scale.get(), rs.data(), sizeof(double) * rs.size(), cudaMemcpyHostToDevice));
  S->rows_host = std::move(h.rows);
  S->sign_bits_host = std::move(h.sign_bits);
  prepare_srdct_tables(c, *S);
  return S.release();
}

void sketch_apply(Context& c, const SketchDev& S, const double* x, i64 nloc, i64 row_begin, double* out_host) {
  DeviceBuffer<double> out(S.s);
  launch_sketch(c, S, x, nloc, row_begin, out.get());
  c.allreduce_sum(out.get(), S.s);
  SDR_CUDA(cudaMemcpyAsync(out_host, out.get(), sizeof(double) * static_cast<size_t>(S.s), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
}

void refresh_recycle(Context& c, Recycle& sp, const DeviceOperator& A, const SketchDev& S, bool exact, Counters* cnt) {
  if (sp.empty()) return;  // recycle.hpp:297-318
  if (sp.n != A.cols)
    throw invalid("refresh_for_new_matrix: space has " + std::to_string(sp.n) + " rows but the operator takes " +
                  std::to_string(A.cols));
  if (!exact) {
    sp.provenance = 4;
    return;
  }
  // SAU(:, q) = S (A u_q) for every column: the k products and sketches are
  // queued back to back (no host round trip per column) and the k sketched
  // images come back in one copy. u_q = uscale_q * buf[slot_q]: the scale is
  // applied to the image (A and S are linear), so U is read in place when the
  // operator needs no halo (one GPU); otherwise through a halo'd staging vector.
  const VecLayout lay = A.layout();
  const i64 k = sp.dim();
  const bool in_place = lay.halo_lo == 0 && lay.halo_hi == 0 && lay.own_off == 0;
  // (small scratch from the context: a cudaFree per refresh would synchronise the device)
  DeviceBuffer<double> ubuf(in_place ? 0 : lay.ld), au(std::max<i64>(lay.nloc, 1) * k);
  struct {
    double* p;
    double* get() const { return p; }
  } sk{c.stage(S.s * k)};  // (not partials(): the one-vector sketch path below folds through it)
  if (!in_place) SDR_CUDA(cudaMemsetAsync(ubuf.get(), 0, sizeof(double) * static_cast<size_t>(lay.ld), c.stream));
  const i64 ldau = std::max<i64>(lay.nloc, 1);
  if (in_place) {  // one pass over A per 8 columns (batched SpMM)
    for (i64 q0 = 0; q0 < k; q0 += kSpmmMax) {
      const int nb = static_cast<int>(std::min<i64>(kSpmmMax, k - q0));
      SpmmCols X;
      for (int q = 0; q < nb; ++q) X.x[q] = sp.col(q0 + q);
      launch_spmm(c, A.view(), X, nb, au.get() + q0 * ldau, ldau);
    }
  }
  // the k sketches are small, latency-bound launches (C3: 15 us + a 6 us
  // fold each, back to back 0.86 ms per refresh): with the SRDCT tile kernel
  // they run on kSides streams at once, each into its own CTA partials, and
  // u_q's scale is applied to the folded image on the host
  static const bool side_on = [] {
    const char* e = std::getenv("SDR_REFRESH_STREAMS");
    return !e || std::atoi(e) != 0;
  }();
  const bool side = side_on && in_place && k > 1 && sketch_partials_eligible(S, lay.nloc, A.row_begin);
  if (side) {
    constexpr int kSides = Context::kAuxStreams;
    const i64 psz = sketch_partials_size(S, c.num_sms);
    struct {
      double* p;
      double* get() const { return p; }
    } parts{c.partials2(psz * k)};
    c.aux_fork(kSides);
    cudaStream_t own = c.stream;
    try {
      for (i64 q = 0; q < k; ++q) {
        c.stream = c.aux_stream(static_cast<int>(q % kSides));
        int G = 0, ld = 0;
        launch_sketch_partials(c, S, au.get() + q * ldau, lay.nloc, A.row_begin, parts.get() + q * psz, &G, &ld);
        launch_sketch_fold_partials(c, S, parts.get() + q * psz, G, ld, sk.get() + q * S.s);
        if (cnt) ++cnt->matvecs, ++cnt->sketch_applies;
      }
    } catch (...) {
      c.stream = own;
      throw;
    }
    c.stream = own;
    c.aux_join(kSides);
    c.allreduce_sum(sk.get(), S.s * k);
    std::vector<double> h(static_cast<size_t>(S.s * k));
    SDR_CUDA(cudaMemcpyAsync(h.data(), sk.get(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    for (i64 q = 0; q < k; ++q) {
      const double us = sp.uscale[static_cast<size_t>(q)];
      for (i64 r = 0; r < S.s; ++r) sp.SAU(r, q) = us * h[static_cast<size_t>(q * S.s + r)];
    }
    sp.provenance = 3;
    return;
  }
  for (i64 q = 0; q < k; ++q) {
    double* aq = au.get() + q * ldau;
    if (!in_place) {
      launch_scale_copy(c, 1.0, sp.col(q), ubuf.get() + lay.own_off, lay.nloc);
      operator_apply(c, A, ubuf.get(), aq);
    }
    if (cnt) ++cnt->matvecs;
    launch_sketch_scaled(c, S, aq, sp.uscale[static_cast<size_t>(q)], lay.nloc, A.row_begin, sk.get() + q * S.s);
    if (cnt) ++cnt->sketch_applies;
  }
  c.allreduce_sum(sk.get(), S.s * k);
  std::vector<double> h(static_cast<size_t>(S.s * k));
  SDR_CUDA(cudaMemcpyAsync(h.data(), sk.get(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  for (i64 q = 0; q < k; ++q) std::copy(h.begin() + q * S.s, h.begin() + (q + 1) * S.s, sp.SAU.col(q));
  sp.provenance = 3;
}

}  // namespace sdr
