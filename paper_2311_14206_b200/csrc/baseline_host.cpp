// Host driver of the device classical restarted GMRES (baseline.hpp:51-216):
// same cycle structure, statuses, notes, counters and report streams as the
// reference; the Arnoldi steps run as device passes (baseline.cu) enqueued
// speculatively in chunks and cut short on the device by the stop flag the
// rotation kernel sets (target reached, breakdown, or m steps).
#include "baseline.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

extern "C" void scipy_dgelsy_(const int* m, const int* n, const int* nrhs, double* a, const int* lda, double* b,
                              const int* ldb, int* jpvt, const double* rcond, int* rank, double* work,
                              const int* lwork, int* info);

namespace sdr {

void BaselineConfig::validate() const {  // baseline.hpp:30-38
  if (m < 1) throw invalid("BaselineConfig: m must be at least 1");
  if (!(tol > 0.0 && tol < 1.0)) throw invalid("BaselineConfig: tol must lie in (0, 1)");
  if (max_restarts < 1) throw invalid("BaselineConfig: max_restarts must be at least 1");
  if (!(breakdown_tol >= 0.0)) throw invalid("BaselineConfig: breakdown_tol must be >= 0");
}

namespace {

/// min ||H y - rhs|| by column-pivoted QR with the basic solution for a
/// rank-deficient H (the zero-pivot fallback, baseline.hpp:171-177).
std::vector<double> lstsq_pivoted(HMat H, std::vector<double> rhs) {
  const int mm = static_cast<int>(H.rows), nn = static_cast<int>(H.cols), one = 1;
  const int ldb = std::max(mm, nn);
  rhs.resize(static_cast<size_t>(ldb), 0.0);
  std::vector<int> jpvt(static_cast<size_t>(nn), 0);
  const double rcond = std::numeric_limits<double>::epsilon() * std::min(mm, nn);
  int rank = 0, info = 0, lwork = -1;
  double wq = 0.0;
  scipy_dgelsy_(&mm, &nn, &one, H.a.data(), &mm, rhs.data(), &ldb, jpvt.data(), &rcond, &rank, &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(static_cast<size_t>(lwork));
  scipy_dgelsy_(&mm, &nn, &one, H.a.data(), &mm, rhs.data(), &ldb, jpvt.data(), &rcond, &rank, work.data(), &lwork,
                &info);
  if (info != 0) throw runtime("baseline_gmres: least-squares fallback failed (dgelsy info " + std::to_string(info) + ")");
  rhs.resize(static_cast<size_t>(nn));
  return rhs;
}

struct MappedFlags {
  int* host = nullptr;
  int* dev = nullptr;
  MappedFlags() {
    SDR_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host), 4 * sizeof(int), cudaHostAllocMapped));
    SDR_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
    std::fill(host, host + 4, 0);
  }
  ~MappedFlags() { cudaFreeHost(host); }
};

struct Events {
  cudaEvent_t e[2] = {nullptr, nullptr};
  Events() {
    for (auto& x : e) SDR_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  }
  ~Events() {
    for (auto& x : e) cudaEventDestroy(x);
  }
};

}  // namespace

void baseline_solve(Context& c, const DeviceOperator& A, const double* b, const double* x0, bool x0_nonzero,
                    const BaselineConfig& cfg, double* x_out, Report& rep) {
  cfg.validate();
  if (A.rows != A.cols)
    throw invalid("baseline_gmres: operator must be square, got " + std::to_string(A.rows) + " x " +
                  std::to_string(A.cols));
  if (cfg.m > kBaselineMaxM)
    throw invalid("baseline_gmres: restart length " + std::to_string(cfg.m) + " exceeds the device limit of " +
                  std::to_string(kBaselineMaxM));
  const auto t_start = std::chrono::steady_clock::now();
  const VecLayout lay = A.layout();
  const i64 nloc = lay.nloc, m = cfg.m, ldh = m + 1;
  const bool dist = c.distributed();

  // fixed row ranges per CTA: about two CTAs per SM, 256-row multiples; on
  // several ranks the grid is the same everywhere (partials allreduce
  // elementwise), empty ranges write zero partials
  const i64 want = 2 * static_cast<i64>(c.num_sms);
  i64 rpc = std::max<i64>(1, (nloc + want - 1) / want);
  rpc = (rpc + 255) / 256 * 256;
  const int G = dist ? static_cast<int>(want) : static_cast<int>(std::max<i64>(1, (nloc + rpc - 1) / rpc));

  DeviceBuffer<double> U((m + 1) * lay.ld), y(std::max<i64>(nloc, 1)), r(std::max<i64>(nloc, 1)),
      x(std::max<i64>(nloc, 1)), corr(lay.ld), acorr(std::max<i64>(nloc, 1)), small(4 * ldh * m + 8 * ldh + 8),
      part(2 * (m + 1) * G + G);
  MappedFlags flags;
  DeviceBuffer<int> ctl(4);
  SDR_CUDA(cudaMemsetAsync(ctl.get(), 0, 4 * sizeof(int), c.stream));
  BaselineStep s;
  s.U = U.get();
  s.ldu = lay.ld;
  s.own_off = lay.own_off;
  s.nloc = nloc;
  s.rows_per_cta = rpc;
  s.G = G;
  s.y = y.get();
  double* sm = small.get();
  s.H = sm;
  s.R = sm + ldh * m;
  s.vs = sm + 2 * ldh * m;
  s.cs = s.vs + ldh;
  s.sn = s.cs + ldh;
  s.g = s.sn + ldh;
  s.est = s.g + ldh;
  double* scal = s.est + ldh;  // 2 doubles
  s.p1 = part.get();
  s.p2 = s.p1 + (m + 1) * G;
  s.p3 = s.p2 + (m + 1) * G;
  s.ctl = ctl.get();
  s.ctl_host = flags.dev;
  s.m = m;
  s.breakdown_tol = cfg.breakdown_tol;
  double* u0 = U.get() + lay.own_off;

  auto read_scalar = [&](const double* dev) {
    double* h = c.pinned(1);
    SDR_CUDA(cudaMemcpyAsync(h, dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return h[0];
  };

  // rhs norm (1 IP), r = b or b - A x0 (baseline.hpp:67-81); u_0 = r
  launch_copy_norm(c, b, r.get(), nloc, scal);
  c.allreduce_sum(scal, 1);
  rep.rhs_norm = std::sqrt(read_scalar(scal));
  ++rep.counters.inner_products;
  const double tol_abs = cfg.tol * rep.rhs_norm;
  s.tol_abs = tol_abs;
  if (x0)
    SDR_CUDA(cudaMemcpyAsync(x.get(), x0, sizeof(double) * static_cast<size_t>(nloc), cudaMemcpyDeviceToDevice, c.stream));
  else
    SDR_CUDA(cudaMemsetAsync(x.get(), 0, sizeof(double) * static_cast<size_t>(std::max<i64>(nloc, 1)), c.stream));
  if (x0 && x0_nonzero) {
    SDR_CUDA(cudaMemcpyAsync(corr.get() + lay.own_off, x0, sizeof(double) * static_cast<size_t>(nloc),
                             cudaMemcpyDeviceToDevice, c.stream));
    c.halo_exchange(A.plan, corr.get() + lay.ext_shift(), A.ext_begin, corr.get() + lay.own_off, A.row_begin);
    launch_residual(c, A.view(), corr.get() + lay.ext_shift(), b, r.get(), scal);
    ++rep.counters.matvecs;
  }
  launch_copy_norm(c, r.get(), u0, nloc, scal + 1);
  c.allreduce_sum(scal + 1, 1);
  double beta2 = read_scalar(scal + 1);

  Events ev;
  std::vector<double> Rh, gh, esth, vsh, Hh;
  double res_norm = std::numeric_limits<double>::quiet_NaN();
  bool have = false;
  constexpr int kChunk = 8;
  for (int cycle = 1; cycle <= cfg.max_restarts; ++cycle) {
    const double beta = std::sqrt(beta2);  // r.norm() (1 IP)
    ++rep.counters.inner_products;
    if (beta == 0.0) {
      rep.status = 0;
      res_norm = 0.0;
      have = true;
      break;
    }
    rep.cycles = cycle;
    SDR_CUDA(cudaMemsetAsync(s.H, 0, sizeof(double) * static_cast<size_t>(ldh * m), c.stream));
    std::fill(flags.host, flags.host + 4, 0);
    baseline_cycle_init(c, s, beta);

    // Arnoldi + rotations, enqueued kChunk steps at a time; the host looks at
    // the stop flag of the chunk before the one just enqueued
    int q = 0, k = 0;
    while (q < m) {
      const int qend = static_cast<int>(std::min<i64>(q + kChunk, m));
      for (; q < qend; ++q) {
        double* uq = U.get() + q * lay.ld;
        c.halo_exchange(A.plan, uq + lay.ext_shift(), A.ext_begin, uq + lay.own_off, A.row_begin);
        launch_spmv_guarded(c, A.view(), uq + lay.ext_shift(), s.y, s.ctl);
        baseline_pass(c, s, q, 0);
        if (dist) c.allreduce_sum(s.p1, static_cast<i64>(q + 1) * G);
        baseline_pass(c, s, q, 1);
        if (dist) c.allreduce_sum(s.p2, static_cast<i64>(q + 1) * G);
        baseline_pass(c, s, q, 2);
        if (dist) c.allreduce_sum(s.p3, G);
        baseline_givens(c, s, q);
      }
      SDR_CUDA(cudaEventRecord(ev.e[k & 1], c.stream));
      if (k >= 1) {
        SDR_CUDA(cudaEventSynchronize(ev.e[(k - 1) & 1]));
        if (reinterpret_cast<volatile int*>(flags.host)[0]) break;
      }
      ++k;
    }
    c.sync();
    const i64 p = reinterpret_cast<volatile int*>(flags.host)[1];
    const bool breakdown = reinterpret_cast<volatile int*>(flags.host)[2] != 0;
    for (i64 qq = 0; qq < p; ++qq) {
      ++rep.counters.matvecs;
      rep.counters.inner_products += qq + 2;  // q+1 MGS dots and ||w||
    }

    // R, g, est, scales of the p steps (one D2H)
    double* h = c.pinned(ldh * p + 3 * ldh);
    SDR_CUDA(cudaMemcpyAsync(h, s.R, sizeof(double) * static_cast<size_t>(ldh * p), cudaMemcpyDeviceToHost, c.stream));
    SDR_CUDA(cudaMemcpyAsync(h + ldh * p, s.g, sizeof(double) * static_cast<size_t>(ldh), cudaMemcpyDeviceToHost, c.stream));
    SDR_CUDA(cudaMemcpyAsync(h + ldh * p + ldh, s.est, sizeof(double) * static_cast<size_t>(ldh), cudaMemcpyDeviceToHost,
                             c.stream));
    SDR_CUDA(cudaMemcpyAsync(h + ldh * p + 2 * ldh, s.vs, sizeof(double) * static_cast<size_t>(ldh),
                             cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    Rh.assign(h, h + ldh * p);
    gh.assign(h + ldh * p, h + ldh * p + ldh);
    esth.assign(h + ldh * p + ldh, h + ldh * p + 2 * ldh);
    vsh.assign(h + ldh * p + 2 * ldh, h + ldh * p + 3 * ldh);
    for (i64 qq = 0; qq < p; ++qq) rep.sketched.emplace_back(rep.iterations + qq + 1, esth[static_cast<size_t>(qq)]);
    const double est = p > 0 ? esth[static_cast<size_t>(p - 1)] : beta;

    // cycle iterate: R y = g, least squares on H if a pivot vanished
    std::vector<double> yv(static_cast<size_t>(p), 0.0);
    bool diag_ok = true;
    for (i64 i = 0; i < p; ++i) diag_ok = diag_ok && Rh[static_cast<size_t>(i + i * ldh)] != 0.0;
    if (diag_ok) {
      for (i64 i = p - 1; i >= 0; --i) {
        double acc = gh[static_cast<size_t>(i)];
        for (i64 j = i + 1; j < p; ++j) acc -= Rh[static_cast<size_t>(i + j * ldh)] * yv[static_cast<size_t>(j)];
        yv[static_cast<size_t>(i)] = acc / Rh[static_cast<size_t>(i + i * ldh)];
      }
    } else {
      HMat Hp(p + 1, p);
      Hh.resize(static_cast<size_t>(ldh * p));
      SDR_CUDA(cudaMemcpy(Hh.data(), s.H, sizeof(double) * Hh.size(), cudaMemcpyDeviceToHost));
      for (i64 j = 0; j < p; ++j)
        for (i64 i = 0; i <= p; ++i) Hp(i, j) = Hh[static_cast<size_t>(i + j * ldh)];
      std::vector<double> rhs(static_cast<size_t>(p + 1), 0.0);
      rhs[0] = beta;
      yv = lstsq_pivoted(std::move(Hp), std::move(rhs));
    }
    // correction = V y = U (vs .* y); x += correction; r -= A correction
    double* coef_h = c.pinned(std::max<i64>(p, 1));
    for (i64 j = 0; j < p; ++j) coef_h[j] = vsh[static_cast<size_t>(j)] * yv[static_cast<size_t>(j)];
    double* coef_d = s.est;  // est already read back: reuse as the coefficient vector
    SDR_CUDA(cudaMemcpyAsync(coef_d, coef_h, sizeof(double) * static_cast<size_t>(std::max<i64>(p, 1)),
                             cudaMemcpyHostToDevice, c.stream));
    if (p > 0 && nloc > 0) {
      TimedLaunch t(c, "baseline_correction");
      c.dgemm_tall(nloc, 1, p, u0, lay.ld, coef_d, std::max<i64>(p, 1), 0.0, corr.get() + lay.own_off, lay.ld);
    } else if (nloc > 0) {
      SDR_CUDA(cudaMemsetAsync(corr.get() + lay.own_off, 0, sizeof(double) * static_cast<size_t>(nloc), c.stream));
    }
    launch_axpy(c, 1.0, corr.get() + lay.own_off, x.get(), nloc);
    c.halo_exchange(A.plan, corr.get() + lay.ext_shift(), A.ext_begin, corr.get() + lay.own_off, A.row_begin);
    launch_spmv(c, A.view(), corr.get() + lay.ext_shift(), acorr.get());
    ++rep.counters.matvecs;
    launch_axpy(c, -1.0, acorr.get(), r.get(), nloc);
    launch_copy_norm(c, r.get(), u0, nloc, scal + 1);  // ||r|| (1 IP) and u_0 of the next cycle
    c.allreduce_sum(scal + 1, 1);
    beta2 = read_scalar(scal + 1);
    res_norm = std::sqrt(beta2);
    ++rep.counters.inner_products;
    have = true;
    rep.iterations += p;
    rep.truth.emplace_back(rep.iterations, res_norm);
    CycleStat st;
    st.steps = p;
    st.entry_residual = beta;
    st.sketched_entry = beta;
    st.exit_sres = est;
    st.exit_residual = res_norm;
    st.safety_after = 1.0;
    rep.cycle_stats.push_back(st);
    if (res_norm < tol_abs) {
      rep.status = 0;
      break;
    }
    if (breakdown) {
      rep.status = 2;
      rep.notes.push_back("cycle " + std::to_string(cycle) + ": basis exhausted before reaching the target");
      break;
    }
    if (p == m && est > 0.99 * beta) {
      rep.status = 3;
      rep.notes.push_back("cycle " + std::to_string(cycle) +
                          ": residual estimate improved by less than 1% over a full cycle");
      break;
    }
    if (cycle == cfg.max_restarts) rep.status = 1;
  }
  if (have) rep.final_relative_residual = rep.rhs_norm > 0.0 ? res_norm / rep.rhs_norm : res_norm;
  if (x_out && nloc > 0)
    SDR_CUDA(cudaMemcpyAsync(x_out, x.get(), sizeof(double) * static_cast<size_t>(nloc), cudaMemcpyDefault, c.stream));
  c.sync();
  rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

}  // namespace sdr
