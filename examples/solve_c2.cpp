// A plain C++ caller of the C-ABI, no Python: the BASELINE C2 solve (128^3
// convection-diffusion, m=100 k=20 t=2 s=240, tol 1e-8) with host b / x, then
// a second right-hand side that reuses the recycle space (solver.hpp:269-365,
// recycle.hpp:31-72). This is the call sequence the reference's C++ shim in
// INTEGRATION.md makes.
//
//   make examples && ./examples/solve_c2 [n]
#include <sdr_b200.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

static void check(int rc, const char* what) {
  if (rc != SDR_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, sdr_last_error());
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 128, N = n * n * n;
  sdr_ctx* ctx = nullptr;
  check(sdr_ctx_create(0, &ctx), "sdr_ctx_create");
  sdr_csr* A = nullptr;
  check(sdr_csr_create_convdiff3d(ctx, n, n, n, 100.0, 50.0, 25.0, 0, n, &A), "sdr_csr_create_convdiff3d");
  sdr_config cfg;
  check(sdr_config_default(&cfg), "sdr_config_default");
  cfg.m = 100, cfg.k = 20, cfg.t = 2, cfg.s = 240, cfg.tol = 1e-8;
  sdr_sketch* S = nullptr;
  check(sdr_sketch_create_srdct(ctx, N, cfg.s, cfg.sketch_seed, &S), "sdr_sketch_create_srdct");
  sdr_recycle* space = nullptr;
  check(sdr_recycle_create(ctx, &space), "sdr_recycle_create");
  std::vector<double> b(static_cast<size_t>(N)), x(static_cast<size_t>(N));
  for (int sys = 0; sys < 2; ++sys) {
    check(sdr_gaussian_vector(N, 1 + sys, b.data()), "sdr_gaussian_vector");
    sdr_report* rep = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    check(sdr_solve(ctx, A, b.data(), nullptr, &cfg, space, S, nullptr, x.data(), &rep), "sdr_solve");
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    int status = 0;
    int64_t it = 0;
    int32_t cycles = 0;
    double rhs = 0, frr = 0, secs = 0;
    check(sdr_report_summary(rep, &status, &it, &cycles, &rhs, &frr, &secs), "sdr_report_summary");
    int64_t mv = 0, ip = 0, sa = 0;
    check(sdr_report_counters(rep, &mv, &ip, &sa), "sdr_report_counters");
    // verify on the host-visible result: ||b - A x|| / ||b|| through the device SpMV
    std::vector<double> ax(static_cast<size_t>(N));
    check(sdr_spmv(ctx, A, x.data(), N, ax.data()), "sdr_spmv");
    double rr = 0, bb = 0;
    for (int64_t i = 0; i < N; ++i) {
      const double d = b[static_cast<size_t>(i)] - ax[static_cast<size_t>(i)];
      rr += d * d;
      bb += b[static_cast<size_t>(i)] * b[static_cast<size_t>(i)];
    }
    std::printf("system %d: status %d, %lld iterations, %d cycles, rel. residual %.3e (verified %.3e), "
                "%lld matvecs / %lld inner products, %.2f ms (%.0f steps/s)\n",
                sys, status, static_cast<long long>(it), cycles, frr, std::sqrt(rr / bb), static_cast<long long>(mv),
                static_cast<long long>(ip), ms, 1e3 * static_cast<double>(it) / ms);
    sdr_report_destroy(rep);
    if (status != SDR_CONVERGED || std::sqrt(rr / bb) > 1.01 * cfg.tol) return 2;
  }
  sdr_recycle_destroy(space);
  sdr_sketch_destroy(S);
  sdr_csr_destroy(A);
  sdr_ctx_destroy(ctx);
  return 0;
}
