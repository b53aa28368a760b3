// Host driver of the B200 GMRES-SDR hot path: solve_cycle / solve /
// solve_sequence (solver.hpp:128-459) over device kernels, with the
// recycle space's U resident in HBM and SU/SAU on the host.
#pragma once

#include "context.hpp"
#include "host_linalg.hpp"
#include "kernels.hpp"
#include "operator.hpp"
#include "sketch.hpp"

#include <chrono>
#include <limits>
#include <map>
#include <string>
#include <vector>

namespace sdr {

struct Config {  // SolverConfig, solver.hpp:48-79
  i64 m = 100, t = 2, k = 20, s = 0;
  double tol = 1e-6, safety_init = 1.4;
  int max_restarts = 10, variant = 0;  // 0 reuse, 1 exact, 2 inexact
  std::uint64_t sketch_seed = 0x5eedULL;
  double rank_tol = 1e-12, breakdown_tol = 1e-14;
  void validate() const;
};

struct Counters {
  i64 matvecs = 0, inner_products = 0, sketch_applies = 0;
  Counters& operator+=(const Counters& o) {
    matvecs += o.matvecs, inner_products += o.inner_products, sketch_applies += o.sketch_applies;
    return *this;
  }
};

struct CycleStat {
  i64 steps = 0;
  double entry_residual = 0, sketched_entry = 0, exit_sres = 0, exit_residual = 0, safety_after = 0, basis_cond = 0;
  i64 deflation_rank = 0;
};

struct Report {  // SolveReport, report.hpp:50-63
  int status = 1;  // max_restarts
  i64 iterations = 0;
  int cycles = 0;
  double rhs_norm = 0.0, final_relative_residual = std::numeric_limits<double>::quiet_NaN();
  Counters counters;
  std::vector<std::pair<i64, double>> sketched, truth;
  std::vector<CycleStat> cycle_stats;
  std::vector<std::string> notes;
  std::string error;
  double seconds = 0.0, device_ms = 0.0, host_wait_ms = 0.0;
  std::map<std::string, double> phase_ms;  // wall-clock breakdown (host view)
};

/// Adds the scope's wall time to rep.phase_ms[name].
struct PhaseTimer {
  Report& r;
  const char* name;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  PhaseTimer(Report& rep, const char* n) : r(rep), name(n) {}
  ~PhaseTimer() { r.phase_ms[name] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
};

/// RecycleSpace (recycle.hpp:31-72): U stays on the device, unnormalised,
/// with per-column scales (u_q = uscale[q] * buf[slot[q]]); SU, SAU on host.
struct Recycle {
  i64 n = 0, nloc = 0, s = 0, ld = 0, cap = 0;
  int provenance = 0;
  DeviceBuffer<double> buf[2];
  int cur = 0;
  std::vector<int> slot;
  std::vector<double> uscale;
  HMat SU, SAU;
  i64 dim() const { return static_cast<i64>(slot.size()); }
  bool empty() const { return slot.empty(); }
  double* col(i64 q) const { return buf[cur].get() + static_cast<i64>(slot[static_cast<size_t>(q)]) * ld; }
  void drop_columns(const std::vector<i64>& cols);
  void clear() {
    slot.clear();
    uscale.clear();
    SU = HMat(s, 0);
    SAU = HMat(s, 0);
    provenance = 0;
  }
  void ensure(i64 nloc_, i64 capacity);
};

struct Callbacks {
  void (*on_iteration)(const void* ev, void* user) = nullptr;
  void (*on_residual)(const void* ev, void* user) = nullptr;
  void* user = nullptr;
};

/// One solve. b, x0: device pointers to this rank's block (x0 may be null).
void solve(Context& c, const DeviceOperator& A, const double* b, const double* x0, bool x0_nonzero, const Config& cfg,
           Recycle& space, const SketchDev* sketch, const Callbacks* cb, double* x_out, Report& rep);

/// refresh_for_new_matrix (recycle.hpp:297-318); exact = true recomputes SAU.
void refresh_recycle(Context& c, Recycle& space, const DeviceOperator& A, const SketchDev& S, bool exact, Counters* cnt);

/// init_krylov + `steps` arnoldi_step through the device pipeline (tests).
void krylov_run(Context& c, const DeviceOperator& A, const SketchDev& S, const double* r0, i64 t, i64 m, i64 steps,
                double breakdown_tol, double* V, double* H, double* SV, double* SAV, i64* j_out, int* breakdown,
                double* r0_norm, i64* counters3);

/// Measurement hook: init + `steps` pipelined Arnoldi steps, then CUDA-event
/// timing of `reps` back-to-back relaunches of the last step's K1 and K2.
void time_step_kernels(Context& c, const DeviceOperator& A, const SketchDev& S, const double* r0, i64 t, i64 m,
                       i64 steps, int reps, double* k1_us, double* k2_us);

/// Builds the default SRDCT sketch of the reference (solver.hpp:283-287).
SketchDev* create_sketch(Context& c, int kind, i64 n, i64 s, std::uint64_t seed, i64 zeta);

/// S x for x (device, this rank's block) -> host out (s values, allreduced).
void sketch_apply(Context& c, const SketchDev& S, const double* x, i64 nloc, i64 row_begin, double* out_host);

}  // namespace sdr
