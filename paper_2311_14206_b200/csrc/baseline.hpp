// Classical restarted GMRES on the device: the reference's comparison point
// (baseline.hpp:24-216), run on the same box as the GMRES-SDR path so the
// inner-product / synchronisation gap shows up as time.
#pragma once

#include "operator.hpp"
#include "solver.hpp"

namespace sdr {

struct BaselineConfig {  // baseline.hpp:24-39
  i64 m = 100;
  double tol = 1e-6;
  int max_restarts = 10;
  double breakdown_tol = 1e-14;
  void validate() const;
};

/// Largest restart length the device passes support (column accumulators per warp).
constexpr i64 kBaselineMaxM = 255;

/// baseline_gmres (baseline.hpp:51-216). b, x0: device pointers to this
/// rank's block (x0 may be null); x_out: host or device.
void baseline_solve(Context& c, const DeviceOperator& A, const double* b, const double* x0, bool x0_nonzero,
                    const BaselineConfig& cfg, double* x_out, Report& rep);

// ---- device passes (baseline.cu)
struct BaselineStep {
  double* U = nullptr;  // m+1 columns in the operator layout, unnormalised: v_i = vs[i] u_i
  i64 ldu = 0, own_off = 0, nloc = 0, rows_per_cta = 0;
  int G = 0;             // CTAs of every pass (fixed across ranks when distributed)
  double* y = nullptr;   // A u_q, then the once-orthogonalised vector (own rows)
  double* vs = nullptr;  // column scales
  double* H = nullptr;   // (m+1) x m Hessenberg, column-major
  double* R = nullptr;   // rotated copy
  double* cs = nullptr;
  double* sn = nullptr;
  double* g = nullptr;    // rotated rhs (m+1)
  double* est = nullptr;  // |g(q+1)| per step
  double* p1 = nullptr;   // [nv][G] partials, pass 1
  double* p2 = nullptr;   // [nv][G] partials, pass 2
  double* p3 = nullptr;   // [G] norm partials
  int* ctl = nullptr;     // device: {stop, p, breakdown}
  int* ctl_host = nullptr;  // mapped host mirror of ctl
  i64 m = 0;
  double tol_abs = 0.0, breakdown_tol = 0.0;
};
void baseline_cycle_init(Context& c, const BaselineStep& s, double beta);
/// The three orthogonalisation passes of step q (after y = A u_q); between
/// them the caller allreduces the partials on several ranks (`between`).
void baseline_pass(Context& c, const BaselineStep& s, int q, int kind);
void baseline_givens(Context& c, const BaselineStep& s, int q);

}  // namespace sdr
