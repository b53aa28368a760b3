// MGS window coefficients from the step records (single thread).
//
// With p_i = v_i.(A v_j) (K1 window dots) and the window Gram entries
// G(l,i) = v_l.v_i (earlier K2 passes), the reference's MGS loop
// (arnoldi.hpp:91-97) h_i = v_i.(A v_j - sum_{l<i} h_l v_l) equals
// h_i = p_i - sum_{l<i} h_l G(l,i) in exact arithmetic (inverse compact-WY
// MGS). Basis vectors are stored unnormalised, v_i = c_i w_i.
//
// Record layout (RecLayout in kernels.hpp), record q = step q-1 / column q:
//   A [0, T+1)  ||y||^2, y.w_{j-d}      H [T+1, 2T+3) ||A v_j||, h_{j-d,j}, c_j
//   B [2T+3, ..) ||w||^2, w.w_{-g}, S w
// Outputs coef[0] = c_j (scale of y = A w_j), coef[1+d] = -h_{j-d,j} c_{j-d}.
#pragma once

#include <cstdint>

namespace sdr {

/// recA_in: the step's A values (||y||^2, y.w_{j-d}); null = record row j+1.
/// curB_in: column j's B values (||w_j||^2, w_j.w_{j-g}); null = record row j.
/// Both are given when the caller folded them itself (the deferred path, in
/// which the rows are written by CTA 0 of the same launch).
/// preB / preC: the earlier window columns' B entries
/// (preB[(d-1) MAXT + g] = B entry g of column j-d) and scales
/// (preC[d-1] = cvec[j-d]), when the caller loaded them already.
template <int MAXT>
__device__ __forceinline__ void mgs_coefficients(double* __restrict__ rec, int64_t rstride, int T, int j, int nwin,
                                                 double* __restrict__ cvec, double* __restrict__ coef, bool write_rec,
                                                 const double* recA_in = nullptr, const double* curB_in = nullptr,
                                                 const double* preB = nullptr, const double* preC = nullptr) {
  const int b_off = 2 * T + 3;
  const double* recA = recA_in ? recA_in : rec + static_cast<int64_t>(j + 1) * rstride;
  auto colB = [&](int i, int g) {  // B entry g of column i (g = 0: norm, g >= 1: Gram with column i - g)
    if (i == j && curB_in) return curB_in[g];
    if (i != j && preB) return preB[(j - i - 1) * MAXT + g];
    return rec[static_cast<int64_t>(i) * rstride + b_off + g];
  };
  const double wn2 = colB(j, 0);
  const double cj = 1.0 / sqrt(wn2);
  double ci[MAXT], h[MAXT];
#pragma unroll
  for (int d = 0; d < MAXT; ++d) {
    ci[d] = d == 0 ? cj : (d < nwin ? (preC ? preC[d - 1] : cvec[j - d]) : 0.0);
    h[d] = 0.0;
  }
  // MGS order i = j-nwin+1 .. j  <=>  d = nwin-1 .. 0
#pragma unroll
  for (int d = MAXT - 1; d >= 0; --d) {
    if (d < nwin) {
      const int i = j - d;
      double acc = cj * ci[d] * recA[1 + d];
#pragma unroll
      for (int d2 = MAXT - 1; d2 > d; --d2) {
        if (d2 < nwin) {
          const double gram = colB(i, d2 - d);
          acc -= h[d2] * (ci[d2] * ci[d] * gram);
        }
      }
      h[d] = acc;
    }
  }
  coef[0] = cj;
#pragma unroll
  for (int d = 0; d < MAXT; ++d) coef[1 + d] = d < nwin ? -h[d] * ci[d] : 0.0;
  if (write_rec) {
    double* recH = rec + static_cast<int64_t>(j + 1) * rstride + (T + 1);
    recH[0] = cj * sqrt(recA[0]);
#pragma unroll
    for (int d = 0; d < MAXT; ++d)
      if (d < T) recH[1 + d] = d < nwin ? h[d] : 0.0;
    for (int d = MAXT; d < T; ++d) recH[1 + d] = 0.0;
    recH[1 + T] = cj;
    cvec[j] = cj;
  }
}

}  // namespace sdr
