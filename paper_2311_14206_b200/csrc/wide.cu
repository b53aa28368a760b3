// Arnoldi steps with a long truncation window (min(t, m) > kFusedWindowMax),
// sm_100a.
//
// The fused step kernels (K1's window-dot epilogue, K2 / K2s) keep the
// window's dots, Gram entries and MGS coefficients in registers and are
// compiled for windows of at most kFusedWindowMax vectors; they form the
// coefficients in one pass from Gram entries (inverse compact-WY MGS, equal
// to MGS in exact arithmetic). The reference accepts any t >= 1
// (solver.hpp:61-70; its acceptance test runs t = m, tests/acceptance.cpp:72),
// and over long windows the one-pass coefficients drift from sequential MGS
// by the basis' loss of orthogonality (3e-11 relative in H at a 50-vector
// window). Longer windows therefore run the reference's literal modified
// Gram-Schmidt loop (arnoldi.hpp:91-97) as streaming passes:
//   y = A w_j                         K1 without epilogue / the caller's apply
//   z = A v_j = c_j y, d_0 = w_i0.z   pass 0 (also ||y||^2)
//   z -= h_{i-1} v_{i-1}, d = w_i.z   pass k, i = j-nwin+1+k (in place: z is
//                                     column j+1 of the basis buffer)
//   z -= h_j v_j                      last pass
//   record H part, c_j                k_mgs_record (one thread)
//   ||w_{j+1}||^2, Gram               k_mdot
//   S w_{j+1}                         the standalone sketch kernel
// h_i = c_i (w_i . z) with v_i = c_i w_i (unnormalised basis, device scales).
// Each dot is a fixed-order fold (and one allreduce per pass on several
// ranks) before the next pass reads it: bitwise reproducible.
#include "kernels.hpp"
#include "reduce.cuh"

namespace sdr {

namespace {

constexpr int kThreads = 256;
constexpr int kChunk = 8;  // window columns per k_mdot pass

/// out-partials for [x.x (if self)] and x.col(c0 - q) for q < nq, value-major.
template <int NQ>
__global__ void __launch_bounds__(kThreads) k_mdot(const double* __restrict__ x, const double* __restrict__ V,
                                                   int64_t ldv, int64_t own_off, int c0, int nq, int self, int64_t n,
                                                   double* __restrict__ partials) {
  double acc[NQ + 1];
#pragma unroll
  for (int k = 0; k <= NQ; ++k) acc[k] = 0.0;
  const double* col[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) col[q] = V + static_cast<int64_t>(c0 - (q < nq ? q : 0)) * ldv + own_off;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double xv = x[r];
    if (self) acc[0] = fma(xv, xv, acc[0]);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q < nq) acc[1 + q] = fma(xv, __ldg(col[q] + r), acc[1 + q]);
  }
  // outputs: [self ? x.x : -] then the nq dots, packed from slot 0
  double packed[NQ + 1];
#pragma unroll
  for (int k = 0; k <= NQ; ++k) packed[k] = 0.0;
  if (self) {
#pragma unroll
    for (int k = 0; k <= NQ; ++k) packed[k] = acc[k];
  } else {
#pragma unroll
    for (int k = 0; k < NQ; ++k) packed[k] = acc[k + 1];
  }
  block_partials<NQ + 1>(packed, nq + (self ? 1 : 0), partials);
}

/// Pass k of the MGS loop on z (column j+1's own part). dots = [||y||^2,
/// d_0, d_1, ...] (reduced values of the earlier passes); pass 0 forms
/// z = c_j y. wprev / iprev: the column the previous dot was taken with
/// (z -= c_i^2 d_{k-1} w_i); wnext: the column of this pass's dot (null on
/// the last pass). Partials: pass 0 [||y||^2, d_0], later passes [d_k].
__global__ void __launch_bounds__(kThreads) k_mgs_pass(const double* __restrict__ y, double* __restrict__ z,
                                                       const double* __restrict__ wprev, const double* __restrict__ wnext,
                                                       int64_t n, int k, int iprev, int j,
                                                       const double* __restrict__ recBj,
                                                       const double* __restrict__ cvec, const double* __restrict__ dots,
                                                       double* __restrict__ partials) {
  const double cj = 1.0 / sqrt(recBj[0]);
  double a = 0.0;
  if (k > 0) {
    const double ci = iprev == j ? cj : cvec[iprev];
    a = (ci * dots[k]) * ci;  // h_i c_i, h_i = c_i (w_i . z)
  }
  double acc[2] = {0.0, 0.0};
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double zv;
    if (k == 0) {
      const double yv = y[r];
      acc[0] = fma(yv, yv, acc[0]);
      zv = cj * yv;
    } else {
      zv = fma(-a, __ldg(wprev + r), z[r]);
    }
    z[r] = zv;
    if (wnext) acc[1] = fma(__ldg(wnext + r), zv, acc[1]);
  }
  double out[2] = {k == 0 ? acc[0] : acc[1], acc[1]};
  const int nv = wnext ? (k == 0 ? 2 : 1) : 0;
  if (nv) block_partials<2>(out, nv, partials);
}

/// Record H part of step j (||A v_j||, h_{j-d,j}, c_j) and cvec[j] from the
/// reduced MGS dots: h_i = c_i d_k for the window column i = j - nwin + 1 + k.
__global__ void k_mgs_record(double* __restrict__ rec, int64_t rstride, int T, int j, int nwin,
                             double* __restrict__ cvec, const double* __restrict__ dots) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int b_off = 2 * T + 3;
  const double cj = 1.0 / sqrt(rec[static_cast<int64_t>(j) * rstride + b_off]);
  double* recj = rec + static_cast<int64_t>(j + 1) * rstride;
  recj[0] = dots[0];  // ||y||^2 (the window dots of the A part are not formed on this path)
  double* recH = recj + (T + 1);
  recH[0] = cj * sqrt(dots[0]);
  for (int d = 0; d < T; ++d) {
    double h = 0.0;
    if (d < nwin) {
      const int i = j - d;
      h = (i == j ? cj : cvec[i]) * dots[1 + (nwin - 1 - d)];
    }
    recH[1 + d] = h;
  }
  recH[1 + T] = cj;
  cvec[j] = cj;
}

int stream_grid(const Context& c, int64_t n) {
  const int64_t want = (n + kThreads - 1) / kThreads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(c.num_sms) * 8)));
}

}  // namespace

void launch_window_dots_wide(Context& c, const double* x, const double* V, int64_t ldv, int64_t own_off, int c0,
                             int nq, bool self, int64_t n, double* out) {
  const int g = stream_grid(c, n);
  int done = 0;
  bool first = true;
  while (first || done < nq) {
    const int q = std::min(kChunk, nq - done);
    const bool s = first && self;
    const int nv = q + (s ? 1 : 0);
    if (nv > 0) {
      double* part = c.partials(static_cast<int64_t>(kChunk + 1) * g);
      {
        TimedLaunch t(c, "window_dots");
        k_mdot<kChunk><<<g, kThreads, 0, c.stream>>>(x, V, ldv, own_off, c0 - done, q, s ? 1 : 0, n, part);
        SDR_KERNEL_CHECK();
      }
      launch_fold_partials(c, part, g, nv, true, out);
      out += nv;
    }
    done += q;
    first = false;
  }
}

void launch_mgs_wide(Context& c, const double* y, double* V, int64_t ldv, const VecLayout& lay, int j, int nwin,
                     double* rec, int64_t rstride, int T, double* cvec, double* dots) {
  const int64_t n = lay.nloc;
  const int g = stream_grid(c, n);
  double* z = V + static_cast<int64_t>(j + 1) * ldv + lay.own_off;
  const double* recBj = rec + static_cast<int64_t>(j) * rstride + (2 * T + 3);
  auto col = [&](int i) { return V + static_cast<int64_t>(i) * ldv + lay.own_off; };
  const int i0 = j - nwin + 1;
  for (int k = 0; k <= nwin; ++k) {
    const double* wnext = k < nwin ? col(i0 + k) : nullptr;
    const double* wprev = k > 0 ? col(i0 + k - 1) : nullptr;
    double* part = c.partials(2 * static_cast<int64_t>(g));
    {
      TimedLaunch t(c, "mgs_pass");
      k_mgs_pass<<<g, kThreads, 0, c.stream>>>(y, z, wprev, wnext, n, k, i0 + k - 1, j, recBj, cvec, dots, part);
      SDR_KERNEL_CHECK();
    }
    if (wnext) {
      const int nv = k == 0 ? 2 : 1;
      double* slot = dots + (k == 0 ? 0 : 1 + k);
      launch_fold_partials(c, part, g, nv, true, slot);
      c.allreduce_sum(slot, nv);
    }
  }
  TimedLaunch t(c, "mgs_record");
  k_mgs_record<<<1, 32, 0, c.stream>>>(rec, rstride, T, j, nwin, cvec, dots);
  SDR_KERNEL_CHECK();
}

}  // namespace sdr
