// Device passes of the classical restarted GMRES baseline (baseline.hpp:98-150
// of the reference): one Arnoldi step orthogonalises A v_q against the whole
// basis. The reference runs modified Gram-Schmidt — q+1 dependent dot/axpy
// pairs, each a grid-wide reduction on a GPU. Here the same projection is
// classical Gram-Schmidt applied twice (CGS2, orthogonal to working precision
// like MGS), which needs three streaming passes per step whatever q is:
//   pass 0  d_i  = u_i . y                          (y = A u_q, raw)
//   pass 1  w'   = vs_q y - sum_i c1_i v_i,   e_i = u_i . w'
//   pass 2  w''  = w' - sum_i c2_i v_i -> u_{q+1},  ||w''||^2,  H(:,q) = c1 + c2
// then one single-warp kernel folds the norm, applies the Givens rotations to
// the new Hessenberg column and sets the stop flag the next steps test.
// Basis columns stay unnormalised (v_i = vs[i] u_i) so no pass waits on a
// norm before it can start. Inner products are counted as the reference
// counts them (one per MGS dot), see baseline_host.cpp.
//
// Every CTA owns a fixed row range and walks it in 256-row sub-chunks: the
// update pass reads u_i[row] thread-per-row (coalesced), the dot pass reads
// the same sub-chunk column by column (warp per column, from L2), so the basis
// is streamed from HBM once per pass. Reductions are deterministic: CTA
// partials [value][G], folded in a fixed order by the consumer.
#include "baseline.hpp"
#include "reduce.cuh"

namespace sdr {

namespace {

constexpr int kT = 256;
constexpr int kWarps = kT / 32;

__device__ __forceinline__ bool stopped(const int* ctl) { return *reinterpret_cast<const volatile int*>(ctl) != 0; }

/// c[v] = sum_g p[v * G + g] for v < nv (warp per value, fixed order).
__device__ __forceinline__ void fold_values(const double* __restrict__ p, int nv, int G, double* c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = warp; v < nv; v += kWarps) {
    double s = 0.0;
    for (int g = lane; g < G; g += 32) s += __ldcg(p + static_cast<int64_t>(v) * G + g);
    s = warp_sum(s);
    if (lane == 0) c[v] = s;
  }
}

template <int KIND, int NVW>
__global__ void __launch_bounds__(kT) k_bl_pass(BaselineStep a, int q) {
  __shared__ double mult[8 * NVW];  // multiplier of raw u_i in the update
  __shared__ double hsum[8 * NVW];  // pass 2, CTA 0: c1 for H(:, q)
  __shared__ double wsub[kT];
  if (stopped(a.ctl)) return;
  const int nv = q + 1, G = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double vq = a.vs[q];
  if constexpr (KIND >= 1) {
    fold_values(KIND == 1 ? a.p1 : a.p2, nv, G, mult);
    if (KIND == 2 && blockIdx.x == 0) fold_values(a.p1, nv, G, hsum);
    __syncthreads();
    for (int i = threadIdx.x; i < nv; i += kT) {
      const double vi = a.vs[i];
      // projection coefficient on the normalised v_i: pass 1 sees w = vs_q y
      const double h = KIND == 1 ? vi * (vq * mult[i]) : vi * mult[i];
      mult[i] = h * vi;
      if (KIND == 2 && blockIdx.x == 0) a.H[i + static_cast<int64_t>(q) * (a.m + 1)] = vi * (vq * hsum[i]) + h;
    }
    __syncthreads();
  }
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * a.rows_per_cta;
  const int64_t r1 = min(r0 + a.rows_per_cta, a.nloc);
  const double* __restrict__ U = a.U + a.own_off;
  double acc[NVW];
#pragma unroll
  for (int k = 0; k < NVW; ++k) acc[k] = 0.0;
  double nacc = 0.0;
  for (int64_t base = r0; base < r1; base += kT) {
    const int64_t row = base + threadIdx.x;
    const bool live = row < r1;
    double w = live ? a.y[row] : 0.0;
    if constexpr (KIND >= 1) {
      if (KIND == 1) w *= vq;
      if (live) {
        const double* up = U + row;
        int i = 0;
        for (; i + 8 <= nv; i += 8) {
          double u[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) u[k] = up[static_cast<int64_t>(i + k) * a.ldu];
#pragma unroll
          for (int k = 0; k < 8; ++k) w = fma(-mult[i + k], u[k], w);
        }
        for (; i < nv; ++i) w = fma(-mult[i], up[static_cast<int64_t>(i) * a.ldu], w);
        if (KIND == 1) a.y[row] = w;
        if (KIND == 2) a.U[static_cast<int64_t>(q + 1) * a.ldu + a.own_off + row] = w;
      }
      if (KIND == 2) nacc = fma(w, w, nacc);
    }
    if constexpr (KIND <= 1) {
      wsub[threadIdx.x] = w;
      __syncthreads();
      const int nrows = r1 - base < kT ? static_cast<int>(r1 - base) : kT;
#pragma unroll
      for (int k = 0; k < NVW; ++k) {
        const int i = warp + kWarps * k;
        if (i < nv) {
          const double* up = U + static_cast<int64_t>(i) * a.ldu + base;
          double s = 0.0;
#pragma unroll
          for (int t = 0; t < kT / 32; ++t) {
            const int rr = lane + 32 * t;
            if (rr < nrows) s = fma(up[rr], wsub[rr], s);
          }
          acc[k] += s;
        }
      }
      __syncthreads();
    }
  }
  if constexpr (KIND <= 1) {
    double* out = KIND == 0 ? a.p1 : a.p2;
#pragma unroll
    for (int k = 0; k < NVW; ++k) {
      const int i = warp + kWarps * k;
      if (i < nv) {
        const double s = warp_sum(acc[k]);
        if (lane == 0) out[static_cast<int64_t>(i) * G + blockIdx.x] = s;
      }
    }
  } else {
    const double v[1] = {nacc};
    block_partials<1>(v, 1, a.p3);
  }
}

/// Norm fold, breakdown test, Givens rotations of column q (baseline.hpp:116-152).
__global__ void k_bl_givens(BaselineStep a, int q) {
  if (stopped(a.ctl)) return;
  const int lane = threadIdx.x;
  double nn = 0.0;
  for (int g = lane; g < a.G; g += 32) nn += __ldcg(a.p3 + g);
  nn = warp_sum(nn);
  if (lane != 0) return;
  const int64_t ldh = a.m + 1;
  double* Hq = a.H + q * ldh;
  double* Rq = a.R + q * ldh;
  const double hn = sqrt(nn);
  double cn2 = hn * hn;
  for (int i = 0; i <= q; ++i) cn2 = fma(Hq[i], Hq[i], cn2);
  const bool bd = hn <= a.breakdown_tol * sqrt(cn2);
  const double hlast = bd ? 0.0 : hn;
  Hq[q + 1] = hlast;
  if (!bd) a.vs[q + 1] = 1.0 / hn;
  double cur = Hq[0];
  for (int i = 0; i < q; ++i) {  // earlier rotations
    const double nxt = Hq[i + 1], c = a.cs[i], s = a.sn[i];
    Rq[i] = c * cur + s * nxt;
    cur = -s * cur + c * nxt;
  }
  const double rr = hypot(cur, hlast);
  const double c = rr > 0.0 ? cur / rr : 1.0, s = rr > 0.0 ? hlast / rr : 0.0;
  a.cs[q] = c;
  a.sn[q] = s;
  Rq[q] = rr;
  Rq[q + 1] = 0.0;
  const double ga = a.g[q];
  a.g[q] = c * ga;
  a.g[q + 1] = -s * ga;
  const double est = fabs(a.g[q + 1]);
  a.est[q] = est;
  const int stop = (est < a.tol_abs || bd || q + 1 == a.m) ? 1 : 0;
  a.ctl[1] = q + 1;
  a.ctl[2] = bd ? 1 : 0;
  a.ctl[0] = stop;
  volatile int* h = a.ctl_host;
  h[1] = q + 1;
  h[2] = bd ? 1 : 0;
  __threadfence_system();
  h[0] = stop;
}

__global__ void k_bl_cycle_init(BaselineStep a, double beta) {
  for (int64_t i = threadIdx.x; i <= a.m; i += blockDim.x) a.g[i] = i == 0 ? beta : 0.0;
  if (threadIdx.x == 0) {
    a.vs[0] = 1.0 / beta;
    a.ctl[0] = 0;
    a.ctl[1] = 0;
    a.ctl[2] = 0;
  }
}

template <int KIND>
void pass_nvw(Context& c, const BaselineStep& s, int q) {
  const int nv = q + 1;
  if (nv <= 8 * 4)
    k_bl_pass<KIND, 4><<<s.G, kT, 0, c.stream>>>(s, q);
  else if (nv <= 8 * 13)
    k_bl_pass<KIND, 13><<<s.G, kT, 0, c.stream>>>(s, q);
  else if (nv <= 8 * 32)
    k_bl_pass<KIND, 32><<<s.G, kT, 0, c.stream>>>(s, q);
  else
    throw invalid("baseline_gmres: restart length exceeds the device limit of " + std::to_string(kBaselineMaxM));
  SDR_KERNEL_CHECK();
}

}  // namespace

void baseline_cycle_init(Context& c, const BaselineStep& s, double beta) {
  TimedLaunch t(c, "baseline_init");
  k_bl_cycle_init<<<1, 128, 0, c.stream>>>(s, beta);
  SDR_KERNEL_CHECK();
}

void baseline_pass(Context& c, const BaselineStep& s, int q, int kind) {
  static const char* names[3] = {"baseline_dots", "baseline_update_dots", "baseline_update_norm"};
  TimedLaunch t(c, names[kind]);
  if (kind == 0)
    pass_nvw<0>(c, s, q);
  else if (kind == 1)
    pass_nvw<1>(c, s, q);
  else
    pass_nvw<2>(c, s, q);
}

void baseline_givens(Context& c, const BaselineStep& s, int q) {
  TimedLaunch t(c, "baseline_givens");
  k_bl_givens<<<1, 32, 0, c.stream>>>(s, q);
  SDR_KERNEL_CHECK();
}

}  // namespace sdr
