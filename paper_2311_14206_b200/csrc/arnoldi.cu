// K2: truncated-Arnoldi update pass, plus small vector kernels and the
// tall-skinny basis recombination (K4/K7), sm_100a.
//
// Replaces arnoldi.hpp:91-114 (MGS window, normalisation) and the N-length
// products of solver.hpp:197-198 / recycle.hpp:257-286.
//
// MGS as one pass (inverse-compact-WY form, Swirydowicz et al., "Low
// synchronization Gram-Schmidt and GMRES algorithms", NLAA 2020): with the
// window dots p_i = v_i.(A v_j) from K1 and the window Gram entries
// G(l,i) = v_l.v_i produced by the previous steps' K2, the MGS coefficients
// are h_i = p_i - sum_{l<i} h_l G(l,i) — equal to the reference's
// h_i = v_i.(A v_j - sum_{l<i} h_l v_l) in exact arithmetic, with MGS-class
// loss of orthogonality. Basis vectors are stored unnormalised (w_i) with
// device scales c_i = 1/||w_i||, so normalisation costs no extra pass.
// Algorithmic bytes per row: y + window vectors read, w_{j+1} written.
#include "kernels.hpp"

#include <map>
#include <mutex>
#include <tuple>
#include "mgs.cuh"
#include "reduce.cuh"

#include <map>

namespace sdr {

namespace {

constexpr int kThreads = 256;

template <int MAXT>
__global__ void __launch_bounds__(kThreads) k_update(const double* __restrict__ y, double* __restrict__ V, int64_t ldv,
                                                      int64_t own_off, int64_t n, int j, int nwin, int ngram,
                                                      double* __restrict__ rec, int64_t rstride, int T,
                                                      double* __restrict__ cvec, const double* __restrict__ coef_ready,
                                                      double* __restrict__ partials, unsigned* __restrict__ counter) {
  __shared__ double coef[MAXT + 1];
  const int b_off = 2 * T + 3;
  const double* W[MAXT];
#pragma unroll
  for (int d = 0; d < MAXT; ++d) W[d] = V + static_cast<int64_t>(j - (d < nwin ? d : 0)) * ldv + own_off;
  double* wout = V + static_cast<int64_t>(j + 1) * ldv + own_off;
  // two rows per thread through 16-byte accesses (own_off and ldv are 32-aligned);
  // the first pair is fetched before the coefficient barrier and every later
  // pair one iteration ahead (software pipelining: 2 pairs in flight).
  const int64_t npair = n >> 1;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double2 yv = make_double2(0.0, 0.0), wv[MAXT];
  auto fetch = [&](int64_t q, double2& yo, double2 (&wo)[MAXT]) {
    yo = __ldcs(reinterpret_cast<const double2*>(y) + q);
#pragma unroll
    for (int d = MAXT - 1; d >= 0; --d)
      if (d < nwin) wo[d] = __ldg(reinterpret_cast<const double2*>(W[d]) + q);
  };
  if (p < npair) fetch(p, yv, wv);
  if (coef_ready) {
    if (threadIdx.x <= MAXT) coef[threadIdx.x] = threadIdx.x <= nwin ? coef_ready[threadIdx.x] : 0.0;
  } else if (threadIdx.x == 0) {
    // multi-GPU: records were allreduced after K1; every CTA forms the same
    // coefficients, CTA 0 publishes them in the record
    mgs_coefficients<MAXT>(rec, rstride, T, j, nwin, cvec, coef, blockIdx.x == 0);
  }
  __syncthreads();

  double acc[MAXT];
#pragma unroll
  for (int k = 0; k < MAXT; ++k) acc[k] = 0.0;
  double cf[MAXT + 1];
#pragma unroll
  for (int k = 0; k <= MAXT; ++k) cf[k] = coef[k];

  while (p < npair) {
    const int64_t pn = p + stride;
    double2 yn = make_double2(0.0, 0.0), wn[MAXT];
    if (pn < npair) fetch(pn, yn, wn);
    double w0 = cf[0] * yv.x, w1 = cf[0] * yv.y;
#pragma unroll
    for (int d = MAXT - 1; d >= 0; --d)
      if (d < nwin) {
        w0 = fma(cf[1 + d], wv[d].x, w0);
        w1 = fma(cf[1 + d], wv[d].y, w1);
      }
    reinterpret_cast<double2*>(wout)[p] = make_double2(w0, w1);
    acc[0] = fma(w0, w0, fma(w1, w1, acc[0]));
#pragma unroll
    for (int g = 1; g < MAXT; ++g)
      if (g <= ngram) acc[g] = fma(w0, wv[g - 1].x, fma(w1, wv[g - 1].y, acc[g]));
    p = pn;
    yv = yn;
#pragma unroll
    for (int d = 0; d < MAXT; ++d) wv[d] = wn[d];
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t r = n - 1;
    double w = cf[0] * y[r];
    double wv[MAXT];
#pragma unroll
    for (int d = MAXT - 1; d >= 0; --d)
      if (d < nwin) {
        wv[d] = W[d][r];
        w = fma(cf[1 + d], wv[d], w);
      }
    wout[r] = w;
    acc[0] = fma(w, w, acc[0]);
#pragma unroll
    for (int g = 1; g < MAXT; ++g)
      if (g <= ngram) acc[g] = fma(w, wv[g - 1], acc[g]);
  }
  block_partials<MAXT>(acc, 1 + ngram, partials);
  if (last_block_done(counter)) {
    double* recB = rec + static_cast<int64_t>(j + 1) * rstride + b_off;
    fold_partials(partials, gridDim.x, 1 + ngram, recB);
    if (threadIdx.x == 0) {
      for (int g = 1 + ngram; g < T; ++g) recB[g] = 0.0;
      *counter = 0u;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_copy_norm(const double* __restrict__ src, double* __restrict__ dst,
                                                         int64_t n, double* __restrict__ partials,
                                                         unsigned* __restrict__ counter, double* __restrict__ out) {
  double acc[1] = {0.0};
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = src[i];
    dst[i] = v;
    acc[0] = fma(v, v, acc[0]);
  }
  block_partials<1>(acc, 1, partials);
  if (last_block_done(counter)) {
    fold_partials(partials, gridDim.x, 1, out);
    if (threadIdx.x == 0) *counter = 0u;
  }
}

/// Column sums of squares of C (n x ncol, ldc): grid (chunks, ncol), CTA
/// partials then a per-column ordered fold (second kernel) — deterministic.
__global__ void __launch_bounds__(kThreads) k_col_sumsq(const double* __restrict__ C, int64_t ldc, int64_t n,
                                                         int64_t chunk, double* __restrict__ partials) {
  const int col = blockIdx.y;
  const double* x = C + static_cast<int64_t>(col) * ldc;
  const int64_t beg = static_cast<int64_t>(blockIdx.x) * chunk, end = min(n, beg + chunk);
  double acc[1] = {0.0};
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) acc[0] = fma(x[i], x[i], acc[0]);
  __shared__ double red[kThreads / 32];
  const double w = warp_sum(acc[0]);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) v += red[k];
    partials[static_cast<int64_t>(col) * gridDim.x + blockIdx.x] = v;
  }
}

__global__ void k_col_fold(const double* __restrict__ partials, int nchunks, int ncol, double* __restrict__ out) {
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (col >= ncol) return;
  double v = 0.0;
  for (int k = lane; k < nchunks; k += 32) v += partials[static_cast<int64_t>(col) * nchunks + k];
  v = warp_sum(v);
  if (lane == 0) out[col] = v;
}

__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) y[i] += a * x[i];
}

__global__ void k_scale_copy(double a, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = a * x[i];
}

/// out_o = sum_i coef[i*nout + o] * in_i, o < nout (<= NOUT); optional
/// ||out_o||^2 via the deterministic grid fold. Each thread owns RPT
/// consecutive rows (RPT-wide vector loads) and keeps U input columns in
/// flight; input pointers and coefficients are broadcast from shared memory,
/// so every input column is streamed from HBM exactly once.
template <int NOUT, int RPT, int U>
__global__ void __launch_bounds__(kThreads) k_tallskinny(const double* const* __restrict__ in, int nin,
                                                          const double* __restrict__ coef, int nout,
                                                          double* const* __restrict__ out, int64_t n,
                                                          double* __restrict__ partials,
                                                          unsigned* __restrict__ counter, double* __restrict__ norms) {
  extern __shared__ double cs[];  // nin * NOUT coefficients, then nin pointers
  const double** ptr = reinterpret_cast<const double**>(cs + nin * NOUT);
  for (int q = threadIdx.x; q < nin * NOUT; q += blockDim.x) {
    const int i = q / NOUT, o = q % NOUT;
    cs[q] = o < nout ? coef[i * nout + o] : 0.0;
  }
  for (int i = threadIdx.x; i < nin; i += blockDim.x) ptr[i] = in[i];
  __syncthreads();
  double nrm[NOUT];
#pragma unroll
  for (int o = 0; o < NOUT; ++o) nrm[o] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * RPT;
  const int64_t nfull = n / RPT * RPT;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * RPT; r < n; r += stride) {
    double a[NOUT][RPT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
#pragma unroll
      for (int q = 0; q < RPT; ++q) a[o][q] = 0.0;
    const bool full = r < nfull;
    for (int i0 = 0; i0 < nin; i0 += U) {
      double v[U][RPT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u < nin) {
          const double* src = ptr[i0 + u] + r;
          if (full && RPT == 2) {
            const double2 t = __ldcs(reinterpret_cast<const double2*>(src));
            v[u][0] = t.x;
            v[u][RPT - 1] = t.y;
          } else if (full && RPT == 4) {
            const double2 t0 = __ldcs(reinterpret_cast<const double2*>(src));
            const double2 t1 = __ldcs(reinterpret_cast<const double2*>(src) + 1);
            v[u][0] = t0.x;
            v[u][1 % RPT] = t0.y;
            v[u][2 % RPT] = t1.x;
            v[u][3 % RPT] = t1.y;
          } else {
#pragma unroll
            for (int q = 0; q < RPT; ++q) v[u][q] = r + q < n ? __ldcs(src + q) : 0.0;
          }
        } else {
#pragma unroll
          for (int q = 0; q < RPT; ++q) v[u][q] = 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u < nin) {
#pragma unroll
          for (int o = 0; o < NOUT; ++o) {
            const double cf = cs[(i0 + u) * NOUT + o];
#pragma unroll
            for (int q = 0; q < RPT; ++q) a[o][q] = fma(cf, v[u][q], a[o][q]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      if (o < nout) {
        double* dst = out[o] + r;
        if (full && RPT == 2) {
          *reinterpret_cast<double2*>(dst) = make_double2(a[o][0], a[o][RPT - 1]);
        } else if (full && RPT == 4) {
          reinterpret_cast<double2*>(dst)[0] = make_double2(a[o][0], a[o][1 % RPT]);
          reinterpret_cast<double2*>(dst)[1] = make_double2(a[o][2 % RPT], a[o][3 % RPT]);
        } else {
#pragma unroll
          for (int q = 0; q < RPT; ++q)
            if (r + q < n) dst[q] = a[o][q];
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q)
          if (r + q < n) nrm[o] = fma(a[o][q], a[o][q], nrm[o]);
      }
    }
  }
  if (norms) {
    block_partials<NOUT>(nrm, nout, partials);
    if (last_block_done(counter)) {
      fold_partials(partials, gridDim.x, nout, norms);
      if (threadIdx.x == 0) *counter = 0u;
    }
  }
}

/// Dense tall-skinny product of the recycle update, one pass over the inputs:
/// C (n x nout, ldc) = [A1 (n x k1) | A2 (n x k2)] B ((k1+k2) x nout), plus the
/// CTA partials of the column sums of squares (CTA-major, folded by
/// k_col_fold). Each thread owns two rows (one 16-byte load per input
/// column); UD input columns are in flight one group ahead of the FMAs, so
/// the HBM stream does not wait on the arithmetic. Coefficients are read from
/// shared memory as 16-byte pairs.
template <int NOUT, int UD>
__global__ void __launch_bounds__(kThreads, NOUT > 12 ? 1 : 2) k_tsgemm(const double* __restrict__ A1, int64_t lda1, int k1,
                                                        const double* __restrict__ A2, int64_t lda2, int k2,
                                                        const double* __restrict__ B, int nout, double* __restrict__ C,
                                                        int64_t ldc, int64_t npairs, double* __restrict__ partials) {
  extern __shared__ double bs[];  // (k1 + k2) x NOUT, row-major by input
  const int kk = k1 + k2;
  for (int q = threadIdx.x; q < kk * NOUT; q += blockDim.x) {
    const int i = q / NOUT, o = q % NOUT;
    bs[q] = o < nout ? B[static_cast<int64_t>(o) * kk + i] : 0.0;
  }
  __syncthreads();
  double nrm[NOUT];
#pragma unroll
  for (int o = 0; o < NOUT; ++o) nrm[o] = 0.0;
  auto col = [&](int i) -> const double2* {
    return reinterpret_cast<const double2*>(i < k1 ? A1 + static_cast<int64_t>(i) * lda1
                                                   : A2 + static_cast<int64_t>(i - k1) * lda2);
  };
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t pr = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; pr < npairs; pr += stride) {
    double2 acc[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) acc[o] = make_double2(0.0, 0.0);
    double2 cur[UD], nxt[UD];
#pragma unroll
    for (int u = 0; u < UD; ++u) cur[u] = u < kk ? __ldcs(col(u) + pr) : make_double2(0.0, 0.0);
    for (int i0 = 0; i0 < kk; i0 += UD) {
#pragma unroll
      for (int u = 0; u < UD; ++u) nxt[u] = i0 + UD + u < kk ? __ldcs(col(i0 + UD + u) + pr) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < UD; ++u) {
        if (i0 + u < kk) {
          const double2* cf2 = reinterpret_cast<const double2*>(bs + (i0 + u) * NOUT);
#pragma unroll
          for (int o2 = 0; o2 < NOUT / 2; ++o2) {
            const double2 cf = cf2[o2];
            acc[2 * o2] = make_double2(fma(cf.x, cur[u].x, acc[2 * o2].x), fma(cf.x, cur[u].y, acc[2 * o2].y));
            acc[2 * o2 + 1] = make_double2(fma(cf.y, cur[u].x, acc[2 * o2 + 1].x), fma(cf.y, cur[u].y, acc[2 * o2 + 1].y));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UD; ++u) cur[u] = nxt[u];
    }
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      if (o < nout) {
        reinterpret_cast<double2*>(C + static_cast<int64_t>(o) * ldc)[pr] = acc[o];
        nrm[o] = fma(acc[o].x, acc[o].x, fma(acc[o].y, acc[o].y, nrm[o]));
      }
    }
  }
  __shared__ double red[NOUT][kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 0; o < NOUT; ++o) {
    const double v = warp_sum(nrm[o]);
    if (lane == 0) red[o][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < nout) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += red[threadIdx.x][w];
    partials[static_cast<int64_t>(threadIdx.x) * gridDim.x + blockIdx.x] = v;
  }
}

/// Recycle product for many outputs (U_new = [A1 A2] B, nout <= NO <= 24),
/// norm partials fused. Shared-memory tiled: persistent CTAs (two per SM)
/// walk 256-row tiles; each tile's inputs stream through a double-buffered
/// 16-input x 256-row chunk filled by cp.async (16-byte pieces, zero-filled
/// past the last row and input), so the HBM stream runs ahead of the
/// arithmetic. The arithmetic is fp64 tensor-core mma (m8n8k4, DMMA): a warp
/// owns 32 rows x NO outputs = 4 x NO/8 accumulator tiles, one 8-byte shared
/// load per m-tile and per n-tile feeds 32·NO/8 FMAs per lane. One pass over
/// the inputs, one write of the outputs (cuBLAS took two GEMMs, the second
/// re-reading and re-writing the outputs).
constexpr int kRgRows = 256, kRgKC = 16, kRgLda = kRgRows + 8;  // padded: k-rows alternate bank halves

__device__ __forceinline__ void cp_async16z(void* dst, const void* src, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}

template <int NO>
__global__ void __launch_bounds__(kThreads, 2) k_rgemm(const double* __restrict__ A1, int64_t lda1, int k1,
                                                       const double* __restrict__ A2, int64_t lda2, int k2,
                                                       const double* __restrict__ B, int nout, double* __restrict__ C,
                                                       int64_t ldc, int64_t n, double* __restrict__ partials) {
  constexpr int NT = NO / 8;  // 8-output tiles
  extern __shared__ __align__(16) double rg_sm[];
  double* As = rg_sm;                        // [2][kRgKC][kRgLda]
  double* Bs = rg_sm + 2 * kRgKC * kRgLda;   // [K + 4][NO], zero rows past K
  const int K = k1 + k2, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Kp = (K + 3) & ~3;
  for (int q = tid; q < Kp * NO; q += blockDim.x) {
    const int i = q / NO, o = q % NO;
    Bs[q] = (o < nout && i < K) ? B[static_cast<int64_t>(o) * K + i] : 0.0;
  }
  const int g8 = lane >> 2, t4 = lane & 3;  // mma fragment coordinates
  const int64_t ntiles = (n + kRgRows - 1) / kRgRows;
  const int nch = (K + kRgKC - 1) / kRgKC;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nstage = my_tiles * nch;
  auto issue = [&](int64_t st, int buf) {
    const int64_t tile = blockIdx.x + (st / nch) * gridDim.x;
    const int ch = static_cast<int>(st % nch);
    const int64_t row0 = tile * kRgRows;
    double* dstb = As + buf * (kRgKC * kRgLda);
    // a warp copies 32 consecutive 16-byte pieces (512 B) of one input column
    // per instruction; each thread keeps its row pair and walks the inputs
    const int pc = tid & (kRgRows / 2 - 1), iw = tid / (kRgRows / 2);
    const int64_t r = row0 + 2 * pc;
    const int rbytes = r + 1 < n ? 16 : (r < n ? 8 : 0);
#pragma unroll
    for (int u = 0; u < kRgKC * (kRgRows / 2) / kThreads; ++u) {
      const int ii = iw + u * (kThreads / (kRgRows / 2));
      const int i = ch * kRgKC + ii;
      const double* src = A1;
      int bytes = 0;
      if (i < K && rbytes) {
        src = (i < k1 ? A1 + static_cast<int64_t>(i) * lda1 : A2 + static_cast<int64_t>(i - k1) * lda2) + r;
        bytes = rbytes;
      }
      cp_async16z(dstb + ii * kRgLda + 2 * pc, src, bytes);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][NT][2], nrm[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) nrm[nt][0] = nrm[nt][1] = 0.0;
  if (nstage > 0) issue(0, 0);
  for (int64_t st = 0; st < nstage; ++st) {
    const int buf = static_cast<int>(st & 1);
    const int ch = static_cast<int>(st % nch);
    if (st + 1 < nstage) {
      issue(st + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // chunk st (and, at st = 0, the coefficients) visible to every thread
    if (ch == 0) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    }
    // warp = 32 rows (4 m-tiles of 8) x NO outputs; fp64 mma m8n8k4 per
    // (m-tile, n-tile, 4 inputs); rows past K are zero in Bs, so partial
    // k-steps add nothing
    const double* ab = As + buf * (kRgKC * kRgLda) + warp * 32 + g8;
    const double* bb = Bs + (ch * kRgKC) * NO + g8;
    const int ksteps = (min(kRgKC, K - ch * kRgKC) + 3) >> 2;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int kr = ks * 4 + t4;
      double a[4], b[NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = ab[kr * kRgLda + mt * 8];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = bb[kr * NO + nt * 8];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
                       : "d"(a[mt]), "d"(b[nt]));
    }
    if (ch == nch - 1) {  // tile complete: C(row, col) = acc[mt][nt][e], row = 8 mt + g8, col = 8 nt + 2 t4 + e
      const int64_t row = (blockIdx.x + (st / nch) * gridDim.x) * kRgRows + warp * 32 + g8;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        if (row + mt * 8 < n) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = nt * 8 + 2 * t4 + e;
              if (col < nout) {
                C[static_cast<int64_t>(col) * ldc + row + mt * 8] = acc[mt][nt][e];
                nrm[nt][e] = fma(acc[mt][nt][e], acc[mt][nt][e], nrm[nt][e]);
              }
            }
        }
      }
    }
    __syncthreads();  // buffer buf is refilled by the issue of stage st + 2
  }
  // norms: lanes with the same t4 hold the same columns; fold over g8, then warps
  __shared__ double red[NO][kThreads / 32];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = nrm[nt][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (g8 == 0) red[nt * 8 + 2 * t4 + e][warp] = v;
    }
  __syncthreads();
  if (tid < nout) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += red[tid][w];
    partials[static_cast<int64_t>(tid) * gridDim.x + blockIdx.x] = v;
  }
}

template <int NO>
void rgemm_impl(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                const double* B, int nout, double* C, int64_t ldc, int64_t n, double* norms2, double* scratch) {
  auto kern = k_rgemm<NO>;
  const size_t smem = sizeof(double) * (static_cast<size_t>(2 * kRgKC * kRgLda) + static_cast<size_t>(k1 + k2 + 4) * NO);
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  const int64_t ntiles = (n + kRgRows - 1) / kRgRows;
  const int per_sm = std::max(1, blocks_per_sm(reinterpret_cast<const void*>(kern), kThreads, smem));
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, static_cast<int64_t>(c.num_sms) * per_sm)));
  double* part = scratch ? scratch : c.partials(static_cast<int64_t>(nout) * g);
  {
    TimedLaunch t(c, "recycle_gemm");
    kern<<<g, kThreads, smem, c.stream>>>(A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, part);
    SDR_KERNEL_CHECK();
  }
  TimedLaunch t(c, "col_norms");
  k_col_fold<<<(nout + 7) / 8, 256, 0, c.stream>>>(part, g, nout, norms2);
  SDR_KERNEL_CHECK();
}

int stream_grid(const Context& c, int64_t n, int per_thread = 1) {
  const int64_t want = (n / per_thread + kThreads - 1) / kThreads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(c.num_sms) * 8)));
}

template <int MAXT>
void update_impl(Context& c, const double* y, double* V, int64_t ldv, const VecLayout& lay, int j, int nwin,
                 int ngram, double* rec, const RecLayout& L, double* cvec, const double* coef_ready) {
  // persistent: one resident wave, each thread streams several pairs
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(k_update<MAXT>), kThreads, 0);
  const int64_t want = (lay.nloc / 2 + kThreads - 1) / kThreads;
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(c.num_sms) * per_sm)));
  TimedLaunch t(c, "update");
  k_update<MAXT><<<g, kThreads, 0, c.stream>>>(y, V, ldv, lay.own_off, lay.nloc, j, nwin, ngram, rec, L.stride, L.T,
                                               cvec, coef_ready, c.partials(static_cast<int64_t>(MAXT) * g),
                                               c.counters() + 2);
  SDR_KERNEL_CHECK();
}

template <int NOUT, int RPT, int U>
void tallskinny_impl(Context& c, const double* const* in, int nin, const double* coef, int nout, double* const* out,
                     int64_t n, double* norms2) {
  auto kern = k_tallskinny<NOUT, RPT, U>;
  const size_t smem = sizeof(double) * static_cast<size_t>(nin) * NOUT + sizeof(void*) * static_cast<size_t>(nin);
  if (smem > 48 * 1024)
    SDR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), kThreads, smem);
  const int64_t want = (n / RPT + kThreads - 1) / kThreads;
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(c.num_sms) * per_sm)));
  TimedLaunch t(c, NOUT == 1 ? "correction" : "tallskinny");
  kern<<<g, kThreads, smem, c.stream>>>(in, nin, coef, nout, out, n, c.partials(static_cast<int64_t>(NOUT) * g),
                                        c.counters() + 3, norms2);
  SDR_KERNEL_CHECK();
}

}  // namespace

int blocks_per_sm(const void* kernel, int threads, size_t smem) {
  // shared by every context / thread of the process: guarded, keyed by device
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, kernel, smem * 4096 + static_cast<size_t>(threads));
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  cache[key] = n;
  return n;
}

void ensure_dyn_smem(const void* kernel, size_t bytes) {
  // the 48 KB default covers static + dynamic shared memory together: opt in
  // early enough for kernels with a few KB of static buffers
  if (bytes <= 32 * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  SDR_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  size_t& have = done[std::make_pair(dev, kernel)];
  if (bytes > have) {
    SDR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    have = bytes;
  }
}

void launch_update(Context& c, const double* y, double* V, int64_t ldv, const VecLayout& lay, int j, int nwin,
                   int ngram, double* rec, const RecLayout& L, double* cvec, const double* coef_ready) {
  const int need = std::max(nwin, ngram + 1);
  if (need <= 4)
    update_impl<4>(c, y, V, ldv, lay, j, nwin, ngram, rec, L, cvec, coef_ready);
  else if (need <= 8)
    update_impl<8>(c, y, V, ldv, lay, j, nwin, ngram, rec, L, cvec, coef_ready);
  else if (need <= 33)
    update_impl<33>(c, y, V, ldv, lay, j, nwin, ngram, rec, L, cvec, coef_ready);
  else
    throw invalid("Arnoldi window of " + std::to_string(nwin) + " vectors exceeds the device limit of 33");
}

void launch_copy_norm(Context& c, const double* src, double* dst, int64_t n, double* norm2) {
  const int g = stream_grid(c, n);
  TimedLaunch t(c, "copy_norm");
  k_copy_norm<<<g, kThreads, 0, c.stream>>>(src, dst, n, c.partials(g), c.counters() + 4, norm2);
  SDR_KERNEL_CHECK();
}

template <int NOUT>
void tsgemm_impl(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                 const double* B, int nout, double* C, int64_t ldc, int64_t n, double* norms2, double* scratch) {
  constexpr int UD = NOUT <= 8 ? 8 : (NOUT <= 12 ? 4 : 2);
  auto kern = k_tsgemm<NOUT, UD>;
  const size_t smem = sizeof(double) * static_cast<size_t>(k1 + k2) * NOUT;
  if (smem > 48 * 1024)
    SDR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), kThreads, smem);
  const int64_t npairs = n / 2;
  const int g = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((npairs + kThreads - 1) / kThreads, static_cast<int64_t>(c.num_sms) * per_sm)));
  double* part = scratch ? scratch : c.partials(static_cast<int64_t>(nout) * g);
  {
    TimedLaunch t(c, "recycle_gemm");
    kern<<<g, kThreads, smem, c.stream>>>(A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, npairs, part);
    SDR_KERNEL_CHECK();
  }
  TimedLaunch t(c, "col_norms");
  k_col_fold<<<(nout + 7) / 8, 256, 0, c.stream>>>(part, g, nout, norms2);
  SDR_KERNEL_CHECK();
}

namespace {
__global__ void k_fold_partials(const double* __restrict__ partials, int G, int nv, int value_major,
                                double* __restrict__ out) {
  const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (v >= nv) return;
  double a = 0.0;
  a = warp_sum(value_major ? strided_sum(partials + static_cast<int64_t>(v) * G, 1, lane, G, 32)
                           : strided_sum(partials + v, nv, lane, G, 32));
  if (lane == 0) out[v] = a;
}
}  // namespace

namespace {
__global__ void k_fold_partials2(const double* __restrict__ p1, int G1, const double* __restrict__ p2, int G2, int nv,
                                 double* __restrict__ out) {
  const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (v >= nv) return;
  double a = 0.0;
  a = strided_sum(p1 + static_cast<int64_t>(v) * G1, 1, lane, G1, 32);
  a = strided_sum(p2 + static_cast<int64_t>(v) * G2, 1, lane, G2, 32, a);
  a = warp_sum(a);
  if (lane == 0) out[v] = a;
}
}  // namespace

void launch_fold_partials2(Context& c, const double* p1, int G1, const double* p2, int G2, int nv, double* out) {
  TimedLaunch t(c, "fold_partials");
  k_fold_partials2<<<(nv + 7) / 8, 256, 0, c.stream>>>(p1, G1, p2, G2, nv, out);
  SDR_KERNEL_CHECK();
}

void launch_fold_partials(Context& c, const double* partials, int G, int nv, bool value_major, double* out) {
  TimedLaunch t(c, "fold_partials");
  k_fold_partials<<<(nv + 7) / 8, 256, 0, c.stream>>>(partials, G, nv, value_major ? 1 : 0, out);
  SDR_KERNEL_CHECK();
}

bool rgemm_supported(int nout, int k, int64_t lda1, int64_t lda2) {
  const size_t smem = sizeof(double) * (static_cast<size_t>(2 * kRgKC * kRgLda) + static_cast<size_t>(k + 4) * 24);
  return nout >= 1 && nout <= 24 && k >= 1 && lda1 % 2 == 0 && lda2 % 2 == 0 && smem <= 227 * 1024;
}

void launch_rgemm(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                  const double* B, int nout, double* C, int64_t ldc, int64_t n, double* norms2, double* scratch) {
  if (!rgemm_supported(nout, k1 + k2, lda1, lda2)) throw invalid("recycle product: unsupported shape");
  if (nout <= 8)
    rgemm_impl<8>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
  else if (nout <= 16)
    rgemm_impl<16>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
  else
    rgemm_impl<24>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
}

bool tsgemm_supported(int nout, int64_t n, int64_t lda1, int64_t lda2, int64_t ldc) {
  return nout >= 1 && nout <= 24 && n % 2 == 0 && lda1 % 2 == 0 && lda2 % 2 == 0 && ldc % 2 == 0;
}

int64_t tsgemm_scratch_size(int num_sms) { return static_cast<int64_t>(24) * num_sms * 8; }  // also k_rgemm (<= 2 CTAs / SM)

void launch_tsgemm(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                   const double* B, int nout, double* C, int64_t ldc, int64_t n, double* norms2, double* scratch) {
  if (!tsgemm_supported(nout, n, lda1, lda2, ldc)) throw invalid("tall-skinny product: unsupported shape");
  if (nout <= 4)
    tsgemm_impl<4>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
  else if (nout <= 8)
    tsgemm_impl<8>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
  else if (nout <= 12)
    tsgemm_impl<12>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
  else if (nout <= 16)
    tsgemm_impl<16>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
  else
    tsgemm_impl<24>(c, A1, lda1, k1, A2, lda2, k2, B, nout, C, ldc, n, norms2, scratch);
}

void launch_col_norms2(Context& c, const double* C, int64_t ldc, int64_t n, int ncol, double* norms2, double* scratch) {
  if (ncol == 0) return;
  const int chunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, 4 * c.num_sms / std::max(1, ncol) + 1)));
  const int64_t chunk = (n + chunks - 1) / chunks;
  double* part = scratch ? scratch : c.partials(static_cast<int64_t>(chunks) * ncol);
  {
    TimedLaunch t(c, "col_norms");
    k_col_sumsq<<<dim3(chunks, ncol), kThreads, 0, c.stream>>>(C, ldc, n, chunk, part);
    SDR_KERNEL_CHECK();
  }
  TimedLaunch t(c, "col_norms");
  k_col_fold<<<(ncol + 7) / 8, 256, 0, c.stream>>>(part, chunks, ncol, norms2);
  SDR_KERNEL_CHECK();
}

void launch_axpy(Context& c, double a, const double* x, double* y, int64_t n) {
  if (n == 0) return;
  TimedLaunch t(c, "axpy");
  k_axpy<<<stream_grid(c, n), kThreads, 0, c.stream>>>(a, x, y, n);
  SDR_KERNEL_CHECK();
}

void launch_scale_copy(Context& c, double a, const double* x, double* y, int64_t n) {
  if (n == 0) return;
  TimedLaunch t(c, "scale_copy");
  k_scale_copy<<<stream_grid(c, n), kThreads, 0, c.stream>>>(a, x, y, n);
  SDR_KERNEL_CHECK();
}

void launch_tallskinny(Context& c, const double* const* in, int nin, const double* coef, int nout,
                       double* const* out, int64_t n, double* norms2) {
  if (nout <= 1)
    tallskinny_impl<1, 4, 8>(c, in, nin, coef, nout, out, n, norms2);
  else if (nout <= 8)
    tallskinny_impl<8, 2, 8>(c, in, nin, coef, nout, out, n, norms2);
  else if (nout <= 16)
    tallskinny_impl<16, 2, 4>(c, in, nin, coef, nout, out, n, norms2);
  else if (nout <= 24)
    tallskinny_impl<24, 2, 4>(c, in, nin, coef, nout, out, n, norms2);
  else if (nout <= 32)
    tallskinny_impl<32, 1, 8>(c, in, nin, coef, nout, out, n, norms2);
  else
    throw invalid("tall-skinny product with " + std::to_string(nout) + " outputs exceeds 32 per launch");
}

}  // namespace sdr
