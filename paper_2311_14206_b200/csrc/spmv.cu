// K1 / K6: SELL-32 SpMV with fused epilogues (sm_100a).
//
// Replaces SparseMatrix::apply (sparse.hpp:84-98) and the first half of
// arnoldi_step (arnoldi.hpp:87-97): one warp owns a 32-row slice, every k
// step of the slice loads 32 int32 column indices (128 B) and 32 fp64 values
// (256 B) fully coalesced; x is gathered through the read-only path (the
// whole vector stays L2-resident up to ~60 M rows, so HBM reads x once).
// The slice loop is software-pipelined: the next slice's column indices are
// in flight while the current slice's values and x gathers are consumed.
// Epilogue variants fuse the reductions the step needs into the same pass:
//   MODE 0  y = A x
//   MODE 1  y = A w_j, plus ||y||^2 and y.w_{j-d} for the MGS window (K1);
//           on one GPU the last CTA also forms the MGS coefficients (mgs.cuh)
//   MODE 2  r = b - A x, plus ||r||^2                (verification, K6)
// Algorithmic bytes per row: 12 B per stored entry + 8 B x + 8 B y (+8 B
// per extra window vector in MODE 1, +8 B b in MODE 2).
#include "kernels.hpp"
#include "mgs.cuh"
#include "reduce.cuh"

#include <cstdlib>

namespace sdr {

namespace {

constexpr int kThreads = 256;
constexpr int kBatch = 8;

struct MgsArgs {
  double* rec = nullptr;
  int64_t rstride = 0;
  int T = 0;
  double* cvec = nullptr;
  double* coef = nullptr;  // null: coefficients are formed later (after an allreduce)
};

template <int MODE, int NV, bool PIPE>
__global__ void __launch_bounds__(kThreads, NV > 8 ? 1 : (PIPE ? 2 : 3)) k_sell_spmv(SellView A, const double* __restrict__ x_ext,
                                                         double* __restrict__ y, const double* __restrict__ aux,
                                                         int64_t ldv, int64_t own_off, int64_t halo_lo, int j,
                                                         int nwin, double* __restrict__ partials,
                                                         unsigned* __restrict__ counter, double* __restrict__ out,
                                                         MgsArgs mg) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;

  auto fetch_idx = [&](int64_t sl, int32_t (&cc)[kBatch], int& ll, int64_t& pp) {
    ll = 0;
    pp = 0;
    if (sl < A.nslices) {
      pp = A.slice_ptr[sl];
      ll = static_cast<int>((A.slice_ptr[sl + 1] - pp) >> 5);
    }
#pragma unroll
    for (int k = 0; k < kBatch; ++k) cc[k] = k < ll ? __ldcs(A.cols + pp + k * kSlice + lane) : 0;
  };

  int64_t sl = gw;
  int32_t c[kBatch];
  int len;
  int64_t p0;
  if constexpr (PIPE) fetch_idx(sl, c, len, p0);
  while (sl < A.nslices) {
    if constexpr (!PIPE) fetch_idx(sl, c, len, p0);
    const int64_t row = sl * kSlice + lane;
    const bool live = row < A.nrows;
    // epilogue operands are independent of the product: fetch them first
    double e0 = 0.0, ew[NV > 2 ? NV - 2 : 1];
    if constexpr (MODE == 1) {
      e0 = live ? x_ext[halo_lo + row] : 0.0;
#pragma unroll
      for (int d = 1; d < NV - 1; ++d) ew[d - 1] = (live && d < nwin) ? __ldcs(aux + (j - d) * ldv + own_off + row) : 0.0;
    } else if constexpr (MODE == 2) {
      e0 = live ? __ldcs(aux + row) : 0.0;
    }
    double v[kBatch], xv[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      v[k] = k < len ? __ldcs(A.vals + p0 + k * kSlice + lane) : 0.0;
      xv[k] = k < len ? __ldg(x_ext + c[k]) : 0.0;
    }
    const int64_t sn = sl + nwarps;
    int32_t cn[kBatch];
    int lenn = 0;
    int64_t p0n = 0;
    if constexpr (PIPE) fetch_idx(sn, cn, lenn, p0n);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kBatch; ++k)
      if (k < len) s = fma(v[k], xv[k], s);
    for (int k0 = kBatch; k0 < len; k0 += kBatch) {  // rows longer than one batch
      int32_t c2[kBatch];
      double v2[kBatch], x2[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const bool ok = k0 + k < len;
        c2[k] = ok ? __ldcs(A.cols + p0 + (k0 + k) * kSlice + lane) : 0;
        v2[k] = ok ? __ldcs(A.vals + p0 + (k0 + k) * kSlice + lane) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k) x2[k] = k0 + k < len ? __ldg(x_ext + c2[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < kBatch; ++k)
        if (k0 + k < len) s = fma(v2[k], x2[k], s);
    }
    if (live) {
      if constexpr (MODE == 0) {
        y[row] = s;
      } else if constexpr (MODE == 1) {
        y[row] = s;
        acc[0] = fma(s, s, acc[0]);
        acc[1] = fma(s, e0, acc[1]);
#pragma unroll
        for (int d = 1; d < NV - 1; ++d)
          if (d < nwin) acc[1 + d] = fma(s, ew[d - 1], acc[1 + d]);
      } else {
        const double r = e0 - s;
        y[row] = r;
        acc[0] = fma(r, r, acc[0]);
      }
    }
    sl = sn;
    if constexpr (PIPE) {
      len = lenn;
      p0 = p0n;
#pragma unroll
      for (int k = 0; k < kBatch; ++k) c[k] = cn[k];
    }
  }
  if constexpr (MODE != 0) {
    const int nv = MODE == 1 ? 1 + nwin : 1;
    block_partials<NV>(acc, nv, partials);
    if (last_block_done(counter)) {
      fold_partials(partials, gridDim.x, nv, out);
      if constexpr (MODE == 1) {
        if (mg.coef) {
          __syncthreads();
          if (threadIdx.x == 0) mgs_coefficients<NV - 1>(mg.rec, mg.rstride, mg.T, j, nwin, mg.cvec, mg.coef, true);
        }
      }
      if (threadIdx.x == 0) *counter = 0u;
    }
  }
}

template <class K>
int resident_grid(const Context& c, K kernel, int64_t want_blocks) {
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kernel), kThreads, 0);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want_blocks, static_cast<int64_t>(c.num_sms) * per_sm)));
}

int64_t blocks_for(int64_t nslices) { return (nslices + (kThreads / 32) - 1) / (kThreads / 32); }

/// SDR_K1_PIPE=1 selects the software-pipelined slice loop (fewer resident
/// warps, more bytes in flight per warp); default is the 4-CTA/SM variant.
bool use_pipe() {
  static const int v = [] {
    const char* e = std::getenv("SDR_K1_PIPE");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

template <int NV, bool PIPE>
void spmv_arnoldi_impl(Context& c, const SellView& A, const double* V, int64_t ldv, const VecLayout& lay, int j,
                       int nwin, double* y, double* recA, const MgsArgs& mg) {
  const int g = resident_grid(c, k_sell_spmv<1, NV, PIPE>, blocks_for(A.nslices));
  const double* x_ext = V + j * ldv + lay.ext_shift();
  TimedLaunch t(c, "spmv_arnoldi");
  k_sell_spmv<1, NV, PIPE><<<g, kThreads, 0, c.stream>>>(A, x_ext, y, V, ldv, lay.own_off, lay.halo_lo, j, nwin,
                                                         c.partials(static_cast<int64_t>(NV) * g), c.counters() + 0,
                                                         recA, mg);
  SDR_KERNEL_CHECK();
}

}  // namespace

void launch_spmv(Context& c, const SellView& A, const double* x_ext, double* y) {
  if (A.nrows == 0) return;
  const int g = resident_grid(c, k_sell_spmv<0, 1, false>, blocks_for(A.nslices));
  TimedLaunch t(c, "spmv");
  k_sell_spmv<0, 1, false><<<g, kThreads, 0, c.stream>>>(A, x_ext, y, nullptr, 0, 0, 0, 0, 0, nullptr, nullptr,
                                                         nullptr, MgsArgs{});
  SDR_KERNEL_CHECK();
}

void launch_spmv_arnoldi(Context& c, const SellView& A, const double* V, int64_t ldv, const VecLayout& lay, int j,
                         int nwin, double* y, double* recA, double* rec, int64_t rstride, int T, double* cvec,
                         double* coef) {
  const MgsArgs mg{rec, rstride, T, cvec, coef};
  if (nwin <= 3) {
    if (use_pipe())
      spmv_arnoldi_impl<4, true>(c, A, V, ldv, lay, j, nwin, y, recA, mg);
    else
      spmv_arnoldi_impl<4, false>(c, A, V, ldv, lay, j, nwin, y, recA, mg);
  } else if (nwin <= 7) {
    spmv_arnoldi_impl<8, false>(c, A, V, ldv, lay, j, nwin, y, recA, mg);
  } else if (nwin <= 33) {
    spmv_arnoldi_impl<34, false>(c, A, V, ldv, lay, j, nwin, y, recA, mg);
  } else {
    throw invalid("Arnoldi window of " + std::to_string(nwin) + " vectors exceeds the device limit of 33");
  }
}

void launch_residual(Context& c, const SellView& A, const double* x_ext, const double* b, double* r, double* norm2) {
  const int g = resident_grid(c, k_sell_spmv<2, 1, false>, blocks_for(A.nslices));
  TimedLaunch t(c, "residual");
  k_sell_spmv<2, 1, false><<<g, kThreads, 0, c.stream>>>(A, x_ext, r, b, 0, 0, 0, 0, 0, c.partials(g),
                                                         c.counters() + 1, norm2, MgsArgs{});
  SDR_KERNEL_CHECK();
}

}  // namespace sdr
