// K1 / K6: SELL-32 SpMV with fused epilogues (sm_100a).
//
// Replaces SparseMatrix::apply (sparse.hpp:84-98) and the first half of
// arnoldi_step (arnoldi.hpp:87-97). One warp owns a 32-row slice; every k
// step of the slice loads 32 fp64 values (256 B) fully coalesced.
// Two storage forms (operator.cu chooses per matrix):
//   SELL      32 int32 column indices per k step; x gathered through them.
//   SELL-DIA  when every slice's entries lie on <= 16 distinct diagonals
//             (banded / stencil operators; gaps stored as explicit zeros),
//             D diagonals per slice (padded to the operator's maximum), one
//             int32 offset per (slice, k): 8 instead of 12 bytes per entry,
//             and x[row + off] is a coalesced load that does not wait on an
//             index load (offsets are fetched a slice ahead, one per lane,
//             and broadcast with shuffles).
// Row sums run in CSR (increasing column) order like the reference.
// Epilogue variants fuse the reductions the step needs into the same pass:
//   MODE 0  y = A x
//   MODE 1  y = A w_j, plus ||y||^2 and y.w_{j-d} for the MGS window (K1);
//           on one GPU the last CTA also forms the MGS coefficients (mgs.cuh)
//   MODE 2  r = b - A x, plus ||r||^2                (verification, K6)
//   MODE 3  y = A x unless the int flag at aux is set (speculatively
//           enqueued steps of the classical baseline, baseline.cu)
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
  // window columns loaded without the evict-first hint: on one GPU when a
  // step's vectors fit in L2, so the update kernel that follows re-reads
  // w_{j-1} from L2 (C2: K2 26.5 -> 25.1 us in-solve; C3 14.7 -> 14.5 us)
  int wkeep = 0;
};

/// Row sums of one 32-row slice (lane = row), CSR order.
/// FMT 0: SELL (column index per entry); FMT > 0: SELL-DIA with FMT
/// diagonals (compile-time, loop fully unrolled so every load of the slice
/// is in flight at once); FMT < 0: SELL-DIA with A.dia_d diagonals.
template <int FMT>
__device__ __forceinline__ double slice_row_sum(const SellView& A, const double* __restrict__ x_ext, int64_t sl,
                                                int64_t row, int64_t halo_lo, int lane, int cur_off) {
  double s = 0.0;
  if constexpr (FMT > 0) {
    const double* vp = A.vals + sl * kSlice * FMT + lane;
    const int64_t rx = halo_lo + row;
    double v[FMT], xv[FMT];
#pragma unroll
    for (int k = 0; k < FMT; ++k) {
      const int o = __shfl_sync(0xffffffffu, cur_off, k);
      int64_t cidx = rx + o;
      cidx = cidx < 0 ? 0 : (cidx >= A.ext_len ? A.ext_len - 1 : cidx);
      v[k] = __ldcs(vp + k * kSlice);
      xv[k] = __ldg(x_ext + cidx);
    }
#pragma unroll
    for (int k = 0; k < FMT; ++k) s = fma(v[k], xv[k], s);
  } else if constexpr (FMT < 0) {
    const int len = A.dia_d;
    const double* vp = A.vals + sl * kSlice * len + lane;
    const int64_t rx = halo_lo + row;
    for (int k0 = 0; k0 < len; k0 += kBatch) {
      double v[kBatch], xv[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const bool ok = k0 + k < len;
        const int o = __shfl_sync(0xffffffffu, cur_off, (k0 + k) & 31);
        int64_t cidx = rx + o;
        cidx = cidx < 0 ? 0 : (cidx >= A.ext_len ? A.ext_len - 1 : cidx);
        v[k] = ok ? __ldcs(vp + (k0 + k) * kSlice) : 0.0;
        xv[k] = ok ? __ldg(x_ext + cidx) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k)
        if (k0 + k < len) s = fma(v[k], xv[k], s);
    }
  } else {
    const int64_t p0 = A.slice_ptr[sl];
    const int len = static_cast<int>((A.slice_ptr[sl + 1] - p0) >> 5);
    const double* vp = A.vals + p0 + lane;
    const int32_t* cp = A.cols + p0 + lane;
    // all index/value loads of a batch are issued before the dependent gathers
    for (int k0 = 0; k0 < len; k0 += kBatch) {
      int32_t c[kBatch];
      double v[kBatch], xv[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const bool ok = k0 + k < len;
        c[k] = ok ? __ldcs(cp + (k0 + k) * kSlice) : 0;
        v[k] = ok ? __ldcs(vp + (k0 + k) * kSlice) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k) xv[k] = k0 + k < len ? __ldg(x_ext + c[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < kBatch; ++k)
        if (k0 + k < len) s = fma(v[k], xv[k], s);
    }
  }
  return s;
}

template <int MODE, int NV, int FMT, int MB = 3>
__global__ void __launch_bounds__(kThreads, NV > 8 ? 1 : MB) k_sell_spmv(SellView A, const double* __restrict__ x_ext,
                                                                         double* __restrict__ y,
                                                                         const double* __restrict__ aux, int64_t ldv,
                                                                         int64_t own_off, int64_t halo_lo, int j,
                                                                         int nwin, double* __restrict__ partials,
                                                                         unsigned* __restrict__ counter,
                                                                         double* __restrict__ out, MgsArgs mg,
                                                                         unsigned long long* stamp, int64_t sl_begin,
                                                                         int64_t sl_end) {
  stamp_begin(stamp);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;

  // DIA: the next slice's diagonal offsets (one per lane) are fetched an
  // iteration ahead, so no load of the current slice waits on an index load
  const int D = FMT > 0 ? FMT : (FMT < 0 ? A.dia_d : 0);
  int nx_off = 0;
  const bool wkeep = mg.wkeep != 0;
  pdl_trigger();  // the next kernel may start its constant-data prologue
  pdl_wait();     // x / the window vectors come from the previous kernel
  if constexpr (MODE == 3)
    if (*reinterpret_cast<const volatile int*>(aux)) return;
  // [sl_begin, sl_end) may run past nslices: slice indices wrap (a boundary
  // launch covers the last slices and then the first ones)
  auto wrap = [&](int64_t q) { return q >= A.nslices ? q - A.nslices : q; };
  if (FMT != 0 && sl_begin + gw < sl_end && lane < D) nx_off = __ldg(A.doff + wrap(sl_begin + gw) * D + lane);
  for (int64_t slv = sl_begin + gw; slv < sl_end; slv += nwarps) {
    const int64_t sl = wrap(slv);
    const int cur_off = nx_off;
    if (FMT != 0 && slv + nwarps < sl_end && lane < D) nx_off = __ldg(A.doff + wrap(slv + nwarps) * D + lane);
    const int64_t row = sl * kSlice + lane;
    const bool live = row < A.nrows;
    // epilogue operands are independent of the product: fetch them first
    double e0 = 0.0, ew[NV > 2 ? NV - 2 : 1];
    if constexpr (MODE == 1) {
      e0 = live ? x_ext[halo_lo + row] : 0.0;
#pragma unroll
      for (int d = 1; d < NV - 1; ++d) {
        const double* wp = aux + (j - d) * ldv + own_off + row;
        ew[d - 1] = (live && d < nwin) ? (wkeep ? __ldg(wp) : __ldcs(wp)) : 0.0;
      }
    } else if constexpr (MODE == 2) {
      e0 = live ? __ldcs(aux + row) : 0.0;
    }
    const double s = slice_row_sum<FMT>(A, x_ext, sl, row, halo_lo, lane, cur_off);
    if (live) {
      if constexpr (MODE == 0 || MODE == 3) {
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
  }
  if constexpr (MODE == 1 || MODE == 2) {
    const int nv = MODE == 1 ? 1 + nwin : 1;
    block_partials<NV>(acc, nv, partials);
    if (counter == nullptr) {  // deferred: the consumer folds the partials
      stamp_end(stamp);
      return;
    }
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

/// Y(:, q) = A X(:, q) for q < nb (<= NB) in one pass over the operator
/// (the exact recycle refresh, recycle.hpp:309-316: k products of one
/// matrix). Per column the row sums run in the same order as
/// slice_row_sum, so each column equals the single-vector SpMV bit for bit.
template <int NB, int FMT>
__global__ void __launch_bounds__(kThreads) k_sell_spmm(SellView A, SpmmCols X, int nb, double* __restrict__ Y,
                                                        int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int D = FMT > 0 ? FMT : (FMT < 0 ? A.dia_d : 0);
  for (int64_t sl = gw; sl < A.nslices; sl += nwarps) {
    const int64_t row = sl * kSlice + lane;
    double acc[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) acc[q] = 0.0;
    if constexpr (FMT != 0) {
      const int cur_off = lane < D ? __ldg(A.doff + sl * D + lane) : 0;
      const double* vp = A.vals + sl * kSlice * D + lane;
      const int64_t rx = A.halo_lo + row;
      for (int k = 0; k < D; ++k) {
        const int o = __shfl_sync(0xffffffffu, cur_off, k & 31);
        int64_t cidx = rx + o;
        cidx = cidx < 0 ? 0 : (cidx >= A.ext_len ? A.ext_len - 1 : cidx);
        const double v = __ldcs(vp + k * kSlice);
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < nb) acc[q] = fma(v, __ldg(X.x[q] + cidx), acc[q]);
      }
    } else {
      const int64_t p0 = A.slice_ptr[sl];
      const int len = static_cast<int>((A.slice_ptr[sl + 1] - p0) >> 5);
      for (int k = 0; k < len; ++k) {
        const int32_t c = __ldcs(A.cols + p0 + k * kSlice + lane);
        const double v = __ldcs(A.vals + p0 + k * kSlice + lane);
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < nb) acc[q] = fma(v, __ldg(X.x[q] + c), acc[q]);
      }
    }
    if (row < A.nrows) {
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (q < nb) Y[q * ldy + row] = acc[q];
    }
  }
}

/// ZSELL (complex-structured operator, interleaved vectors): lane = complex
/// row p (real rows 2p, 2p+1), one 16-byte value and one 16-byte x gather per
/// complex entry. The real / imaginary sums run over the entries in the order
/// of the real CSR rows (a·xr then −b·xi; b·xr then a·xi per column), so the
/// result equals the real SELL path's bit for bit. Same MODEs / epilogues as
/// k_sell_spmv, on double2 rows.
template <int MODE, int NV>
__global__ void __launch_bounds__(kThreads, NV > 8 ? 1 : 3) k_zsell_spmv(SellView A, const double* __restrict__ x_ext,
                                                                          double* __restrict__ y,
                                                                          const double* __restrict__ aux, int64_t ldv,
                                                                          int64_t own_off, int64_t halo_lo, int j,
                                                                          int nwin, double* __restrict__ partials,
                                                                          unsigned* __restrict__ counter,
                                                                          double* __restrict__ out, MgsArgs mg,
                                                                          unsigned long long* stamp, int64_t,
                                                                          int64_t) {  // slice range: one-rank only
  stamp_begin(stamp);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t nrc = A.nrows / 2, hlc = halo_lo / 2;
  const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x_ext);
  const double2* __restrict__ v2 = reinterpret_cast<const double2*>(A.vals);
  double2* __restrict__ y2 = reinterpret_cast<double2*>(y);
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  pdl_trigger();
  pdl_wait();
  if constexpr (MODE == 3)
    if (*reinterpret_cast<const volatile int*>(aux)) return;
  for (int64_t sl = gw; sl < A.nslices; sl += nwarps) {
    const int64_t p = sl * kSlice + lane;
    const bool live = p < nrc;
    double2 e0 = make_double2(0.0, 0.0), ew[NV > 2 ? NV - 2 : 1];
    if constexpr (MODE == 1) {
      if (live) e0 = x2[hlc + p];
#pragma unroll
      for (int d = 1; d < NV - 1; ++d)
        ew[d - 1] = (live && d < nwin) ? __ldcs(reinterpret_cast<const double2*>(aux + (j - d) * ldv + own_off) + p)
                                       : make_double2(0.0, 0.0);
    } else if constexpr (MODE == 2) {
      if (live) e0 = __ldcs(reinterpret_cast<const double2*>(aux) + p);
    }
    const int64_t p0 = A.slice_ptr[sl];
    const int len = static_cast<int>((A.slice_ptr[sl + 1] - p0) >> 5);
    double sr = 0.0, si = 0.0;
    for (int k0 = 0; k0 < len; k0 += kBatch) {
      int32_t c[kBatch];
      double2 v[kBatch], xv[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const bool ok = k0 + k < len;
        c[k] = ok ? __ldcs(A.cols + p0 + (k0 + k) * kSlice + lane) : 0;
        v[k] = ok ? __ldcs(v2 + p0 + (k0 + k) * kSlice + lane) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k) xv[k] = k0 + k < len ? __ldg(x2 + c[k]) : make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < kBatch; ++k)
        if (k0 + k < len) {
          sr = fma(v[k].x, xv[k].x, sr);
          sr = fma(-v[k].y, xv[k].y, sr);
          si = fma(v[k].y, xv[k].x, si);
          si = fma(v[k].x, xv[k].y, si);
        }
    }
    if (live) {
      if constexpr (MODE == 0 || MODE == 3) {
        y2[p] = make_double2(sr, si);
      } else if constexpr (MODE == 1) {
        y2[p] = make_double2(sr, si);
        acc[0] = fma(sr, sr, fma(si, si, acc[0]));
        acc[1] = fma(sr, e0.x, fma(si, e0.y, acc[1]));
#pragma unroll
        for (int d = 1; d < NV - 1; ++d)
          if (d < nwin) acc[1 + d] = fma(sr, ew[d - 1].x, fma(si, ew[d - 1].y, acc[1 + d]));
      } else {
        const double rr = e0.x - sr, ri = e0.y - si;
        y2[p] = make_double2(rr, ri);
        acc[0] = fma(rr, rr, fma(ri, ri, acc[0]));
      }
    }
  }
  if constexpr (MODE == 1 || MODE == 2) {
    const int nv = MODE == 1 ? 1 + nwin : 1;
    block_partials<NV>(acc, nv, partials);
    if (counter == nullptr) {
      stamp_end(stamp);
      return;
    }
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

/// Epilogues of K1 / K6 for a callable operator, whose product y = A x the
/// caller's function already wrote: MODE 1 — ||y||^2 and y.w_{j-d} (window
/// dots), MODE 2 — r = b - y in place, ||r||^2. Same partial layouts, folds
/// and MGS coefficients as k_sell_spmv.
template <int MODE, int NV>
__global__ void __launch_bounds__(kThreads) k_product_epilogue(double* __restrict__ y, int64_t n,
                                                               const double* __restrict__ x_own,
                                                               const double* __restrict__ aux, int64_t ldv,
                                                               int64_t own_off, int j, int nwin,
                                                               double* __restrict__ partials,
                                                               unsigned* __restrict__ counter, double* __restrict__ out,
                                                               MgsArgs mg) {
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if constexpr (MODE == 1) {
      const double s = y[row];
      acc[0] = fma(s, s, acc[0]);
      acc[1] = fma(s, x_own[row], acc[1]);
#pragma unroll
      for (int d = 1; d < NV - 1; ++d)
        if (d < nwin) acc[1 + d] = fma(s, aux[(j - d) * ldv + own_off + row], acc[1 + d]);
    } else {
      const double r = aux[row] - y[row];
      y[row] = r;
      acc[0] = fma(r, r, acc[0]);
    }
  }
  const int nv = MODE == 1 ? 1 + nwin : 1;
  block_partials<NV>(acc, nv, partials);
  if (counter == nullptr) return;  // deferred: the consumer folds the partials
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

/// The caller's y = A x (not one of this library's kernels: not counted as a launch).
void call_apply(Context& c, const SellView& A, const double* x, double* y) {
  if (c.timing) c.time_begin("operator_apply");
  const int rc = A.apply(x, y, c.stream, A.apply_user);
  if (c.timing) c.time_end();
  if (rc != 0) throw runtime("OperatorRef: the apply callback reported failure");
}

template <class K>
int resident_grid(const Context& c, K kernel, int64_t want_blocks, int max_per_sm = 0) {
  int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kernel), kThreads, 0);
  if (max_per_sm < 0) return c.num_sms * per_sm;  // fixed grid (CTAs past the work write zero partials)
  if (max_per_sm > 0) per_sm = std::min(per_sm, max_per_sm);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want_blocks, static_cast<int64_t>(c.num_sms) * per_sm)));
}

int64_t blocks_for(int64_t nslices) { return (nslices + (kThreads / 32) - 1) / (kThreads / 32); }

template <int MODE, int NV, int FMT>
int launch_impl(Context& c, const char* name, const SellView& A, const double* x_ext, double* y, const double* aux,
                int64_t ldv, int64_t own_off, int64_t halo_lo, int j, int nwin, unsigned* counter, double* out,
                const MgsArgs& mg, double* partials_out, int max_per_sm, int64_t sl_begin, int64_t sl_end) {
  // CTAs per SM: 4 (64 registers) when each warp has few slices to walk —
  // latency-bound (C3 1 M rows: K1 16.1 -> 14.2 us; C2: 33.2 -> 31.2 us in-solve),
  // 3 (77 registers, deeper per-warp pipelining) on long sweeps (C5: 1848 vs
  // 1908 us). SDR_K1_MINB=3/4 forces one.
  static const int minb_env = [] {
    const char* e = std::getenv("SDR_K1_MINB");
    return e ? std::atoi(e) : 0;
  }();
  const int64_t nsl = std::max<int64_t>(sl_end - sl_begin, 1);
  // (several ranks: always 3 — slab sizes differ per rank and grids / partial
  // layouts must not depend on them)
  const int minb = minb_env ? minb_env
                            : (!c.distributed() && nsl <= static_cast<int64_t>(c.num_sms) * 32 * 64 ? 4 : 3);
  auto kern = A.cplx ? k_zsell_spmv<MODE, NV> : (minb == 4 ? k_sell_spmv<MODE, NV, FMT, 4> : k_sell_spmv<MODE, NV, FMT>);
  const int g = resident_grid(c, kern, blocks_for(nsl), max_per_sm);
  double* part = partials_out ? partials_out : ((MODE == 1 || MODE == 2) ? c.partials(static_cast<int64_t>(NV) * g) : nullptr);
  TimedLaunch t(c, name);
  if (partials_out) {  // deferred step pipeline: programmatic dependent launch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1] = {pdl_attribute()};
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    SDR_CUDA(cudaLaunchKernelEx(&cfg, kern, A, x_ext, y, aux, ldv, own_off, halo_lo, j, nwin, part,
                                static_cast<unsigned*>(nullptr), out, mg, c.launch_stamp(name), sl_begin, sl_end));
  } else {
    kern<<<g, kThreads, 0, c.stream>>>(A, x_ext, y, aux, ldv, own_off, halo_lo, j, nwin, part, counter, out, mg,
                                       static_cast<unsigned long long*>(nullptr), sl_begin, sl_end);
    SDR_KERNEL_CHECK();
  }
  return g;
}

template <int MODE, int NV>
int launch_fmt(Context& c, const char* name, const SellView& A, const double* x_ext, double* y, const double* aux,
               int64_t ldv, int64_t own_off, int64_t halo_lo, int j, int nwin, unsigned* counter, double* out,
               const MgsArgs& mg, double* partials_out = nullptr, int max_per_sm = 0, int64_t sl_begin = 0,
               int64_t sl_end = -1) {
  if (sl_end < 0) sl_end = A.nslices;
#define SDR_SPMV_FMT(F) return launch_impl<MODE, NV, F>(c, name, A, x_ext, y, aux, ldv, own_off, halo_lo, j, nwin, counter, out, mg, partials_out, max_per_sm, sl_begin, sl_end)
  if (!A.doff)
    SDR_SPMV_FMT(0);
  else if (A.dia_d == 7)  // 3-D 7-point stencils
    SDR_SPMV_FMT(7);
  else if (A.dia_d == 5)  // 2-D 5-point stencils
    SDR_SPMV_FMT(5);
  else
    SDR_SPMV_FMT(-1);
#undef SDR_SPMV_FMT
}

}  // namespace

void launch_spmv(Context& c, const SellView& A, const double* x_ext, double* y) {
  if (A.nrows == 0) return;
  if (A.apply) return call_apply(c, A, x_ext + A.halo_lo, y);
  launch_fmt<0, 1>(c, "spmv", A, x_ext, y, nullptr, 0, 0, A.halo_lo, 0, 0, nullptr, nullptr, MgsArgs{});
}

int launch_spmv_arnoldi(Context& c, const SellView& A, const double* V, int64_t ldv, const VecLayout& lay, int j,
                        int nwin, double* y, double* recA, double* rec, int64_t rstride, int T, double* cvec,
                        double* coef, double* partials_out, int max_per_sm, int64_t sl_begin, int64_t sl_end) {
  static const int wkeep_env = [] {
    const char* e = std::getenv("SDR_K1_WKEEP");
    return e ? std::atoi(e) : -1;
  }();
  static const int64_t l2_bytes = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) != cudaSuccess) {
      cudaGetLastError();
      return int64_t{0};
    }
    return static_cast<int64_t>(v);
  }();
  MgsArgs mg{rec, rstride, T, cvec, coef};
  mg.wkeep = wkeep_env >= 0 ? wkeep_env : (!c.distributed() && 4 * 8 * lay.nloc <= l2_bytes ? 1 : 0);
  const double* x_ext = V + j * ldv + lay.ext_shift();
  if (A.apply) {  // y = A w_j by the caller's function, then the window dots
    if (sl_begin != 0 || (sl_end >= 0 && sl_end != A.nslices)) throw logic("callable operator: no split SpMV");
    call_apply(c, A, V + j * ldv + lay.own_off, y);
    auto go = [&](auto kern, int nv_cap) -> int {
      const int g = resident_grid(c, kern, (A.nrows + kThreads - 1) / kThreads, max_per_sm);
      double* part = partials_out ? partials_out : c.partials(static_cast<int64_t>(nv_cap) * g);
      TimedLaunch t(c, "spmv_arnoldi");
      kern<<<g, kThreads, 0, c.stream>>>(y, A.nrows, V + j * ldv + lay.own_off, V, ldv, lay.own_off, j, nwin, part,
                                         partials_out ? nullptr : c.counters() + 0, recA, mg);
      SDR_KERNEL_CHECK();
      return g;
    };
    if (nwin <= 3) return go(k_product_epilogue<1, 4>, 4);
    if (nwin <= 7) return go(k_product_epilogue<1, 8>, 8);
    if (nwin <= 33) return go(k_product_epilogue<1, 34>, 34);
    throw invalid("Arnoldi window of " + std::to_string(nwin) + " vectors exceeds the device limit of 33");
  }
  if (nwin <= 3)
    return launch_fmt<1, 4>(c, "spmv_arnoldi", A, x_ext, y, V, ldv, lay.own_off, lay.halo_lo, j, nwin, c.counters() + 0,
                            recA, mg, partials_out, max_per_sm, sl_begin, sl_end);
  else if (nwin <= 7)
    return launch_fmt<1, 8>(c, "spmv_arnoldi", A, x_ext, y, V, ldv, lay.own_off, lay.halo_lo, j, nwin, c.counters() + 0,
                            recA, mg, partials_out, max_per_sm, sl_begin, sl_end);
  else if (nwin <= 33)
    return launch_fmt<1, 34>(c, "spmv_arnoldi", A, x_ext, y, V, ldv, lay.own_off, lay.halo_lo, j, nwin,
                             c.counters() + 0, recA, mg, partials_out, max_per_sm, sl_begin, sl_end);
  else
    throw invalid("Arnoldi window of " + std::to_string(nwin) + " vectors exceeds the device limit of 33");
}

void launch_spmm(Context& c, const SellView& A, const SpmmCols& X, int nb, double* Y, int64_t ldy) {
  if (A.nrows == 0 || nb == 0) return;
  if (A.cplx || A.apply) {  // ZSELL / callable operator: one product per column
    for (int q = 0; q < nb; ++q) launch_spmv(c, A, X.x[q], Y + q * ldy);
    return;
  }
  if (nb > kSpmmMax) throw invalid("launch_spmm: at most 8 columns per launch");
  auto go = [&](auto kern) {
    const int g = resident_grid(c, kern, blocks_for(A.nslices));
    TimedLaunch t(c, "spmm");
    kern<<<g, kThreads, 0, c.stream>>>(A, X, nb, Y, ldy);
    SDR_KERNEL_CHECK();
  };
  if (!A.doff)
    go(k_sell_spmm<kSpmmMax, 0>);
  else if (A.dia_d == 7)
    go(k_sell_spmm<kSpmmMax, 7>);
  else if (A.dia_d == 5)
    go(k_sell_spmm<kSpmmMax, 5>);
  else
    go(k_sell_spmm<kSpmmMax, -1>);
}

void launch_spmv_guarded(Context& c, const SellView& A, const double* x_ext, double* y, const int* stop) {
  if (A.nrows == 0) return;
  if (A.apply) return call_apply(c, A, x_ext + A.halo_lo, y);  // no device-side skip: the product is unused past a stop
  launch_fmt<3, 1>(c, "baseline_spmv", A, x_ext, y, reinterpret_cast<const double*>(stop), 0, 0, A.halo_lo, 0, 0,
                   nullptr, nullptr, MgsArgs{});
}

void launch_residual(Context& c, const SellView& A, const double* x_ext, const double* b, double* r, double* norm2) {
  if (A.apply) {
    call_apply(c, A, x_ext + A.halo_lo, r);
    const int g = resident_grid(c, k_product_epilogue<2, 1>, (A.nrows + kThreads - 1) / kThreads);
    TimedLaunch t(c, "residual");
    k_product_epilogue<2, 1><<<g, kThreads, 0, c.stream>>>(r, A.nrows, nullptr, b, 0, 0, 0, 0, c.partials(g),
                                                           c.counters() + 1, norm2, MgsArgs{});
    SDR_KERNEL_CHECK();
    return;
  }
  launch_fmt<2, 1>(c, "residual", A, x_ext, r, b, 0, 0, A.halo_lo, 0, 0, c.counters() + 1, norm2, MgsArgs{});
}

}  // namespace sdr
