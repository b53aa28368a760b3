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

// ------------------------------------------------- K1 with bulk-copy staging
// Groups of kGroup slices (kGroup warps, one slice each). A single thread
// streams each group's SELL values and column indices into a kStages-deep
// shared-memory ring with cp.async.bulk (SASS UBLKCP, the TMA engine's 1-D
// path) completing on an mbarrier; warps wait on the stage's barrier, gather
// x through L1/L2, and release the stage at a CTA barrier. Matrix bytes — 85%
// of K1's traffic — thereby stream with no register cost and a deep queue.
constexpr int kGroup = kThreads / 32;
constexpr int kStages = 3;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int NV>
__global__ void __launch_bounds__(kThreads) k_sell_spmv_bulk(SellView A, const double* __restrict__ x_ext,
                                                              double* __restrict__ y, const double* __restrict__ V,
                                                              int64_t ldv, int64_t own_off, int64_t halo_lo, int j,
                                                              int nwin, int64_t stage_entries,
                                                              double* __restrict__ partials,
                                                              unsigned* __restrict__ counter, double* __restrict__ out,
                                                              MgsArgs mg) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sval = reinterpret_cast<double*>(smem_raw);                       // [kStages][stage_entries]
  int32_t* scol = reinterpret_cast<int32_t*>(sval + kStages * stage_entries);  // [kStages][stage_entries]
  __shared__ __align__(8) uint64_t full[kStages];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ngroups = (A.nslices + kGroup - 1) / kGroup;
  const int64_t per = (ngroups + gridDim.x - 1) / gridDim.x;
  const int64_t g0 = blockIdx.x * per, g1 = min(ngroups, g0 + per);
  auto issue = [&](int64_t g) {
    const int st = static_cast<int>((g - g0) % kStages);
    const int64_t s0 = g * kGroup, s1 = min(A.nslices, s0 + kGroup);
    const int64_t e0 = A.slice_ptr[s0], e1 = A.slice_ptr[s1];
    const unsigned ne = static_cast<unsigned>(e1 - e0);
    mbar_arrive_tx(&full[st], ne * 12u);
    bulk_g2s(sval + st * stage_entries, A.vals + e0, ne * 8u, &full[st]);
    bulk_g2s(scol + st * stage_entries, A.cols + e0, ne * 4u, &full[st]);
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int64_t g = g0; g < min(g1, g0 + kStages); ++g) issue(g);
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int64_t g = g0; g < g1; ++g) {
    const int st = static_cast<int>((g - g0) % kStages);
    const unsigned parity = static_cast<unsigned>(((g - g0) / kStages) & 1);
    const int64_t sl = g * kGroup + warp;
    const int64_t row = sl * kSlice + lane;
    const bool live = sl < A.nslices && row < A.nrows;
    // operands independent of the staged matrix data first
    double e0 = 0.0, ew[NV > 2 ? NV - 2 : 1];
    if (live) {
      e0 = x_ext[halo_lo + row];
#pragma unroll
      for (int d = 1; d < NV - 1; ++d) ew[d - 1] = d < nwin ? __ldcs(V + (j - d) * ldv + own_off + row) : 0.0;
    }
    int64_t base = 0;
    int len = 0;
    if (sl < A.nslices) {
      const int64_t gbase = A.slice_ptr[g * kGroup];
      const int64_t p0 = A.slice_ptr[sl];
      base = p0 - gbase;
      len = static_cast<int>((A.slice_ptr[sl + 1] - p0) >> 5);
    }
    mbar_wait(&full[st], parity);
    const double* sv = sval + st * stage_entries + base + lane;
    const int32_t* sc = scol + st * stage_entries + base + lane;
    double s = 0.0;
    for (int k0 = 0; k0 < len; k0 += kBatch) {
      double xv[kBatch], vv[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const bool ok = k0 + k < len;
        xv[k] = ok ? __ldg(x_ext + sc[(k0 + k) * kSlice]) : 0.0;
        vv[k] = ok ? sv[(k0 + k) * kSlice] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k)
        if (k0 + k < len) s = fma(vv[k], xv[k], s);
    }
    if (live) {
      y[row] = s;
      acc[0] = fma(s, s, acc[0]);
      acc[1] = fma(s, e0, acc[1]);
#pragma unroll
      for (int d = 1; d < NV - 1; ++d)
        if (d < nwin) acc[1 + d] = fma(s, ew[d - 1], acc[1 + d]);
    }
    __syncthreads();  // stage st fully consumed
    if (threadIdx.x == 0 && g + kStages < g1) issue(g + kStages);
  }
  block_partials<NV>(acc, 1 + nwin, partials);
  if (last_block_done(counter)) {
    fold_partials(partials, gridDim.x, 1 + nwin, out);
    if (mg.coef) {
      __syncthreads();
      if (threadIdx.x == 0) mgs_coefficients<NV - 1>(mg.rec, mg.rstride, mg.T, j, nwin, mg.cvec, mg.coef, true);
    }
    if (threadIdx.x == 0) *counter = 0u;
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
  // bulk-staged variant when a group's stage fits comfortably in shared memory
  static const bool bulk_on = [] {
    const char* e = std::getenv("SDR_K1_BULK");
    return !e || std::atoi(e) != 0;
  }();
  const int64_t stage = round_up(std::max<int64_t>(A.max_group, 32), 32);
  const size_t smem = static_cast<size_t>(kStages) * static_cast<size_t>(stage) * 12;
  if (bulk_on && nwin <= 7 && A.nslices > 0 && smem <= 150 * 1024) {
    auto launch = [&](auto kern, int nv) {
      static size_t configured[2] = {0, 0};
      size_t& cfgd = configured[nv > 4];
      if (smem > cfgd) {
        SDR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        cfgd = smem;
      }
      const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), kThreads, smem);
      const int64_t ngroups = (A.nslices + kGroup - 1) / kGroup;
      const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ngroups, static_cast<int64_t>(c.num_sms) * per_sm)));
      const double* x_ext = V + j * ldv + lay.ext_shift();
      TimedLaunch t(c, "spmv_arnoldi");
      kern<<<g, kThreads, smem, c.stream>>>(A, x_ext, y, V, ldv, lay.own_off, lay.halo_lo, j, nwin, stage,
                                            c.partials(static_cast<int64_t>(nv) * g), c.counters() + 0, recA, mg);
      SDR_KERNEL_CHECK();
    };
    if (nwin <= 3)
      launch(k_sell_spmv_bulk<4>, 4);
    else
      launch(k_sell_spmv_bulk<8>, 8);
    return;
  }
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
