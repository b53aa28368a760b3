// Deterministic block / grid reductions for the streaming kernels.
//
// Every HBM-bound kernel here produces a handful of fp64 sums (norms, MGS
// dots, Gram entries, sketch rows). They are reduced without floating-point
// atomics: each CTA writes its block sum into partials[v * gridDim.x + b],
// and the last CTA to finish (atomic ticket) folds those partials in a fixed
// order. Results are therefore bitwise reproducible run to run, matching the
// reference's determinism guarantee (tests/test_solver.cpp:244-259).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace sdr {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

/// sum of p[b * ld] over b = b0, b0 + step, ... < G, added in that order,
/// with eight loads in flight per round (a fold over a few hundred CTA
/// partials is one or two L2 round trips instead of one per partial);
/// `a` is the running sum to continue.
__device__ __forceinline__ double strided_sum(const double* __restrict__ p, int64_t ld, int b0, int G, int step,
                                              double a = 0.0) {
  for (int b = b0; b < G; b += 8 * step) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b + u * step < G ? __ldcg(p + static_cast<int64_t>(b + u * step) * ld) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) a += v[u];
  }
  return a;
}

/// strided_sum over (re, im) pairs p[b * ld], p[b * ld + 1].
__device__ __forceinline__ double2 strided_sum2(const double* __restrict__ p, int64_t ld, int b0, int G, int step) {
  double re = 0.0, im = 0.0;
  for (int b = b0; b < G; b += 8 * step) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = b + u * step < G ? __ldcg(reinterpret_cast<const double2*>(p + static_cast<int64_t>(b + u * step) * ld))
                              : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      re += v[u].x;
      im += v[u].y;
    }
  }
  return make_double2(re, im);
}

/// Block-reduce nv (<= NV) per-thread values; thread 0's warp writes
/// partials[k * gridDim.x + blockIdx.x]. Requires blockDim.x % 32 == 0.
template <int NV>
__device__ __forceinline__ void block_partials(const double (&v)[NV], int nv, double* __restrict__ partials) {
  __shared__ double red[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (k < nv) {
      const double s = warp_sum(v[k]);
      if (lane == 0) red[k][warp] = s;
    }
  }
  __syncthreads();
  for (int k = warp; k < nv; k += nw) {
    double s = lane < nw ? red[k][lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) partials[static_cast<int64_t>(k) * gridDim.x + blockIdx.x] = s;
  }
}

/// Ticket over `expected` arriving CTAs: true in exactly one CTA, after every
/// arriving CTA's global writes have reached L2. Thread 0's release atomic
/// publishes the CTA's writes (cumulative through the preceding bar.sync);
/// the last CTA reads them with L1-bypassing loads (ld.cg) only after its
/// atomic returned — the threadFenceReduction pattern. No acquire fence on
/// the reader side: an acquire invalidates L1 (CCTL.IVALL), after which
/// every spilled-register reload of the folding CTA misses to L2/HBM, which
/// showed up as a multi-µs kernel tail. The caller resets *ctr.
__device__ __forceinline__ bool ticket(unsigned* ctr, unsigned expected) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
    last = prev == expected - 1u;
  }
  __syncthreads();
  return last;
}

__device__ __forceinline__ bool last_block_done(unsigned* counter) { return ticket(counter, gridDim.x); }

/// In the last CTA: out[k * out_stride] = sum_b partials[k * nblocks + b] for
/// k < nv, in a fixed order. Wide two-level fold: the CTA's threads split
/// (value, block-group) pairs so every thread issues a handful of
/// independent loads (one or two L2 round trips in total instead of one per
/// value), then each value's group sums are combined in group order.
/// Requires blockDim.x <= 1024 and a multiple of 32.
__device__ __forceinline__ void fold_partials(const double* partials, int nblocks, int nv, double* out,
                                           int out_stride = 1) {
  __shared__ double red[1024];
  const int T = blockDim.x, t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5, nw = T >> 5;
  for (int k0 = 0; k0 < nv; k0 += T) {
    const int nk = min(T, nv - k0);
    const int G = T / nk;  // block groups per value
    const int k = t % nk, g = t / nk;
    if (g < G) {
      const double* p = partials + static_cast<int64_t>(k0 + k) * nblocks;
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = 0.0;
      int b = g;
      for (; b + 7 * G < nblocks; b += 8 * G) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += __ldcg(p + b + u * G);
      }
      for (; b < nblocks; b += G) a[0] += __ldcg(p + b);
      red[g * nk + k] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    __syncthreads();
    if (nk <= nw) {
      if (warp < nk) {
        double v = 0.0;
        for (int gg = lane; gg < G; gg += 32) v += red[gg * nk + warp];
        v = warp_sum(v);
        if (lane == 0) out[static_cast<int64_t>(k0 + warp) * out_stride] = v;
      }
    } else if (t < nk) {
      double v = 0.0;
      for (int gg = 0; gg < G; ++gg) v += red[gg * nk + t];
      out[static_cast<int64_t>(k0 + t) * out_stride] = v;
    }
    __syncthreads();
  }
}

}  // namespace sdr
