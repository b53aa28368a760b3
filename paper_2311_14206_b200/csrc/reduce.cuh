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

/// Atomic ticket: true in exactly one CTA, after every CTA's partials are
/// globally visible. The ticket counter is reset by the caller's last CTA.
__device__ __forceinline__ bool last_block_done(unsigned* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned ticket = atomicAdd(counter, 1u);
    am_last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

/// In the last CTA: out[k * out_stride] = sum_b partials[k * nblocks + b] for
/// k < nv, in a fixed lane/tree order. One warp per value.
__device__ __forceinline__ void fold_partials(const double* partials, int nblocks, int nv, double* out,
                                              int out_stride = 1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = warp; k < nv; k += nw) {
    const double* p = partials + static_cast<int64_t>(k) * nblocks;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = lane;
    for (; b + 96 < nblocks; b += 128) {
      a0 += __ldcg(p + b);
      a1 += __ldcg(p + b + 32);
      a2 += __ldcg(p + b + 64);
      a3 += __ldcg(p + b + 96);
    }
    for (; b < nblocks; b += 32) a0 += __ldcg(p + b);
    double s = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) out[static_cast<int64_t>(k) * out_stride] = s;
  }
}

}  // namespace sdr
