// Tall-skinny products of the restart boundary on a bulk-copy ring, sm_100a:
//   out[o] (n rows) = sum_i A_i B(i, o),  A = [A1 (k1 cols) | A2 (k2 cols)],
// plus ||out[o]||^2 (deterministic CTA partials). Replaces the basis
// recombinations x += [U V] y (solver.hpp:197-198) and U_new = [U V] P
// (recycle.hpp:257-265) — and, fused, both at once (one pass over [V U]
// writing the correction and the new recycle columns).
//
// HBM-bound: every input column is read once. A producer warp streams
// 8-column x 256-row chunks through a 4-stage shared-memory ring with
// cp.async.bulk (one 2 KB copy per column, mbarrier transaction counts), so
// the bytes in flight do not depend on registers or occupancy (the
// register-staged k_tsgemm / k_rgemm kept 32-64 KB per SM in flight and ran
// at 0.55-0.62 of HBM). Eight consumer warps own 32 rows each and
// accumulate all outputs on the fp64 tensor cores (mma.sync m8n8k4, DMMA):
// 4 m-tiles x NO/8 n-tiles per warp. A 64-bit shared load is served per
// half-warp (lanes 4 g + t, g < 4): fragment rows t of stride 4 mod 16
// doubles put its 16 addresses in 16 distinct bank pairs, so the ring's
// columns are padded by 32 bytes and the coefficient rows to NO + 4
// (measured at C5: strides 264 / NO = 16 made the A loads 2-way and the B
// loads 4-way conflicted, 63 % of all shared wavefronts).
#include "kernels.hpp"
#include "reduce.cuh"
#include "tma.cuh"

#include <algorithm>

namespace sdr {

namespace {

constexpr int kTmRows = 256;             // rows per tile (8 consumer warps x 32)
constexpr int kTmKC = 8;                 // input columns per ring stage
constexpr int kTmLd = kTmRows + 4;       // padded column stride in shared memory (== 4 mod 16 doubles)
constexpr int kTmStages = 4;
constexpr int kTmConsumers = 8;
constexpr int kTmThreads = 32 * (1 + kTmConsumers);
constexpr int kTmMaxOut = 40;

struct TsmmArgs {
  const double* A1;
  int64_t lda1;
  int k1;
  const double* A2;
  int64_t lda2;
  int k2;
  const double* B;  // (k1 + k2) x nout, column-major
  int nout;
  double* out[kTmMaxOut];
  int64_t n;
  double* partials;  // [nout][grid]
};

template <int NO>
__global__ void __launch_bounds__(kTmThreads) k_tsmm(TsmmArgs a) {
  constexpr int NT = NO / 8;
  extern __shared__ __align__(128) double tm_sm[];
  __shared__ __align__(8) uint64_t full[kTmStages], empty[kTmStages];
  const int K = a.k1 + a.k2;
  const int nch = (K + kTmKC - 1) / kTmKC;
  const int Kp = nch * kTmKC;
  constexpr int LDB = NO + 4;
  double* ring = tm_sm;                                   // [stage][kTmKC][kTmLd]
  double* Bs = tm_sm + kTmStages * kTmKC * kTmLd;         // [Kp][LDB], zero past K / nout
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int q = tid; q < Kp * LDB; q += blockDim.x) {
    const int i = q / LDB, o = q % LDB;
    Bs[q] = (o < a.nout && i < K) ? a.B[static_cast<int64_t>(o) * K + i] : 0.0;
  }
  if (tid == 0) {
    for (int s = 0; s < kTmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmConsumers);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t ntiles = (a.n + kTmRows - 1) / kTmRows;
  const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
  double nrm[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) nrm[nt][0] = nrm[nt][1] = 0.0;

  if (warp == 0) {
    // ---- producer: chunk (tile, ch) -> stage; one elected lane issues the copies
    int st = 0;
    uint32_t ph = 0;
    int64_t it = 0;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t r0 = t * kTmRows;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kTmRows), a.n - r0) * 8);
      for (int ch = 0; ch < nch; ++ch, ++it) {
        if (it >= kTmStages) mbar_wait_sleep(&empty[st], ph ^ 1u);
        if (lane == 0) {
          double* dst = ring + st * (kTmKC * kTmLd);
          mbar_arrive_expect_tx(&full[st], bytes * kTmKC);
#pragma unroll
          for (int u = 0; u < kTmKC; ++u) {
            // padding columns past K repeat the last input (finite data; its B rows are zero)
            const int i = min(ch * kTmKC + u, K - 1);
            const double* src = i < a.k1 ? a.A1 + static_cast<int64_t>(i) * a.lda1 : a.A2 + static_cast<int64_t>(i - a.k1) * a.lda2;
            bulk_g2s(dst + u * kTmLd, src + r0, bytes, &full[st]);
          }
        }
        __syncwarp();
        if (++st == kTmStages) st = 0, ph ^= 1u;
      }
    }
  } else {
    // ---- consumers: warp cw owns rows [32 cw, 32 cw + 32) of each tile
    const int cw = warp - 1, g8 = lane >> 2, t4 = lane & 3;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      double acc[4][NT][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
      for (int ch = 0; ch < nch; ++ch) {
        mbar_wait(&full[st], ph);
        const double* ab = ring + st * (kTmKC * kTmLd) + cw * 32 + g8;
        const double* bb = Bs + (ch * kTmKC) * LDB + g8;
#pragma unroll
        for (int ks = 0; ks < kTmKC / 4; ++ks) {
          const int kr = ks * 4 + t4;
          double af[4], bf[NT];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) af[mt] = ab[kr * kTmLd + mt * 8];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) bf[nt] = bb[kr * LDB + nt * 8];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
                           : "d"(af[mt]), "d"(bf[nt]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == kTmStages) st = 0, ph ^= 1u;
      }
      // tile complete: out(row, col) = acc[mt][nt][e], row = 8 mt + g8, col = 8 nt + 2 t4 + e
      const int64_t row = t * kTmRows + cw * 32 + g8;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        if (row + mt * 8 < a.n) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = nt * 8 + 2 * t4 + e;
              if (col < a.nout) {
                __stcs(a.out[col] + row + mt * 8, acc[mt][nt][e]);
                nrm[nt][e] = fma(acc[mt][nt][e], acc[mt][nt][e], nrm[nt][e]);
              }
            }
        }
      }
    }
  }
  // norms: lanes with the same t4 hold the same columns; fold over g8, then warps
  __shared__ double red[NO][kTmConsumers + 1];
  const int g8 = lane >> 2, t4 = lane & 3;
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
  if (tid < a.nout) {
    double v = 0.0;
    for (int w = 1; w <= kTmConsumers; ++w) v += red[tid][w];
    a.partials[static_cast<int64_t>(tid) * gridDim.x + blockIdx.x] = v;
  }
}

size_t tsmm_smem(int K, int NO) {
  const int Kp = (K + kTmKC - 1) / kTmKC * kTmKC;
  return sizeof(double) * (static_cast<size_t>(kTmStages) * kTmKC * kTmLd + static_cast<size_t>(Kp) * (NO + 4));
}

template <int NO>
void tsmm_impl(Context& c, TsmmArgs a, double* norms2, double* scratch) {
  auto kern = k_tsmm<NO>;
  const size_t smem = tsmm_smem(a.k1 + a.k2, NO);
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  const int64_t ntiles = (a.n + kTmRows - 1) / kTmRows;
  const int per_sm = std::max(1, blocks_per_sm(reinterpret_cast<const void*>(kern), kTmThreads, smem));
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, static_cast<int64_t>(c.num_sms) * per_sm)));
  a.partials = scratch ? scratch : c.partials(static_cast<int64_t>(a.nout) * g);
  {
    TimedLaunch t(c, "recycle_gemm");
    kern<<<g, kTmThreads, smem, c.stream>>>(a);
    SDR_KERNEL_CHECK();
  }
  launch_fold_partials(c, a.partials, g, a.nout, true, norms2);
}

}  // namespace

int64_t tsmm_scratch_size(int num_sms) { return static_cast<int64_t>(kTmMaxOut) * num_sms * 4; }

bool tsmm_supported(int nout, int k, int64_t n, int64_t lda1, int64_t lda2) {
  const int NO = nout <= 8 ? 8 : (nout <= 16 ? 16 : (nout <= 24 ? 24 : 40));
  return nout >= 1 && nout <= kTmMaxOut && k >= 1 && n % 2 == 0 && lda1 % 2 == 0 && lda2 % 2 == 0 &&
         tsmm_smem(k, NO) <= 200 * 1024;
}

void launch_tsmm(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                 const double* B, int nout, double* const* out, int64_t n, double* norms2, double* scratch) {
  if (!tsmm_supported(nout, k1 + k2, n, lda1, lda2)) throw invalid("tall-skinny product: unsupported shape");
  TsmmArgs a{};
  a.A1 = A1;
  a.lda1 = lda1;
  a.k1 = k1;
  a.A2 = A2 ? A2 : A1;
  a.lda2 = lda2;
  a.k2 = k2;
  a.B = B;
  a.nout = nout;
  for (int o = 0; o < nout; ++o) a.out[o] = out[o];
  a.n = n;
  if (nout <= 8)
    tsmm_impl<8>(c, a, norms2, scratch);
  else if (nout <= 16)
    tsmm_impl<16>(c, a, norms2, scratch);
  else if (nout <= 24)
    tsmm_impl<24>(c, a, norms2, scratch);
  else
    tsmm_impl<40>(c, a, norms2, scratch);
}

}  // namespace sdr
