// KF: one launch per Arnoldi step on one GPU with the sparse-sign sketch —
// the update + sketch of step j (K2s) and the SpMV + window dots of step
// j + 1 (K1) in a single streaming pass, sm_100a.
//
// Replaces, for step j, arnoldi.hpp:91-114 (MGS window update of w_{j+1},
// its norm / Gram, S w_{j+1}) and, for step j + 1, arnoldi.hpp:87-90 and the
// window dots of :91-97 (y_{j+1} = A w_{j+1}, ||y||^2, y.w_{j+1-d}).
//
// Why: K1 is HBM-bound (0.89 of peak) and K2s is bound by instruction issue
// and the shared-memory pipe (0.63 of peak); run back to back they cannot
// hide each other. Here every CTA carries both roles:
//   warps 0..2  the K2s pipeline (producer warp with bulk copies into a
//               2-stage ring, two consumer warps: update, norm / Gram,
//               sparse-sign scatter into lane-private bins);
//   warps 3..   SpMV warps over 32-row slices of the same operator storage K1
//               streams (SELL-DIA), reading w_{j+1} as the update writes it.
// The update walks its 512-row tiles in global order, chunk by chunk (chunk
// c = tiles [c G, (c + 1) G), tile c G + b to CTA b); consumer warp 0 of a
// CTA counts the chunk done once its stores of w_{j+1} are fenced. An SpMV
// warp about to compute a slice waits until every chunk up to the one
// holding its last stencil row (row + the slice's largest diagonal offset)
// is done. The SpMV front therefore trails the update front by about one
// stencil reach (one 512 x 512 plane at C5, 2 MB), so w_{j+1} is read back
// from L2, and w_j — the update's window column — is still in L2 when the
// SpMV's dot y.w_j needs it. HBM traffic per step: A, y_j, w_j, w_{j-1} read,
// w_{j+1}, y_{j+1} written (C5: 12.98 GB vs 15.14 GB for K1 + K2s).
//
// Deadlock freedom: update warps never wait on SpMV warps, and every CTA is
// resident at once (cooperative launch of an occupancy-sized grid), so every
// chunk is eventually counted. A wait that exceeds 4 s traps (the process
// fails loudly instead of hanging the GPU).
//
// Status: opt-in (SDR_FUSE_STEP=1), parity-green, and measured SLOWER than
// K1 + K2s at C5 (512^3, in-solve CUDA events, µs per step): KF 3381 vs
// 1775 + 903 (+ fold). ncu: 14.4 GB DRAM read per launch (the SpMV front
// falls behind and w_{j+1}, w_j no longer come from L2), DRAM 60 % of peak,
// warps active 35 %, long-scoreboard 42 %. The two roles share one register
// budget (80 / thread at 24 warps per SM), so each gets fewer warps than its
// own kernel; the update alone in this shape takes 1.77 ms (K2s: 0.92), and
// a producer throttle that keeps the fronts within a stencil reach (so the
// re-reads hit L2; SDR_KF_MODE=32) made it slower still (4.25 ms): the chunk
// counters couple every CTA to the slowest one. DESIGN.md §4 records it.
//
// Determinism: the update / sketch / dots are the K2s and K1 arithmetic
// (row sums in CSR order, lane-private bins, fixed-order folds); only which
// CTA accumulates which tile differs from K2s, so results are bitwise
// reproducible run to run and within rounding of the two-kernel step.
#include "kernels.hpp"
#include "mgs.cuh"
#include "reduce.cuh"
#include "sketch.hpp"
#include "tma.cuh"

#include <climits>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdlib>

namespace sdr {

namespace {

constexpr int kTR = 512;  // update tile rows (as K2s)
constexpr int kNS = 2;    // ring stages
constexpr int kUpdWarps = 3;
constexpr int kNV1 = 4;  // SpMV dots: ||y||^2, y.w_{j+1}, y.w_j, y.w_{j-1}

struct FusedArgs {
  // update + sketch of step j (writes column j + 1)
  const double* y;  // y_j
  double* V;
  int64_t ldv, own_off, n;
  int j, T;
  const double* coef;  // step j's MGS coefficients (nwin + 1)
  int64_t row_begin;
  uint64_t key;
  int s;
  int64_t ntiles, nchunks;
  unsigned* chunk_done;
  double* vpart;  // [8][G] value-major: norm / Gram (T), then the SpMV dots (1 + nwin1)
  double* skpart;  // [G][s]
  // SpMV of step j + 1
  SellView A;
  const double* x_ext;  // w_{j+1} in the extended layout
  double* y_out;        // y_{j+1}
  int nwin1;
  unsigned long long* stamp;
  // the fold after the launch
  double* rec;
  int64_t R;
  double* cvec;
  double* coef_out;  // step j + 1's coefficients (may alias coef: the fold runs after the launch)
  int64_t lagc;  // producer throttle: feed chunk c once the CTA's SpMV warps reached row (c - lagc) G kTR
  int mode;  // SDR_KF_MODE (measurement only): 1 no SpMV, 2 no scatter, 4 no chunk waits, 8 x via ld.global.nc,
             // 16 no fence before the chunk count, 32 producer throttle on
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

/// Row sum of one SELL-DIA slice (lane = row), CSR order; x through L2
/// (ld.cg): w_{j+1} is written by this launch.
template <int FMT>
__device__ __forceinline__ double dia_row_sum_cg(const SellView& A, const double* __restrict__ x_ext, int64_t sl,
                                                 int64_t row, int lane, int cur_off) {
  double s = 0.0;
  const int64_t rx = A.halo_lo + row;
  if constexpr (FMT > 0) {
    const double* vp = A.vals + sl * kSlice * FMT + lane;
    double v[FMT], xv[FMT];
#pragma unroll
    for (int k = 0; k < FMT; ++k) {
      const int o = __shfl_sync(0xffffffffu, cur_off, k);
      int64_t cidx = rx + o;
      cidx = cidx < 0 ? 0 : (cidx >= A.ext_len ? A.ext_len - 1 : cidx);
      v[k] = __ldcs(vp + k * kSlice);
      xv[k] = __ldcg(x_ext + cidx);
    }
#pragma unroll
    for (int k = 0; k < FMT; ++k) s = fma(v[k], xv[k], s);
  } else {
    constexpr int kB = 8;
    const int len = A.dia_d;
    const double* vp = A.vals + sl * kSlice * len + lane;
    for (int k0 = 0; k0 < len; k0 += kB) {
      double v[kB], xv[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const bool ok = k0 + k < len;
        const int o = __shfl_sync(0xffffffffu, cur_off, (k0 + k) & 31);
        int64_t cidx = rx + o;
        cidx = cidx < 0 ? 0 : (cidx >= A.ext_len ? A.ext_len - 1 : cidx);
        v[k] = ok ? __ldcs(vp + (k0 + k) * kSlice) : 0.0;
        xv[k] = ok ? __ldcg(x_ext + cidx) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kB; ++k)
        if (k0 + k < len) s = fma(v[k], xv[k], s);
    }
  }
  return s;
}

/// Measurement variant: x through the non-coherent path (SDR_KF_MODE & 8).
template <int FMT>
__device__ __forceinline__ double dia_row_sum_nc(const SellView& A, const double* __restrict__ x_ext, int64_t sl,
                                                 int64_t row, int lane, int cur_off) {
  double s = 0.0;
  const int64_t rx = A.halo_lo + row;
  constexpr int F = FMT > 0 ? FMT : 16;
  const int len = FMT > 0 ? FMT : A.dia_d;
  const double* vp = A.vals + sl * kSlice * len + lane;
  double v[F], xv[F];
#pragma unroll
  for (int k = 0; k < F; ++k) {
    const bool ok = k < len;
    const int o = __shfl_sync(0xffffffffu, cur_off, k);
    int64_t cidx = rx + o;
    cidx = cidx < 0 ? 0 : (cidx >= A.ext_len ? A.ext_len - 1 : cidx);
    v[k] = ok ? __ldcs(vp + k * kSlice) : 0.0;
    xv[k] = ok ? __ldg(x_ext + cidx) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < F; ++k)
    if (k < len) s = fma(v[k], xv[k], s);
  return s;
}

/// NW / NG: window and Gram entries of the update (compile time, as K2s);
/// FMT: SELL-DIA diagonals (7, 5, or -1 = A.dia_d); PW SpMV warps per CTA;
/// BS: compile-time sketch block size (15 for s = 120) or 0.
template <int NW, int NG, int FMT, int PW, int MINB, int BS>
__global__ void __launch_bounds__(32 * (kUpdWarps + PW), MINB) k_fused_step(FusedArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[kNS], empty[kNS];
  __shared__ double coef[NW + 1];
  __shared__ volatile long long sprog[PW];  // row of the slice each SpMV warp is on (LLONG_MAX: done)
  stamp_begin(a.stamp);
  const int s = a.s;
  double* bins = smem;                                 // [s][32]
  double* ring = smem + static_cast<int64_t>(s) * 32;  // [stage][1 + NW][kTR]
  constexpr int kNvec = 1 + NW;
  constexpr int kStageElems = kNvec * kTR;
  constexpr int kRowsPerLane = kTR / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, b = blockIdx.x;

  for (int i = threadIdx.x; i < s * 32; i += blockDim.x) bins[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kNS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 2);
    }
    mbar_fence_init();
  }
  if (threadIdx.x <= NW) coef[threadIdx.x] = a.coef[threadIdx.x];
  if (threadIdx.x < PW) sprog[threadIdx.x] = (a.mode & 1) || !(a.mode & 32) ? LLONG_MAX : 0;
  __syncthreads();

  double acc[8];  // [0, 4): ||w||^2, Gram (consumer 0); [4, 8): SpMV dots
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;

  if (warp == 0) {
    // ---- producer: tile c G + b of every chunk c, one elected lane
    int st = 0;
    uint32_t ph = 0;
    int64_t k = 0;
    for (int64_t c = 0; c < a.nchunks; ++c) {
      const int64_t t = c * G + b;
      if (t >= a.ntiles) break;
      if (k >= kNS) mbar_wait_sleep(&empty[st], ph ^ 1u);
      // do not run ahead of this CTA's SpMV warps by more than lagc chunks
      // (one stencil reach + one chunk: the rows between the two fronts stay
      // in L2; lagc > reach / chunk keeps every SpMV wait satisfiable)
      const int64_t need = (c - a.lagc) * static_cast<int64_t>(G) * kTR;
      if (need > 0 && lane == 0) {
        unsigned long long t0 = 0;
        for (int spins = 0;; ++spins) {
          long long mn = LLONG_MAX;
#pragma unroll
          for (int q = 0; q < PW; ++q) mn = min(mn, sprog[q]);
          if (mn >= need) break;
          __nanosleep(256);
          if (spins == 64) {
            t0 = global_ns();
          } else if (spins > 64 && (spins & 1023) == 0 && global_ns() - t0 > 4000000000ull) {
            printf("k_fused_step: producer throttle stuck at chunk %lld (CTA %d)\n", static_cast<long long>(c), b);
            __trap();
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        const int64_t r0 = t * kTR;
        const int64_t rows = min(static_cast<int64_t>(kTR), a.n - r0);
        const uint32_t bytes = static_cast<uint32_t>((rows & ~int64_t{1}) * 8);
        double* dst = ring + st * kStageElems;
        mbar_arrive_expect_tx(&full[st], bytes * kNvec);
        if (bytes) {
          bulk_g2s(dst, a.y + r0, bytes, &full[st]);
#pragma unroll
          for (int d = 0; d < NW; ++d)
            bulk_g2s(dst + (1 + d) * kTR, a.V + static_cast<int64_t>(a.j - d) * a.ldv + a.own_off + r0, bytes,
                     &full[st]);
        }
      }
      __syncwarp();
      ++k;
      if (++st == kNS) st = 0, ph ^= 1u;
    }
  } else if (warp < kUpdWarps) {
    // ---- consumers (K2s arithmetic)
    const int cw = warp - 1;
    double cf[NW + 1];
#pragma unroll
    for (int q = 0; q <= NW; ++q) cf[q] = coef[q];
    uint32_t rbB[4];
    int bsz[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int l = 4 * cw + e;
      const int r = (l * s) / 8;
      bsz[e] = ((l + 1) * s) / 8 - r;
      rbB[e] = smem_addr(bins + r * 32 + lane);
    }
    const uint64_t d_row = 64ull * kPhi64;
    double* wout = a.V + static_cast<int64_t>(a.j + 1) * a.ldv + a.own_off;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t c = 0; c < a.nchunks; ++c) {
      const int64_t t = c * G + b;
      if (t < a.ntiles) {
        const double* ys = ring + st * kStageElems + lane;
        const int64_t r0 = t * kTR;
        const int rows = static_cast<int>(min(static_cast<int64_t>(kTR), a.n - r0));
        const uint64_t arg0 =
            a.key + (static_cast<uint64_t>(a.row_begin + r0 + lane) * 2u + static_cast<uint64_t>(cw) + 1u) * kPhi64;
        mbar_wait(&full[st], ph);
        // two halves of 8 rows per lane: update (ring -> w), then the hashes
        // and the scatter; the stage is released after the second half's
        // ring reads. 16 + 16 live registers for w and the hashes.
        constexpr int kH = kRowsPerLane / 2;
        const bool fullt = rows == kTR;
        const int even = rows & ~1;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          double w[kH];
#pragma unroll
          for (int uu = 0; uu < kH; ++uu) {
            const int u = hf * kH + uu;
            const int r = 32 * u + lane;
            double yv, wv[NW];
            if (fullt || r < even) {
              yv = ys[32 * u];
#pragma unroll
              for (int d = 0; d < NW; ++d) wv[d] = ys[(1 + d) * kTR + 32 * u];
            } else {
              yv = 0.0;
#pragma unroll
              for (int d = 0; d < NW; ++d) wv[d] = 0.0;
              if (r < rows) {  // odd last row of the vector: not in the bulk copy
                yv = a.y[r0 + r];
#pragma unroll
                for (int d = 0; d < NW; ++d) wv[d] = a.V[static_cast<int64_t>(a.j - d) * a.ldv + a.own_off + r0 + r];
              }
            }
            double x = cf[0] * yv;
#pragma unroll
            for (int d = NW - 1; d >= 0; --d) x = fma(cf[1 + d], wv[d], x);
            w[uu] = x;  // rows past the end carry w = 0 and store nothing
            if (cw == 0 && (fullt || r < rows)) {
              __stcg(wout + r0 + r, x);
              acc[0] = fma(x, x, acc[0]);
#pragma unroll
              for (int g = 1; g <= NG; ++g) acc[g] = fma(x, wv[g - 1], acc[g]);
            }
          }
          if (hf == 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == kNS) st = 0, ph ^= 1u;
          }
          if (a.mode & 2) continue;
          uint64_t h[kH];
#pragma unroll
          for (int uu = 0; uu < kH; ++uu) h[uu] = mix64(arg0 + (hf * kH + uu) * d_row);
#pragma unroll
          for (int uu = 0; uu < kH; ++uu) {
            const uint32_t nwhi = static_cast<uint32_t>(__double2hiint(w[uu])) ^ 0x80000000u;
            const int wlo = __double2loint(w[uu]);
            const uint32_t hw[2] = {static_cast<uint32_t>(h[uu]), static_cast<uint32_t>(h[uu] >> 32)};
            uint32_t addr[4];
            double sv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t f = hw[e >> 1] >> (16 * (e & 1));  // sign bit 0, row bits 1..15
              const uint32_t xb = (f & 0xFFFEu) * static_cast<uint32_t>(BS > 0 ? BS : bsz[e]);
              addr[e] = rbB[e] + ((xb >> 16) << 8);
              sv[e] = __hiloint2double(static_cast<int>(nwhi ^ (f << 31)), wlo);
            }
            double tv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(tv[e]) : "r"(addr[e]));
#pragma unroll
            for (int e = 0; e < 4; ++e)
              asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr[e]), "d"(tv[e] + sv[e]) : "memory");
          }
        }
      }
      if (cw == 0) {
        // the tile's stores of w_{j+1} were issued before the scatter: by now
        // the fence has little left to wait for
        if (!(a.mode & 16)) __threadfence();
        __syncwarp();
        if (lane == 0) red_release_add(a.chunk_done + c, 1u);
      }
    }
    const int rlo = (4 * cw * s) / 8, rhi = ((4 * cw + 4) * s) / 8;
    for (int r = rlo; r < rhi; ++r) {
      const double v = warp_sum(bins[r * 32 + lane]);
      if (lane == 0) a.skpart[static_cast<int64_t>(b) * s + r] = v;
    }
  } else if (!(a.mode & 1)) {
    // ---- SpMV warps: slices in global order, each behind the update front
    const SellView& A = a.A;
    const int D = FMT > 0 ? FMT : A.dia_d;
    const int64_t sw = static_cast<int64_t>(b) * PW + (warp - kUpdWarps);
    const int64_t nsw = static_cast<int64_t>(G) * PW;
    const int64_t ns = A.nslices;
    const double* __restrict__ x_ext = a.x_ext;
    const double* wj = a.V + static_cast<int64_t>(a.j) * a.ldv + a.own_off;
    int nx_off = (sw < ns && lane < D) ? __ldg(A.doff + sw * D + lane) : 0;
    int64_t ready = 0;  // chunks [0, ready) are known complete
    const int64_t tiles_per_chunk = G;
    volatile long long* my = sprog + (warp - kUpdWarps);
    for (int64_t sl = sw; sl < ns; sl += nsw) {
      if (lane == 0) *my = sl * kSlice;
      const int cur_off = nx_off;
      if (sl + nsw < ns && lane < D) nx_off = __ldg(A.doff + (sl + nsw) * D + lane);
      const int mo = __reduce_max_sync(0xffffffffu, lane < D ? cur_off : INT_MIN);
      int64_t need = sl * kSlice + (kSlice - 1) + (mo > 0 ? mo : 0);
      if (need > a.n - 1) need = a.n - 1;
      const int64_t need_chunk = (need / kTR) / tiles_per_chunk;
      if (need_chunk >= ready && !(a.mode & 4)) {
        unsigned long long t0 = 0;
        int spins = 0;
        while (need_chunk >= ready) {
          unsigned v = 0;
          if (lane == 0) v = ld_acquire_u32(a.chunk_done + ready);
          v = __shfl_sync(0xffffffffu, v, 0);
          if (v >= static_cast<unsigned>(G)) {
            ++ready;
            continue;
          }
          __nanosleep(128);
          if (++spins == 64) {
            t0 = global_ns();
          } else if (spins > 64 && (spins & 1023) == 0 && global_ns() - t0 > 4000000000ull) {
            if (lane == 0) printf("k_fused_step: chunk %lld never completed (CTA %d)\n", static_cast<long long>(ready), b);
            __trap();
          }
        }
        __syncwarp();
      }
      const int64_t row = sl * kSlice + lane;
      const bool live = row < a.n;
      const double e0 = live ? __ldcg(x_ext + A.halo_lo + row) : 0.0;  // w_{j+1}
      double ew[kNV1 - 2];
#pragma unroll
      for (int d = 1; d < kNV1 - 1; ++d)
        ew[d - 1] = (live && d < a.nwin1) ? __ldcs(wj - static_cast<int64_t>(d - 1) * a.ldv + row) : 0.0;
      const double sum = (a.mode & 8) ? dia_row_sum_nc<FMT>(A, x_ext, sl, row, lane, cur_off)
                                      : dia_row_sum_cg<FMT>(A, x_ext, sl, row, lane, cur_off);
      if (live) {
        __stcs(a.y_out + row, sum);
        acc[4] = fma(sum, sum, acc[4]);
        acc[5] = fma(sum, e0, acc[5]);
#pragma unroll
        for (int d = 1; d < kNV1 - 1; ++d)
          if (d < a.nwin1) acc[5 + d] = fma(sum, ew[d - 1], acc[5 + d]);
      }
    }
  }
  if (warp >= kUpdWarps && lane == 0) sprog[warp - kUpdWarps] = LLONG_MAX;
  block_partials<8>(acc, 8, a.vpart);
  stamp_end(a.stamp);
}

/// One CTA folds a KF launch's partials in a fixed order: record row j+1's B
/// part (norm / Gram, sketch rows x 1/sqrt(zeta)) and row j+2's A part (the
/// SpMV dots), then forms step j+1's MGS coefficients (mgs.cuh) — the values
/// k_fold_update_sparse and K1's last CTA give in the two-kernel step.
__global__ void __launch_bounds__(1024) k_fused_fold(const double* __restrict__ vp, const double* __restrict__ sk, int G,
                                                     int s, int T, int nwin1, double scale, double* __restrict__ rec,
                                                     int64_t R, int j, double* __restrict__ cvec,
                                                     double* __restrict__ coef, unsigned long long* stamp) {
  stamp_begin(stamp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* recB = rec + static_cast<int64_t>(j + 1) * R + (2 * T + 3);  // RecLayout::b_off
  double* recA = rec + static_cast<int64_t>(j + 2) * R;                  // RecLayout::a_off
  const int nv = T + s + 1 + nwin1;
  for (int q = warp; q < nv; q += nw) {
    double v;
    if (q < T) {
      v = warp_sum(strided_sum(vp + static_cast<int64_t>(q) * G, 1, lane, G, 32));
      if (lane == 0) recB[q] = v;
    } else if (q < T + s) {
      const int r = q - T;
      v = warp_sum(strided_sum(sk + r, s, lane, G, 32));
      if (lane == 0) recB[T + r] = v * scale;
    } else {
      const int d = q - T - s;
      v = warp_sum(strided_sum(vp + static_cast<int64_t>(4 + d) * G, 1, lane, G, 32));
      if (lane == 0) recA[d] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) mgs_coefficients<3>(rec, R, T, j + 1, nwin1, cvec, coef, true);
  stamp_end(stamp);
}

/// Largest SELL-DIA diagonal offset of the operator (its forward stencil reach).
__global__ void k_max_offset(const int32_t* __restrict__ doff, int64_t n, int* __restrict__ out) {
  int m = INT_MIN;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = max(m, doff[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

/// Forward reach of an operator, computed once per storage (cached by the
/// offsets' address and size: operators are immutable once created).
int64_t forward_reach(Context& c, const SellView& A) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int64_t>, int64_t> cache;
  const auto key = std::make_pair(static_cast<const void*>(A.doff), A.nslices * A.dia_d);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  DeviceBuffer<int> d(1);
  const int init = INT_MIN;
  SDR_CUDA(cudaMemcpyAsync(d.get(), &init, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  k_max_offset<<<c.num_sms * 4, 256, 0, c.stream>>>(A.doff, A.nslices * A.dia_d, d.get());
  SDR_KERNEL_CHECK();
  int h = 0;
  SDR_CUDA(cudaMemcpyAsync(&h, d.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SDR_CUDA(cudaStreamSynchronize(c.stream));
  const int64_t r = std::max(0, h);
  std::lock_guard<std::mutex> g(mu);
  cache[key] = r;
  return r;
}

constexpr int kPW = 5;  // 8 warps per CTA, 3 CTAs per SM: 6 warps per scheduler, <= 80 registers
constexpr int kMinB = 3;

size_t fused_smem(int s, int nw) { return sizeof(double) * (static_cast<size_t>(s) * 32 + static_cast<size_t>(kNS) * (1 + nw) * kTR); }

template <int NW, int NG, int FMT>
void fused_impl(Context& c, FusedArgs a) {
  static const bool bs_on = [] {
    const char* e = std::getenv("SDR_K2S_BS");
    return !e || std::atoi(e) != 0;
  }();
  auto kern = (bs_on && a.s == 120) ? k_fused_step<NW, NG, FMT, kPW, kMinB, 15> : k_fused_step<NW, NG, FMT, kPW, kMinB, 0>;
  const int threads = 32 * (kUpdWarps + kPW);
  const size_t smem = fused_smem(a.s, NW);
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), threads, smem);
  if (per_sm < 1) throw logic("fused step: kernel does not fit on an SM");
  const int G = c.num_sms * per_sm;
  a.ntiles = (a.n + kTR - 1) / kTR;
  a.nchunks = (a.ntiles + G - 1) / G;
  const int64_t crow = static_cast<int64_t>(G) * kTR;
  a.lagc = !(a.mode & 32) ? (int64_t{1} << 40) : (forward_reach(c, a.A) + kSlice - 1 + crow - 1) / crow + 1;
  a.vpart = c.partials(8 * static_cast<int64_t>(G));
  a.skpart = c.partials2(static_cast<int64_t>(G) * a.s);
  SDR_CUDA(cudaMemsetAsync(a.chunk_done, 0, sizeof(unsigned) * static_cast<size_t>(a.nchunks), c.stream));
  a.stamp = c.launch_stamp("fused_step");
  {
    TimedLaunch t(c, "fused_step");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the chunk waits always resolve
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SDR_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  }
  {
    TimedLaunch t(c, "fused_fold");
    k_fused_fold<<<1, 1024, 0, c.stream>>>(a.vpart, a.skpart, G, a.s, a.T, a.nwin1, 1.0 / std::sqrt(8.0), a.rec, a.R,
                                           a.j, a.cvec, a.coef_out, c.launch_stamp("fused_fold"));
    SDR_KERNEL_CHECK();
  }
}

template <int NW, int NG>
void fused_fmt(Context& c, const FusedArgs& a) {
  if (a.A.dia_d == 7) return fused_impl<NW, NG, 7>(c, a);
  if (a.A.dia_d == 5) return fused_impl<NW, NG, 5>(c, a);
  return fused_impl<NW, NG, -1>(c, a);
}

}  // namespace

bool fused_step_eligible(const SellView& A, const SketchDev& S, const VecLayout& lay, const RecLayout& RL, int t,
                         bool distributed) {
  static const bool on = [] {
    const char* e = std::getenv("SDR_FUSE_STEP");  // opt-in: measured slower than K1 + K2s
    return e && std::atoi(e) != 0;
  }();
  return on && !distributed && !A.apply && !A.cplx && A.doff != nullptr && A.halo_lo == 0 &&
         S.kind == kSparseSign && S.zeta == 8 && S.s >= 8 && S.s <= 128 && t >= 1 && t <= 3 && RL.T <= 3 &&
         lay.own_off % 2 == 0 && lay.ld % 2 == 0 && lay.nloc >= kTR && fused_smem(static_cast<int>(S.s), 3) <= 64 * 1024;
}

int64_t fused_step_chunks(const Context& c, int64_t nloc) {
  // upper bound on the chunk count of any instantiation (grid >= one CTA per SM)
  const int64_t ntiles = (nloc + kTR - 1) / kTR;
  return (ntiles + c.num_sms - 1) / c.num_sms;
}

void launch_fused_step(Context& c, const SellView& A, const SketchDev& S, const double* y_in, double* y_out, double* V,
                       int64_t ldv, const VecLayout& lay, int j, int nwin, int ngram, int nwin1, double* rec,
                       const RecLayout& RL, double* cvec, double* coef, int64_t row_begin, unsigned* chunk_done) {
  if (nwin < 1 || nwin > 3 || ngram < 0 || ngram > 2 || ngram > nwin || nwin1 < 1 || nwin1 > 3)
    throw logic("launch_fused_step: window outside the compiled range");
  FusedArgs a{};
  a.y = y_in;
  a.V = V;
  a.ldv = ldv;
  a.own_off = lay.own_off;
  a.n = lay.nloc;
  a.j = j;
  a.T = RL.T;
  a.coef = coef;
  a.row_begin = row_begin;
  a.key = S.key;
  a.s = static_cast<int>(S.s);
  a.chunk_done = chunk_done;
  a.A = A;
  a.x_ext = V + static_cast<int64_t>(j + 1) * ldv + lay.ext_shift();
  a.y_out = y_out;
  a.nwin1 = nwin1;
  static const int mode = [] {
    const char* e = std::getenv("SDR_KF_MODE");
    return e ? std::atoi(e) : 0;
  }();
  a.mode = mode;
  a.rec = rec;
  a.R = RL.stride;
  a.cvec = cvec;
  a.coef_out = coef;
  switch (nwin * 3 + ngram) {
    case 3: fused_fmt<1, 0>(c, a); break;
    case 4: fused_fmt<1, 1>(c, a); break;
    case 6: fused_fmt<2, 0>(c, a); break;
    case 7: fused_fmt<2, 1>(c, a); break;
    case 8: fused_fmt<2, 2>(c, a); break;
    case 9: fused_fmt<3, 0>(c, a); break;
    case 10: fused_fmt<3, 1>(c, a); break;
    default: fused_fmt<3, 2>(c, a); break;
  }
}

}  // namespace sdr
