// K3a / K3b: sketch kernels (sm_100a).
//
// K3a — subsampled randomized DCT (SketchOperator::subsampled_dct,
// sketch.hpp:105-162). The reference runs a full length-n FFTW DCT-II and
// keeps s outputs; here only the s selected rows are formed, by a four-step
// factorisation of the length-2N transform:
//   X[k]   = sum_j z_j cos(pi k (2j+1) / 2N) = Re(e^{i pi k/2N} Z(k)),
//   Z(k)   = sum_{a<L} e^{i pi k (r0+a)/N} T(a, k mod F),
//   T(a,u) = sum_{b<M} z_{r0+a+L b} e^{2 pi i u b / F},   F = 2N/L,
// with z = sign ⊙ x, the rank's block [r0, r0 + L·M). A CTA takes a tile of
// 32 consecutive a and all M b (M coalesced 256-byte rows), runs sixteen
// length-F complex FFTs (two real columns per complex sequence) in shared
// memory, then accumulates the s selected rows with exact-integer-reduced
// twiddles. HBM traffic is one read of x (+ n/8 sign bytes); the selected
// rows are folded over CTAs deterministically.
//
// K3b — sparse sign embedding (new; BASELINE C1/C5), block construction,
// generated on the fly from a counter hash (no index storage). Each thread
// owns one (lane, row-block) pair and accumulates into private shared-memory
// bins, so the result is deterministic without atomics.
#include "kernels.hpp"
#include "mgs.cuh"
#include "reduce.cuh"
#include "sketch.hpp"

#include <cooperative_groups.h>

namespace sdr {

namespace {

constexpr int kThreads = 256;
constexpr int kTileA = 32;
constexpr int kMaxF = 256;

struct SrdctPlan {
  int64_t M = 1, L = 1, F = 2;
  int logF = 1;
};

/// Largest power-of-two M dividing nloc with F = 2N·M/nloc a power of two
/// no larger than kMaxF; M = 1 (direct evaluation) always qualifies.
SrdctPlan plan_srdct(int64_t N, int64_t nloc) {
  SrdctPlan p;
  for (int64_t M = 128; M >= 1; M >>= 1) {
    if (nloc % M) continue;
    const int64_t L = nloc / M;
    if ((2 * N) % L) continue;
    const int64_t F = 2 * N / L;
    if (F > kMaxF || (F & (F - 1))) continue;
    p.M = M, p.L = L, p.F = F;
    break;
  }
  if (p.M == 1) {
    p.L = nloc;
    p.F = 2;
  }
  p.logF = 0;
  while ((int64_t{1} << p.logF) < p.F) ++p.logF;
  return p;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void __launch_bounds__(kThreads) k_srdct(const double* __restrict__ x, double xscale, int64_t N, int64_t r0,
                                                     int64_t M, int64_t L, int F, int logF,
                                                     const uint32_t* __restrict__ sign_bits,
                                                     const int64_t* __restrict__ rows, const double* __restrict__ row_scale,
                                                     int s, int64_t ntiles, double* __restrict__ partials,
                                                     unsigned* __restrict__ counter, double* __restrict__ fold,
                                                     double* __restrict__ out) {
  extern __shared__ double2 smem[];
  double2* buf = smem;                          // [16][F]
  double2* tw = buf + (kTileA / 2) * F;         // [F/2] e^{+2 pi i k / F}
  double2* acc = tw + F / 2;                    // [s]
  const int tid = threadIdx.x;
  for (int k = tid; k < F / 2; k += blockDim.x) {
    double sn, cs;
    sincospi(2.0 * static_cast<double>(k) / static_cast<double>(F), &sn, &cs);
    tw[k] = make_double2(cs, sn);
  }
  for (int q = tid; q < s; q += blockDim.x) acc[q] = make_double2(0.0, 0.0);
  const uint64_t twoN = 2u * static_cast<uint64_t>(N);

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t a0 = tile * kTileA;
    __syncthreads();
    // load z = sign ⊙ x into bit-reversed positions; b >= M is zero padding
    for (int idx = tid; idx < F * kTileA; idx += blockDim.x) {
      const int b = idx / kTileA, da = idx % kTileA;
      const int64_t a = a0 + da;
      double z = 0.0;
      if (b < M && a < L) {
        const int64_t jl = a + L * b;
        const int64_t jg = r0 + jl;
        const bool pos = (__ldg(sign_bits + (jg >> 5)) >> (jg & 31)) & 1u;
        const double v = __ldcs(x + jl) * xscale;
        z = pos ? v : -v;
      }
      const int pos_b = static_cast<int>(__brev(static_cast<unsigned>(b)) >> (32 - logF));
      double* slot = reinterpret_cast<double*>(buf + (da >> 1) * F + pos_b);
      slot[da & 1] = z;
    }
    __syncthreads();
    // radix-2 DIT over the 16 sequences
    for (int half = 1; half < F; half <<= 1) {
      const int tstep = F / (2 * half);
      for (int t = tid; t < (kTileA / 2) * (F / 2); t += blockDim.x) {
        const int p = t / (F / 2), bt = t % (F / 2);
        const int grp = bt / half, pos = bt % half;
        const int i0 = grp * 2 * half + pos, i1 = i0 + half;
        double2* sq = buf + p * F;
        const double2 u = sq[i0];
        const double2 v = cmul(sq[i1], tw[pos * tstep]);
        sq[i0] = make_double2(u.x + v.x, u.y + v.y);
        sq[i1] = make_double2(u.x - v.x, u.y - v.y);
      }
      __syncthreads();
    }
    // accumulate the selected rows
    for (int q = tid; q < s; q += blockDim.x) {
      const uint64_t k = static_cast<uint64_t>(rows[q]);
      const int u = static_cast<int>(k & static_cast<uint64_t>(F - 1));
      const int um = (F - u) & (F - 1);
      double sn, cs;
      const uint64_t ph = (k * static_cast<uint64_t>(r0 + a0)) % twoN;
      sincospi(static_cast<double>(ph) / static_cast<double>(N), &sn, &cs);
      double2 t = make_double2(cs, sn);
      sincospi(static_cast<double>(k) / static_cast<double>(N), &sn, &cs);
      const double2 step = make_double2(cs, sn);
      double2 a = acc[q];
#pragma unroll 4
      for (int p = 0; p < kTileA / 2; ++p) {
        const double2 C = buf[p * F + u], Cm = buf[p * F + um];
        const double2 T0 = make_double2(0.5 * (C.x + Cm.x), 0.5 * (C.y - Cm.y));
        const double2 T1 = make_double2(0.5 * (C.y + Cm.y), -0.5 * (C.x - Cm.x));
        double2 m = cmul(t, T0);
        a.x += m.x, a.y += m.y;
        t = cmul(t, step);
        m = cmul(t, T1);
        a.x += m.x, a.y += m.y;
        t = cmul(t, step);
      }
      acc[q] = a;
    }
  }
  __syncthreads();
  double* part = partials;
  for (int q = tid; q < s; q += blockDim.x) {
    part[static_cast<int64_t>(2 * q) * gridDim.x + blockIdx.x] = acc[q].x;
    part[static_cast<int64_t>(2 * q + 1) * gridDim.x + blockIdx.x] = acc[q].y;
  }
  if (last_block_done(counter)) {
    fold_partials(partials, gridDim.x, 2 * s, fold);
    __syncthreads();
    for (int q = tid; q < s; q += blockDim.x) {
      const int64_t k = rows[q];
      double sn, cs;
      sincospi(static_cast<double>(k) / (2.0 * static_cast<double>(N)), &sn, &cs);
      const double re = fold[2 * q], im = fold[2 * q + 1];
      out[q] = (cs * re - sn * im) * row_scale[q];
    }
    if (tid == 0) *counter = 0u;
  }
}

// ---------------------------------------------------------------- F = 256 path
// Register four-step FFT: 256 = 16 x 16. Thread (p, t) owns pair p of the
// tile (columns a0+2p, a0+2p+1 packed as one complex sequence) and row
// class t: stage 1 is a 16-point DFT over b = t + 16 i held in registers,
// stage 2 (after one padded shared-memory transpose) a 16-point DFT over t.
// Only M/16 of the 16 stage-1 inputs are nonzero (zero padding b >= M).

constexpr int kPairs = 16;   // 32 columns a per tile
constexpr int kXS = 257;     // padded row stride (double2) -> conflict-free transposes

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

/// x * e^{+2 pi i K / 16}; K is a compile-time constant after unrolling.
__device__ __forceinline__ double2 rot16(double2 x, int K) {
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173, R2 = 0.70710678118654752440;
  switch (K) {
    case 0: return x;
    case 1: return cmul(x, make_double2(C1, S1));
    case 2: return make_double2(R2 * (x.x - x.y), R2 * (x.x + x.y));
    case 3: return cmul(x, make_double2(S1, C1));
    case 4: return make_double2(-x.y, x.x);
    case 5: return cmul(x, make_double2(-S1, C1));
    case 6: return make_double2(-R2 * (x.x + x.y), R2 * (x.x - x.y));
    default: return cmul(x, make_double2(-C1, S1));
  }
}

template <int LEN>
__device__ __forceinline__ void dit_stage(double2 (&b)[16]) {
#pragma unroll
  for (int i = 0; i < 16; i += LEN) {
#pragma unroll
    for (int k = 0; k < LEN / 2; ++k) {
      const double2 u = b[i + k];
      const double2 v = rot16(b[i + k + LEN / 2], k * (16 / LEN));
      b[i + k] = cadd(u, v);
      b[i + k + LEN / 2] = csub(u, v);
    }
  }
}

/// a[k] <- sum_n a[n] e^{+2 pi i k n / 16} (radix-2 DIT, fully unrolled).
__device__ __forceinline__ void dft16(double2 (&a)[16]) {
  double2 b[16];
#pragma unroll
  for (int n = 0; n < 16; ++n) b[((n & 1) << 3) | ((n & 2) << 1) | ((n & 4) >> 1) | ((n & 8) >> 3)] = a[n];
  dit_stage<2>(b);
  dit_stage<4>(b);
  dit_stage<8>(b);
  dit_stage<16>(b);
#pragma unroll
  for (int n = 0; n < 16; ++n) a[n] = b[n];
}

/// dft16 for inputs a[8..15] == 0 (zero-padded stage 1 when M = 128): after
/// the bit-reversal every first-stage butterfly pairs a value with a zero.
__device__ __forceinline__ void dft16_half(double2 (&a)[16]) {
  double2 b[16];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int n = ((2 * m) & 1) << 3 | ((2 * m) & 2) << 1 | ((2 * m) & 4) >> 1 | ((2 * m) & 8) >> 3;
    b[2 * m] = a[n];
    b[2 * m + 1] = a[n];
  }
  dit_stage<4>(b);
  dit_stage<8>(b);
  dit_stage<16>(b);
#pragma unroll
  for (int n = 0; n < 16; ++n) a[n] = b[n];
}

// ------------------------------------------------ fused K2 + K3a (F = 256)
// One pass over the step's vectors: the Arnoldi update
//   w_{j+1} = c_j y - sum_d h_{j-d} c_{j-d} w_{j-d}          (arnoldi.hpp:91-114)
// is evaluated in the SRDCT tile order (it is elementwise, so any order is
// valid), w_{j+1} is stored once, its norm / Gram partials are accumulated,
// and the sign-flipped values go straight from registers into the stage-1
// FFT. HBM traffic is the update's alone (y + window reads, one write); the
// sketch's FFT and row accumulation overlap with it instead of re-reading
// w_{j+1} in a second kernel. Requires M = 128 (F = 256) and an even block.
template <int MAXT>
__global__ void __launch_bounds__(kThreads, 2) k_update_srdct256(
    const double* __restrict__ y, double* __restrict__ V, int64_t ldv, int64_t own_off, int j, int nwin, int ngram,
    double* __restrict__ rec, int64_t rstride, int T, double* __restrict__ cvec, const double* __restrict__ coef_ready,
    int64_t N, int64_t r0, int64_t L, const uint32_t* __restrict__ sign_bits, const int64_t* __restrict__ rows,
    const double* __restrict__ row_scale, int s, int64_t ntiles, int csize, double* __restrict__ partials,
    unsigned* __restrict__ counter, double* __restrict__ fold) {
  extern __shared__ double2 sm[];
  double2* X = sm;                    // [16][257]
  double2* acc = X + kPairs * kXS;    // [s] sketch rows, then [MAXT] norm/Gram (as .x)
  double2* zq = acc + s + MAXT;
  double2* ga = zq + s;
  double2* gb = ga + s;
  double2* tw = gb + s;
  int* uq = reinterpret_cast<int*>(tw + 256);
  __shared__ double coef[MAXT + 1];
  __shared__ double nred[MAXT][kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t twoN = 2u * static_cast<uint64_t>(N);
  const int b_off = 2 * T + 3;
  for (int k = tid; k < 256; k += blockDim.x) {
    double sn, cs;
    sincospi(static_cast<double>(k) / 128.0, &sn, &cs);
    tw[k] = make_double2(cs, sn);
  }
  for (int q = tid; q < s; q += blockDim.x) {
    const int64_t k = rows[q];
    double sn, cs;
    sincospi(static_cast<double>(k) / static_cast<double>(N), &sn, &cs);
    ga[q] = make_double2(0.5 * (1.0 + sn), -0.5 * cs);
    gb[q] = make_double2(0.5 * (1.0 - sn), 0.5 * cs);
    sincospi(static_cast<double>((2 * static_cast<uint64_t>(k)) % twoN) / static_cast<double>(N), &sn, &cs);
    zq[q] = make_double2(cs, sn);
    uq[q] = static_cast<int>(k & 255);
    acc[q] = make_double2(0.0, 0.0);
  }
  if (coef_ready) {
    if (tid <= MAXT) coef[tid] = tid <= nwin ? coef_ready[tid] : 0.0;
  } else if (tid == 0) {
    mgs_coefficients<MAXT>(rec, rstride, T, j, nwin, cvec, coef, blockIdx.x == 0);
  }
  __syncthreads();
  double cf[MAXT + 1];
#pragma unroll
  for (int k = 0; k <= MAXT; ++k) cf[k] = coef[k];
  const double* W[MAXT];
#pragma unroll
  for (int d = 0; d < MAXT; ++d) W[d] = V + static_cast<int64_t>(j - (d < nwin ? d : 0)) * ldv + own_off;
  double* wout = V + static_cast<int64_t>(j + 1) * ldv + own_off;
  double nacc[MAXT];
#pragma unroll
  for (int g = 0; g < MAXT; ++g) nacc[g] = 0.0;
  const int p = tid & 15, t = tid >> 4;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t a0 = tile * (2 * kPairs);
    const int64_t aa = a0 + 2 * p;
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = make_double2(0.0, 0.0);
    if (aa < L) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t jl = aa + L * static_cast<int64_t>(t + 16 * i);
        const double2 yv = __ldcs(reinterpret_cast<const double2*>(y + jl));
        double2 wv[MAXT];
#pragma unroll
        for (int d = MAXT - 1; d >= 0; --d)
          if (d < nwin) wv[d] = __ldg(reinterpret_cast<const double2*>(W[d] + jl));
        double w0 = cf[0] * yv.x, w1 = cf[0] * yv.y;
#pragma unroll
        for (int d = MAXT - 1; d >= 0; --d)
          if (d < nwin) {
            w0 = fma(cf[1 + d], wv[d].x, w0);
            w1 = fma(cf[1 + d], wv[d].y, w1);
          }
        *reinterpret_cast<double2*>(wout + jl) = make_double2(w0, w1);
        nacc[0] = fma(w0, w0, fma(w1, w1, nacc[0]));
#pragma unroll
        for (int g = 1; g < MAXT; ++g)
          if (g <= ngram) nacc[g] = fma(w0, wv[g - 1].x, fma(w1, wv[g - 1].y, nacc[g]));
        const int64_t jg = r0 + jl;
        const uint32_t bits = __ldg(sign_bits + (jg >> 5));
        v[i] = make_double2((bits >> (jg & 31)) & 1u ? w0 : -w0, (bits >> ((jg + 1) & 31)) & 1u ? w1 : -w1);
      }
    }
    dft16_half(v);
#pragma unroll
    for (int vv = 1; vv < 16; ++vv) v[vv] = cmul(v[vv], tw[(vv * t) & 255]);
    __syncthreads();
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) X[p * kXS + vv * 16 + t] = v[vv];
    __syncthreads();
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) v[tt] = X[p * kXS + t * 16 + tt];
    dft16(v);
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 16; ++w) X[p * kXS + t + 16 * w] = v[w];
    __syncthreads();
    for (int q = tid; q < s; q += blockDim.x) {
      const uint64_t k = static_cast<uint64_t>(rows[q]);
      const int u = uq[q], um = (256 - u) & 255;
      const double2 zz = zq[q];
      double2 S1 = X[(kPairs - 1) * kXS + u];
      double2 Cm = X[(kPairs - 1) * kXS + um];
      double2 S2 = make_double2(Cm.x, -Cm.y);
#pragma unroll
      for (int pp = kPairs - 2; pp >= 0; --pp) {
        const double2 C = X[pp * kXS + u];
        Cm = X[pp * kXS + um];
        S1 = make_double2(fma(S1.x, zz.x, fma(-S1.y, zz.y, C.x)), fma(S1.x, zz.y, fma(S1.y, zz.x, C.y)));
        S2 = make_double2(fma(S2.x, zz.x, fma(-S2.y, zz.y, Cm.x)), fma(S2.x, zz.y, fma(S2.y, zz.x, -Cm.y)));
      }
      double sn, cs;
      const uint64_t ph = (k * static_cast<uint64_t>(r0 + a0)) % twoN;
      sincospi(static_cast<double>(ph) / static_cast<double>(N), &sn, &cs);
      const double2 tsum = cadd(cmul(ga[q], S1), cmul(gb[q], S2));
      acc[q] = cadd(acc[q], cmul(make_double2(cs, sn), tsum));
    }
  }
  // norm / Gram partials of this CTA into acc[s + g].x
#pragma unroll
  for (int g = 0; g < MAXT; ++g) {
    const double v = warp_sum(nacc[g]);
    if (lane == 0) nred[g][warp] = v;
  }
  __syncthreads();
  if (tid < MAXT) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += nred[tid][w];
    acc[s + tid] = make_double2(v, 0.0);
  }
  __syncthreads();
  const int nacc_tot = s + MAXT;
  int nparts = gridDim.x, part = blockIdx.x;
  if (csize > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const bool leader = cl.block_rank() == 0;
    if (leader) {
      for (int q = tid; q < nacc_tot; q += blockDim.x) {
        double2 sum = acc[q];
        for (int r = 1; r < csize; ++r) sum = cadd(sum, cl.map_shared_rank(acc, r)[q]);
        acc[q] = sum;
      }
    }
    cl.sync();
    if (!leader) return;
    nparts = gridDim.x / csize;
    part = blockIdx.x / csize;
  }
  for (int q = tid; q < s; q += blockDim.x) {
    partials[static_cast<int64_t>(2 * q) * nparts + part] = acc[q].x;
    partials[static_cast<int64_t>(2 * q + 1) * nparts + part] = acc[q].y;
  }
  for (int g = tid; g < MAXT; g += blockDim.x) partials[static_cast<int64_t>(2 * s + g) * nparts + part] = acc[s + g].x;
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(counter, 1u) == static_cast<unsigned>(nparts - 1);
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  fold_partials(partials, nparts, 2 * s + MAXT, fold);
  __syncthreads();
  double* recB = rec + static_cast<int64_t>(j + 1) * rstride + b_off;
  for (int q = tid; q < s; q += blockDim.x) {
    const int64_t k = rows[q];
    double sn, cs;
    sincospi(static_cast<double>(k) / (2.0 * static_cast<double>(N)), &sn, &cs);
    recB[T + q] = (cs * fold[2 * q] - sn * fold[2 * q + 1]) * row_scale[q];
  }
  for (int g = tid; g < T; g += blockDim.x) recB[g] = (g <= ngram && g < MAXT) ? fold[2 * s + g] : 0.0;
  if (tid == 0) *counter = 0u;
}

template <int NI, bool PAIRED>
__global__ void __launch_bounds__(kThreads) k_srdct256(const double* __restrict__ x, double xscale, int64_t N, int64_t r0,
                                                        int M, int64_t L, const uint32_t* __restrict__ sign_bits,
                                                        const int64_t* __restrict__ rows,
                                                        const double* __restrict__ row_scale, int s, int64_t ntiles,
                                                        int csize, double* __restrict__ partials,
                                                        unsigned* __restrict__ counter, double* __restrict__ fold,
                                                        double* __restrict__ out) {
  extern __shared__ double2 sm[];
  double2* X = sm;                    // [16][257]
  double2* acc = X + kPairs * kXS;    // [s]
  double2* zq = acc + s;              // [s] e^{2 i pi k_q / N}  (two columns per pair)
  double2* ga = zq + s;               // [s] (1 - i e^{i pi k/N}) / 2
  double2* gb = ga + s;               // [s] (1 + i e^{i pi k/N}) / 2
  double2* tw = gb + s;               // [256] e^{2 pi i k / 256}
  int* uq = reinterpret_cast<int*>(tw + 256);
  const int tid = threadIdx.x;
  const uint64_t twoN = 2u * static_cast<uint64_t>(N);
  for (int k = tid; k < 256; k += blockDim.x) {
    double sn, cs;
    sincospi(static_cast<double>(k) / 128.0, &sn, &cs);
    tw[k] = make_double2(cs, sn);
  }
  for (int q = tid; q < s; q += blockDim.x) {
    const int64_t k = rows[q];
    double sn, cs;
    sincospi(static_cast<double>(k) / static_cast<double>(N), &sn, &cs);
    ga[q] = make_double2(0.5 * (1.0 + sn), -0.5 * cs);
    gb[q] = make_double2(0.5 * (1.0 - sn), 0.5 * cs);
    sincospi(static_cast<double>((2 * static_cast<uint64_t>(k)) % twoN) / static_cast<double>(N), &sn, &cs);
    zq[q] = make_double2(cs, sn);
    uq[q] = static_cast<int>(k & 255);
    acc[q] = make_double2(0.0, 0.0);
  }
  const int p = tid & 15, t = tid >> 4;
  const int nI = NI ? NI : (M >> 4);  // <= 8 nonzero stage-1 inputs
  // Raw tile data in registers, fetched one tile ahead: the loads for tile
  // k+1 are in flight while tile k's accumulation runs.
  double2 z[8];
  uint32_t wb0[8], wb1[PAIRED ? 1 : 8];
  auto issue = [&](int64_t tile) {
    const int64_t aa = tile * (2 * kPairs) + 2 * p;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      z[i] = make_double2(0.0, 0.0);
      wb0[i] = 0u;
      if constexpr (!PAIRED) wb1[i] = 0u;
      if (tile < ntiles && i < nI && aa < L) {
        const int64_t jl = aa + L * static_cast<int64_t>(t + 16 * i);
        const int64_t jg = r0 + jl;
        if constexpr (PAIRED) {
          z[i] = __ldcs(reinterpret_cast<const double2*>(x + jl));
          wb0[i] = __ldg(sign_bits + (jg >> 5));
        } else {
          z[i].x = __ldcs(x + jl);
          z[i].y = aa + 1 < L ? __ldcs(x + jl + 1) : 0.0;
          wb0[i] = __ldg(sign_bits + (jg >> 5));
          wb1[i] = __ldg(sign_bits + ((jg + 1) >> 5));
        }
      }
    }
  };
  issue(blockIdx.x);
  __syncthreads();

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t a0 = tile * (2 * kPairs);
    const int64_t aa = a0 + 2 * p;
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = make_double2(0.0, 0.0);
      if (i < 8) {
        const int64_t jg = r0 + aa + L * static_cast<int64_t>(t + 16 * i);
        const uint32_t b0 = (wb0[i] >> (jg & 31)) & 1u;
        uint32_t b1;
        if constexpr (PAIRED) b1 = (wb0[i] >> ((jg + 1) & 31)) & 1u;
        else b1 = (wb1[i] >> ((jg + 1) & 31)) & 1u;
        const double zx = z[i].x * xscale, zy = z[i].y * xscale;
        v[i] = make_double2(b0 ? zx : -zx, b1 ? zy : -zy);
      }
    }
    if constexpr (NI == 8) dft16_half(v);
    else dft16(v);
#pragma unroll
    for (int vv = 1; vv < 16; ++vv) v[vv] = cmul(v[vv], tw[(vv * t) & 255]);
    __syncthreads();  // previous tile's accumulation has finished reading X
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) X[p * kXS + vv * 16 + t] = v[vv];
    __syncthreads();
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) v[tt] = X[p * kXS + t * 16 + tt];
    dft16(v);
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 16; ++w) X[p * kXS + t + 16 * w] = v[w];
    issue(tile + gridDim.x);
    __syncthreads();
    // accumulate the selected rows: sum_a e^{i pi k (r0+a)/N} T(a, k mod 256).
    // With the pair unpacking folded into g_alpha / g_beta, a tile contributes
    //   r0 (g_alpha sum_p z^p C_p[u] + g_beta sum_p z^p conj(C_p[-u])),
    // z = e^{2 i pi k / N}: two Horner recurrences over the 16 pairs.
    for (int q = tid; q < s; q += blockDim.x) {
      const uint64_t k = static_cast<uint64_t>(rows[q]);
      const int u = uq[q], um = (256 - u) & 255;
      const double2 zz = zq[q];
      double2 S1 = X[(kPairs - 1) * kXS + u];
      double2 Cm = X[(kPairs - 1) * kXS + um];
      double2 S2 = make_double2(Cm.x, -Cm.y);
#pragma unroll
      for (int pp = kPairs - 2; pp >= 0; --pp) {
        const double2 C = X[pp * kXS + u];
        Cm = X[pp * kXS + um];
        S1 = make_double2(fma(S1.x, zz.x, fma(-S1.y, zz.y, C.x)), fma(S1.x, zz.y, fma(S1.y, zz.x, C.y)));
        S2 = make_double2(fma(S2.x, zz.x, fma(-S2.y, zz.y, Cm.x)), fma(S2.x, zz.y, fma(S2.y, zz.x, -Cm.y)));
      }
      double sn, cs;
      const uint64_t ph = (k * static_cast<uint64_t>(r0 + a0)) % twoN;
      sincospi(static_cast<double>(ph) / static_cast<double>(N), &sn, &cs);
      const double2 tsum = cadd(cmul(ga[q], S1), cmul(gb[q], S2));
      acc[q] = cadd(acc[q], cmul(make_double2(cs, sn), tsum));
    }
  }
  __syncthreads();
  // cluster reduction of the per-CTA accumulators through distributed shared memory
  int nparts = gridDim.x, part = blockIdx.x;
  if (csize > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const bool leader = cl.block_rank() == 0;
    if (leader) {
      for (int q = tid; q < s; q += blockDim.x) {
        double2 sum = acc[q];
        for (int r = 1; r < csize; ++r) sum = cadd(sum, cl.map_shared_rank(acc, r)[q]);
        acc[q] = sum;
      }
    }
    cl.sync();
    if (!leader) return;
    nparts = gridDim.x / csize;
    part = blockIdx.x / csize;
  }
  for (int q = tid; q < s; q += blockDim.x) {
    partials[static_cast<int64_t>(2 * q) * nparts + part] = acc[q].x;
    partials[static_cast<int64_t>(2 * q + 1) * nparts + part] = acc[q].y;
  }
  // last-arriving CTA (ticket over nparts) folds in a fixed order
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(counter, 1u) == static_cast<unsigned>(nparts - 1);
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  fold_partials(partials, nparts, 2 * s, fold);
  __syncthreads();
  for (int q = tid; q < s; q += blockDim.x) {
    const int64_t k = rows[q];
    double sn, cs;
    sincospi(static_cast<double>(k) / (2.0 * static_cast<double>(N)), &sn, &cs);
    out[q] = (cs * fold[2 * q] - sn * fold[2 * q + 1]) * row_scale[q];
  }
  if (tid == 0) *counter = 0u;
}

__global__ void __launch_bounds__(kThreads) k_sparse_sign(const double* __restrict__ x, double xscale, int64_t nloc,
                                                           int64_t r0, uint64_t key, int s, int zeta, double inv_sqrt_zeta,
                                                           int64_t chunk, double* __restrict__ partials,
                                                           unsigned* __restrict__ counter, double* __restrict__ out) {
  extern __shared__ double bins[];  // [s][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < s * 32; i += blockDim.x) bins[i] = 0.0;
  __syncthreads();
  const int64_t beg = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t end = min(nloc, beg + chunk);
  for (int64_t jl = beg + lane; jl < end; jl += 32) {
    const double v = __ldg(x + jl) * xscale;
    const int64_t jg = r0 + jl;
    for (int l = w; l < zeta; l += nw) {
      int64_t row;
      bool positive;
      sparse_sign_entry(key, s, zeta, jg, l, &row, &positive);
      double* b = bins + row * 32 + lane;
      *b += positive ? v : -v;
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < s; r += blockDim.x) {
    double acc = 0.0;
    for (int e = 0; e < 32; ++e) acc += bins[r * 32 + e];
    partials[static_cast<int64_t>(r) * gridDim.x + blockIdx.x] = acc;
  }
  if (last_block_done(counter)) {
    fold_partials(partials, gridDim.x, s, out);
    __syncthreads();
    for (int r = threadIdx.x; r < s; r += blockDim.x) out[r] *= inv_sqrt_zeta;
    if (threadIdx.x == 0) *counter = 0u;
  }
}

}  // namespace

bool launch_update_sketch(Context& c, const SketchDev& S, const double* y, double* V, int64_t ldv, const VecLayout& lay,
                          int j, int nwin, int ngram, double* rec, const RecLayout& RL, double* cvec,
                          const double* coef_ready, int64_t row_begin) {
  constexpr int MAXT = 4;
  if (S.kind != kSrdct || std::max(nwin, ngram + 1) > MAXT) return false;
  const SrdctPlan p = plan_srdct(S.n, lay.nloc);
  if (p.F != 256 || p.M != 128 || p.L % 2 || row_begin % 2 || lay.own_off % 2 || ldv % 2) return false;
  const int64_t ntiles = (p.L + kTileA - 1) / kTileA;
  int csize = ntiles >= 16 ? 8 : 1;
  const int64_t per = (ntiles + 2 * c.num_sms - 1) / (2 * c.num_sms);
  int grid = static_cast<int>((ntiles + per - 1) / per);
  if (csize > 1) grid = std::max(csize, (grid + csize - 1) / csize * csize);
  grid = static_cast<int>(std::min<int64_t>(grid, ntiles));
  if (csize > 1 && grid % csize) csize = 1;
  const size_t smem = sizeof(double2) * static_cast<size_t>(kPairs * kXS + 4 * S.s + MAXT + 256) + sizeof(int) * S.s;
  static size_t configured = 0;
  if (smem > configured) {
    SDR_CUDA(cudaFuncSetAttribute(k_update_srdct256<MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(csize);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TimedLaunch t(c, "update_sketch");
  SDR_CUDA(cudaLaunchKernelEx(&cfg, k_update_srdct256<MAXT>, y, V, ldv, lay.own_off, j, nwin, ngram, rec, RL.stride,
                              RL.T, cvec, coef_ready, S.n, row_begin, p.L, static_cast<const uint32_t*>(S.sign_bits.get()),
                              static_cast<const int64_t*>(S.rows.get()), static_cast<const double*>(S.row_scale.get()),
                              static_cast<int>(S.s), ntiles, csize, c.partials((2 * S.s + MAXT) * grid),
                              c.counters() + 7, c.partials2(2 * S.s + MAXT)));
  return true;
}

void launch_sketch(Context& c, const SketchDev& S, const double* x_own, int64_t nloc, int64_t row_begin, double* out) {
  launch_sketch_scaled(c, S, x_own, 1.0, nloc, row_begin, out);
}

void launch_sketch_scaled(Context& c, const SketchDev& S, const double* x_own, double xscale, int64_t nloc,
                          int64_t row_begin, double* out) {
  if (S.kind == kIdentity) {
    if (c.distributed()) throw invalid("identity sketch is not supported in a distributed context");
    launch_scale_copy(c, xscale, x_own, out, nloc);
    return;
  }
  if (S.kind == kSrdct) {
    const SrdctPlan p = plan_srdct(S.n, nloc);
    const int64_t ntiles = (p.L + kTileA - 1) / kTileA;
    if (p.F == 256 && p.M % 16 == 0) {
      // fast path: persistent CTAs in clusters of 8, ~2 per SM
      int csize = ntiles >= 16 ? 8 : 1;
      // equal tiles per CTA (no tail wave), at most ~2 CTAs per SM
      const int64_t per = (ntiles + 2 * c.num_sms - 1) / (2 * c.num_sms);
      int grid = static_cast<int>((ntiles + per - 1) / per);
      if (csize > 1) grid = std::max(csize, (grid + csize - 1) / csize * csize);
      grid = static_cast<int>(std::min<int64_t>(grid, ntiles));
      if (csize > 1 && grid % csize) csize = 1;
      const size_t smem = sizeof(double2) * static_cast<size_t>(kPairs * kXS + 4 * S.s + 256) + sizeof(int) * S.s;
      const bool fast = p.M == 128 && p.L % 2 == 0 && row_begin % 2 == 0;
      auto kern = fast ? k_srdct256<8, true> : k_srdct256<0, false>;
      static size_t configured[2] = {0, 0};
      if (smem > configured[fast]) {
        SDR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        configured[fast] = smem;
      }
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = c.stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = static_cast<unsigned>(csize);
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      TimedLaunch t(c, "sketch");
      SDR_CUDA(cudaLaunchKernelEx(&cfg, kern, x_own, xscale, S.n, row_begin, static_cast<int>(p.M), p.L,
                                  static_cast<const uint32_t*>(S.sign_bits.get()), static_cast<const int64_t*>(S.rows.get()),
                                  static_cast<const double*>(S.row_scale.get()), static_cast<int>(S.s), ntiles, csize,
                                  c.partials(2 * S.s * grid), c.counters() + 5, c.partials2(2 * S.s), out));
      return;
    }
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, 2 * c.num_sms)));
    const size_t smem = sizeof(double2) * static_cast<size_t>((kTileA / 2) * p.F + p.F / 2 + S.s);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      SDR_CUDA(cudaFuncSetAttribute(k_srdct, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      configured = smem;
    }
    TimedLaunch t(c, "sketch");
    k_srdct<<<grid, kThreads, smem, c.stream>>>(x_own, xscale, S.n, row_begin, p.M, p.L, static_cast<int>(p.F), p.logF,
                                                S.sign_bits.get(), S.rows.get(), S.row_scale.get(),
                                                static_cast<int>(S.s), ntiles, c.partials(2 * S.s * grid),
                                                c.counters() + 5, c.partials2(2 * S.s), out);
    SDR_KERNEL_CHECK();
    return;
  }
  // sparse sign
  const int64_t want = (nloc + 1023) / 1024;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 4 * c.num_sms)));
  const int64_t chunk = round_up((nloc + grid - 1) / grid, 32);
  const size_t smem = sizeof(double) * 32 * static_cast<size_t>(S.s);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    SDR_CUDA(cudaFuncSetAttribute(k_sparse_sign, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = smem;
  }
  TimedLaunch t(c, "sketch");
  k_sparse_sign<<<grid, kThreads, smem, c.stream>>>(x_own, xscale, nloc, row_begin, S.key, static_cast<int>(S.s),
                                                    static_cast<int>(S.zeta), 1.0 / std::sqrt(static_cast<double>(S.zeta)),
                                                    chunk, c.partials(S.s * grid), c.counters() + 6, out);
  SDR_KERNEL_CHECK();
}

}  // namespace sdr
