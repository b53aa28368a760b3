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

#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include <vector>

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

// ------------------------------------------------ F = 256 tile kernels
// One kernel template serves the plain sketch (SRC = kSrcSketch, input z =
// sign ⊙ xscale·x) and the fused Arnoldi update (SRC = kSrcUpdate):
//   w_{j+1} = c_j y - sum_d h_{j-d} c_{j-d} w_{j-d}          (arnoldi.hpp:91-114)
// evaluated in the SRDCT tile order (elementwise, so any order is valid);
// w_{j+1} is stored once, its norm / Gram partials are accumulated, and the
// sign-flipped values go from registers straight into the stage-1 FFT. HBM
// traffic is the update's alone (y + window reads, one write).
//
// Work split: one CTA per SM owns the contiguous tile range [tb, te); each of
// its kGroups tile groups walks its share downwards, so the two Horner
// recurrences over column pairs (z = e^{2 i pi k / N} per pair) continue from
// tile to tile (jumping over the other groups' tiles with a precomputed
// z^{8 (kGroups-1)}); the phase of a group's lowest tile,
// e^{i pi k (r0 + 16 t_low) / N}, is applied once at the end with an exact
// integer reduction. Per-row constants come precomputed with the sketch
// (SketchDev::tab). CTA partials go out CTA-major and a separate small
// kernel (k_srdct_fold) folds them in a fixed order — deterministic, no
// floating-point atomics, and no serial last-CTA tail.
enum { kSrcSketch = 0, kSrcUpdate = 1 };

struct TileArgs {
  int64_t N = 0, r0 = 0, L = 0, ntiles = 0;
  int M = 0, s = 0;
  const uint32_t* sign_bits = nullptr;
  const int64_t* rows = nullptr;
  const double* row_scale = nullptr;
  const double2* tab = nullptr;  // [g_alpha s][g_beta s][z s][half-phase s][jump z^24, z^8, z^28, z^16 (4s)][twiddle 256]
  const int* uq = nullptr;       // k mod 256
  const int* uperm = nullptr;    // rows in increasing k mod 256
  double* partials = nullptr;    // [G][nvp] CTA partials
  unsigned long long* trace = nullptr;  // SDR_TRACE=1: per-CTA phase timestamps [G][16]
  unsigned long long* stamp = nullptr;  // SDR_TRACE=2: launch timeline
};

__device__ __forceinline__ void trace_mark(unsigned long long* tr, int slot) {
  if (tr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[blockIdx.x * 16 + slot] = t;
  }
}

struct UpdateArgs {
  const double* y = nullptr;
  double* V = nullptr;
  int64_t ldv = 0, own_off = 0, rstride = 0;
  int j = 0, nwin = 0, ngram = 0, T = 0;
  double* rec = nullptr;
  double* cvec = nullptr;
  const double* coef_ready = nullptr;
  // deferred folds (one GPU), all in the prologue:
  //   K1's value-major window-dot partials [1 + nwin][k1_G];
  //   column j's norm / Gram partials (CTA-major rows of ng_ld, entry g at
  //   ng_off + g), null at j = 0;
  //   sketch partials (CTA-major rows of sk_ld, row q at 2q, 2q+1) of column
  //   sk_row, folded once (one warp per sketch row), or null.
  const double* k1_partials = nullptr;
  int k1_G = 0;
  const double* prev_ng = nullptr;
  int prev_ng_G = 0, prev_ng_ld = 0, prev_ng_off = 0, prev_ngram = 0;
  const double* prev_sk = nullptr;
  int prev_sk_G = 0, prev_sk_ld = 0, sk_row = 0;
};

/// Sketch row q from CTA-major tile partials [G][nvp]: lane-strided sums over
/// CTAs, a fixed xor tree, then Re(e^{i pi k/2N} Z) scaled — deterministic.
__device__ __forceinline__ void sketch_row_fold(const double* __restrict__ partials, int G, int nvp, int q, int lane,
                                                int s, const double2* __restrict__ tab,
                                                const double* __restrict__ row_scale, double* __restrict__ dst) {
  const double2 v = strided_sum2(partials + 2 * q, nvp, lane, G, 32);
  const double re = warp_sum(v.x), im = warp_sum(v.y);
  if (lane == 0) {
    const double2 hp = tab[3 * s + q];
    dst[q] = (hp.x * re - hp.y * im) * row_scale[q];
  }
}


/// Deferred-pipeline prologue of an update kernel (NT threads per CTA, every
/// CTA): folds K1's window dots and column j's norm / Gram in the same fixed
/// order in every CTA, folds a pending set of sketch rows (spread over all
/// warps of the grid), forms the MGS coefficients into coef[0..MAXT]; CTA 0
/// writes record rows j+1 (A, H), j (norm / Gram) and cvec[j].
/// The first half of the warps folds the dots, the second half the sketch
/// rows and loads the earlier window columns' MGS inputs, so every global
/// load of the prologue is in flight at once (one L2 round trip between
/// the previous kernel's completion and the coefficients, not three).
template <int MAXT, int NT>
__device__ __forceinline__ void deferred_prologue(const UpdateArgs& ua, int s, const double2* __restrict__ tab,
                                                  const double* __restrict__ row_scale, double* coef) {
  constexpr int NW = NT / 32, NWH = NW / 2;
  __shared__ double red[2 * MAXT + 1][NWH];
  __shared__ double sA[MAXT + 1], sB[MAXT], preB[MAXT * MAXT], preC[MAXT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x, G = gridDim.x;
  const int nA = 1 + ua.nwin;
  const bool prev = ua.prev_ng != nullptr;
  const int64_t R = ua.rstride;
  const int b_off = 2 * ua.T + 3;
  if (warp < NWH) {
    double a[MAXT + 1], bs[MAXT];
#pragma unroll
    for (int v = 0; v <= MAXT; ++v)
      a[v] = v < nA ? strided_sum(ua.k1_partials + static_cast<int64_t>(v) * ua.k1_G, 1, tid, ua.k1_G, NT / 2) : 0.0;
#pragma unroll
    for (int v = 0; v < MAXT; ++v)
      bs[v] = prev ? strided_sum(ua.prev_ng + ua.prev_ng_off + v, ua.prev_ng_ld, tid, ua.prev_ng_G, NT / 2) : 0.0;
#pragma unroll
    for (int v = 0; v <= MAXT; ++v) {
      const double r = warp_sum(a[v]);
      if (lane == 0) red[v][warp] = r;
    }
#pragma unroll
    for (int v = 0; v < MAXT; ++v) {
      const double r = warp_sum(bs[v]);
      if (lane == 0) red[MAXT + 1 + v][warp] = r;
    }
  } else {
    const int w2 = warp - NWH;
    if (w2 == NWH - 1 && MAXT > 1) {
      // B entries and scales of columns j-1 .. j-MAXT+1 (written by earlier steps)
      if (lane < (MAXT - 1) * MAXT) {
        const int d = 1 + lane / MAXT, g = lane % MAXT;
        preB[lane] = d < ua.nwin ? __ldcg(ua.rec + static_cast<int64_t>(ua.j - d) * R + b_off + g) : 0.0;
      } else if (lane >= 16 && lane < 16 + MAXT - 1) {
        const int d = lane - 15;
        preC[d - 1] = d < ua.nwin ? __ldcg(ua.cvec + ua.j - d) : 0.0;
      }
    }
    if (ua.prev_sk) {
      double* dst = ua.rec + static_cast<int64_t>(ua.sk_row) * R + b_off + ua.T;
      for (int q = w2 * G + b; q < s; q += G * NWH)  // at most a row or two per CTA
        sketch_row_fold(ua.prev_sk, ua.prev_sk_G, ua.prev_sk_ld, q, lane, s, tab, row_scale, dst);
    }
  }
  __syncthreads();
  if (tid < 2 * MAXT + 1) {
    double r = 0.0;
    for (int w = 0; w < NWH; ++w) r += red[tid][w];
    if (tid <= MAXT) sA[tid] = r;
    else sB[tid - MAXT - 1] = (tid - MAXT - 1 <= ua.prev_ngram) ? r : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    mgs_coefficients<MAXT>(ua.rec, R, ua.T, ua.j, ua.nwin, ua.cvec, coef, b == 0, sA, prev ? sB : nullptr,
                           MAXT > 1 ? preB : nullptr, MAXT > 1 ? preC : nullptr);
    if (b == 0) {
      double* recA = ua.rec + static_cast<int64_t>(ua.j + 1) * R;
      for (int v = 0; v < nA; ++v) recA[v] = sA[v];
      if (prev) {
        double* recj = ua.rec + static_cast<int64_t>(ua.j) * R + b_off;
        for (int g2 = 0; g2 < ua.T; ++g2) recj[g2] = g2 < MAXT ? sB[g2] : 0.0;
      }
    }
  }
}

// Tile-group layout: a CTA of kGroups x 128 threads per SM. Each group of
// four warps owns its own tiles (8 column pairs x 128 rows), transpose
// buffer and Horner state and synchronises on its own named barrier, so the
// groups' load, FFT and accumulation phases interleave on the SM.
constexpr int kGPairs = 8;                       // column pairs per tile (16 columns)
constexpr int kGroupsMax = 4;                    // tile groups per CTA (GRP template: 4, or 2 to co-reside)

template <int NT>
__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(NT) : "memory");
}

/// Table slot of the group jump z^{PR (GRP - 1)} (k_srdct_tables).
constexpr int jump_slot(int pr, int grp) {
  return pr * (grp - 1) == 24 ? 4 : (pr * (grp - 1) == 8 ? 5 : (pr * (grp - 1) == 28 ? 6 : 7));
}

template <int SRC, int NI, bool PAIRED, int MAXT, int GRP, int CHK = 0, int PR = kGPairs>
// GRP = 2 sketches run beside K1 / K2' on the same SMs (split pipeline): <= 85 registers.
__global__ void __launch_bounds__(GRP * PR * 16, (GRP == 2 && SRC == kSrcSketch) ? 3 : 1) k_srdct_tiles(TileArgs ta, const double* __restrict__ x,
                                                                 double xscale, double* __restrict__ out,
                                                                 UpdateArgs ua) {
  constexpr int kGT = PR * 16;  // threads per group
  constexpr int kCta = GRP * kGT;
  extern __shared__ double2 sm[];
  const int s = ta.s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = tid / kGT, lt = tid % kGT;
  double2* X = sm + g * (PR * kXS);                  // [8][257] per group
  double2* S1s = sm + GRP * (PR * kXS) + g * 2 * s;  // [s] per group
  double2* S2s = S1s + s;                                  // [s] per group
  double2* zq = sm + GRP * (PR * kXS + 2 * s);   // [s]  z = e^{2 i pi k/N}
  double2* zj = zq + s;                                    // [s]  z^{8 (GRP - 1)}: jump over the other groups' tiles
  double2* tw = zj + s;                                    // [256]
  // per-row tables in Horner order i (rows sorted by u = k mod 256, so a
  // warp's gathers X[pp][u], X[pp][-u] hit consecutive u: no bank conflicts)
  int* uq = reinterpret_cast<int*>(tw + 256);              // [s]
  int* pm = uq + s;                                        // [s] row of Horner slot i
  __shared__ double coef[MAXT + 1];
  __shared__ double nred[MAXT][kCta / 32];
  const int G = gridDim.x, b = blockIdx.x;
  const uint64_t twoN = 2u * static_cast<uint64_t>(ta.N);
  stamp_begin(ta.stamp);
  trace_mark(ta.trace, 0);
  for (int k = tid; k < 256; k += kCta) tw[k] = ta.tab[8 * s + k];
  for (int i = tid; i < s; i += kCta) {
    const int q = ta.uperm[i];
    zq[i] = ta.tab[2 * s + q];
    zj[i] = ta.tab[jump_slot(PR, GRP) * s + q];
    uq[i] = ta.uq[q];
    pm[i] = q;
  }
  for (int q = tid; q < GRP * 2 * s; q += kCta) S1s[q - g * 2 * s] = make_double2(0.0, 0.0);
  pdl_trigger();
  pdl_wait();  // everything below reads the previous kernels' output
  trace_mark(ta.trace, 4);
  if constexpr (SRC == kSrcUpdate) {
    if (ua.k1_partials) {
      deferred_prologue<MAXT, kCta>(ua, s, ta.tab, ta.row_scale, coef);
    } else if (ua.coef_ready) {
      if (tid <= MAXT) coef[tid] = tid <= ua.nwin ? ua.coef_ready[tid] : 0.0;
    } else if (tid == 0) {
      mgs_coefficients<MAXT>(ua.rec, ua.rstride, ua.T, ua.j, ua.nwin, ua.cvec, coef, b == 0);
    }
  }
  __syncthreads();
  trace_mark(ta.trace, 1);
  double cf[MAXT + 1];
  const double* W[MAXT];
  double* wout = nullptr;
  double nacc[MAXT];
#pragma unroll
  for (int k = 0; k < MAXT; ++k) nacc[k] = 0.0;
  if constexpr (SRC == kSrcUpdate) {
#pragma unroll
    for (int k = 0; k <= MAXT; ++k) cf[k] = coef[k];
#pragma unroll
    for (int d = 0; d < MAXT; ++d)
      W[d] = ua.V + static_cast<int64_t>(ua.j - (d < ua.nwin ? d : 0)) * ua.ldv + ua.own_off;
    wout = ua.V + static_cast<int64_t>(ua.j + 1) * ua.ldv + ua.own_off;
  }
  const int p = lt & (PR - 1), t = lt / PR;
  const int nI = NI ? NI : (ta.M >> 4);  // <= 8 nonzero stage-1 inputs
  // CTA b owns tiles [tb, te); group g takes te-1-g, te-1-g-GRP, ... (descending)
  const int64_t tb = static_cast<int64_t>(b) * ta.ntiles / G, te = static_cast<int64_t>(b + 1) * ta.ntiles / G;
  int64_t tlow = -1;

  for (int64_t tile = te - 1 - g; tile >= tb; tile -= GRP) {
    const int64_t aa = tile * (2 * PR) + 2 * p;
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = make_double2(0.0, 0.0);
    if (aa < ta.L) {
      if constexpr (SRC == kSrcUpdate) {
        // loads in chunks of CH rows, all issued before the chunk's math
        // NI = M/16 rows of 16 per column pair (M = 128 on one GPU; 64, 32, 16
        // on 2, 4, 8 ranks, where F = 2N/L stays 256)
        constexpr int CH0 = CHK > 0 ? CHK : (MAXT <= 2 ? 2 : 1);
        constexpr int CH = CH0 < NI ? CH0 : NI;
#pragma unroll
        for (int i0 = 0; i0 < NI; i0 += CH) {
          double2 yv[CH], wv[CH][MAXT];
          uint32_t bits[CH];
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int64_t jl = aa + ta.L * static_cast<int64_t>(t + 16 * (i0 + c));
            yv[c] = __ldcs(reinterpret_cast<const double2*>(ua.y + jl));
#pragma unroll
            for (int d = 0; d < MAXT; ++d)
              if (d < ua.nwin) wv[c][d] = __ldg(reinterpret_cast<const double2*>(W[d] + jl));
            bits[c] = __ldg(ta.sign_bits + ((ta.r0 + jl) >> 5));
          }
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int64_t jl = aa + ta.L * static_cast<int64_t>(t + 16 * (i0 + c));
            double w0 = cf[0] * yv[c].x, w1 = cf[0] * yv[c].y;
#pragma unroll
            for (int d = MAXT - 1; d >= 0; --d)
              if (d < ua.nwin) {
                w0 = fma(cf[1 + d], wv[c][d].x, w0);
                w1 = fma(cf[1 + d], wv[c][d].y, w1);
              }
            *reinterpret_cast<double2*>(wout + jl) = make_double2(w0, w1);
            nacc[0] = fma(w0, w0, fma(w1, w1, nacc[0]));
#pragma unroll
            for (int k = 1; k < MAXT; ++k)
              if (k <= ua.ngram) nacc[k] = fma(w0, wv[c][k - 1].x, fma(w1, wv[c][k - 1].y, nacc[k]));
            const int64_t jg = ta.r0 + jl;
            v[i0 + c] = make_double2((bits[c] >> (jg & 31)) & 1u ? w0 : -w0, (bits[c] >> ((jg + 1) & 31)) & 1u ? w1 : -w1);
          }
        }
      } else {
        double2 zv[8];
        uint32_t b0[8], b1[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          zv[i] = make_double2(0.0, 0.0);
          b0[i] = b1[i] = 0u;
          if (i < nI) {
            const int64_t jl = aa + ta.L * static_cast<int64_t>(t + 16 * i);
            const int64_t jg = ta.r0 + jl;
            if constexpr (PAIRED) {
              zv[i] = __ldcs(reinterpret_cast<const double2*>(x + jl));
              b0[i] = __ldg(ta.sign_bits + (jg >> 5));
              b1[i] = b0[i];
            } else {
              zv[i].x = __ldcs(x + jl);
              zv[i].y = aa + 1 < ta.L ? __ldcs(x + jl + 1) : 0.0;
              b0[i] = __ldg(ta.sign_bits + (jg >> 5));
              b1[i] = __ldg(ta.sign_bits + ((jg + 1) >> 5));
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t jg = ta.r0 + aa + ta.L * static_cast<int64_t>(t + 16 * i);
          const double zx = zv[i].x * xscale, zy = zv[i].y * xscale;
          v[i] = make_double2((b0[i] >> (jg & 31)) & 1u ? zx : -zx, (b1[i] >> ((jg + 1) & 31)) & 1u ? zy : -zy);
        }
      }
    }
    if constexpr (NI == 8) dft16_half(v);
    else dft16(v);
#pragma unroll
    for (int vv = 1; vv < 16; ++vv) v[vv] = cmul(v[vv], tw[(vv * t) & 255]);
    group_sync<kGT>(g);  // the group's previous Horner pass has finished reading X
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) X[p * kXS + vv * 16 + t] = v[vv];
    group_sync<kGT>(g);
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) v[tt] = X[p * kXS + t * 16 + tt];
    dft16(v);
    group_sync<kGT>(g);
#pragma unroll
    for (int w = 0; w < 16; ++w) X[p * kXS + t + 16 * w] = v[w];
    group_sync<kGT>(g);
    // Horner over the tile's 8 pairs, continuing the group's recurrence;
    // the first step also jumps over the GRP - 1 tiles in between
    const bool first = tlow < 0;
    for (int q = lt; q < s; q += kGT) {
      const int u = uq[q], um = (256 - u) & 255;
      const double2 zz = zq[q];
      double2 S1 = S1s[q], S2 = S2s[q];
      if (!first) {
        const double2 jz = zj[q];
        S1 = cmul(S1, jz);
        S2 = cmul(S2, jz);
      }
#pragma unroll
      for (int pp = PR - 1; pp >= 0; --pp) {
        const double2 C = X[pp * kXS + u];
        const double2 Cm = X[pp * kXS + um];
        S1 = make_double2(fma(S1.x, zz.x, fma(-S1.y, zz.y, C.x)), fma(S1.x, zz.y, fma(S1.y, zz.x, C.y)));
        S2 = make_double2(fma(S2.x, zz.x, fma(-S2.y, zz.y, Cm.x)), fma(S2.x, zz.y, fma(S2.y, zz.x, -Cm.y)));
      }
      S1s[q] = S1;
      S2s[q] = S2;
    }
    tlow = tile;
  }
  // publish each group's lowest tile, then combine the groups per row:
  // sum_g e^{i pi k (r0 + 16 tlow_g)/N} (g_alpha S1_g + g_beta S2_g)
  __shared__ int64_t glow[GRP];
  if (lt == 0) glow[g] = tlow;
  if constexpr (SRC == kSrcUpdate) {
#pragma unroll
    for (int k = 0; k < MAXT; ++k) {
      const double v = warp_sum(nacc[k]);
      if (lane == 0) nred[k][warp] = v;
    }
  }
  __syncthreads();
  trace_mark(ta.trace, 2);
  // CTA-major partials [b][nvp] so that both the writes here and the folds'
  // reads are coalesced (a value-major layout made every fold load its own
  // L2 request: a multi-µs tail)
  const int nv = 2 * s + (SRC == kSrcUpdate ? MAXT : 0);
  const int nvp = (nv + 1) & ~1;
  for (int i = tid; i < s; i += kCta) {
    const int q = pm[i];
    const uint64_t k = static_cast<uint64_t>(ta.rows[q]);
    const double2 ga = ta.tab[q], gb = ta.tab[s + q];
    double2 acc = make_double2(0.0, 0.0);
    for (int gg = 0; gg < GRP; ++gg) {
      if (glow[gg] < 0) continue;
      const double2* S = sm + GRP * (PR * kXS) + gg * 2 * s;
      double sn, cs;
      const uint64_t kx = k * static_cast<uint64_t>(ta.r0 + glow[gg] * 2 * PR);
      const uint64_t ph = (twoN & (twoN - 1)) == 0 ? (kx & (twoN - 1)) : kx % twoN;
      sincospi(static_cast<double>(ph) / static_cast<double>(ta.N), &sn, &cs);
      acc = cadd(acc, cmul(make_double2(cs, sn), cadd(cmul(ga, S[i]), cmul(gb, S[s + i]))));
    }
    *reinterpret_cast<double2*>(ta.partials + static_cast<int64_t>(b) * nvp + 2 * q) = acc;
  }
  if constexpr (SRC == kSrcUpdate) {
    if (tid < MAXT) {
      double v = 0.0;
      for (int w = 0; w < kCta / 32; ++w) v += nred[tid][w];
      ta.partials[static_cast<int64_t>(b) * nvp + 2 * s + tid] = v;
    }
  }
  trace_mark(ta.trace, 3);
  stamp_end(ta.stamp);
}

/// Fold of the tile kernels' CTA partials ([G][nvp], CTA-major), one warp per
/// sketch row (plus one per norm / Gram entry for the update source): lane
/// sums over CTAs lane, lane+32, ... then a fixed xor-tree — deterministic.
/// A separate small kernel instead of a last-CTA fold: the in-kernel version
/// ran serially on one SM with cold code and cost ~10 µs per launch.
template <int SRC>
__global__ void __launch_bounds__(256) k_srdct_fold(const double* __restrict__ partials, int G, int nvp, int s,
                                                     const double2* __restrict__ tab,
                                                     const double* __restrict__ row_scale, double* __restrict__ out,
                                                     UpdateArgs ua, int maxt) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q < s) {
    double* dst = out;
    if constexpr (SRC == kSrcUpdate) dst = ua.rec + static_cast<int64_t>(ua.j + 1) * ua.rstride + (2 * ua.T + 3) + ua.T;
    sketch_row_fold(partials, G, nvp, q, lane, s, tab, row_scale, dst);
  } else if (SRC == kSrcUpdate && q < s + ua.T) {
    const int g = q - s;
    double a = 0.0;
    if (g <= ua.ngram && g < maxt)
      a = strided_sum(partials + 2 * s + g, nvp, lane, G, 32);
    a = warp_sum(a);
    if (lane == 0) ua.rec[static_cast<int64_t>(ua.j + 1) * ua.rstride + (2 * ua.T + 3) + g] = a;
  }
}

// ----------------------------------------- split step pipeline (one GPU)
// K2' = the Arnoldi update alone (HBM streaming, deferred prologue); the
// SRDCT of w_{j+1} runs on a side stream concurrently with K1(j+1) / K2'(j+1)
// and its partials are folded two steps later (kernels.hpp SplitFold).
constexpr int kUpdThreads = 256;
constexpr int kNgLd = 4;  // norm / Gram partial row length (MAXT <= 4)

template <int MAXT>
__global__ void __launch_bounds__(kUpdThreads) k_update_split(UpdateArgs ua, int s, const double2* __restrict__ tab,
                                                              const double* __restrict__ row_scale, int64_t npairs,
                                                              double* __restrict__ partials,
                                                              unsigned long long* stamp) {
  stamp_begin(stamp);
  __shared__ double coef[MAXT + 1];
  __shared__ double nred[MAXT][kUpdThreads / 32];
  pdl_trigger();
  pdl_wait();
  deferred_prologue<MAXT, kUpdThreads>(ua, s, tab, row_scale, coef);
  __syncthreads();
  double cf[MAXT + 1];
#pragma unroll
  for (int k = 0; k <= MAXT; ++k) cf[k] = coef[k];
  const double2* W[MAXT];
#pragma unroll
  for (int d = 0; d < MAXT; ++d)
    W[d] = reinterpret_cast<const double2*>(ua.V + static_cast<int64_t>(ua.j - (d < ua.nwin ? d : 0)) * ua.ldv + ua.own_off);
  double2* wout = reinterpret_cast<double2*>(ua.V + static_cast<int64_t>(ua.j + 1) * ua.ldv + ua.own_off);
  const double2* y2 = reinterpret_cast<const double2*>(ua.y);
  double nacc[MAXT];
#pragma unroll
  for (int g = 0; g < MAXT; ++g) nacc[g] = 0.0;
  constexpr int U = 4;  // pairs in flight per thread
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kUpdThreads;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * kUpdThreads + threadIdx.x; i0 < npairs; i0 += U * stride) {
    double2 yv[U], wv[U][MAXT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      const bool ok = i < npairs;
      yv[u] = ok ? __ldcs(y2 + i) : make_double2(0.0, 0.0);
#pragma unroll
      for (int d = 0; d < MAXT; ++d) wv[u][d] = (ok && d < ua.nwin) ? __ldg(W[d] + i) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < npairs) {
        double w0 = cf[0] * yv[u].x, w1 = cf[0] * yv[u].y;
#pragma unroll
        for (int d = MAXT - 1; d >= 0; --d)
          if (d < ua.nwin) {
            w0 = fma(cf[1 + d], wv[u][d].x, w0);
            w1 = fma(cf[1 + d], wv[u][d].y, w1);
          }
        wout[i] = make_double2(w0, w1);
        nacc[0] = fma(w0, w0, fma(w1, w1, nacc[0]));
#pragma unroll
        for (int g = 1; g < MAXT; ++g)
          if (g <= ua.ngram) nacc[g] = fma(w0, wv[u][g - 1].x, fma(w1, wv[u][g - 1].y, nacc[g]));
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < MAXT; ++g) {
    const double v = warp_sum(nacc[g]);
    if (lane == 0) nred[g][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < kNgLd) {
    double v = 0.0;
    if (threadIdx.x < MAXT)
      for (int w = 0; w < kUpdThreads / 32; ++w) v += nred[threadIdx.x][w];
    partials[static_cast<int64_t>(blockIdx.x) * kNgLd + threadIdx.x] = v;
  }
  stamp_end(stamp);
}

/// End of a split cycle (no K2' follows step j): folds the pending sketch
/// partials of columns j (a) and j+1 (b) and K2'(j)'s norm / Gram (row j+1).
__global__ void __launch_bounds__(256) k_split_flush(const double* __restrict__ ska, int Ga, int lda,
                                                     const double* __restrict__ skb, int Gb, int ldb,
                                                     const double* __restrict__ ng, int Gn, int s,
                                                     const double2* __restrict__ tab,
                                                     const double* __restrict__ row_scale, double* __restrict__ rec,
                                                     int64_t rstride, int T, int j, int ngram, int maxt) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b_off = 2 * T + 3;
  if (q < s) {
    if (ska) sketch_row_fold(ska, Ga, lda, q, lane, s, tab, row_scale, rec + static_cast<int64_t>(j) * rstride + b_off + T);
  } else if (q < 2 * s) {
    sketch_row_fold(skb, Gb, ldb, q - s, lane, s, tab, row_scale, rec + static_cast<int64_t>(j + 1) * rstride + b_off + T);
  } else if (q < 2 * s + T) {
    const int g = q - 2 * s;
    double a = 0.0;
    if (g <= ngram && g < maxt)
      for (int bb = lane; bb < Gn; bb += 32) a += ng[static_cast<int64_t>(bb) * kNgLd + g];
    a = warp_sum(a);
    if (lane == 0) rec[static_cast<int64_t>(j + 1) * rstride + b_off + g] = a;
  }
}

/// Per-row constants of an SRDCT: g_alpha, g_beta, z = e^{2 i pi k/N},
/// half-phase e^{i pi k/2N}, the group jumps z^{8 (GRP-1)}, k mod 256, and
/// the 256 stage twiddles.
__global__ void k_srdct_tables(int64_t N, const int64_t* __restrict__ rows, int s, double2* __restrict__ tab,
                               int* __restrict__ uq) {
  const uint64_t twoN = 2u * static_cast<uint64_t>(N);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < s + 256; q += gridDim.x * blockDim.x) {
    double sn, cs;
    if (q < s) {
      const uint64_t k = static_cast<uint64_t>(rows[q]);
      sincospi(static_cast<double>(k) / static_cast<double>(N), &sn, &cs);
      tab[q] = make_double2(0.5 * (1.0 + sn), -0.5 * cs);
      tab[s + q] = make_double2(0.5 * (1.0 - sn), 0.5 * cs);
      sincospi(static_cast<double>((2 * k) % twoN) / static_cast<double>(N), &sn, &cs);
      tab[2 * s + q] = make_double2(cs, sn);
      sincospi(static_cast<double>(k) / (2.0 * static_cast<double>(N)), &sn, &cs);
      tab[3 * s + q] = make_double2(cs, sn);
      // group jumps z^E = e^{2 i pi k E / N}, E = pairs (groups - 1) in {24, 8, 28}, exact reduction
      for (int gi = 0; gi < 4; ++gi) {
        const uint64_t E = gi == 0 ? 24 : (gi == 1 ? 8 : (gi == 2 ? 28 : 16));
        const uint64_t e = (2 * k * E) % twoN;
        sincospi(static_cast<double>(e) / static_cast<double>(N), &sn, &cs);
        tab[(4 + gi) * s + q] = make_double2(cs, sn);
      }
      uq[q] = static_cast<int>(k & 255);
    } else {
      const int k = q - s;
      sincospi(static_cast<double>(k) / 128.0, &sn, &cs);
      tab[8 * s + k] = make_double2(cs, sn);
    }
  }
}

// Sparse sign, one warp per CTA: each lane owns a private column of the
// warp's [s][32] shared bins, so the ζ scatter-adds per element need neither
// atomics nor ordering; one hash serves four entries. CTA partials (row
// sums over lanes, CTA-major) are folded by k_sparse_fold in a fixed order.
template <int ZETA>  // 0: runtime zeta (<= 64)
__global__ void __launch_bounds__(32) k_sparse_sign_lanes(const double* __restrict__ x, double xscale, int64_t nloc,
                                                          int64_t r0, uint64_t key, int s, int zeta_rt,
                                                          double* __restrict__ partials) {
  extern __shared__ double bins[];  // [s][32]
  __shared__ int b0s[64], bss[64];
  const int zeta = ZETA ? ZETA : zeta_rt;
  const int lane = threadIdx.x;
  for (int i = lane; i < s * 32; i += 32) bins[i] = 0.0;
  for (int l = lane; l < zeta; l += 32) {
    b0s[l] = static_cast<int>((static_cast<int64_t>(l) * s) / zeta);
    bss[l] = static_cast<int>((static_cast<int64_t>(l + 1) * s) / zeta) - b0s[l];
  }
  __syncwarp();
  constexpr int NCH = ZETA ? (ZETA + 3) / 4 : 16;
  int b0r[ZETA ? ZETA : 1], bsr[ZETA ? ZETA : 1];
  if constexpr (ZETA > 0) {
#pragma unroll
    for (int l = 0; l < ZETA; ++l) {
      b0r[l] = b0s[l];
      bsr[l] = bss[l];
    }
  }
  const uint64_t nc = static_cast<uint64_t>(sparse_sign_chunks(zeta));
  const int64_t stride = static_cast<int64_t>(gridDim.x) * 32;
  if constexpr (ZETA > 0) {
    // UE elements per lane per iteration, loaded one iteration ahead: the
    // hash chains of the UE elements overlap each other and the loads
    constexpr int UE = 4;
    const int64_t step = UE * stride;
    int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32 + lane;
    double vn[UE];
#pragma unroll
    for (int u = 0; u < UE; ++u) vn[u] = j0 + u * stride < nloc ? __ldcs(x + j0 + u * stride) : 0.0;
    for (; j0 < nloc; j0 += step) {
      double v[UE];
#pragma unroll
      for (int u = 0; u < UE; ++u) {
        v[u] = vn[u] * xscale;
        const int64_t jn = j0 + step + u * stride;
        vn[u] = jn < nloc ? __ldcs(x + jn) : 0.0;
      }
      int row[UE][ZETA];
      double sv[UE][ZETA];
#pragma unroll
      for (int u = 0; u < UE; ++u) {
        const uint64_t jg = static_cast<uint64_t>(r0 + j0 + u * stride);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const uint64_t h = mix64(key + (jg * nc + static_cast<uint64_t>(c) + 1u) * kPhi64);
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const int l = 4 * c + e4;
            if (l < ZETA) {
              const uint32_t f = static_cast<uint32_t>(h >> (16 * e4)) & 0xFFFFu;
              row[u][l] = (b0r[l] + static_cast<int>(((f >> 1) & 0x7FFFu) * static_cast<uint32_t>(bsr[l]) >> 15)) * 32 + lane;
              sv[u][l] = (f & 1u) ? v[u] : -v[u];  // elements past the end carry v = 0
            }
          }
        }
      }
      // a column's ZETA rows lie in distinct blocks: its read-modify-writes
      // touch distinct bins; consecutive elements go one after the other
#pragma unroll
      for (int u = 0; u < UE; ++u) {
        double t[ZETA];
#pragma unroll
        for (int l = 0; l < ZETA; ++l) t[l] = bins[row[u][l]];
#pragma unroll
        for (int l = 0; l < ZETA; ++l) bins[row[u][l]] = t[l] + sv[u][l];
      }
    }
  } else {
    for (int64_t jl = static_cast<int64_t>(blockIdx.x) * 32 + lane; jl < nloc; jl += stride) {
      const double v = __ldcs(x + jl) * xscale;
      const uint64_t jg = static_cast<uint64_t>(r0 + jl);
      for (int c = 0; c < static_cast<int>(nc); ++c) {
        const uint64_t h = mix64(key + (jg * nc + static_cast<uint64_t>(c) + 1u) * kPhi64);
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const int l = 4 * c + e4;
          if (l < zeta) {
            const uint32_t f = static_cast<uint32_t>(h >> (16 * e4)) & 0xFFFFu;
            const int row = b0s[l] + static_cast<int>(((f >> 1) & 0x7FFFu) * static_cast<uint32_t>(bss[l]) >> 15);
            bins[row * 32 + lane] += (f & 1u) ? v : -v;
          }
        }
      }
    }
  }
  __syncwarp();
  for (int r = lane; r < s; r += 32) {
    double acc = 0.0;
    for (int e = 0; e < 32; ++e) acc += bins[r * 32 + e];
    partials[static_cast<int64_t>(blockIdx.x) * s + r] = acc;
  }
}

/// Sparse sign with one warp per 4-entry hash chunk (ZETA = 4·NCH): warp c
/// evaluates h_c for its lanes' columns and scatters entries 4c..4c+3, whose
/// rows lie in blocks 4c..4c+3 — a contiguous row range no other warp
/// touches. The CTA's lane-private bins are the same [s][32] doubles as in
/// k_sparse_sign_lanes, shared by NCH warps instead of one, so twice (ζ = 8)
/// the warps fit on an SM and each thread does half the hashing and
/// scattering per column. Same map, same deterministic fold.
template <int ZETA>
__global__ void __launch_bounds__(32 * (ZETA / 4)) k_sparse_sign_chunks(const double* __restrict__ x, double xscale,
                                                                        int64_t nloc, int64_t r0, uint64_t key, int s,
                                                                        double* __restrict__ partials) {
  constexpr int NCH = ZETA / 4;
  extern __shared__ double bins[];  // [s][32]
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < s * 32; i += blockDim.x) bins[i] = 0.0;
  int b0r[4], bsr[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int l = 4 * c + e;
    b0r[e] = static_cast<int>((static_cast<int64_t>(l) * s) / ZETA);
    bsr[e] = static_cast<int>((static_cast<int64_t>(l + 1) * s) / ZETA) - b0r[e];
  }
  const int rlo = b0r[0], rhi = b0r[3] + bsr[3];  // this warp's rows
  int rb[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) rb[e] = b0r[e] * 32 + lane;
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * 32;
  constexpr int UE = 4;
  const int64_t step = UE * stride;
  int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  double vn[UE];
#pragma unroll
  for (int u = 0; u < UE; ++u) vn[u] = j0 + u * stride < nloc ? __ldcs(x + j0 + u * stride) : 0.0;
  // hash arguments key + (jg*NCH + c + 1)*phi advance by step*NCH*phi per
  // iteration and stride*NCH*phi per element of the batch (mod 2^64, exact)
  const uint64_t d_u = static_cast<uint64_t>(stride) * NCH * kPhi64;
  const uint64_t d_it = static_cast<uint64_t>(step) * NCH * kPhi64;
  uint64_t arg0 = key + (static_cast<uint64_t>(r0 + j0) * NCH + static_cast<uint64_t>(c) + 1u) * kPhi64;
  for (; j0 < nloc; j0 += step, arg0 += d_it) {
    double v[UE];
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      v[u] = vn[u] * xscale;
      const int64_t jn = j0 + step + u * stride;
      vn[u] = jn < nloc ? __ldcs(x + jn) : 0.0;
    }
    int row[UE][4];
    double sv[UE][4];
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      const uint64_t h = mix64(arg0 + static_cast<uint64_t>(u) * d_u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t f = static_cast<uint32_t>(h >> (16 * e)) & 0xFFFFu;
        row[u][e] = rb[e] + static_cast<int>(((f >> 1) & 0x7FFFu) * static_cast<uint32_t>(bsr[e]) >> 15) * 32;
        // sign bit flipped when the entry's sign bit is clear
        sv[u][e] = __longlong_as_double(__double_as_longlong(v[u]) ^ (static_cast<long long>(~f & 1u) << 63));
      }
    }
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      double t[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) t[e] = bins[row[u][e]];
#pragma unroll
      for (int e = 0; e < 4; ++e) bins[row[u][e]] = t[e] + sv[u][e];
    }
  }
  __syncwarp();
  for (int r = rlo + lane; r < rhi; r += 32) {
    double acc = 0.0;
    for (int e = 0; e < 32; ++e) acc += bins[r * 32 + e];
    partials[static_cast<int64_t>(blockIdx.x) * s + r] = acc;
  }
}

/// out[r] = inv_sqrt_zeta * sum_b partials[b][r]: one warp per row, lane-
/// strided sums then a fixed xor tree.
__global__ void __launch_bounds__(256) k_sparse_fold(const double* __restrict__ partials, int G, int s,
                                                     double inv_sqrt_zeta, double* __restrict__ out,
                                                     const double* __restrict__ row_scale = nullptr) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= s) return;
  double a = 0.0;
  a = warp_sum(strided_sum(partials + r, s, lane, G, 32));
  if (lane == 0) out[r] = a * (row_scale ? row_scale[r] : inv_sqrt_zeta);
}

// ------------------------------------------------------- direct SRDCT rows
// For blocks whose length has no four-step factorisation with F = 256 (odd
// or otherwise awkward n, e.g. the 103^2 acceptance grid): every selected
// row evaluated term by term, X[k] = sum_j z_j cos(pi k (2j+1) / 2N), the
// cosine generated by a unit-complex rotation z <- z e^{i pi k / N} that is
// re-anchored from an exactly reduced integer phase every kAnchor terms
// (rounding grows ~kAnchor·eps, not with n). CTA = (256 selected rows, one
// column chunk staged in shared memory with the signs applied); partials
// [chunk][row] are folded per row in a fixed order by k_sparse_fold.
// Cost s·n·5 fp64 ops, no O(s·G) serial fold.
constexpr int kAnchor = 64;

__global__ void __launch_bounds__(kThreads) k_srdct_direct(const double* __restrict__ x, double xscale, int64_t N,
                                                           int64_t r0, int64_t nloc, int64_t chunk,
                                                           const uint32_t* __restrict__ sign_bits,
                                                           const int64_t* __restrict__ rows, int s,
                                                           double* __restrict__ partials) {
  extern __shared__ double zs[];  // chunk values sign ⊙ x
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * chunk;
  const int64_t c1 = min(nloc, c0 + chunk);
  for (int64_t jl = c0 + threadIdx.x; jl < c1; jl += blockDim.x) {
    const int64_t jg = r0 + jl;
    const bool pos = (__ldg(sign_bits + (jg >> 5)) >> (jg & 31)) & 1u;
    const double v = __ldg(x + jl) * xscale;
    zs[jl - c0] = pos ? v : -v;
  }
  __syncthreads();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= s) return;
  const uint64_t k = static_cast<uint64_t>(__ldg(rows + q));
  const uint64_t fourN = 4u * static_cast<uint64_t>(N);
  const double inv2N = 0.5 / static_cast<double>(N);
  double sn, cs;
  sincospi(static_cast<double>((2u * k) % fourN) * inv2N, &sn, &cs);
  const double2 step = make_double2(cs, sn);
  const uint64_t jump = (static_cast<uint64_t>(2 * kAnchor) * k) % fourN;  // phase advance per anchor block
  uint64_t ph = (k * (2u * static_cast<uint64_t>(r0 + c0) + 1u)) % fourN;
  double acc = 0.0;
  for (int64_t a = c0; a < c1; a += kAnchor) {
    sincospi(static_cast<double>(ph) * inv2N, &sn, &cs);
    double2 z = make_double2(cs, sn);
    const int len = c1 - a < kAnchor ? static_cast<int>(c1 - a) : kAnchor;
    const double* zp = zs + (a - c0);
    if (len == kAnchor) {
#pragma unroll 8
      for (int t = 0; t < kAnchor; ++t) {
        acc = fma(zp[t], z.x, acc);
        z = cmul(z, step);
      }
    } else {
      for (int t = 0; t < len; ++t) {
        acc = fma(zp[t], z.x, acc);
        z = cmul(z, step);
      }
    }
    ph += jump;
    if (ph >= fourN) ph -= fourN;
  }
  partials[static_cast<int64_t>(blockIdx.y) * s + q] = acc;
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

namespace {


size_t tiles_smem(int64_t s, int grp = kGroupsMax, int pr = kGPairs) {
  return sizeof(double2) * static_cast<size_t>(grp * (pr * kXS + 2 * s) + 2 * s + 256) +
         sizeof(int) * static_cast<size_t>(2 * s);
}

bool tiles_eligible(const SketchDev& S, const SrdctPlan& p) {
  return p.F == 256 && p.M % 16 == 0 && S.tab.size() > 0 && tiles_smem(S.s) <= 227 * 1024;
}

template <int SRC, int NI, bool PAIRED, int MAXT, int GRP = kGroupsMax, int CHK = 0, int PR = kGPairs>
void launch_tiles(Context& c, const char* name, const SketchDev& S, const SrdctPlan& p, int64_t row_begin,
                  const double* x, double xscale, double* out, const UpdateArgs& ua, StepFold* sf = nullptr) {
  const int64_t ntiles = (p.L + 2 * PR - 1) / (2 * PR);
  const int G = (sf && sf->fixed_grid)
                    ? c.num_sms
                    : static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((ntiles + GRP - 1) / GRP, c.num_sms)));
  const int64_t nv = (2 * S.s + (SRC == kSrcUpdate ? MAXT : 0) + 1) & ~int64_t{1};
  TileArgs ta;
  ta.N = S.n;
  ta.r0 = row_begin;
  ta.L = p.L;
  ta.ntiles = ntiles;
  ta.M = static_cast<int>(p.M);
  ta.s = static_cast<int>(S.s);
  ta.sign_bits = S.sign_bits.get();
  ta.rows = S.rows.get();
  ta.row_scale = S.row_scale.get();
  ta.tab = S.tab.get();
  ta.uq = S.uq.get();
  ta.uperm = S.uperm.get();
  ta.partials = sf ? sf->out_partials : c.partials(nv * G);
  ta.trace = c.trace(16 * static_cast<int64_t>(G));
  ta.stamp = c.launch_stamp(name);
  const size_t smem = tiles_smem(S.s, GRP, PR);
  auto kern = k_srdct_tiles<SRC, NI, PAIRED, MAXT, GRP, CHK, PR>;
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  {
    TimedLaunch t(c, name);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(GRP * PR * 16);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1] = {pdl_attribute()};
    cfg.attrs = at;
    cfg.numAttrs = (sf && pdl_enabled()) ? 1 : 0;  // deferred step pipeline: programmatic dependent launch
    SDR_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, x, xscale, out, ua));
  }
  if (sf) {  // the next step's update (or the pipeline flush) folds these
    sf->out_G = G;
    sf->out_nvp = static_cast<int>(nv);
    return;
  }
  const int nwarps = static_cast<int>(S.s) + (SRC == kSrcUpdate ? ua.T : 0);
  TimedLaunch t(c, "sketch_fold");
  k_srdct_fold<SRC><<<(nwarps + 7) / 8, 256, 0, c.stream>>>(ta.partials, G, static_cast<int>(nv), static_cast<int>(S.s),
                                                           S.tab.get(), S.row_scale.get(), out, ua, MAXT);
  SDR_KERNEL_CHECK();
}

}  // namespace

void launch_sparse_fold(Context& c, const double* partials, int G, int s, double scale, double* out) {
  TimedLaunch t(c, "sketch_fold");
  k_sparse_fold<<<(s + 7) / 8, 256, 0, c.stream>>>(partials, G, s, scale, out);
  SDR_KERNEL_CHECK();
}

void prepare_srdct_tables(Context& c, SketchDev& S) {
  S.tab.resize(8 * S.s + 256);
  S.uq.resize(S.s);
  k_srdct_tables<<<static_cast<int>((S.s + 256 + 255) / 256), 256, 0, c.stream>>>(S.n, S.rows.get(), static_cast<int>(S.s),
                                                                                 S.tab.get(), S.uq.get());
  SDR_KERNEL_CHECK();
  std::vector<int> perm(static_cast<size_t>(S.s));
  for (int q = 0; q < static_cast<int>(S.s); ++q) perm[static_cast<size_t>(q)] = q;
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) {
    return (S.rows_host[static_cast<size_t>(a)] & 255) < (S.rows_host[static_cast<size_t>(b)] & 255);
  });
  S.uperm.resize(S.s);
  SDR_CUDA(cudaMemcpyAsync(S.uperm.get(), perm.data(), sizeof(int) * perm.size(), cudaMemcpyHostToDevice, c.stream));
  c.sync();
}

bool update_sketch_eligible(const SketchDev& S, const VecLayout& lay, int need, int64_t row_begin, int64_t ldv) {
  if (S.kind != kSrdct || need > 4) return false;
  const SrdctPlan p = plan_srdct(S.n, lay.nloc);
  return tiles_eligible(S, p) && (p.M == 128 || p.M == 64 || p.M == 32 || p.M == 16) && p.L % 2 == 0 &&
         row_begin % 2 == 0 && lay.own_off % 2 == 0 &&
         ldv % 2 == 0;
}

int64_t update_sketch_partials_size(const SketchDev& S, int num_sms) { return (2 * S.s + 8) * num_sms; }

bool launch_update_sketch(Context& c, const SketchDev& S, const double* y, double* V, int64_t ldv, const VecLayout& lay,
                          int j, int nwin, int ngram, double* rec, const RecLayout& RL, double* cvec,
                          const double* coef_ready, int64_t row_begin, StepFold* sf) {
  const int need = std::max(nwin, ngram + 1);
  if (!update_sketch_eligible(S, lay, need, row_begin, ldv)) return false;
  const SrdctPlan p = plan_srdct(S.n, lay.nloc);
  UpdateArgs ua;
  ua.y = y;
  ua.V = V;
  ua.ldv = ldv;
  ua.own_off = lay.own_off;
  ua.rstride = RL.stride;
  ua.j = j;
  ua.nwin = nwin;
  ua.ngram = ngram;
  ua.T = RL.T;
  ua.rec = rec;
  ua.cvec = cvec;
  ua.coef_ready = coef_ready;
  if (sf) {
    ua.k1_partials = sf->k1_partials;
    ua.k1_G = sf->k1_G;
    if (sf->prev_partials) {  // the previous fused update's partials hold both norm / Gram and sketch rows
      ua.prev_ng = ua.prev_sk = sf->prev_partials;
      ua.prev_ng_G = ua.prev_sk_G = sf->prev_G;
      ua.prev_ng_ld = ua.prev_sk_ld = sf->prev_nvp;
      ua.prev_ng_off = 2 * static_cast<int>(S.s);
      ua.prev_ngram = sf->prev_ngram;
      ua.sk_row = j;
    }
  }
  // t <= 2: two tile groups per CTA with eight rows of loads in flight per
  // thread (242 registers) measured 2.5 % faster per step than four groups
  // with two rows (128 registers); SDR_K2_VARIANT=1 selects the latter.
  // Also measured slower (C2, isolated / step period): three groups of 168
  // registers (22.9 us / 52.0 us vs 19.1 / 48.4), an L2 prefetch of each
  // group's next tile (20.0 us), and a cp.async staging of the next tile in
  // per-thread shared-memory slots (21.4 us; its 201 KB of shared memory
  // also keeps K1 from starting early: 60.8 us step).
  static const int variant = [] {
    const char* e = std::getenv("SDR_K2_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  if (p.M == 128) {
    if (need <= 2 && variant == 1)
      launch_tiles<kSrcUpdate, 8, true, 2>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
    else if (need <= 2)
      launch_tiles<kSrcUpdate, 8, true, 2, 2, 8>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
    else
      launch_tiles<kSrcUpdate, 8, true, 4>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
  } else if (p.M == 64) {  // the per-rank row blocks of a 2..8-rank z-slab run
    if (need <= 2)
      launch_tiles<kSrcUpdate, 4, true, 2>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
    else
      launch_tiles<kSrcUpdate, 4, true, 4>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
  } else if (p.M == 32) {
    if (need <= 2)
      launch_tiles<kSrcUpdate, 2, true, 2>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
    else
      launch_tiles<kSrcUpdate, 2, true, 4>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
  } else {
    if (need <= 2)
      launch_tiles<kSrcUpdate, 1, true, 2>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
    else
      launch_tiles<kSrcUpdate, 1, true, 4>(c, "update_sketch", S, p, row_begin, nullptr, 1.0, nullptr, ua, sf);
  }
  return true;
}

void launch_update_sketch_flush(Context& c, const SketchDev& S, const StepFold& sf, double* rec, const RecLayout& RL,
                                int j, int ngram) {
  UpdateArgs ua;
  ua.rstride = RL.stride;
  ua.j = j;
  ua.ngram = ngram;
  ua.T = RL.T;
  ua.rec = rec;
  const int nwarps = static_cast<int>(S.s) + RL.T;
  TimedLaunch t(c, "sketch_fold");
  k_srdct_fold<kSrcUpdate><<<(nwarps + 7) / 8, 256, 0, c.stream>>>(sf.out_partials, sf.out_G, sf.out_nvp,
                                                                   static_cast<int>(S.s), S.tab.get(), S.row_scale.get(),
                                                                   nullptr, ua, (sf.out_nvp - 2 * static_cast<int>(S.s)));
  SDR_KERNEL_CHECK();
}

bool sketch_partials_eligible(const SketchDev& S, int64_t nloc, int64_t row_begin) {
  if (S.kind != kSrdct) return false;
  const SrdctPlan p = plan_srdct(S.n, nloc);
  return tiles_eligible(S, p) && tiles_smem(S.s, 2) <= 100 * 1024 && p.M == 128 && p.L % 2 == 0 && row_begin % 2 == 0;
}

int64_t sketch_partials_size(const SketchDev& S, int num_sms) { return (2 * S.s + 2) * num_sms; }

void launch_sketch_partials(Context& c, const SketchDev& S, const double* x_own, int64_t nloc, int64_t row_begin,
                            double* partials, int* G, int* ld) {
  const SrdctPlan p = plan_srdct(S.n, nloc);
  StepFold sf;
  sf.out_partials = partials;
  // two tile groups (256 threads, ~90 KB shared memory): co-resides with K1 / K2'
  launch_tiles<kSrcSketch, 8, true, 1, 2>(c, "sketch_side", S, p, row_begin, x_own, 1.0, nullptr, UpdateArgs{}, &sf);
  *G = sf.out_G;
  *ld = sf.out_nvp;
}

void launch_sketch_fold_partials(Context& c, const SketchDev& S, const double* partials, int G, int ld, double* out) {
  TimedLaunch t(c, "sketch_fold");
  k_srdct_fold<kSrcSketch><<<static_cast<int>((S.s + 7) / 8), 256, 0, c.stream>>>(
      partials, G, ld, static_cast<int>(S.s), S.tab.get(), S.row_scale.get(), out, UpdateArgs{}, 1);
  SDR_KERNEL_CHECK();
}

int64_t update_split_partials_size(int num_sms) { return static_cast<int64_t>(kNgLd) * num_sms * 8; }

int launch_update_split(Context& c, const SketchDev& S, const double* y, double* V, int64_t ldv, const VecLayout& lay,
                        int j, int nwin, int ngram, double* rec, const RecLayout& RL, double* cvec, const SplitFold& sf) {
  const int need = std::max(nwin, ngram + 1);
  if (need > 4 || lay.nloc % 2 || lay.own_off % 2 || ldv % 2)
    throw invalid("split step pipeline: update needs an even block and a window of at most 4");
  UpdateArgs ua;
  ua.y = y;
  ua.V = V;
  ua.ldv = ldv;
  ua.own_off = lay.own_off;
  ua.rstride = RL.stride;
  ua.j = j;
  ua.nwin = nwin;
  ua.ngram = ngram;
  ua.T = RL.T;
  ua.rec = rec;
  ua.cvec = cvec;
  ua.k1_partials = sf.k1_partials;
  ua.k1_G = sf.k1_G;
  if (sf.prev_ng) {
    ua.prev_ng = sf.prev_ng;
    ua.prev_ng_G = sf.prev_ng_G;
    ua.prev_ng_ld = kNgLd;
    ua.prev_ng_off = 0;
    ua.prev_ngram = sf.prev_ngram;
  }
  if (sf.prev_sk) {
    ua.prev_sk = sf.prev_sk;
    ua.prev_sk_G = sf.prev_sk_G;
    ua.prev_sk_ld = sf.prev_sk_ld;
    ua.sk_row = sf.sk_row;
  }
  const int64_t npairs = lay.nloc / 2;
  const int G = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((npairs + kUpdThreads - 1) / kUpdThreads,
                                                                        static_cast<int64_t>(c.num_sms) * 2)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kUpdThreads);
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1] = {pdl_attribute()};
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TimedLaunch t(c, "update");
  if (need <= 2)
    SDR_CUDA(cudaLaunchKernelEx(&cfg, k_update_split<2>, ua, static_cast<int>(S.s), static_cast<const double2*>(S.tab.get()),
                                static_cast<const double*>(S.row_scale.get()), npairs, sf.out_ng, c.launch_stamp("update")));
  else
    SDR_CUDA(cudaLaunchKernelEx(&cfg, k_update_split<4>, ua, static_cast<int>(S.s), static_cast<const double2*>(S.tab.get()),
                                static_cast<const double*>(S.row_scale.get()), npairs, sf.out_ng, c.launch_stamp("update")));
  return G;
}

void launch_split_flush(Context& c, const SketchDev& S, const double* ska, int Ga, int lda, const double* skb, int Gb,
                        int ldb, const double* ng, int Gn, double* rec, const RecLayout& RL, int j, int ngram, int maxt) {
  const int nwarps = 2 * static_cast<int>(S.s) + RL.T;
  TimedLaunch t(c, "sketch_fold");
  k_split_flush<<<(nwarps + 7) / 8, 256, 0, c.stream>>>(ska, Ga, lda, skb, Gb, ldb, ng, Gn, static_cast<int>(S.s),
                                                       S.tab.get(), S.row_scale.get(), rec, RL.stride, RL.T, j, ngram,
                                                       maxt);
  SDR_KERNEL_CHECK();
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
    if (tiles_eligible(S, p)) {
      if (p.M == 128 && p.L % 2 == 0 && row_begin % 2 == 0)
        launch_tiles<kSrcSketch, 8, true, 1>(c, "sketch", S, p, row_begin, x_own, xscale, out, UpdateArgs{});
      else
        launch_tiles<kSrcSketch, 0, false, 1>(c, "sketch", S, p, row_begin, x_own, xscale, out, UpdateArgs{});
      return;
    }
    if (p.F < 32 || static_cast<double>(S.s) * static_cast<double>(nloc) <= 4e9) {
      // direct rows: (row blocks) x (column chunks) ~ 2 CTAs per SM
      const int rb = static_cast<int>((S.s + kThreads - 1) / kThreads);
      const int64_t cb_want = std::max<int64_t>(1, (2 * c.num_sms + rb - 1) / rb);
      const int64_t chunk = std::min<int64_t>(round_up((nloc + cb_want - 1) / cb_want, kAnchor), 6144);  // <= 48 KB shared
      const int cb = static_cast<int>(std::max<int64_t>(1, (nloc + chunk - 1) / chunk));
      double* part = c.partials(static_cast<int64_t>(cb) * S.s);
      {
        TimedLaunch t(c, "sketch");
        k_srdct_direct<<<dim3(rb, cb), kThreads, sizeof(double) * static_cast<size_t>(chunk), c.stream>>>(
            x_own, xscale, S.n, row_begin, nloc, chunk, S.sign_bits.get(), S.rows.get(), static_cast<int>(S.s), part);
        SDR_KERNEL_CHECK();
      }
      TimedLaunch t(c, "sketch_fold");
      k_sparse_fold<<<static_cast<int>((S.s + 7) / 8), 256, 0, c.stream>>>(part, cb, static_cast<int>(S.s), 0.0, out,
                                                                          S.row_scale.get());
      SDR_KERNEL_CHECK();
      return;
    }
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, 2 * c.num_sms)));
    const size_t smem = sizeof(double2) * static_cast<size_t>((kTileA / 2) * p.F + p.F / 2 + S.s);
    ensure_dyn_smem(reinterpret_cast<const void*>(k_srdct), smem);
    TimedLaunch t(c, "sketch");
    k_srdct<<<grid, kThreads, smem, c.stream>>>(x_own, xscale, S.n, row_begin, p.M, p.L, static_cast<int>(p.F), p.logF,
                                                S.sign_bits.get(), S.rows.get(), S.row_scale.get(),
                                                static_cast<int>(S.s), ntiles, c.partials(2 * S.s * grid),
                                                c.counters() + 5, c.partials2(2 * S.s), out);
    SDR_KERNEL_CHECK();
    return;
  }
  // sparse sign
  const size_t lane_smem = sizeof(double) * 32 * static_cast<size_t>(S.s);
  if (lane_smem <= 48 * 1024 && S.zeta <= 64) {
    const int per_sm = static_cast<int>(std::max<size_t>(1, (200 * 1024) / (lane_smem + 1024)));
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((nloc + 255) / 256, static_cast<int64_t>(c.num_sms) * std::min(per_sm, 16))));
    double* part = c.partials(static_cast<int64_t>(grid) * S.s);
    {
      TimedLaunch t(c, "sketch");
      static const bool chunk_warps = [] {
        const char* e = std::getenv("SDR_SPARSE_CHUNKS");
        return !e || std::atoi(e) != 0;
      }();
      if (S.zeta == 8 && chunk_warps)
        k_sparse_sign_chunks<8><<<grid, 64, lane_smem, c.stream>>>(x_own, xscale, nloc, row_begin, S.key,
                                                                   static_cast<int>(S.s), part);
      else if (S.zeta == 8)
        k_sparse_sign_lanes<8><<<grid, 32, lane_smem, c.stream>>>(x_own, xscale, nloc, row_begin, S.key,
                                                                  static_cast<int>(S.s), 8, part);
      else
        k_sparse_sign_lanes<0><<<grid, 32, lane_smem, c.stream>>>(x_own, xscale, nloc, row_begin, S.key,
                                                                  static_cast<int>(S.s), static_cast<int>(S.zeta), part);
      SDR_KERNEL_CHECK();
    }
    TimedLaunch t(c, "sketch_fold");
    k_sparse_fold<<<static_cast<int>((S.s + 7) / 8), 256, 0, c.stream>>>(
        part, grid, static_cast<int>(S.s), 1.0 / std::sqrt(static_cast<double>(S.zeta)), out);
    SDR_KERNEL_CHECK();
    return;
  }
  const int64_t want = (nloc + 1023) / 1024;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 4 * c.num_sms)));
  const int64_t chunk = round_up((nloc + grid - 1) / grid, 32);
  const size_t smem = sizeof(double) * 32 * static_cast<size_t>(S.s);
  ensure_dyn_smem(reinterpret_cast<const void*>(k_sparse_sign), smem);
  TimedLaunch t(c, "sketch");
  k_sparse_sign<<<grid, kThreads, smem, c.stream>>>(x_own, xscale, nloc, row_begin, S.key, static_cast<int>(S.s),
                                                    static_cast<int>(S.zeta), 1.0 / std::sqrt(static_cast<double>(S.zeta)),
                                                    chunk, c.partials(S.s * grid), c.counters() + 6, out);
  SDR_KERNEL_CHECK();
}

}  // namespace sdr
