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
#include "reduce.cuh"
#include "sketch.hpp"

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
