// K2s: truncated-Arnoldi update fused with the ζ = 8 sparse-sign sketch of
// the new basis vector (BASELINE C1/C5), sm_100a.
//
// Replaces arnoldi.hpp:91-114 (MGS window update, normalisation) plus the
// sketch application S v_{j+1} (arnoldi.hpp:110-114 / sketch.hpp:139-162)
// for the sparse-sign map of DESIGN.md §4 — one HBM pass instead of two
// (the separate sketch re-read w_{j+1} and was issue-bound at 0.15 of HBM).
//
// Data movement: a producer warp streams y = A w_j and the window columns
// w_{j-d} tile by tile (512 rows) into a 2-stage shared-memory ring with
// bulk-async copies (cp.async.bulk, mbarrier transaction counts), so the
// bytes in flight do not depend on how many warps are resident — the
// sketch's lane-private bins (s x 32 doubles per CTA) cap residency at four
// CTAs per SM. (Measured alternative, slower: no producer warp, the second
// consumer to release a stage issuing its refill — 1.17 vs 1.11 ms at C5.)
// Consumer warp c (0, 1) evaluates chunk hash h_c of its lanes' rows
// (entries 4c..4c+3, blocks 4c..4c+3: a row range no other warp touches)
// and scatters them; both recompute the (bitwise identical) update, warp 0
// stores w_{j+1} and accumulates ||w||^2 and the Gram entries. Per tile a
// warp first forms all its rows' hashes and updates (independent chains,
// issued back to back), releases the stage, then runs the scatter.
// Determinism: bins are lane-private, CTA rows are reduced in a fixed xor
// tree, CTA partials folded in a fixed order (k_sparse_fold / fold_partials).
#include "kernels.hpp"
#include "mgs.cuh"
#include "reduce.cuh"
#include "sketch.hpp"
#include "tma.cuh"

#include <cstdlib>

namespace sdr {

namespace {

// rows per ring stage (4 KB per vector) and stages: C5 sweep (t = 2, isolated,
// us per launch): 256/3 1108, 256/2 1209, 256/4 1110, 128/4 1356, 128/6 1272,
// 512/2 1006, 512/3 1252, 768/2 1203, 1024/2 2165 — larger tiles halve the
// per-tile bookkeeping, more stages cost a resident CTA per SM. One consumer
// warp per CTA doing all eight entries (no duplicated ring reads / update,
// four consumer warps per SM) measured 1766 us in-solve vs 1120 us: too few
// warps to cover the bin read-modify-writes (it did keep the GPU off its
// power cap, 1965 vs 1717 MHz, which is where K1's 1794 vs 1850 us came from)
constexpr int kTileRows = 512;
constexpr int kStages = 2;
constexpr int kConsumers = 2;  // one warp per 4-entry hash chunk (ζ = 8)
constexpr int kThreadsUS = 32 * (1 + kConsumers);  // producer + consumers

struct UpdSparseArgs {
  const double* y;
  double* V;
  int64_t ldv, own_off, n;
  int j, nwin, ngram;
  double* rec;
  int64_t rstride;
  int T;
  double* cvec;
  const double* coef_ready;
  double* ng_partials;
  double* sk_partials;  // [grid][s]
  int64_t row_begin;
  uint64_t key;
  int s;
  int64_t ntiles;
  unsigned long long* stamp;
};

/// NW = nwin window columns, NG = ngram Gram entries (compile time: the
/// per-row code has no window predicates).
template <int NW, int NG, int TR = kTileRows, int NS = kStages, int BS = 0>
__global__ void __launch_bounds__(kThreadsUS) k_update_sparse8(UpdSparseArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  __shared__ double coef[NW + 1];
  stamp_begin(a.stamp);
  const int s = a.s;
  double* bins = smem;                                 // [s][32]
  double* ring = smem + static_cast<int64_t>(s) * 32;  // [stage][1 + NW][TR]
  constexpr int kNvec = 1 + NW;
  constexpr int kStageElems = kNvec * TR;
  constexpr int kRowsPerLane = TR / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < s * 32; i += blockDim.x) bins[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kConsumers);
    }
    mbar_fence_init();
  }
  if (a.coef_ready) {
    if (threadIdx.x <= NW) coef[threadIdx.x] = a.coef_ready[threadIdx.x];
  } else if (threadIdx.x == 0) {
    // several ranks: records were allreduced after K1; every CTA forms the
    // same coefficients, CTA 0 publishes them in the record
    if constexpr (NW > 0) {
      double cfull[NW + 1];
      mgs_coefficients<NW>(a.rec, a.rstride, a.T, a.j, NW, a.cvec, cfull, blockIdx.x == 0);
      for (int k = 0; k <= NW; ++k) coef[k] = cfull[k];
    }
  }
  __syncthreads();

  // this CTA's contiguous tile range
  const int64_t t0 = a.ntiles * blockIdx.x / gridDim.x, t1 = a.ntiles * (blockIdx.x + 1) / gridDim.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // ||w||^2 and Gram entries (consumer 0; zero elsewhere)
  // Bulk copy of tile t into ring stage st (one thread): y and the window
  // columns, a 16-byte multiple (an odd last row of the vector is read directly).
  auto feed = [&](int64_t t, int st) {
    const int64_t r0 = t * TR;
    const int64_t rows = min(static_cast<int64_t>(TR), a.n - r0);
    const uint32_t bytes = static_cast<uint32_t>((rows & ~int64_t{1}) * 8);
    double* dst = ring + st * kStageElems;
    mbar_arrive_expect_tx(&full[st], bytes * kNvec);
    if (bytes) {
      bulk_g2s(dst, a.y + r0, bytes, &full[st]);
#pragma unroll
      for (int d = 0; d < NW; ++d)
        bulk_g2s(dst + (1 + d) * TR, a.V + static_cast<int64_t>(a.j - d) * a.ldv + a.own_off + r0, bytes,
                 &full[st]);
    }
  };
  if (warp == 0) {
    // ---- producer: the warp walks the tiles, one elected lane feeds the ring
    int st = 0;
    uint32_t ph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      if (t - t0 >= NS) mbar_wait_sleep(&empty[st], ph ^ 1u);
      if (lane == 0) feed(t, st);
      __syncwarp();
      if (++st == NS) st = 0, ph ^= 1u;
    }
  } else {
    // ---- consumers
    const int c = warp - 1;
    double cf[NW + 1];
#pragma unroll
    for (int k = 0; k <= NW; ++k) cf[k] = coef[k];
    int rb[4], bsz[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int l = 4 * c + e;
      rb[e] = (l * s) / 8;
      bsz[e] = ((l + 1) * s) / 8 - rb[e];
      rb[e] = rb[e] * 32 + lane;
    }
    // shared-memory byte address of bin row 0 of each entry's block (this lane)
    uint32_t rbB[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) rbB[e] = smem_addr(bins + rb[e]);
    // hash argument key + (jg*2 + c + 1)*phi; 32 rows further = 64 phi
    const uint64_t d_row = 64ull * kPhi64;
    double* wout = a.V + static_cast<int64_t>(a.j + 1) * a.ldv + a.own_off;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      const double* ys = ring + st * kStageElems + lane;
      const int64_t r0 = t * TR;
      const int rows = static_cast<int>(min(static_cast<int64_t>(TR), a.n - r0));
      const uint64_t arg0 =
          a.key + (static_cast<uint64_t>(a.row_begin + r0 + lane) * 2u + static_cast<uint64_t>(c) + 1u) * kPhi64;
      uint64_t h[kRowsPerLane];
#pragma unroll
      for (int u = 0; u < kRowsPerLane; ++u) h[u] = mix64(arg0 + u * d_row);
      mbar_wait(&full[st], ph);
      double w[kRowsPerLane];
      if (rows == TR) {  // full tile: no bounds checks
#pragma unroll
        for (int u = 0; u < kRowsPerLane; ++u) {
          double wv[NW > 0 ? NW : 1];
#pragma unroll
          for (int d = 0; d < NW; ++d) wv[d] = ys[(1 + d) * TR + 32 * u];
          double x = cf[0] * ys[32 * u];
#pragma unroll
          for (int d = NW - 1; d >= 0; --d) x = fma(cf[1 + d], wv[d], x);
          w[u] = x;
          if (c == 0) {
            __stcs(wout + r0 + 32 * u + lane, x);
            acc[0] = fma(x, x, acc[0]);
#pragma unroll
            for (int g = 1; g <= NG; ++g) acc[g] = fma(x, wv[g - 1], acc[g]);
          }
        }
      } else {  // the vector's last, partial tile
        const int even = rows & ~1;
        for (int u = 0; u < kRowsPerLane; ++u) {
          const int r = 32 * u + lane;
          double yv = 0.0, wv[NW > 0 ? NW : 1];
#pragma unroll
          for (int d = 0; d < NW; ++d) wv[d] = 0.0;
          if (r < even) {
            yv = ys[32 * u];
#pragma unroll
            for (int d = 0; d < NW; ++d) wv[d] = ys[(1 + d) * TR + 32 * u];
          } else if (r < rows) {  // odd last row of the vector: not in the bulk copy
            yv = a.y[r0 + r];
#pragma unroll
            for (int d = 0; d < NW; ++d) wv[d] = a.V[static_cast<int64_t>(a.j - d) * a.ldv + a.own_off + r0 + r];
          }
          // rows past the end carry w = 0 and store nothing
          double x = cf[0] * yv;
#pragma unroll
          for (int d = NW - 1; d >= 0; --d) x = fma(cf[1 + d], wv[d], x);
          w[u] = x;
          if (c == 0 && r < rows) {
            __stcs(wout + r0 + r, x);
            acc[0] = fma(x, x, acc[0]);
#pragma unroll
            for (int g = 1; g <= NG; ++g) acc[g] = fma(x, wv[g - 1], acc[g]);
          }
        }
      }
      // the stage's inputs are in registers now: release it to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == NS) st = 0, ph ^= 1u;
#pragma unroll
      for (int u = 0; u < kRowsPerLane; ++u) {
        // w with its sign bit flipped: an entry whose sign bit f & 1 is clear
        // takes -w, i.e. nwhi ^ (f << 31)
        const uint32_t nwhi = static_cast<uint32_t>(__double2hiint(w[u])) ^ 0x80000000u;
        const int wlo = __double2loint(w[u]);
        const uint32_t hw[2] = {static_cast<uint32_t>(h[u]), static_cast<uint32_t>(h[u] >> 32)};
        uint32_t addr[4];
        double sv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t f = hw[e >> 1] >> (16 * (e & 1));  // sign bit 0, row bits 1..15
          // bin ((f >> 1) & 0x7FFF) * bsz >> 15 == ((f & 0xFFFE) * bsz) >> 16 of
          // the block; 256 bytes (32 lane columns) per bin row
          const uint32_t xb = (f & 0xFFFEu) * static_cast<uint32_t>(BS > 0 ? BS : bsz[e]);
          addr[e] = rbB[e] + ((xb >> 16) << 8);
          sv[e] = __hiloint2double(static_cast<int>(nwhi ^ (f << 31)), wlo);
        }
        // a row's four entries lie in four distinct blocks: distinct bins
        double tv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(tv[e]) : "r"(addr[e]));
#pragma unroll
        for (int e = 0; e < 4; ++e) asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr[e]), "d"(tv[e] + sv[e]) : "memory");
      }
    }
    // CTA sketch rows of this warp's blocks: lane-ordered xor tree per row
    const int rlo = (4 * c * s) / 8, rhi = ((4 * c + 4) * s) / 8;
    for (int r = rlo; r < rhi; ++r) {
      const double v = warp_sum(bins[r * 32 + lane]);
      if (lane == 0) a.sk_partials[static_cast<int64_t>(blockIdx.x) * s + r] = v;
    }
  }
  // T values (entries past ngram are zero): value-major CTA partials, folded
  // into the record by a separate fixed-order kernel (no last-CTA fold: its
  // 8 KB of shared memory would cost a resident CTA per SM)
  block_partials<4>(acc, a.T, a.ng_partials);
  stamp_end(a.stamp);
}

/// One fold of a K2s launch's CTA partials into the record's B part, which
/// is contiguous: out[0, T) = the norm / Gram values (value-major partials),
/// out[T, T + s) = the sketch rows (CTA-major partials) times 1/sqrt(zeta).
/// Fixed-order sums (strided_sum, then the xor tree): the values
/// k_fold_partials / k_sparse_fold give, in one launch instead of two.
__global__ void __launch_bounds__(256) k_fold_update_sparse(const double* __restrict__ ng, int T,
                                                             const double* __restrict__ sk, int s, int G,
                                                             double scale, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q < T) {
    const double a = warp_sum(strided_sum(ng + static_cast<int64_t>(q) * G, 1, lane, G, 32));
    if (lane == 0) out[q] = a;
  } else if (q < T + s) {
    const int r = q - T;
    const double a = warp_sum(strided_sum(sk + r, s, lane, G, 32));
    if (lane == 0) out[T + r] = a * scale;
  }
}

size_t upd_sparse_smem(int s, int nwin, int tr = kTileRows, int ns = kStages) {
  return sizeof(double) * (static_cast<size_t>(s) * 32 + static_cast<size_t>(ns) * (1 + nwin) * tr);
}

template <int NW, int NG, int TR = kTileRows, int NS = kStages>
void upd_sparse_impl(Context& c, const SketchDev& S, UpdSparseArgs a, const RecLayout& RL, double* out) {
  // s = 120 (BASELINE C1 / C5): eight blocks of 15 rows, a compile-time block size
  static const bool bs_on = [] {
    const char* e = std::getenv("SDR_K2S_BS");
    return !e || std::atoi(e) != 0;
  }();
  auto kern = (bs_on && S.s == 120) ? k_update_sparse8<NW, NG, TR, NS, 15> : k_update_sparse8<NW, NG, TR, NS, 0>;
  const size_t smem = upd_sparse_smem(static_cast<int>(S.s), NW, TR, NS);
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  const int per_sm = std::max(1, blocks_per_sm(reinterpret_cast<const void*>(kern), kThreadsUS, smem));
  a.ntiles = (a.n + TR - 1) / TR;
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(a.ntiles, static_cast<int64_t>(c.num_sms) * per_sm)));
  a.ng_partials = c.partials(4 * static_cast<int64_t>(g));
  a.sk_partials = c.partials2(static_cast<int64_t>(g) * S.s);
  a.stamp = c.launch_stamp("update_sketch");
  {
    TimedLaunch t(c, "update_sketch");
    kern<<<g, kThreadsUS, smem, c.stream>>>(a);
    SDR_KERNEL_CHECK();
  }
  double* recB = a.rec + static_cast<int64_t>(a.j + 1) * RL.stride + RL.b_off();
  if (out == recB + RL.T) {  // the record's B part: norm / Gram, then the sketch rows
    TimedLaunch t(c, "sketch_fold");
    const int nw = RL.T + static_cast<int>(S.s);
    k_fold_update_sparse<<<(nw + 7) / 8, 256, 0, c.stream>>>(a.ng_partials, RL.T, a.sk_partials, static_cast<int>(S.s),
                                                             g, 1.0 / std::sqrt(8.0), recB);
    SDR_KERNEL_CHECK();
  } else {
    launch_fold_partials(c, a.ng_partials, g, RL.T, true, recB);
    launch_sparse_fold(c, a.sk_partials, g, static_cast<int>(S.s), 1.0 / std::sqrt(8.0), out);
  }
}

template <int NW>
void upd_sparse_ng(Context& c, const SketchDev& S, const UpdSparseArgs& a, const RecLayout& RL, double* out) {
  if constexpr (NW == 0) return upd_sparse_impl<0, 0>(c, S, a, RL, out);
  switch (a.ngram) {
    case 0: return upd_sparse_impl<NW, 0>(c, S, a, RL, out);
    case 1:
      return upd_sparse_impl<NW, (NW >= 1 ? 1 : 0)>(c, S, a, RL, out);
    case 2: return upd_sparse_impl<NW, (NW >= 2 ? 2 : 0)>(c, S, a, RL, out);
    default: return upd_sparse_impl<NW, (NW >= 3 ? 3 : 0)>(c, S, a, RL, out);
  }
}

}  // namespace

bool update_sparse_eligible(const SketchDev& S, const VecLayout& lay, const RecLayout& RL, int need, int64_t ldv) {
  static const bool on = [] {
    const char* e = std::getenv("SDR_FUSE_SPARSE");
    return !e || std::atoi(e) != 0;
  }();
  return on && S.kind == kSparseSign && S.zeta == 8 && need <= 4 && RL.T <= 4 && S.s >= 8 && S.s <= 128 &&
         lay.own_off % 2 == 0 && ldv % 2 == 0 && upd_sparse_smem(static_cast<int>(S.s), 4) <= 200 * 1024;
}

void launch_update_sparse(Context& c, const SketchDev& S, const double* y, double* V, int64_t ldv,
                          const VecLayout& lay, int j, int nwin, int ngram, double* rec, const RecLayout& RL,
                          double* cvec, const double* coef_ready, int64_t row_begin) {
  if (nwin < 0 || nwin > 4 || ngram < 0 || ngram > 3 || ngram > nwin || (nwin == 0 && !coef_ready))
    throw logic("launch_update_sparse: window outside the compiled range");
  UpdSparseArgs a{};
  a.y = y;
  a.V = V;
  a.ldv = ldv;
  a.own_off = lay.own_off;
  a.n = lay.nloc;
  a.j = j;
  a.nwin = nwin;
  a.ngram = ngram;
  a.rec = rec;
  a.rstride = RL.stride;
  a.T = RL.T;
  a.cvec = cvec;
  a.coef_ready = coef_ready;
  a.ntiles = (lay.nloc + kTileRows - 1) / kTileRows;
  a.row_begin = row_begin;
  a.key = S.key;
  a.s = static_cast<int>(S.s);
  double* out = rec + static_cast<int64_t>(j + 1) * RL.stride + RL.sketch_off();
  switch (nwin) {
    case 0: return upd_sparse_ng<0>(c, S, a, RL, out);  // w = coef_ready[0] y: a cycle's first column
    case 1: return upd_sparse_ng<1>(c, S, a, RL, out);
    case 2: return upd_sparse_ng<2>(c, S, a, RL, out);
    case 3: return upd_sparse_ng<3>(c, S, a, RL, out);
    default: return upd_sparse_ng<4>(c, S, a, RL, out);
  }
}

}  // namespace sdr
