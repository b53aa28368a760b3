// GMRES-SDR driver: solve_cycle / solve semantics of the reference
// (solver.hpp:128-365) with every N-length operation on the GPU.
//
// Device pipeline per Arnoldi step j (single stream, no host round trip
// inside a step):   [halo(w_j)] K1 spmv+dots(+MGS coefficients) [allreduce A]
//                   K2 update  K3 sketch [allreduce B]  D2H(record j) event
// The host consumes step records strictly in order (incremental QR, LS
// solve, trigger test) while the device runs up to `kLookahead` steps ahead:
// the Arnoldi recurrence never depends on the least-squares result, so
// speculative steps are either consumed exactly as the reference would take
// them or discarded at cycle end.
//
// Cycle overlap: the Krylov basis V is double-buffered. When a cycle ends
// and another follows, the next cycle's init_krylov and first speculative
// steps are enqueued on the other buffer *before* the host runs the
// harmonic-Ritz SVD/Schur of the finished cycle, so the LAPACK work hides
// under device work (the recycle product U_new = [V U] P reads the finished
// buffer, which the new cycle does not touch).
#include "solver.hpp"
#include "peer.hpp"

#include <atomic>
#include <exception>
#include <functional>
#include <thread>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <optional>

namespace sdr {

namespace {
constexpr int kLookahead = 2;
constexpr int kPumpDepth = 3;  // steps kept in flight while the host runs restart bookkeeping

/// SDR_FUSE=0 disables the fused update+sketch kernel (A/B and parity checks).
/// SDR_SPLIT=1 runs the SRDCT on a side stream beside K1 / K2' (SplitFold).
/// Off by default: measured on B200 at C2, the co-resident SRDCT CTAs slowed
/// K1 from 27.5 to 50 us and the step period rose from 52.7 to 55.5 us.
bool split_pipeline() {
  static const bool on = [] {
    const char* e = std::getenv("SDR_SPLIT");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

bool fuse_update_sketch() {
  static const bool on = [] {
    const char* e = std::getenv("SDR_FUSE");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

struct Workspace {
  VecLayout lay;
  i64 m = -1, s = -1;
  int T = 0;
  RecLayout RL;
  DeviceBuffer<double> V[2];
  int nV = 0;
  DeviceBuffer<double> y, rec, cvec, corr, r0, rnew, x, tmp, scal, coef, coef_dev;
  DeviceBuffer<double> y2;            // KF step pipeline: y_{j+1} beside y_j (by step parity)
  DeviceBuffer<unsigned> chunk_done;  // KF: per-chunk completion counters of the update front
  DeviceBuffer<double> unorm;  // ||.||^2 of the fused restart pass's outputs (correction, U_new)
  DeviceBuffer<double> one;    // {1.0}: coefficient of a cycle's first column (w_0 = r0)
  double last_harmonic_ms = -1.0;  // host time of the previous cycle's harmonic pencil
  // several ranks: the step pipeline every rank agreed on (ArnoldiPipeline::setup_deferred)
  // (cache key: values every rank derives from the same call sequence — no
  // addresses, which could match on one rank and not on another)
  std::vector<i64> defer_key;
  bool defer_agreed = false;
  DeviceBuffer<double> p1, p2[2];  // deferred step pipeline: K1 / K2 CTA partials (K2's by step parity)
  // several ranks: the same partials folded over this rank's CTAs before the
  // allreduce; comb[j & 1] = [K2(j) folded (nvp) | K1(j + 1) folded], one
  // allreduce per step
  DeviceBuffer<double> p1f, comb[2];
  DeviceBuffer<double> p1b;                 // several ranks: boundary-slice partials of a split K1
  cudaStream_t halo_stream = nullptr;       // several ranks: halo transfers beside K1's interior
  cudaEvent_t ev_w = nullptr, ev_halo = nullptr;
  DeviceBuffer<double> gcoef;      // recycle-update GEMM coefficients
  DeviceBuffer<double> pside;      // recycle-update norm partials (runs on the side stream)
  DeviceBuffer<double> ps[2], pu[2];  // split pipeline: SRDCT / update partials by step parity
  cudaStream_t sk_stream = nullptr;   // split pipeline: SRDCT beside K1 / K2'
  cudaEvent_t ev_sk[2] = {nullptr, nullptr}, ev_u = nullptr, ev_skq = nullptr;
  PinnedBuffer<double> hgcoef;
  DeviceBuffer<const double*> inptr;
  DeviceBuffer<double*> outptr;
  PinnedBuffer<double> hrec, hscal, hcoef;
  PinnedBuffer<const double*> hin;
  PinnedBuffer<double*> hout;
  std::vector<cudaEvent_t> ev;   // record j copied to the host (copy stream)
  std::vector<cudaEvent_t> evk;  // record j complete on the device (compute stream)
  cudaEvent_t ev_init = nullptr, ev_init_k = nullptr, ev_copies = nullptr;
  // Record read-back runs on its own stream so the compute stream never waits
  // for a device-to-host copy between steps (it did: ~9 µs per step).
  cudaStream_t copy_stream = nullptr;
  // recycle-update product off the compute stream (one GPU, deferred pipeline)
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_side_in = nullptr, ev_side_out = nullptr;
  std::vector<cudaEvent_t> evd;  // K2(j) finished (speculation pump)
  ~Workspace() {
    for (auto e : ev_sk)
      if (e) cudaEventDestroy(e);
    if (ev_u) cudaEventDestroy(ev_u);
    if (ev_skq) cudaEventDestroy(ev_skq);
    if (sk_stream) cudaStreamDestroy(sk_stream);
    for (auto e : evd) cudaEventDestroy(e);
    if (ev_side_in) cudaEventDestroy(ev_side_in);
    if (ev_side_out) cudaEventDestroy(ev_side_out);
    if (side_stream) cudaStreamDestroy(side_stream);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : evk) cudaEventDestroy(e);
    if (ev_init) cudaEventDestroy(ev_init);
    if (ev_init_k) cudaEventDestroy(ev_init_k);
    if (ev_copies) cudaEventDestroy(ev_copies);
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }
  /// D2H copy of n doubles once the compute stream reaches this point; done
  /// is recorded on the copy stream.
  void copy_back(Context& c, double* host, const double* dev, i64 n, cudaEvent_t ready, cudaEvent_t done) {
    SDR_CUDA(cudaEventRecord(ready, c.stream));
    SDR_CUDA(cudaStreamWaitEvent(copy_stream, ready, 0));
    SDR_CUDA(cudaMemcpyAsync(host, dev, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, copy_stream));
    SDR_CUDA(cudaEventRecord(done, copy_stream));
  }
  /// The compute stream waits for every copy issued so far (before rec rows
  /// that a pending copy may still read are rewritten by a new cycle).
  void fence_copies(Context& c) {
    SDR_CUDA(cudaEventRecord(ev_copies, copy_stream));
    SDR_CUDA(cudaStreamWaitEvent(c.stream, ev_copies, 0));
  }
  double* Vcol(int b, i64 i) const { return V[b].get() + i * lay.ld + lay.own_off; }
  double* Vbuf(int b, i64 i) const { return V[b].get() + i * lay.ld; }
};

Workspace& workspace(Context& c, const VecLayout& lay, i64 m, i64 s, int T) {
  auto w = std::static_pointer_cast<Workspace>(c.workspace);
  if (!w) {
    w = std::make_shared<Workspace>();
    c.workspace = w;
  }
  const bool relayout = w->lay.ld != lay.ld || w->lay.own_off != lay.own_off || w->lay.nloc != lay.nloc ||
                        w->lay.halo_lo != lay.halo_lo || w->lay.halo_hi != lay.halo_hi;
  if (relayout || m > w->m || s != w->s || T != w->T) {
    const i64 mm = std::max(m, w->m);
    w->lay = lay;
    w->m = mm;
    w->s = s;
    w->T = T;
    w->RL = RecLayout::make(T, s);
    w->V[1].release();
    w->V[0].resize((mm + 1) * lay.ld);
    SDR_CUDA(cudaMemsetAsync(w->V[0].get(), 0, sizeof(double) * static_cast<size_t>(w->V[0].size()), c.stream));
    w->nV = 1;
    // second basis buffer for cycle overlap, only when it leaves ample headroom
    size_t free_b = 0, total_b = 0;
    SDR_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t need = sizeof(double) * static_cast<size_t>((mm + 1) * lay.ld);
    if (free_b > need + (size_t{4} << 30) + total_b / 16) {
      w->V[1].resize((mm + 1) * lay.ld);
      SDR_CUDA(cudaMemsetAsync(w->V[1].get(), 0, need, c.stream));
      w->nV = 2;
    }
    w->rec.resize((mm + 2) * w->RL.stride);
    SDR_CUDA(cudaMemsetAsync(w->rec.get(), 0, sizeof(double) * static_cast<size_t>(w->rec.size()), c.stream));
    w->cvec.resize(mm + 2);
    w->hrec.ensure((mm + 2) * w->RL.stride);
    while (static_cast<i64>(w->ev.size()) < mm + 2) {
      cudaEvent_t e, k, d;
      SDR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&k, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&d, cudaEventDisableTiming));
      w->ev.push_back(e);
      w->evk.push_back(k);
      w->evd.push_back(d);
    }
    if (!w->ev_init) {
      SDR_CUDA(cudaEventCreateWithFlags(&w->ev_init, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&w->ev_init_k, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&w->ev_copies, cudaEventDisableTiming));
      SDR_CUDA(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
      SDR_CUDA(cudaStreamCreateWithFlags(&w->side_stream, cudaStreamNonBlocking));
      SDR_CUDA(cudaStreamCreateWithFlags(&w->sk_stream, cudaStreamNonBlocking));
      for (auto& e : w->ev_sk) SDR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&w->ev_u, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&w->ev_skq, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&w->ev_side_in, cudaEventDisableTiming));
      SDR_CUDA(cudaEventCreateWithFlags(&w->ev_side_out, cudaEventDisableTiming));
    }
  }
  const i64 nl = std::max<i64>(lay.nloc, 1);
  w->y.ensure(nl);
  w->corr.ensure(lay.ld);
  if (relayout) SDR_CUDA(cudaMemsetAsync(w->corr.get(), 0, sizeof(double) * static_cast<size_t>(lay.ld), c.stream));
  w->r0.ensure(nl);
  w->rnew.ensure(nl);
  w->x.ensure(nl);
  w->tmp.ensure(lay.ld);
  w->scal.ensure(64);
  w->unorm.ensure(32);
  w->coef_dev.ensure(std::max<i64>(64, T + 2));
  w->hscal.ensure(64);
  return *w;
}

void ensure_ptrs(Workspace& w, i64 nin, i64 nout) {
  w.inptr.ensure(nin);
  w.outptr.ensure(nout);
  w.coef.ensure(nin * std::max<i64>(nout, 1));
  w.hin.ensure(nin);
  w.hout.ensure(nout);
  w.hcoef.ensure(nin * std::max<i64>(nout, 1));
}

/// out_o = sum_i coef(i, o) * in_i through the K4 kernel (chunks of 32 outputs).
void tallskinny(Context& c, Workspace& w, const std::vector<const double*>& in, const HMat& coef /* nin x nout */,
                const std::vector<double*>& out, i64 n, double* norms2_dev) {
  const i64 nin = static_cast<i64>(in.size()), nout = static_cast<i64>(out.size());
  if (nout == 0) return;
  if (nin == 0) {
    for (auto* o : out) SDR_CUDA(cudaMemsetAsync(o, 0, sizeof(double) * static_cast<size_t>(n), c.stream));
    if (norms2_dev) SDR_CUDA(cudaMemsetAsync(norms2_dev, 0, sizeof(double) * static_cast<size_t>(nout), c.stream));
    return;
  }
  c.sync();  // staging buffers are reused
  ensure_ptrs(w, nin, nout);
  for (i64 i = 0; i < nin; ++i) w.hin.get()[i] = in[static_cast<size_t>(i)];
  SDR_CUDA(cudaMemcpyAsync(w.inptr.get(), w.hin.get(), sizeof(void*) * nin, cudaMemcpyHostToDevice, c.stream));
  for (i64 o0 = 0; o0 < nout; o0 += 32) {
    const i64 no = std::min<i64>(32, nout - o0);
    if (o0 > 0) c.sync();
    for (i64 i = 0; i < nin; ++i)
      for (i64 o = 0; o < no; ++o) w.hcoef.get()[i * no + o] = coef(i, o0 + o);
    for (i64 o = 0; o < no; ++o) w.hout.get()[o] = out[static_cast<size_t>(o0 + o)];
    SDR_CUDA(cudaMemcpyAsync(w.coef.get(), w.hcoef.get(), sizeof(double) * nin * no, cudaMemcpyHostToDevice, c.stream));
    SDR_CUDA(cudaMemcpyAsync(w.outptr.get(), w.hout.get(), sizeof(void*) * no, cudaMemcpyHostToDevice, c.stream));
    launch_tallskinny(c, w.inptr.get(), static_cast<int>(nin), w.coef.get(), static_cast<int>(no), w.outptr.get(), n,
                      norms2_dev ? norms2_dev + o0 : nullptr);
  }
}

struct HostKrylov {
  HMat H, SV, SAV;
  std::vector<double> cv;  // device scale of each stored column
  i64 j = 0;
  double r0_norm = 0.0;
  bool breakdown = false;
};

/// Harmonic pencil (and basis condition number) of a cycle, started on a host
/// thread as soon as the cycle's trigger fires — before the correction and
/// the verification residual — from copies of the cycle's sketched blocks.
/// Discarded (thread detached, result dropped) if the cycle continues.
struct EarlyHarmonic {
  i64 j = -1, kh = -1;
  Harmonic hp;
  bool have_hp = false, have_cond = false;
  bool product_done = false;  // U_new (and its norms, Workspace::unorm + 1) came out of the fused restart pass
  double cond = 1.0, ms = 0.0, cond_ms = 0.0;
  std::exception_ptr err;
  std::atomic<bool> done{false};
  std::thread th;
  ~EarlyHarmonic() {
    if (th.joinable()) th.join();
  }
};

std::shared_ptr<EarlyHarmonic> start_early_harmonic(const HostKrylov& st, const Recycle& sp, const HostQR* qr, i64 k,
                                                    double rank_tol) {
  auto e = std::make_shared<EarlyHarmonic>();
  const i64 j = st.j, kh = sp.dim(), s = st.SV.rows;
  e->j = j;
  e->kh = kh;
  auto SAW = std::make_shared<HMat>(s, kh + j), SW = std::make_shared<HMat>(s, kh + j);
  for (i64 q = 0; q < kh; ++q) {
    std::copy(sp.SAU.col(q), sp.SAU.col(q) + s, SAW->col(q));
    std::copy(sp.SU.col(q), sp.SU.col(q) + s, SW->col(q));
  }
  for (i64 i = 0; i < j; ++i) {
    std::copy(st.SAV.col(i), st.SAV.col(i) + s, SAW->col(kh + i));
    std::copy(st.SV.col(i), st.SV.col(i) + s, SW->col(kh + i));
  }
  std::shared_ptr<HMat> Q, R;
  if (qr && qr->clean() && qr->cols() == kh + j) {
    Q = std::make_shared<HMat>(s, kh + j);
    R = std::make_shared<HMat>(kh + j, kh + j);
    qr->factors(Q->a.data(), R->a.data());
  }
  std::shared_ptr<HMat> B;
  if (!st.breakdown) {
    B = std::make_shared<HMat>(s, j + 1);
    std::copy(st.SV.a.begin(), st.SV.a.begin() + s * (j + 1), B->a.begin());
  }
  std::weak_ptr<EarlyHarmonic> self = e;
  EarlyHarmonic* raw = e.get();
  // two threads: the basis condition number and the pencil are independent
  raw->th = std::thread([raw, SAW, SW, Q, R, B, k, rank_tol] {
    std::exception_ptr cond_err;
    std::thread tc;
    if (B) {
      tc = std::thread([raw, B, &cond_err] {
        try {
          const auto t0 = std::chrono::steady_clock::now();
          raw->cond = cond2(*B);
          raw->cond_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
          raw->have_cond = true;
        } catch (...) {
          cond_err = std::current_exception();
        }
      });
    }
    try {
      if (k > 0) {
        const auto t0 = std::chrono::steady_clock::now();
        raw->hp = (Q && R) ? harmonic_extract(*SAW, *SW, k, rank_tol, Q.get(), R.get())
                           : harmonic_extract(*SAW, *SW, k, rank_tol);
        raw->have_hp = true;
        raw->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      }
    } catch (...) {
      raw->err = std::current_exception();
    }
    if (tc.joinable()) tc.join();
    if (!raw->err && cond_err) raw->err = cond_err;
    raw->done.store(true, std::memory_order_release);
  });
  return e;
}

struct CycleOut {
  double residual_norm = 0, sres = 0, entry_norm = 0, sketched_entry = 0;
  i64 steps = 0;
  bool converged = false, breakdown = false, have_correction = false;
  double safety = 1.0;
  std::shared_ptr<HostQR> qr;  // the cycle's factorization of [SAU SAV] (reused by the recycle SVD)
  std::shared_ptr<EarlyHarmonic> early;
};

struct StepEvent {  // mirrors sdr_iteration_event in the C-ABI
  int32_t cycle;
  int64_t step, iteration;
  double sres, new_basis_sketch_norm;
  const double* y;
  int64_t y_len, space_dim;
};
struct ResidualEvent {
  int32_t cycle;
  int64_t iteration;
  double sres, true_residual;
};

double d2h_scalar(Context& c, Workspace& w, const double* dev) {
  SDR_CUDA(cudaMemcpyAsync(w.hscal.get(), dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  return w.hscal.get()[0];
}

/// Device Arnoldi pipeline + host bookkeeping of init_krylov / arnoldi_step
/// (arnoldi.hpp:47-119) on basis buffer `vb`: the device produces step
/// records, the host turns them into H, SV, SAV exactly as the reference's
/// KrylovState.
struct ArnoldiPipeline {
  Context& c;
  Workspace& w;
  const DeviceOperator& A;
  const SketchDev& S;
  i64 t, m;
  double breakdown_tol;
  int vb;
  HostKrylov st;
  i64 issued = 0;
  double wait_ms = 0.0;

  ArnoldiPipeline(Context& c_, Workspace& w_, const DeviceOperator& A_, const SketchDev& S_, i64 t_, i64 m_,
                  double btol, int vb_)
      : c(c_), w(w_), A(A_), S(S_), t(t_), m(m_), breakdown_tol(btol), vb(vb_) {}

  /// w_0 = r0, ||r0||^2 and S r0 on the device; the host reads them in init_finish.
  void init_enqueue(const double* r0) {
    const RecLayout& RL = w.RL;
    setup_deferred();
    w.fence_copies(c);
    SDR_CUDA(cudaEventRecord(w.ev_skq, w.sk_stream));  // earlier side-stream sketches are done before reuse
    SDR_CUDA(cudaStreamWaitEvent(c.stream, w.ev_skq, 0));
    if (!A.apply && update_sparse_eligible(S, w.lay, RL, 1, w.lay.ld) && reinterpret_cast<uintptr_t>(r0) % 16 == 0) {
      // sparse sign: w_0 = r0, ||r0||^2 and S r0 in one bulk-copy pass (K2s with an empty window)
      if (w.one.size() == 0) {
        w.one.resize(1);
        const double v = 1.0;
        SDR_CUDA(cudaMemcpy(w.one.get(), &v, sizeof(double), cudaMemcpyHostToDevice));
      }
      launch_update_sparse(c, S, r0, w.V[vb].get(), w.lay.ld, w.lay, -1, 0, 0, w.rec.get(), RL, w.cvec.get(),
                           w.one.get(), A.row_begin);
    } else {
      launch_copy_norm(c, r0, w.Vcol(vb, 0), w.lay.nloc, w.rec.get() + RL.b_off());
      launch_sketch(c, S, w.Vcol(vb, 0), w.lay.nloc, A.row_begin, w.rec.get() + RL.sketch_off());
    }
    c.allreduce_sum(w.rec.get() + RL.b_off(), RL.b_len());
    w.copy_back(c, w.hrec.get(), w.rec.get(), RL.stride, w.ev_init_k, w.ev_init);
    issued = 0;
    done_upto = 0;
  }

  /// init_krylov bookkeeping (arnoldi.hpp:47-72); throws domain on a zero residual.
  void init_finish(Counters& cnt) {
    SDR_CUDA(cudaEventSynchronize(w.ev_init));
    const RecLayout& RL = w.RL;
    const i64 s = S.s;
    st = HostKrylov{};
    st.r0_norm = std::sqrt(w.hrec.get()[RL.b_off()]);
    ++cnt.inner_products;
    if (st.r0_norm == 0.0) throw domain("init_krylov: zero initial residual (already converged)");
    ++cnt.sketch_applies;
    st.H = HMat(m + 1, m);
    st.SV = HMat(s, m + 1);
    st.SAV = HMat(s, m);
    st.cv.assign(static_cast<size_t>(m + 1), 0.0);
    const double* sk = w.hrec.get() + RL.sketch_off();
    for (i64 r = 0; r < s; ++r) st.SV(r, 0) = sk[r] / st.r0_norm;
    st.cv[0] = 1.0 / st.r0_norm;
  }

  // deferred-fold pipeline (one GPU, fused update eligible): record row j is
  // completed by K2(j)'s prologue, so its copy follows K2(j); see StepFold
  bool deferred = false;
  bool split = false;  // deferred + SRDCT on the side stream (SplitFold)
  // several ranks, non-deferred steps: K2(j)'s record part B (norm, Gram,
  // sketch rows of w_{j+1}) is reduced together with K1(j+1)'s dots — one
  // allreduce per step over the contiguous record span [B_{j+1} | A_{j+2}]
  bool merge_b = false;
  bool wide = false;  // min(t, m) > kFusedWindowMax: enqueue_wide
  // one GPU, sparse sign, SELL-DIA: update(j) and SpMV(j+1) in one launch (KF, enqueue_fused)
  bool fused = false;
  StepFold last;  // partials K2(issued - 1) left
  i64 last_ngram = 0, last_j = -1;
  double* pend_buf = nullptr;  // several ranks: K2's folded partials not yet allreduced
  int pend_n = 0;

  /// Slices [b_lo, b_hi) whose rows never read a halo entry (rows
  /// [reach_lo_end, reach_hi_begin), recorded per row when the operator was
  /// created — not the halo widths, which bound only the columns, not which
  /// rows reach them); false when there is no halo or no interior.
  /// SDR_K1_SPLIT=force splits a halo-free operator too (four slices each
  /// side), which exercises the split launches on one rank.
  bool k1_split_range(i64& b_lo, i64& b_hi) const {
    static const int mode = [] {
      const char* e = std::getenv("SDR_K1_SPLIT");
      if (!e) return 1;
      return std::string(e) == "force" ? 2 : std::atoi(e);
    }();
    if (mode == 0) return false;
    const i64 ns = A.view().nslices;
    if (A.plan.empty()) {
      if (mode != 2 || ns < 16) return false;
      b_lo = 4;
      b_hi = ns - 4;
      return true;
    }
    b_lo = (A.reach_lo_end + kSlice - 1) / kSlice;
    b_hi = std::max<i64>(0, A.reach_hi_begin) / kSlice;
    return b_lo < b_hi;
  }

  /// Measurement: CUDA-event time of `reps` back-to-back relaunches of the
  /// last enqueued step's K1 and of its K2 on the library stream. Both are
  /// idempotent for fixed inputs (same y / w_{j+1} / partials / record rows
  /// are rewritten), so the state stays what the step left.
  void time_last_step(int reps, double* k1_us, double* k2_us) {
    if (!deferred || split || last_j < 1) throw logic("time_last_step: needs an enqueued deferred step j >= 1");
    const i64 j = last_j;
    const VecLayout& lay = w.lay;
    const RecLayout& RL = w.RL;
    const int nwin = static_cast<int>(std::min<i64>(t, j + 1));
    const int ngram = static_cast<int>(std::min<i64>(RL.T - 1, j + 1));
    double* Vb = w.V[vb].get();
    cudaEvent_t e[3];
    for (auto& x : e) SDR_CUDA(cudaEventCreate(&x));
    c.sync();
    SDR_CUDA(cudaEventRecord(e[0], c.stream));
    for (int r = 0; r < reps; ++r)
      launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), nullptr, w.rec.get(),
                          RL.stride, RL.T, w.cvec.get(), nullptr, w.p1.get(), 0);
    SDR_CUDA(cudaEventRecord(e[1], c.stream));
    StepFold sf = last;
    for (int r = 0; r < reps; ++r)
      launch_update_sketch(c, S, w.y.get(), Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, w.rec.get(), RL,
                           w.cvec.get(), nullptr, A.row_begin, &sf);
    SDR_CUDA(cudaEventRecord(e[2], c.stream));
    SDR_CUDA(cudaEventSynchronize(e[2]));
    float a = 0.f, b = 0.f;
    SDR_CUDA(cudaEventElapsedTime(&a, e[0], e[1]));
    SDR_CUDA(cudaEventElapsedTime(&b, e[1], e[2]));
    for (auto& x : e) cudaEventDestroy(x);
    *k1_us = 1e3 * a / reps;
    *k2_us = 1e3 * b / reps;
  }
  int pu_G[2] = {0, 0}, ps_G[2] = {0, 0}, ps_ld[2] = {0, 0};

  void setup_deferred() {
    // windows past the fused kernels' register capacity: unfused step (wide.cu)
    wide = std::min(t, m) > kFusedWindowMax;
    fused = false;
    if (wide) {
      deferred = split = merge_b = false;
      return;
    }
    const int need = static_cast<int>(std::max<i64>(std::min(t, m), std::min<i64>(w.RL.T - 1, m) + 1));
    static const bool defer_dist = [] {
      const char* e = std::getenv("SDR_DEFER_DIST");
      return !e || std::atoi(e) != 0;
    }();
    deferred = !A.apply && (!c.distributed() || defer_dist) && fuse_update_sketch() &&
               update_sketch_eligible(S, w.lay, need, A.row_begin, w.lay.ld);
    if (c.distributed() && !A.apply && defer_dist) {
      // the two step pipelines enqueue different collectives: every rank must
      // take the same one (eligibility depends on the rank's slab), agreed
      // once per workspace and sketch
      const std::vector<i64> key = {S.kind, S.n, S.s, S.zeta, need, A.row_begin, w.lay.nloc, w.lay.own_off, w.lay.ld};
      if (w.defer_key != key) {
        const i64 mine = deferred ? 1 : 0;
        std::vector<i64> all(static_cast<size_t>(c.world));
        c.allgather_i64(&mine, 1, all.data());
        w.defer_agreed = *std::min_element(all.begin(), all.end()) == 1;
        w.defer_key = key;
      }
      deferred = w.defer_agreed;
    }
    split = deferred && !c.distributed() && split_pipeline() && sketch_partials_eligible(S, w.lay.nloc, A.row_begin);
    merge_b = !deferred && c.distributed();
    fused = !deferred && m >= 2 && fused_step_eligible(A.view(), S, w.lay, w.RL, static_cast<int>(t), c.distributed());
    if (fused) {
      w.y2.ensure(std::max<i64>(w.lay.nloc, 1));
      w.chunk_done.ensure(fused_step_chunks(c, w.lay.nloc));
    }
    if (!deferred && c.distributed() && !A.apply) {
      // several ranks, non-deferred steps (sparse sign): K1's interior slices
      // still run beside the halo transfer (enqueue)
      w.p1.ensure(34 * static_cast<i64>(c.num_sms) * 8);
      w.p1b.ensure(34 * static_cast<i64>(c.num_sms) * 8);
      if (!w.halo_stream) {
        SDR_CUDA(cudaStreamCreateWithFlags(&w.halo_stream, cudaStreamNonBlocking));
        SDR_CUDA(cudaEventCreateWithFlags(&w.ev_w, cudaEventDisableTiming));
        SDR_CUDA(cudaEventCreateWithFlags(&w.ev_halo, cudaEventDisableTiming));
      }
    }
    if (!deferred) return;
    w.p1.ensure(34 * static_cast<i64>(c.num_sms) * 8);
    for (auto& b : w.p2) b.ensure(update_sketch_partials_size(S, c.num_sms));
    if (c.distributed()) {
      w.p1f.ensure(34);
      w.p1b.ensure(34 * static_cast<i64>(c.num_sms) * 8);
      for (auto& b : w.comb) b.ensure(update_sketch_partials_size(S, 1) + 34);
      if (!w.halo_stream) {
        SDR_CUDA(cudaStreamCreateWithFlags(&w.halo_stream, cudaStreamNonBlocking));
        SDR_CUDA(cudaEventCreateWithFlags(&w.ev_w, cudaEventDisableTiming));
        SDR_CUDA(cudaEventCreateWithFlags(&w.ev_halo, cudaEventDisableTiming));
      }
    }
    if (split) {
      for (auto& b : w.ps) b.ensure(sketch_partials_size(S, c.num_sms));
      for (auto& b : w.pu) b.ensure(update_split_partials_size(c.num_sms));
    }
  }

  void enqueue(i64 j) {
    const VecLayout& lay = w.lay;
    const RecLayout& RL = w.RL;
    const i64 R = RL.stride;
    const int T = RL.T;
    const int nwin = static_cast<int>(std::min<i64>(t, j + 1));
    const int ngram = static_cast<int>(std::min<i64>(T - 1, j + 1));
    double* Vb = w.V[vb].get();
    double* recj = w.rec.get() + (j + 1) * R;
    if (split) {
      enqueue_split(j, nwin, ngram);
      return;
    }
    if (wide) {
      enqueue_wide(j, nwin, ngram);
      return;
    }
    if (fused) {
      enqueue_fused(j, nwin, ngram);
      return;
    }
    if (deferred) {
      const bool dist = c.distributed();
      // several ranks: K1 over the interior slices (no halo rows in their
      // stencils) runs while the halo of w_j moves on its own stream; the
      // boundary slices follow once it has landed
      i64 b_lo = 0, b_hi = 0;
      const bool split_k1 = dist && k1_split_range(b_lo, b_hi);
      if (split_k1) {
        SDR_CUDA(cudaEventRecord(w.ev_w, c.stream));
        SDR_CUDA(cudaStreamWaitEvent(w.halo_stream, w.ev_w, 0));
        c.halo_exchange(A.plan, w.Vbuf(vb, j) + lay.ext_shift(), A.ext_begin, w.Vcol(vb, j), A.row_begin,
                        w.halo_stream);
        SDR_CUDA(cudaEventRecord(w.ev_halo, w.halo_stream));
      } else {
        c.halo_exchange(A.plan, w.Vbuf(vb, j) + lay.ext_shift(), A.ext_begin, w.Vcol(vb, j), A.row_begin);
      }
      // several ranks: each rank folds its own CTA partials (fixed order) and
      // only the folded values cross the NVLink fabric, once per step
      // ([2s + t after K2(j-1) | 1 + nwin after K1(j)] instead of every
      // CTA's row after each kernel); NCCL's allreduce hands every rank the
      // same sums, so all ranks fold identically
      StepFold sf;
      sf.k1_partials = w.p1.get();
      int gb = 0;
      if (split_k1) {
        const i64 ns = A.view().nslices;
        sf.k1_G = launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), nullptr,
                                      w.rec.get(), R, T, w.cvec.get(), nullptr, w.p1.get(), 0, b_lo, b_hi);
        SDR_CUDA(cudaStreamWaitEvent(c.stream, w.ev_halo, 0));
        gb = launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), nullptr,
                                 w.rec.get(), R, T, w.cvec.get(), nullptr, w.p1b.get(), 0, b_hi, ns + b_lo);
      } else {
        sf.k1_G = launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), nullptr,
                                      w.rec.get(), R, T, w.cvec.get(), nullptr, w.p1.get(), 0);
      }
      if (dist) {  // K1(j)'s folded dots ride on the allreduce of K2(j-1)'s folded partials
        double* cb = pend_n > 0 ? pend_buf : w.p1f.get();
        const int off = pend_n;
        fold_allreduce(c, w.p1.get(), sf.k1_G, split_k1 ? w.p1b.get() : nullptr, gb, 1 + nwin, cb, off);
        sf.k1_partials = cb + off;
        sf.k1_G = 1;
        pend_n = 0;
      }
      if (j > 0) {
        sf.prev_partials = last.out_partials;
        sf.prev_G = last.out_G;
        sf.prev_nvp = last.out_nvp;
        sf.prev_ngram = static_cast<int>(last_ngram);
      }
      sf.out_partials = w.p2[j & 1].get();
      if (!launch_update_sketch(c, S, w.y.get(), Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, w.rec.get(), RL,
                                w.cvec.get(), nullptr, A.row_begin, &sf))
        throw logic("deferred step pipeline: fused update became ineligible");
      if (dist) {  // reduced together with K1(j+1)'s dots (or by flush at the cycle's end)
        double* folded = w.comb[j & 1].get();
        launch_fold_partials(c, sf.out_partials, sf.out_G, sf.out_nvp, false, folded);
        sf.out_partials = folded;
        sf.out_G = 1;
        pend_buf = folded;
        pend_n = sf.out_nvp;
      }
      last = sf;
      last_ngram = ngram;
      last_j = j;
      SDR_CUDA(cudaEventRecord(w.evd[static_cast<size_t>(j)], c.stream));
      if (j > 0)  // row j is complete now
        w.copy_back(c, w.hrec.get() + j * R, w.rec.get() + j * R, R, w.evk[static_cast<size_t>(j)],
                    w.ev[static_cast<size_t>(j)]);
      if (j + 1 == m) flush(j);
      return;
    }
    // one GPU: K1's last CTA forms the MGS coefficients; several: K2 forms
    // them after the allreduce of the window dots
    double* coef = c.distributed() ? nullptr : w.coef_dev.get();
    i64 b_lo = 0, b_hi = 0;
    if (c.distributed() && !A.apply && w.halo_stream && k1_split_range(b_lo, b_hi)) {
      // several ranks: the interior slices (no halo row in their stencils)
      // run while the halo of w_j moves on its own stream, the boundary
      // slices once it has landed; both leave CTA partials, folded into the
      // record in a fixed order before the allreduce
      SDR_CUDA(cudaEventRecord(w.ev_w, c.stream));
      SDR_CUDA(cudaStreamWaitEvent(w.halo_stream, w.ev_w, 0));
      c.halo_exchange(A.plan, w.Vbuf(vb, j) + lay.ext_shift(), A.ext_begin, w.Vcol(vb, j), A.row_begin, w.halo_stream);
      SDR_CUDA(cudaEventRecord(w.ev_halo, w.halo_stream));
      const i64 ns = A.view().nslices;
      const int g1 = launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), nullptr,
                                         w.rec.get(), R, T, w.cvec.get(), nullptr, w.p1.get(), 0, b_lo, b_hi);
      SDR_CUDA(cudaStreamWaitEvent(c.stream, w.ev_halo, 0));
      const int g2 = launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), nullptr,
                                         w.rec.get(), R, T, w.cvec.get(), nullptr, w.p1b.get(), 0, b_hi, ns + b_lo);
      launch_fold_partials2(c, w.p1.get(), g1, w.p1b.get(), g2, 1 + nwin, recj + RL.a_off());
    } else {
      c.halo_exchange(A.plan, w.Vbuf(vb, j) + lay.ext_shift(), A.ext_begin, w.Vcol(vb, j), A.row_begin);
      launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), recj + RL.a_off(),
                          w.rec.get(), R, T, w.cvec.get(), coef);
    }
    if (merge_b && j > 0) {
      // row j's B part (left by K2(j-1)), its padding and row j+1's A part
      // are contiguous: one allreduce, after which row j is complete
      c.allreduce_sum(w.rec.get() + j * R + RL.b_off(), (R - RL.b_off()) + (T + 1));
      w.copy_back(c, w.hrec.get() + j * R, w.rec.get() + j * R, R, w.evk[static_cast<size_t>(j)],
                  w.ev[static_cast<size_t>(j)]);
    } else {
      c.allreduce_sum(recj + RL.a_off(), T + 1);
    }
    if (update_sparse_eligible(S, lay, RL, std::max(nwin, ngram + 1), lay.ld)) {
      // sparse sign: update and sketch of w_{j+1} in one pass (sparse_update.cu)
      launch_update_sparse(c, S, w.y.get(), Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, w.rec.get(), RL,
                           w.cvec.get(), coef, A.row_begin);
    } else if (!fuse_update_sketch() ||
               !launch_update_sketch(c, S, w.y.get(), Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, w.rec.get(),
                                     RL, w.cvec.get(), coef, A.row_begin)) {
      launch_update(c, w.y.get(), Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, w.rec.get(), RL, w.cvec.get(),
                    coef);
      launch_sketch(c, S, w.Vcol(vb, j + 1), lay.nloc, A.row_begin, recj + RL.sketch_off());
    }
    if (merge_b && j + 1 < m) {  // reduced with K1(j+1)'s dots
      SDR_CUDA(cudaEventRecord(w.evd[static_cast<size_t>(j)], c.stream));
      return;
    }
    c.allreduce_sum(recj + RL.b_off(), RL.b_len());
    SDR_CUDA(cudaEventRecord(w.evd[static_cast<size_t>(j)], c.stream));
    w.copy_back(c, w.hrec.get() + (j + 1) * R, recj, R, w.evk[static_cast<size_t>(j + 1)],
                w.ev[static_cast<size_t>(j + 1)]);
  }

  /// KF step (one GPU, sparse sign, SELL-DIA): K1(0) alone at j = 0, then
  /// per step one launch doing the update + sketch of step j and the SpMV +
  /// window dots of step j+1 (fused_step.cu) and a one-CTA fold that writes
  /// record rows j+1 (B) and j+2 (A) and forms step j+1's coefficients; the
  /// cycle's last step is K2s alone. y_j alternates between two buffers.
  void enqueue_fused(i64 j, int nwin, int ngram) {
    const VecLayout& lay = w.lay;
    const RecLayout& RL = w.RL;
    const i64 R = RL.stride;
    double* Vb = w.V[vb].get();
    double* yj = (j & 1) ? w.y2.get() : w.y.get();
    double* yn = (j & 1) ? w.y.get() : w.y2.get();
    double* recj = w.rec.get() + (j + 1) * R;
    if (j == 0)  // K1(0); its last CTA forms step 0's coefficients
      launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, 0, nwin, yj, recj + RL.a_off(), w.rec.get(), R, RL.T,
                          w.cvec.get(), w.coef_dev.get());
    if (j + 1 < m) {
      const int nwin1 = static_cast<int>(std::min<i64>(t, j + 2));
      launch_fused_step(c, A.view(), S, yj, yn, Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, nwin1, w.rec.get(),
                        RL, w.cvec.get(), w.coef_dev.get(), A.row_begin, w.chunk_done.get());
    } else {
      launch_update_sparse(c, S, yj, Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, w.rec.get(), RL, w.cvec.get(),
                           w.coef_dev.get(), A.row_begin);
    }
    SDR_CUDA(cudaEventRecord(w.evd[static_cast<size_t>(j)], c.stream));
    w.copy_back(c, w.hrec.get() + (j + 1) * R, recj, R, w.evk[static_cast<size_t>(j + 1)],
                w.ev[static_cast<size_t>(j + 1)]);
  }

  /// Long window (min(t, m) > kFusedWindowMax): the step as separate passes
  /// (wide.cu) — product, the literal MGS loop (one pass and one reduced dot
  /// per window column), norm / Gram, sketch — into the same record layout.
  void enqueue_wide(i64 j, int nwin, int ngram) {
    const VecLayout& lay = w.lay;
    const RecLayout& RL = w.RL;
    const i64 R = RL.stride;
    double* Vb = w.V[vb].get();
    double* recj = w.rec.get() + (j + 1) * R;
    c.halo_exchange(A.plan, w.Vbuf(vb, j) + lay.ext_shift(), A.ext_begin, w.Vcol(vb, j), A.row_begin);
    launch_spmv(c, A.view(), w.Vbuf(vb, j) + lay.ext_shift(), w.y.get());
    launch_mgs_wide(c, w.y.get(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.rec.get(), R, RL.T, w.cvec.get(),
                    w.coef_dev.get());
    launch_window_dots_wide(c, w.Vcol(vb, j + 1), Vb, lay.ld, lay.own_off, static_cast<int>(j), ngram, true, lay.nloc,
                            recj + RL.b_off());
    launch_sketch(c, S, w.Vcol(vb, j + 1), lay.nloc, A.row_begin, recj + RL.sketch_off());
    c.allreduce_sum(recj + RL.b_off(), RL.b_len());
    SDR_CUDA(cudaEventRecord(w.evd[static_cast<size_t>(j)], c.stream));
    w.copy_back(c, w.hrec.get() + (j + 1) * R, recj, R, w.evk[static_cast<size_t>(j + 1)],
                w.ev[static_cast<size_t>(j + 1)]);
  }

  /// Split pipeline step (SplitFold): K1(j) and K2'(j) on the compute
  /// stream, SRDCT(j) of w_{j+1} on the side stream; row j-1 completes here.
  void enqueue_split(i64 j, int nwin, int ngram) {
    const VecLayout& lay = w.lay;
    const RecLayout& RL = w.RL;
    const i64 R = RL.stride;
    const int T = RL.T;
    double* Vb = w.V[vb].get();
    const int par = static_cast<int>(j & 1);
    SplitFold sf;
    sf.k1_partials = w.p1.get();
    sf.k1_G = launch_spmv_arnoldi(c, A.view(), Vb, lay.ld, lay, static_cast<int>(j), nwin, w.y.get(), nullptr,
                                  w.rec.get(), R, T, w.cvec.get(), nullptr, w.p1.get(), 2);
    if (j >= 1) {
      sf.prev_ng = w.pu[1 - par].get();
      sf.prev_ng_G = pu_G[1 - par];
      sf.prev_ngram = static_cast<int>(last_ngram);
    }
    if (j >= 2) {  // SRDCT(j-2) -> sketch rows of column j-1
      SDR_CUDA(cudaStreamWaitEvent(c.stream, w.ev_sk[par], 0));
      sf.prev_sk = w.ps[par].get();
      sf.prev_sk_G = ps_G[par];
      sf.prev_sk_ld = ps_ld[par];
      sf.sk_row = static_cast<int>(j - 1);
    }
    sf.out_ng = w.pu[par].get();
    pu_G[par] = launch_update_split(c, S, w.y.get(), Vb, lay.ld, lay, static_cast<int>(j), nwin, ngram, w.rec.get(), RL,
                                    w.cvec.get(), sf);
    last_ngram = ngram;
    SDR_CUDA(cudaEventRecord(w.evd[static_cast<size_t>(j)], c.stream));
    // SRDCT(j) of w_{j+1} beside the next steps
    SDR_CUDA(cudaEventRecord(w.ev_u, c.stream));
    SDR_CUDA(cudaStreamWaitEvent(w.sk_stream, w.ev_u, 0));
    std::swap(c.stream, w.sk_stream);
    launch_sketch_partials(c, S, w.Vcol(vb, j + 1), lay.nloc, A.row_begin, w.ps[par].get(), &ps_G[par], &ps_ld[par]);
    std::swap(c.stream, w.sk_stream);
    SDR_CUDA(cudaEventRecord(w.ev_sk[par], w.sk_stream));
    if (j >= 2)  // row j-1 is complete now
      w.copy_back(c, w.hrec.get() + (j - 1) * R, w.rec.get() + (j - 1) * R, R, w.evk[static_cast<size_t>(j - 1)],
                  w.ev[static_cast<size_t>(j - 1)]);
    if (j + 1 == m) flush_split(j);
  }

  /// Split pipeline: completes rows j and j + 1 when no K2'(j + 1) follows.
  void flush_split(i64 j) {
    const i64 R = w.RL.stride;
    const int par = static_cast<int>(j & 1);
    SDR_CUDA(cudaStreamWaitEvent(c.stream, w.ev_sk[par], 0));  // SRDCT(j) (and SRDCT(j-1) before it)
    const bool have_a = j >= 1;
    launch_split_flush(c, S, have_a ? w.ps[1 - par].get() : nullptr, ps_G[1 - par], ps_ld[1 - par], w.ps[par].get(),
                       ps_G[par], ps_ld[par], w.pu[par].get(), pu_G[par], w.rec.get(), w.RL, static_cast<int>(j),
                       static_cast<int>(last_ngram), 4);
    if (have_a)
      w.copy_back(c, w.hrec.get() + j * R, w.rec.get() + j * R, R, w.evk[static_cast<size_t>(j)],
                  w.ev[static_cast<size_t>(j)]);
    w.copy_back(c, w.hrec.get() + (j + 1) * R, w.rec.get() + (j + 1) * R, R, w.evk[static_cast<size_t>(j + 1)],
                w.ev[static_cast<size_t>(j + 1)]);
  }

  /// Deferred pipeline: completes row j + 1 when no K2(j + 1) will follow.
  void flush(i64 j) {
    const i64 R = w.RL.stride;
    if (pend_n > 0) {
      c.allreduce_sum(pend_buf, pend_n);
      pend_n = 0;
    }
    launch_update_sketch_flush(c, S, last, w.rec.get(), w.RL, static_cast<int>(j), static_cast<int>(last_ngram));
    w.copy_back(c, w.hrec.get() + (j + 1) * R, w.rec.get() + (j + 1) * R, R, w.evk[static_cast<size_t>(j + 1)],
                w.ev[static_cast<size_t>(j + 1)]);
  }

  i64 done_upto = 0;  // steps [0, done_upto) have finished on the GPU
  void poll_done() {
    while (done_upto < issued && cudaEventQuery(w.evd[static_cast<size_t>(done_upto)]) == cudaSuccess) ++done_upto;
  }

  /// Keep up to kLookahead speculative steps ahead of step j in flight, and
  /// at least two in flight while the host catches up with finished steps.
  void issue_ahead(i64 j) {
    while (issued < m && issued <= j + kLookahead + (split ? 1 : 0)) enqueue(issued++);
    if (lockstep()) return;
    poll_done();
    while (issued < m && issued - done_upto < 2) enqueue(issued++);
  }

  /// Several ranks: every step enqueues collectives (halo send/recv,
  /// allreduce), which NCCL matches by issue order per communicator. Steps
  /// are then issued only at points of the host program that are the same on
  /// every rank (a fixed look-ahead from the consumed step), never by how far
  /// this rank's GPU has progressed: otherwise one rank could enqueue a
  /// step's allreduce where another enqueues the restart's, and the
  /// collectives would pair up across different operations.
  bool lockstep() const { return c.distributed(); }

  /// Speculation while the host is busy elsewhere (restart bookkeeping):
  /// keeps kPumpDepth steps in flight without queueing the whole cycle
  /// (one rank only, see lockstep()).
  void pump() {
    if (lockstep()) return;
    poll_done();
    while (issued < m && issued - done_upto < kPumpDepth) enqueue(issued++);
  }

  /// Consumes step st.j (arnoldi.hpp:87-118 bookkeeping); returns true on
  /// lucky breakdown.
  bool step(Counters& cnt) {
    if (st.breakdown) throw logic("arnoldi_step: basis already broke down");
    if (st.j >= m) throw logic("arnoldi_step: step capacity exhausted");
    const i64 j = st.j;
    issue_ahead(j);
    const auto tw0 = std::chrono::steady_clock::now();
    SDR_CUDA(cudaEventSynchronize(w.ev[static_cast<size_t>(j + 1)]));
    wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw0).count();
    const RecLayout& RL = w.RL;
    const int T = RL.T;
    const i64 s = S.s;
    const double* rj = w.hrec.get() + (j + 1) * RL.stride;
    const int nwin = static_cast<int>(std::min<i64>(t, j + 1));
    const i64 i0 = j - nwin + 1;
    const double norm_before = rj[RL.h_off()];
    for (int d = 0; d < nwin; ++d) st.H(j - d, j) = rj[RL.h_off() + 1 + d];
    st.cv[static_cast<size_t>(j)] = rj[RL.h_off() + 1 + T];
    const double h_next = std::sqrt(rj[RL.b_off()]);
    ++cnt.matvecs;
    cnt.inner_products += 2 + nwin;
    bool brk = false;
    if (h_next <= breakdown_tol * norm_before) {  // arnoldi.hpp:101-108
      st.H(j + 1, j) = 0.0;
      for (i64 r = 0; r < s; ++r) {
        double acc = 0.0;
        for (i64 i = i0; i <= j; ++i) acc += st.SV(r, i) * st.H(i, j);
        st.SAV(r, j) = acc;
      }
      st.breakdown = true;
      brk = true;
    } else {
      st.H(j + 1, j) = h_next;
      st.cv[static_cast<size_t>(j + 1)] = 1.0 / h_next;
      const double* sk = rj + RL.sketch_off();
      const double inv_h = 1.0 / h_next;
      for (i64 r = 0; r < s; ++r) st.SV(r, j + 1) = sk[r] * inv_h;
      ++cnt.sketch_applies;
      for (i64 r = 0; r < s; ++r) {  // arnoldi.hpp:115
        double acc = 0.0;
        for (i64 i = i0; i <= j + 1; ++i) acc += st.SV(r, i) * st.H(i, j);
        st.SAV(r, j) = acc;
      }
    }
    st.j = j + 1;
    return brk;
  }
};

/// Runs `job` on a host thread while the calling thread keeps the GPU fed
/// through `pump` (no CUDA call leaves the calling thread).
template <class F>
void host_job_while_pumping(F&& job, const std::function<void()>* pump) {
  if (!pump) {
    job();
    return;
  }
  std::atomic<bool> done{false};
  std::exception_ptr err;
  std::thread th([&] {
    try {
      job();
    } catch (...) {
      err = std::current_exception();
    }
    done.store(true, std::memory_order_release);
  });
  while (!done.load(std::memory_order_acquire)) {
    (*pump)();
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  th.join();
  if (err) std::rethrow_exception(err);
}

/// pump: keeps the next cycle's speculative steps flowing while the host
/// computes the harmonic pencil (the GPU otherwise idles at every restart).
void update_recycle(Context& c, Workspace& w, const HostKrylov& st, int vb, Recycle& sp, i64 k, double rank_tol,
                    Counters& cnt, std::vector<std::string>* notes, Report& rep,
                    const std::function<void()>* pump = nullptr, bool side_stream = false,
                    const HostQR* qr = nullptr, const Harmonic* pre = nullptr,
                    bool product_done = false) {  // recycle.hpp:226-289
  const i64 j = st.j, kh = sp.dim(), s = st.SV.rows;
  if (j < 1) throw invalid("update_recycle: no Arnoldi steps taken");
  HMat SAW(s, kh + j), SW(s, kh + j);
  for (i64 q = 0; q < kh; ++q) {
    std::copy(sp.SAU.col(q), sp.SAU.col(q) + s, SAW.col(q));
    std::copy(sp.SU.col(q), sp.SU.col(q) + s, SW.col(q));
  }
  for (i64 i = 0; i < j; ++i) {
    std::copy(st.SAV.col(i), st.SAV.col(i) + s, SAW.col(kh + i));
    std::copy(st.SV.col(i), st.SV.col(i) + s, SW.col(kh + i));
  }
  Harmonic hp;
  if (pre) {
    hp = *pre;
  } else {
    double ms = 0.0;
    host_job_while_pumping(
        [&] {
          const auto t0 = std::chrono::steady_clock::now();
          // SAW = [SAU SAV] is exactly the cycle's least-squares matrix: when
          // its incremental QR kept every column, take the SVD of R (p x p)
          if (qr && qr->clean() && qr->cols() == kh + j) {
            HMat Q(s, kh + j), R(kh + j, kh + j);
            qr->factors(Q.a.data(), R.a.data());
            hp = harmonic_extract(SAW, SW, k, rank_tol, &Q, &R);
          } else {
            hp = harmonic_extract(SAW, SW, k, rank_tol);
          }
          ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        },
        pump);
    rep.phase_ms["recycle_harmonic"] += ms;
    rep.phase_ms["harmonic_svd"] += hp.svd_ms;
    rep.phase_ms["harmonic_schur"] += hp.schur_ms;
    rep.phase_ms["harmonic_rest"] += hp.rest_ms;
  }
  if (notes) {
    if (hp.rank_limited)
      notes->push_back("deflation space limited to pencil rank " + std::to_string(hp.rank) + " (requested " +
                       std::to_string(hp.k_requested) + ")");
    if (hp.pair_extended) notes->push_back("deflation space grew by one to keep a conjugate pair together");
  }
  const int prov = sp.empty() ? 1 : sp.provenance;
  const i64 ke = hp.k_eff;
  if (ke == 0) {
    sp.clear();
    sp.provenance = prov;
    return;
  }
  sp.ensure(w.lay.nloc, std::max<i64>(ke, kh));
  // device: U_new = V(:,0:j) C_bot + U C_top with the lazy scales folded into
  // the coefficients — two plain tall-skinny GEMMs (cuBLAS) and a column-norm
  // pass. The U part needs its live columns to be exactly slots [0, kc)
  // (a dead column could hold non-finite data that a zero coefficient would
  // not cancel); otherwise the pointer-list K4 kernel runs instead.
  const i64 nloc = w.lay.nloc;
  i64 kc = 0;
  bool dense_u = true;
  {
    std::vector<char> used(static_cast<size_t>(std::max<i64>(sp.cap, 1)), 0);
    for (i64 p = 0; p < kh; ++p) {
      used[static_cast<size_t>(sp.slot[static_cast<size_t>(p)])] = 1;
      kc = std::max<i64>(kc, sp.slot[static_cast<size_t>(p)] + 1);
    }
    for (i64 q = 0; q < kc; ++q) dense_u = dense_u && used[static_cast<size_t>(q)];
  }
  const int other = 1 - sp.cur;
  // with a side stream the product does not queue behind the speculative
  // steps pumped onto the compute stream (it reads the finished cycle's basis
  // and the old U only; the next cycle's correction waits for it below)
  const bool side = side_stream && dense_u && !c.distributed() && !product_done;
  if (side) {  // ev_side_in: recorded by solve() when the finished cycle's device work was enqueued
    SDR_CUDA(cudaStreamWaitEvent(w.side_stream, w.ev_side_in, 0));
    std::swap(c.stream, w.side_stream);
  }
  static const bool own_gemm = [] {
    const char* e = std::getenv("SDR_TSGEMM");
    return !e || std::atoi(e) != 0;
  }();
  // one HBM pass over [V U] with the norms fused: k_tsgemm for few outputs
  // (C5, k = 10: 17.4 vs 37 ms per restart through cuBLAS), the shared-memory
  // tiled k_rgemm for up to 24 (C2, k = 20); SDR_RGEMM=0 selects cuBLAS there
  static const int rgemm_mode = [] {  // 0: cuBLAS above 12 outputs, 1: default, 2: k_rgemm for every count
    const char* e = std::getenv("SDR_RGEMM");
    return e ? std::atoi(e) : 1;
  }();
  const bool own_rgemm = rgemm_mode != 0;
  const bool use_ts = rgemm_mode != 2 && ke <= 12 && tsgemm_supported(static_cast<int>(ke), nloc, w.lay.ld, sp.ld, sp.ld);
  const bool use_rg = !use_ts && own_rgemm && rgemm_supported(static_cast<int>(ke), static_cast<int>(j + kc), w.lay.ld, sp.ld);
  static const bool tsmm_on = [] {
    const char* e = std::getenv("SDR_TSMM");
    return !e || std::atoi(e) != 0;
  }();
  const bool use_tm = tsmm_on && tsmm_supported(static_cast<int>(ke), static_cast<int>(j + kc), nloc, w.lay.ld, sp.ld);
  if (product_done) {
    // the fused restart pass already wrote U_new into sp.buf[other] and its
    // squared norms after the correction's (run_cycle)
    SDR_CUDA(cudaMemcpyAsync(w.scal.get(), w.unorm.get() + 1, sizeof(double) * static_cast<size_t>(ke),
                             cudaMemcpyDeviceToDevice, c.stream));
  } else if (dense_u && own_gemm && (use_tm || use_ts || use_rg)) {
    const i64 kk = j + kc;
    w.gcoef.ensure(std::max<i64>(kk * ke, 1));
    w.hgcoef.ensure(std::max<i64>(kk * ke, 1));
    double* hb = w.hgcoef.get();
    std::fill(hb, hb + kk * ke, 0.0);
    for (i64 q = 0; q < ke; ++q) {
      for (i64 i = 0; i < j; ++i) hb[q * kk + i] = hp.coeffs(kh + i, q) * st.cv[static_cast<size_t>(i)];
      for (i64 p = 0; p < kh; ++p)
        hb[q * kk + j + sp.slot[static_cast<size_t>(p)]] = hp.coeffs(p, q) * sp.uscale[static_cast<size_t>(p)];
    }
    SDR_CUDA(cudaMemcpyAsync(w.gcoef.get(), hb, sizeof(double) * static_cast<size_t>(kk * ke), cudaMemcpyHostToDevice,
                             c.stream));
    w.pside.ensure(std::max(tsgemm_scratch_size(c.num_sms), tsmm_scratch_size(c.num_sms)));
    if (use_tm) {
      std::vector<double*> outs(static_cast<size_t>(ke));
      for (i64 q = 0; q < ke; ++q) outs[static_cast<size_t>(q)] = sp.buf[other].get() + q * sp.ld;
      launch_tsmm(c, w.Vcol(vb, 0), w.lay.ld, static_cast<int>(j), sp.buf[sp.cur].get(), sp.ld, static_cast<int>(kc),
                  w.gcoef.get(), static_cast<int>(ke), outs.data(), nloc, w.scal.get(), w.pside.get());
    } else if (use_ts)
      launch_tsgemm(c, w.Vcol(vb, 0), w.lay.ld, static_cast<int>(j), sp.buf[sp.cur].get(), sp.ld, static_cast<int>(kc),
                    w.gcoef.get(), static_cast<int>(ke), sp.buf[other].get(), sp.ld, nloc, w.scal.get(), w.pside.get());
    else
      launch_rgemm(c, w.Vcol(vb, 0), w.lay.ld, static_cast<int>(j), sp.buf[sp.cur].get(), sp.ld, static_cast<int>(kc),
                   w.gcoef.get(), static_cast<int>(ke), sp.buf[other].get(), sp.ld, nloc, w.scal.get(), w.pside.get());
  } else if (dense_u) {
    const i64 ncoef = j * ke + kc * ke;
    w.gcoef.ensure(std::max<i64>(ncoef, 1));
    w.hgcoef.ensure(std::max<i64>(ncoef, 1));
    double* hv = w.hgcoef.get();
    for (i64 q = 0; q < ke; ++q)
      for (i64 i = 0; i < j; ++i) hv[q * j + i] = hp.coeffs(kh + i, q) * st.cv[static_cast<size_t>(i)];
    double* hu = hv + j * ke;
    for (i64 p = 0; p < kh; ++p)
      for (i64 q = 0; q < ke; ++q)
        hu[q * kc + sp.slot[static_cast<size_t>(p)]] = hp.coeffs(p, q) * sp.uscale[static_cast<size_t>(p)];
    SDR_CUDA(cudaMemcpyAsync(w.gcoef.get(), hv, sizeof(double) * static_cast<size_t>(ncoef), cudaMemcpyHostToDevice,
                             c.stream));
    double* unew = sp.buf[other].get();
    c.dgemm_tall(nloc, ke, j, w.Vcol(vb, 0), w.lay.ld, w.gcoef.get(), j, 0.0, unew, sp.ld);
    if (kc > 0) c.dgemm_tall(nloc, ke, kc, sp.buf[sp.cur].get(), sp.ld, w.gcoef.get() + j * ke, kc, 1.0, unew, sp.ld);
    w.pside.ensure(tsgemm_scratch_size(c.num_sms));
    launch_col_norms2(c, unew, sp.ld, nloc, static_cast<int>(ke), w.scal.get(), w.pside.get());
  } else {
    std::vector<const double*> in;
    HMat coef(kh + j, ke);
    for (i64 i = 0; i < j; ++i) {
      in.push_back(w.Vcol(vb, i));
      for (i64 q = 0; q < ke; ++q) coef(static_cast<i64>(in.size()) - 1, q) = hp.coeffs(kh + i, q) * st.cv[static_cast<size_t>(i)];
    }
    for (i64 p = 0; p < kh; ++p) {
      in.push_back(sp.col(p));
      for (i64 q = 0; q < ke; ++q) coef(static_cast<i64>(in.size()) - 1, q) = hp.coeffs(p, q) * sp.uscale[static_cast<size_t>(p)];
    }
    std::vector<double*> out;
    for (i64 q = 0; q < ke; ++q) out.push_back(sp.buf[other].get() + q * sp.ld);
    tallskinny(c, w, in, coef, out, nloc, w.scal.get());
  }
  c.allreduce_sum(w.scal.get(), ke);  // (the fused pass's norms are this rank's partial sums too)
  SDR_CUDA(cudaMemcpyAsync(w.hscal.get(), w.scal.get(), sizeof(double) * ke, cudaMemcpyDeviceToHost, c.stream));
  SDR_CUDA(cudaEventRecord(w.ev_side_out, c.stream));
  if (side) {
    std::swap(c.stream, w.side_stream);
    SDR_CUDA(cudaStreamWaitEvent(c.stream, w.ev_side_out, 0));  // later work on the compute stream sees U_new
  }
  // host: SU_new, SAU_new (recycle.hpp:257-265) while the product runs
  HMat SU(s, ke), SAU(s, ke);
  host_job_while_pumping(
      [&] {  // [SU SV] C and [SAU SAV] C as BLAS-3 products (V block, then U block added)
        const int ms = static_cast<int>(s), nk = static_cast<int>(ke), kj = static_cast<int>(j),
                  kk = static_cast<int>(kh), ldc = static_cast<int>(hp.coeffs.rows);
        const double one = 1.0, zero = 0.0;
        if (ms > 0 && nk > 0) {
          scipy_dgemm_("N", "N", &ms, &nk, &kj, &one, st.SV.a.data(), &ms, hp.coeffs.a.data() + kh, &ldc, &zero,
                       SU.a.data(), &ms, 1, 1);
          scipy_dgemm_("N", "N", &ms, &nk, &kj, &one, st.SAV.a.data(), &ms, hp.coeffs.a.data() + kh, &ldc, &zero,
                       SAU.a.data(), &ms, 1, 1);
          if (kk > 0) {
            scipy_dgemm_("N", "N", &ms, &nk, &kk, &one, sp.SU.a.data(), &ms, hp.coeffs.a.data(), &ldc, &one,
                         SU.a.data(), &ms, 1, 1);
            scipy_dgemm_("N", "N", &ms, &nk, &kk, &one, sp.SAU.a.data(), &ms, hp.coeffs.a.data(), &ldc, &one,
                         SAU.a.data(), &ms, 1, 1);
          }
        }
      },
      pump);
  while (cudaEventQuery(w.ev_side_out) == cudaErrorNotReady) {
    if (pump) (*pump)();
    std::this_thread::sleep_for(std::chrono::microseconds(10));
  }
  SDR_CUDA(cudaEventSynchronize(w.ev_side_out));
  sp.cur = other;
  sp.slot.resize(static_cast<size_t>(ke));
  sp.uscale.resize(static_cast<size_t>(ke));
  for (i64 q = 0; q < ke; ++q) sp.slot[static_cast<size_t>(q)] = static_cast<int>(q);
  sp.SU = std::move(SU);
  sp.SAU = std::move(SAU);
  sp.provenance = prov;
  std::vector<i64> bad;
  for (i64 q = 0; q < ke; ++q) {  // recycle.hpp:269-286
    const double nrm = std::sqrt(w.hscal.get()[q]);
    ++cnt.inner_products;
    if (nrm == 0.0 || !std::isfinite(nrm)) {
      bad.push_back(q);
      sp.uscale[static_cast<size_t>(q)] = 0.0;
      continue;
    }
    sp.uscale[static_cast<size_t>(q)] = 1.0 / nrm;
    for (i64 r = 0; r < s; ++r) {
      sp.SU(r, q) /= nrm;
      sp.SAU(r, q) /= nrm;
    }
  }
  if (!bad.empty()) {
    sp.drop_columns(bad);
    if (notes) notes->push_back("dropped " + std::to_string(bad.size()) + " degenerate deflation columns after the harmonic update");
  }
  if (sp.empty()) sp.provenance = 0;
}

/// Restart boundary in one pass over [V U]: when the cycle's harmonic pencil
/// is cheap next to a pass over the basis (C5: ~0.8 ms vs ~13 ms; chosen when
/// the pass is estimated at 1.5x the pencil or more), the host
/// forms it first and one tall-skinny kernel writes both the correction
/// (solver.hpp:197-198) and U_new = [U V] P (recycle.hpp:257-265), reading
/// the basis once instead of twice. SDR_FUSE_RESTART=0/1 forces it off/on.
bool fuse_restart_wanted(const Context& c, const Workspace& w, i64 kh, i64 j) {
  static const int mode = [] {
    const char* e = std::getenv("SDR_FUSE_RESTART");
    return e ? std::atoi(e) : -1;
  }();
  if (mode == 0) return false;
  if (mode == 1) return true;
  const double pass_ms = static_cast<double>(kh + j) * static_cast<double>(w.lay.nloc) * 8.0 / 5.0e9;
  const double p = static_cast<double>(kh + j);
  const double harm_ms = w.last_harmonic_ms >= 0.0 ? w.last_harmonic_ms : 2.5 * (p / 120.0) * (p / 120.0) * (p / 120.0);
  // fused: the GPU waits for the pencil (harm_ms) and saves one read of the
  // basis (~pass_ms); 1.5x margin for the estimates
  return pass_ms > 1.5 * harm_ms;
}

/// Launches the fused pass (outputs: correction, then the k_eff new recycle
/// columns into sp.buf[1 - sp.cur], squared norms into Workspace::unorm);
/// false when the shape is not eligible (the caller runs the two passes).
bool launch_fused_restart(Context& c, Workspace& w, const HostKrylov& st, int vb, Recycle& sp, const Harmonic& hp,
                          const std::vector<double>& y, double* corr_own) {
  const i64 j = st.j, kh = sp.dim(), ke = hp.k_eff, nloc = w.lay.nloc;
  if (ke + 1 > 40 || j < 1) return false;
  sp.ensure(nloc, std::max<i64>(ke, kh));
  i64 kc = 0;
  std::vector<char> used(static_cast<size_t>(std::max<i64>(sp.cap, 1)), 0);
  for (i64 p = 0; p < kh; ++p) {
    used[static_cast<size_t>(sp.slot[static_cast<size_t>(p)])] = 1;
    kc = std::max<i64>(kc, sp.slot[static_cast<size_t>(p)] + 1);
  }
  for (i64 q = 0; q < kc; ++q)
    if (!used[static_cast<size_t>(q)]) return false;  // dead U slots could hold non-finite data
  const int nout = static_cast<int>(1 + ke);
  if (!tsmm_supported(nout, static_cast<int>(j + kc), nloc, w.lay.ld, sp.ld)) return false;
  const i64 kk = j + kc;
  w.gcoef.ensure(kk * nout);
  w.hgcoef.ensure(kk * nout);
  double* hb = w.hgcoef.get();
  std::fill(hb, hb + kk * nout, 0.0);
  for (i64 i = 0; i < j; ++i) hb[i] = y[static_cast<size_t>(kh + i)] * st.cv[static_cast<size_t>(i)];
  for (i64 p = 0; p < kh; ++p)
    hb[j + sp.slot[static_cast<size_t>(p)]] = y[static_cast<size_t>(p)] * sp.uscale[static_cast<size_t>(p)];
  for (i64 q = 0; q < ke; ++q) {
    double* col = hb + (q + 1) * kk;
    for (i64 i = 0; i < j; ++i) col[i] = hp.coeffs(kh + i, q) * st.cv[static_cast<size_t>(i)];
    for (i64 p = 0; p < kh; ++p)
      col[j + sp.slot[static_cast<size_t>(p)]] = hp.coeffs(p, q) * sp.uscale[static_cast<size_t>(p)];
  }
  SDR_CUDA(cudaMemcpyAsync(w.gcoef.get(), hb, sizeof(double) * static_cast<size_t>(kk * nout), cudaMemcpyHostToDevice,
                           c.stream));
  std::vector<double*> outs(static_cast<size_t>(nout));
  outs[0] = corr_own;
  for (i64 q = 0; q < ke; ++q) outs[static_cast<size_t>(q + 1)] = sp.buf[1 - sp.cur].get() + q * sp.ld;
  w.pside.ensure(std::max(tsgemm_scratch_size(c.num_sms), tsmm_scratch_size(c.num_sms)));
  launch_tsmm(c, w.Vcol(vb, 0), w.lay.ld, static_cast<int>(j), sp.buf[sp.cur].get(), sp.ld, static_cast<int>(kc),
              w.gcoef.get(), nout, outs.data(), nloc, w.unorm.get(), w.pside.get());
  return true;
}

/// Steps, least squares and verification of one restart cycle
/// (solver.hpp:128-216). `ap` has its init enqueued (and possibly
/// speculative steps in flight); r0 is the device residual (own part).
CycleOut run_cycle(Context& c, Workspace& w, ArnoldiPipeline& ap, const DeviceOperator& A, const Config& cfg,
                   const double* r0, Recycle& space, double tol_abs, double safety_in, Counters& cnt, Report& rep,
                   const Callbacks* cb, int cycle_index, i64 iteration_base) {
  CycleOut out;
  out.safety = std::max(1.0, safety_in);
  const VecLayout& lay = w.lay;
  const i64 s = ap.S.s, m = cfg.m;
  {
    PhaseTimer pt(rep, "cycle_init");
    ap.init_finish(cnt);
  }
  HostKrylov& st = ap.st;
  out.entry_norm = st.r0_norm;
  std::vector<double> sr0(static_cast<size_t>(s));
  for (i64 r = 0; r < s; ++r) sr0[static_cast<size_t>(r)] = st.SV(r, 0) * st.r0_norm;
  out.sketched_entry = hnorm(sr0.data(), s);

  // ---- seed the QR with the deflation block (solver.hpp:144-159)
  auto qr = std::make_shared<HostQR>(s, space.dim() + m, cfg.rank_tol);
  for (;;) {
    std::vector<i64> bad;
    for (i64 q = 0; q < space.dim(); ++q)
      if (qr->append(space.SAU.col(q), s).rank_deficient) bad.push_back(q);
    if (bad.empty()) break;
    space.drop_columns(bad);
    rep.notes.push_back("cycle " + std::to_string(cycle_index) + ": dropped " + std::to_string(bad.size()) +
                        " deflation columns with rank-deficient sketched images");
    qr = std::make_shared<HostQR>(s, space.dim() + m, cfg.rank_tol);
    if (space.empty()) break;
  }
  const i64 k_hat = space.dim();
  qr->set_rhs(sr0.data(), s);

  std::vector<double> y(static_cast<size_t>(k_hat + m), 0.0);
  double sres = out.sketched_entry;
  bool done = false;
  while (!done && st.j < m && !st.breakdown) {  // solver.hpp:165-216
    const bool step_breakdown = ap.step(cnt);
    PhaseTimer pt_step(rep, "host_step");
    const i64 jj = st.j;
    std::optional<PhaseTimer> pt_qr(std::in_place, rep, "qr_append");
    const auto info = qr->append(st.SAV.col(jj - 1), s);
    pt_qr.reset();
    if (info.rank_deficient) {
      qr->exclude(info.column);
      rep.notes.push_back("cycle " + std::to_string(cycle_index) + ", step " + std::to_string(jj) +
                          ": sketched basis column rank-deficient; excluded from the least-squares problem");
    }
    {
      PhaseTimer pt_ls(rep, "ls_solve");
      sres = qr->solve_cached(y.data());
    }
    const i64 p = qr->cols();
    const i64 global_iter = iteration_base + jj;
    rep.sketched.emplace_back(global_iter, sres);
    if (cb && cb->on_iteration) {
      StepEvent ev{cycle_index, jj, global_iter, sres, step_breakdown ? 1.0 : hnorm(st.SV.col(jj), s), y.data(), p,
                   k_hat};
      cb->on_iteration(&ev, cb->user);
    }
    const bool last = jj == m || st.breakdown;
    if (sres < tol_abs / out.safety || last) {
      // correction = V(:,0:j) y_tail + U y_head (solver.hpp:197-198), on the device
      PhaseTimer pt_check(rep, "check");
      double* corr_own = w.corr.get() + lay.own_off;
      bool fused = false;
      if (cfg.k > 0 && fuse_restart_wanted(c, w, k_hat, jj)) {
        // the cycle very likely ends here: form its harmonic pencil now and
        // write the correction and U_new in one pass over the basis
        auto e = start_early_harmonic(st, space, qr.get(), cfg.k, cfg.rank_tol);
        if (e->th.joinable()) e->th.join();
        if (e->err) std::rethrow_exception(e->err);
        w.last_harmonic_ms = e->ms;
        if (e->have_hp) fused = launch_fused_restart(c, w, st, ap.vb, space, e->hp, y, corr_own);
        e->product_done = fused;
        out.early = e;
      }
      if (!fused) {
        std::vector<const double*> in;
        HMat coef(jj + k_hat, 1);
        for (i64 i = 0; i < jj; ++i) {
          in.push_back(w.Vcol(ap.vb, i));
          coef(i, 0) = y[static_cast<size_t>(k_hat + i)] * st.cv[static_cast<size_t>(i)];
        }
        for (i64 q = 0; q < k_hat; ++q) {
          in.push_back(space.col(q));
          coef(jj + q, 0) = y[static_cast<size_t>(q)] * space.uscale[static_cast<size_t>(q)];
        }
        tallskinny(c, w, in, coef, {corr_own}, lay.nloc, nullptr);
      }
      c.halo_exchange(A.plan, w.corr.get() + lay.ext_shift(), A.ext_begin, corr_own, A.row_begin);
      launch_residual(c, A.view(), w.corr.get() + lay.ext_shift(), r0, w.rnew.get(), w.scal.get());
      c.allreduce_sum(w.scal.get(), 1);
      // the cycle very likely ends here: start its restart bookkeeping (host
      // threads) while the verification runs on the device
      if (!out.early) out.early = start_early_harmonic(st, space, qr.get(), cfg.k, cfg.rank_tol);
      out.residual_norm = std::sqrt(d2h_scalar(c, w, w.scal.get()));
      out.have_correction = true;
      ++cnt.matvecs;
      ++cnt.inner_products;
      rep.truth.emplace_back(global_iter, out.residual_norm);
      if (cb && cb->on_residual) {
        ResidualEvent ev{cycle_index, global_iter, sres, out.residual_norm};
        cb->on_residual(&ev, cb->user);
      }
      if (out.residual_norm < tol_abs) {
        out.converged = true;
        done = true;
      } else {
        if (sres > 0.0) out.safety = std::max(out.safety, out.residual_norm / sres);
        if (last) done = true;
      }
      if (!done && out.early && !out.early->th.joinable()) {  // fused: nothing running, result discarded
        out.early.reset();
      } else if (!done && out.early) {  // the cycle goes on: let the thread finish on its own
        out.early->th.detach();
        auto keep = out.early;
        std::thread([keep] {
          while (!keep->done.load(std::memory_order_acquire)) std::this_thread::sleep_for(std::chrono::microseconds(200));
        }).detach();
        out.early.reset();
      }
    }
  }
  out.steps = st.j;
  out.sres = sres;
  out.breakdown = st.breakdown;
  out.qr = qr;
  rep.host_wait_ms += ap.wait_ms;
  rep.phase_ms["step_wait"] += ap.wait_ms;
  return out;
}

/// Cycle statistics and the harmonic recycle update (solver.hpp:218-253).
void finish_cycle(Context& c, Workspace& w, const ArnoldiPipeline& ap, const CycleOut& out, const Config& cfg,
                  Recycle& space, Counters& cnt, Report& rep, int cycle_index,
                  const std::function<void()>* pump = nullptr, bool side_stream = false) {
  const HostKrylov& st = ap.st;
  const i64 s = ap.S.s;
  CycleStat cs;
  cs.steps = st.j;
  cs.entry_residual = out.entry_norm;
  cs.sketched_entry = out.sketched_entry;
  cs.exit_sres = out.sres;
  cs.exit_residual = out.residual_norm;
  cs.safety_after = out.safety;
  const bool want_bc = st.j >= 1 && !st.breakdown;
  // early pencil from the trigger point (run_cycle) when it matches this cycle
  EarlyHarmonic* early = (out.early && out.early->j == st.j && out.early->kh == space.dim()) ? out.early.get() : nullptr;
  if (early) {
    while (!early->done.load(std::memory_order_acquire)) {
      if (pump) (*pump)();
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    if (early->th.joinable()) early->th.join();
    if (early->err) std::rethrow_exception(early->err);
    if (want_bc && early->have_cond) {
      cs.basis_cond = early->cond;
      rep.phase_ms["basis_cond"] += early->cond_ms;
    }
    if (cfg.k > 0 && st.j >= 1) {
      rep.phase_ms["recycle_harmonic"] += early->ms;
      rep.phase_ms["harmonic_svd"] += early->hp.svd_ms;
      rep.phase_ms["harmonic_schur"] += early->hp.schur_ms;
      rep.phase_ms["harmonic_rest"] += early->hp.rest_ms;
      std::vector<std::string> notes;
      PhaseTimer pt(rep, "recycle");
      update_recycle(c, w, st, ap.vb, space, cfg.k, cfg.rank_tol, cnt, &notes, rep, pump, side_stream, out.qr.get(),
                     early->have_hp ? &early->hp : nullptr, early->product_done);
      if (!early->product_done) w.last_harmonic_ms = early->ms;
      cs.deflation_rank = space.dim();
      for (auto& n : notes) rep.notes.push_back("cycle " + std::to_string(cycle_index) + ": " + n);
    } else if (cfg.k == 0) {
      space.clear();
    }
    rep.cycle_stats.push_back(cs);
    return;
  }
  // otherwise: the basis condition number (an SVD of SV) on its own host
  // thread, concurrently with the harmonic update below
  HMat B;
  double bc_ms = 0.0;
  std::exception_ptr bc_err;
  std::thread bc_thread;
  if (want_bc) {
    B = HMat(s, st.j + 1);
    std::copy(st.SV.a.begin(), st.SV.a.begin() + s * (st.j + 1), B.a.begin());
    bc_thread = std::thread([&] {
      try {
        const auto t0 = std::chrono::steady_clock::now();
        cs.basis_cond = cond2(B);
        bc_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      } catch (...) {
        bc_err = std::current_exception();
      }
    });
  }
  auto join_bc = [&] {
    if (bc_thread.joinable()) bc_thread.join();
  };
  try {
    if (cfg.k > 0 && st.j >= 1) {
      std::vector<std::string> notes;
      PhaseTimer pt(rep, "recycle");
      update_recycle(c, w, st, ap.vb, space, cfg.k, cfg.rank_tol, cnt, &notes, rep, pump, side_stream, out.qr.get());
      cs.deflation_rank = space.dim();
      for (auto& n : notes) rep.notes.push_back("cycle " + std::to_string(cycle_index) + ": " + n);
    } else if (cfg.k == 0) {
      space.clear();
    }
  } catch (...) {
    join_bc();
    throw;
  }
  join_bc();
  if (bc_err) std::rethrow_exception(bc_err);
  if (want_bc) rep.phase_ms["basis_cond"] += bc_ms;
  rep.cycle_stats.push_back(cs);
}

}  // namespace

void krylov_run(Context& c, const DeviceOperator& A, const SketchDev& S, const double* r0, i64 t, i64 m, i64 steps,
                double breakdown_tol, double* V, double* H, double* SV, double* SAV, i64* j_out, int* breakdown,
                double* r0_norm, i64* counters3) {
  if (t < 1) throw invalid("init_krylov: truncation window must be at least 1");
  if (m < 1) throw invalid("init_krylov: m_max must be at least 1");
  if (S.n != A.rows)
    throw invalid("init_krylov: residual length " + std::to_string(A.rows) + " does not match sketch input " +
                  std::to_string(S.n));
  init_host_blas();
  const VecLayout lay = A.layout();
  Workspace& w = workspace(c, lay, m, S.s, static_cast<int>(std::min(t, m)));
  Counters cnt;
  ArnoldiPipeline ap(c, w, A, S, t, m, breakdown_tol, 0);
  ap.init_enqueue(r0);
  ap.init_finish(cnt);
  for (i64 q = 0; q < steps && !ap.st.breakdown && ap.st.j < m; ++q) ap.step(cnt);
  c.sync();
  const HostKrylov& st = ap.st;
  if (V) {
    const i64 cols = st.breakdown ? st.j : st.j + 1;
    DeviceBuffer<double> tmp(std::max<i64>(lay.nloc * (m + 1), 1));
    SDR_CUDA(cudaMemsetAsync(tmp.get(), 0, sizeof(double) * static_cast<size_t>(lay.nloc * (m + 1)), c.stream));
    for (i64 i = 0; i < cols; ++i)
      launch_scale_copy(c, st.cv[static_cast<size_t>(i)], w.Vcol(0, i), tmp.get() + i * lay.nloc, lay.nloc);
    SDR_CUDA(cudaMemcpyAsync(V, tmp.get(), sizeof(double) * static_cast<size_t>(lay.nloc * (m + 1)), cudaMemcpyDefault,
                             c.stream));
    c.sync();
  }
  if (H) std::copy(st.H.a.begin(), st.H.a.end(), H);
  if (SV) std::copy(st.SV.a.begin(), st.SV.a.end(), SV);
  if (SAV) std::copy(st.SAV.a.begin(), st.SAV.a.end(), SAV);
  if (j_out) *j_out = st.j;
  if (breakdown) *breakdown = st.breakdown ? 1 : 0;
  if (r0_norm) *r0_norm = st.r0_norm;
  if (counters3) {
    counters3[0] = cnt.matvecs;
    counters3[1] = cnt.inner_products;
    counters3[2] = cnt.sketch_applies;
  }
}

void time_step_kernels(Context& c, const DeviceOperator& A, const SketchDev& S, const double* r0, i64 t, i64 m,
                       i64 steps, int reps, double* k1_us, double* k2_us) {
  if (steps < 2 || steps > m || reps < 1) throw invalid("time_step_kernels: need 2 <= steps <= m and reps >= 1");
  init_host_blas();
  const VecLayout lay = A.layout();
  Workspace& w = workspace(c, lay, m, S.s, static_cast<int>(std::min(t, m)));
  Counters cnt;
  ArnoldiPipeline ap(c, w, A, S, t, m, 1e-14, 0);
  ap.init_enqueue(r0);
  ap.init_finish(cnt);
  for (i64 q = 0; q < steps && !ap.st.breakdown && ap.st.j < m; ++q) ap.step(cnt);
  c.sync();
  ap.time_last_step(reps, k1_us, k2_us);
}

void solve(Context& c, const DeviceOperator& A, const double* b, const double* x0, bool x0_nonzero, const Config& cfg,
           Recycle& space, const SketchDev* sketch, const Callbacks* cb, double* x_out, Report& rep) {
  cfg.validate();  // solver.hpp:273-298
  if (A.rows != A.cols)
    throw invalid("solve: operator must be square, got " + std::to_string(A.rows) + " x " + std::to_string(A.cols));
  std::unique_ptr<SketchDev> own;
  if (!sketch) {
    own.reset(create_sketch(c, kSrdct, A.rows, cfg.s, cfg.sketch_seed, 0));
    sketch = own.get();
  }
  if (sketch->n != A.rows)
    throw invalid("solve: sketch takes length " + std::to_string(sketch->n) + " but the operator is " +
                  std::to_string(A.rows) + " x " + std::to_string(A.cols));
  if (sketch->s < 2 * (cfg.m + cfg.k))
    throw invalid("solve: sketch size " + std::to_string(sketch->s) + " is below 2 (m + k) = " +
                  std::to_string(2 * (cfg.m + cfg.k)));
  if (!space.empty() && space.n != A.rows)
    throw invalid("solve: recycle space has " + std::to_string(space.n) + " rows but the operator is " +
                  std::to_string(A.rows) + " x " + std::to_string(A.cols));
  if (!space.empty() && space.s != sketch->s)
    throw invalid("solve: recycle space has " + std::to_string(space.s) + " sketch rows but the sketch has " +
                  std::to_string(sketch->s));
  init_host_blas();
  const auto t_start = std::chrono::steady_clock::now();
  auto pt_setup = std::make_unique<PhaseTimer>(rep, "setup");
  const VecLayout lay = A.layout();
  const int T = static_cast<int>(std::min<i64>(cfg.t, cfg.m));
  Workspace& w = workspace(c, lay, cfg.m, sketch->s, T);
  space.n = A.rows;
  space.s = sketch->s;
  space.ensure(lay.nloc, std::max<i64>(cfg.k + 1, space.dim()));
  if (space.SU.rows != space.s) {
    space.SU = HMat(space.s, space.dim());
    space.SAU = HMat(space.s, space.dim());
  }

  // rhs norm (1 IP), tol_abs (solver.hpp:303-305)
  launch_copy_norm(c, b, w.r0.get(), lay.nloc, w.scal.get());
  c.allreduce_sum(w.scal.get(), 1);
  rep.rhs_norm = std::sqrt(d2h_scalar(c, w, w.scal.get()));
  ++rep.counters.inner_products;
  const double tol_abs = cfg.tol * rep.rhs_norm;
  if (x0)
    SDR_CUDA(cudaMemcpyAsync(w.x.get(), x0, sizeof(double) * static_cast<size_t>(lay.nloc), cudaMemcpyDeviceToDevice, c.stream));
  else
    SDR_CUDA(cudaMemsetAsync(w.x.get(), 0, sizeof(double) * static_cast<size_t>(std::max<i64>(lay.nloc, 1)), c.stream));
  if (x0 && x0_nonzero) {  // r = b - A x0 (solver.hpp:307-316)
    SDR_CUDA(cudaMemcpyAsync(w.tmp.get() + lay.own_off, x0, sizeof(double) * static_cast<size_t>(lay.nloc),
                             cudaMemcpyDeviceToDevice, c.stream));
    c.halo_exchange(A.plan, w.tmp.get() + lay.ext_shift(), A.ext_begin, w.tmp.get() + lay.own_off, A.row_begin);
    launch_residual(c, A.view(), w.tmp.get() + lay.ext_shift(), b, w.r0.get(), w.scal.get());
    ++rep.counters.matvecs;
  }

  double safety = cfg.safety_init, res_norm = std::numeric_limits<double>::quiet_NaN();
  bool have = false, x_copied = false;
  pt_setup.reset();
  auto cur = std::make_unique<ArnoldiPipeline>(c, w, A, *sketch, cfg.t, cfg.m, cfg.breakdown_tol, 0);
  cur->init_enqueue(w.r0.get());
  for (int cycle = 1; cycle <= cfg.max_restarts; ++cycle) {  // solver.hpp:321-359
    CycleOut cr;
    try {
      cr = run_cycle(c, w, *cur, A, cfg, w.r0.get(), space, tol_abs, safety, rep.counters, rep, cb, cycle,
                     rep.iterations);
    } catch (const Error& e) {
      if (e.code != 2) throw;
      rep.status = 0;  // zero residual at cycle entry: converged exactly
      res_norm = 0.0;
      have = true;
      break;
    }
    rep.cycles = cycle;
    rep.iterations += cr.steps;
    safety = cr.safety;
    if (cr.have_correction) {
      launch_axpy(c, 1.0, w.corr.get() + lay.own_off, w.x.get(), lay.nloc);
      std::swap(w.r0, w.rnew);
    }
    res_norm = cr.residual_norm;
    have = true;
    // the outcome is known before the recycle update; notes keep the reference order
    int status = -1;
    std::string note;
    if (cr.converged) {
      status = 0;
    } else if (cr.breakdown) {
      status = 2;
      note = "cycle " + std::to_string(cycle) + ": basis exhausted before reaching the target";
    } else if (cr.steps == cfg.m && cr.sres > 0.99 * cr.sketched_entry) {
      status = 3;
      note = "cycle " + std::to_string(cycle) + ": sketched residual improved by less than 1% over a full cycle";
    } else if (cycle == cfg.max_restarts) {
      status = 1;
    }
    // the solve ends with this cycle: x is final, so its copy-out runs while
    // the host computes the last recycle update
    if (status >= 0 && x_out) {
      x_copied = true;
      SDR_CUDA(cudaMemcpyAsync(x_out, w.x.get(), sizeof(double) * static_cast<size_t>(lay.nloc), cudaMemcpyDefault,
                               c.stream));
    }
    // the finished cycle's device work is all enqueued: the recycle product
    // may start as soon as it completes (side stream, see update_recycle)
    SDR_CUDA(cudaEventRecord(w.ev_side_in, c.stream));
    std::unique_ptr<ArnoldiPipeline> next;
    std::function<void()> pump;
    if (status < 0 && w.nV == 2) {
      // overlap: the next cycle's init and steps on the other basis buffer,
      // pumped while the host computes the harmonic pencil of this cycle
      next = std::make_unique<ArnoldiPipeline>(c, w, A, *sketch, cfg.t, cfg.m, cfg.breakdown_tol, 1 - cur->vb);
      next->init_enqueue(w.r0.get());
      next->issue_ahead(0);
      pump = [&next] { next->pump(); };
    }
    finish_cycle(c, w, *cur, cr, cfg, space, rep.counters, rep, cycle, next ? &pump : nullptr,
                 next && next->deferred);
    if (status >= 0) {
      rep.status = status;
      if (!note.empty()) rep.notes.push_back(note);
      break;
    }
    if (!next) {
      next = std::make_unique<ArnoldiPipeline>(c, w, A, *sketch, cfg.t, cfg.m, cfg.breakdown_tol, cur->vb);
      next->init_enqueue(w.r0.get());
    }
    cur = std::move(next);
  }
  if (have) rep.final_relative_residual = rep.rhs_norm > 0.0 ? res_norm / rep.rhs_norm : res_norm;
  if (x_out && !x_copied)
    SDR_CUDA(cudaMemcpyAsync(x_out, w.x.get(), sizeof(double) * static_cast<size_t>(lay.nloc), cudaMemcpyDefault, c.stream));
  c.sync();
  rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

}  // namespace sdr
