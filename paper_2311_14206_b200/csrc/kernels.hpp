// Host-side launchers for the sm_100a kernels (definitions in *.cu).
#pragma once

#include "context.hpp"

namespace sdr {

constexpr int kSlice = 32;  // SELL-C slice height (one warp)

/// Device SELL-32 view of a (rank-local) operator. Column indices address
/// the rank's extended vector (halo_lo rows below the own block first).
struct SellView {
  const int64_t* slice_ptr = nullptr;  // nslices + 1 element offsets
  const int32_t* cols = nullptr;
  const double* vals = nullptr;
  const int32_t* doff = nullptr;  // SELL-DIA: [nslices][dia_d] diagonal offsets; null for plain SELL
  int dia_d = 0;                   // SELL-DIA diagonals per slice (slice_ptr unused)
  int cplx = 0;  // ZSELL: 2x2 [[a, -b], [b, a]] blocks stored as complex a + ib; slices of 32 complex rows,
                 // cols = complex column of the extended vector, vals = (re, im) pairs; vectors interleaved
  int64_t nrows = 0, nslices = 0;
  int64_t halo_lo = 0, ext_len = 0;  // own row r is extended index halo_lo + r
  // callable operator (OperatorRef with an Apply, operator_ref.hpp:22-25):
  // y = A x is the caller's function, enqueued on the given stream; the SpMV
  // launchers run it and then the same epilogues as separate kernels
  int (*apply)(const double* x, double* y, void* stream, void* user) = nullptr;
  void* apply_user = nullptr;
};

/// Layout of every length-N vector a rank stores with halo space:
/// [pad | halo_lo | own (nloc) | halo_hi]; own starts at own_off (32-aligned).
struct VecLayout {
  int64_t nloc = 0, halo_lo = 0, halo_hi = 0, own_off = 0, ld = 0;
  int64_t ext_shift() const { return own_off - halo_lo; }  // buffer index of ext row 0
};

/// Per-step record layout (doubles), T = max window:
///   A  [0, T+1)         : ||y||^2, y.w_{j-d} (d < T)      (K1, allreduced)
///   H  [T+1, 2T+3)      : ||A v_j||, h_{j-d,j} (d < T), c_j (K2 prologue)
///   B  [2T+3, 3T+3+s)   : ||w_{j+1}||^2, w_{j+1}.w_{j+1-g} (1<=g<T), S w_{j+1} (allreduced)
/// Record q holds step q-1 (A,H) and column q (B); record 0 is column 0.
struct RecLayout {
  int T = 1;
  int64_t s = 0, stride = 0;
  int a_off() const { return 0; }
  int h_off() const { return T + 1; }
  int b_off() const { return 2 * T + 3; }
  int sketch_off() const { return 3 * T + 3; }
  int64_t b_len() const { return T + s; }
  static RecLayout make(int T, int64_t s) {
    RecLayout L;
    L.T = T;
    L.s = s;
    L.stride = (3 * T + 3 + s + 3) / 4 * 4;
    return L;
  }
};

struct SketchDev;  // sketch.cu

/// SDR_PDL=0 disables programmatic dependent launch in the step pipeline.
bool pdl_enabled();

/// Occupancy-derived resident CTAs per SM for a kernel (cached per device and
/// kernel; thread-safe).
int blocks_per_sm(const void* kernel, int threads, size_t smem);
/// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the
/// current device (once per device and kernel; thread-safe).
void ensure_dyn_smem(const void* kernel, size_t bytes);

// ---- SpMV family (spmv.cu)
void launch_spmv(Context& c, const SellView& A, const double* x_ext, double* y);
/// K1. When coef != nullptr (single GPU) the last CTA also forms the MGS
/// coefficients of step j into coef[0..nwin] and the record's H part. With
/// partials_out (deferred step pipeline) the CTAs only leave their window
/// dots there, value-major [1 + nwin][grid], and nothing is folded; the
/// return value is the grid size. max_blocks_per_sm < 0: the full resident
/// grid regardless of the local size (identical layouts on every rank).
/// [sl_begin, sl_end): the 32-row slices this launch covers (default all),
/// so the halo-free interior can run while the halo is in flight.
int launch_spmv_arnoldi(Context& c, const SellView& A, const double* V, int64_t ldv, const VecLayout& lay, int j,
                        int nwin, double* y, double* recA, double* rec, int64_t rstride, int T, double* cvec,
                        double* coef, double* partials_out = nullptr, int max_blocks_per_sm = 0,
                        int64_t sl_begin = 0, int64_t sl_end = -1);
void launch_residual(Context& c, const SellView& A, const double* x_ext, const double* b, double* r, double* norm2);
/// Column pointers of a batched product (extended-vector layout, like x_ext).
constexpr int kSpmmMax = 8;
struct SpmmCols {
  const double* x[kSpmmMax] = {};
};
/// Y(:, q) = A X(:, q), q < nb <= 8, one pass over A (Y column-major, ldy).
void launch_spmm(Context& c, const SellView& A, const SpmmCols& X, int nb, double* Y, int64_t ldy);
/// y = A x, skipped (no stores) when *stop != 0 on the device.
void launch_spmv_guarded(Context& c, const SellView& A, const double* x_ext, double* y, const int* stop);

// ---- Arnoldi update (arnoldi.cu). coef_ready: coefficients already formed
// by K1 (single GPU); null: formed in the K2 prologue from allreduced records.
void launch_update(Context& c, const double* y, double* V, int64_t ldv, const VecLayout& lay, int j, int nwin,
                   int ngram, double* rec, const RecLayout& L, double* cvec, const double* coef_ready);
void launch_copy_norm(Context& c, const double* src, double* dst, int64_t n, double* norm2);
// ---- Long truncation windows (wide.cu): min(t, m) > kFusedWindowMax, the
// largest window the fused step kernels keep in registers.
constexpr int kFusedWindowMax = 33;
/// out = [x.x (self)] then x.V(:, c0 - q) for q < nq (own parts), folded.
void launch_window_dots_wide(Context& c, const double* x, const double* V, int64_t ldv, int64_t own_off, int c0,
                             int nq, bool self, int64_t n, double* out);
/// Step j's modified Gram-Schmidt loop (arnoldi.hpp:91-97) as streaming
/// passes: w_{j+1} = A v_j - sum h v over the window, record H part, cvec[j].
/// dots: device scratch of nwin + 1 values (reduced over ranks).
void launch_mgs_wide(Context& c, const double* y, double* V, int64_t ldv, const VecLayout& lay, int j, int nwin,
                     double* rec, int64_t rstride, int T, double* cvec, double* dots);
void launch_axpy(Context& c, double a, const double* x, double* y, int64_t n);
/// C = [A1 A2] B (column-major; B is (k1+k2) x nout with leading dim k1+k2)
/// in one pass over the inputs, norms2[o] = ||C(:, o)||^2 (deterministic).
bool tsgemm_supported(int nout, int64_t n, int64_t lda1, int64_t lda2, int64_t ldc);
/// scratch: tsgemm_scratch_size doubles for the norm partials (null: the
/// context's shared scratch — not safe beside other streams' kernels).
int64_t tsgemm_scratch_size(int num_sms);
void launch_tsgemm(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                   const double* B, int nout, double* C, int64_t ldc, int64_t n, double* norms2,
                   double* scratch = nullptr);
/// Same product for up to 24 outputs and any row count: shared-memory tiled,
/// cp.async double-buffered, one pass over the inputs (k1 + k2 inputs).
bool rgemm_supported(int nout, int k, int64_t lda1, int64_t lda2);
void launch_rgemm(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                  const double* B, int nout, double* C, int64_t ldc, int64_t n, double* norms2,
                  double* scratch = nullptr);
/// Same product on a bulk-copy ring with fp64 tensor-core accumulation
/// (tsmm.cu), outputs through a pointer list (out[o], n rows each; up to 40),
/// so one pass can write the correction and the new recycle columns.
bool tsmm_supported(int nout, int k, int64_t n, int64_t lda1, int64_t lda2);
int64_t tsmm_scratch_size(int num_sms);
void launch_tsmm(Context& c, const double* A1, int64_t lda1, int k1, const double* A2, int64_t lda2, int k2,
                 const double* B, int nout, double* const* out, int64_t n, double* norms2, double* scratch = nullptr);
/// norms2[q] = ||C(:, q)||^2 for q < ncol (column-major, ldc), deterministic.
/// scratch: at least (4 num_sms + ncol) doubles, or null for the context's scratch.
void launch_col_norms2(Context& c, const double* C, int64_t ldc, int64_t n, int ncol, double* norms2,
                       double* scratch = nullptr);
void launch_scale_copy(Context& c, double a, const double* x, double* y, int64_t n);
void launch_tallskinny(Context& c, const double* const* in_dev, int nin, const double* coef_dev, int nout,
                       double* const* out_dev, int64_t n, double* norms2);

// ---- sketches (sketch.cu): out (device, s doubles) = S (xscale * x_own),
// the rank-local contribution of rows [row_begin, row_begin + nloc).
void launch_sketch(Context& c, const SketchDev& S, const double* x_own, int64_t nloc, int64_t row_begin,
                   double* out);
void launch_sketch_scaled(Context& c, const SketchDev& S, const double* x_own, double xscale, int64_t nloc,
                          int64_t row_begin, double* out);
/// out[r] = scale * sum_b partials[b][r] (CTA-major [G][s]), fixed order.
void launch_sparse_fold(Context& c, const double* partials, int G, int s, double scale, double* out);
/// Fused update + ζ = 8 sparse sign (sparse_update.cu): w_{j+1}, the record's
/// norm / Gram entries and S w_{j+1} (record row j+1) in one pass.
bool update_sparse_eligible(const SketchDev& S, const VecLayout& lay, const RecLayout& RL, int need, int64_t ldv);
void launch_update_sparse(Context& c, const SketchDev& S, const double* y, double* V, int64_t ldv,
                          const VecLayout& lay, int j, int nwin, int ngram, double* rec, const RecLayout& RL,
                          double* cvec, const double* coef_ready, int64_t row_begin);
/// KF (fused_step.cu, one GPU, SELL-DIA, sparse sign, t <= 3): the update +
/// sketch of step j and the SpMV + window dots of step j+1 in one launch
/// (y_in = y_j, y_out = y_{j+1}, distinct buffers), then a one-CTA fold into
/// record rows j+1 (B) and j+2 (A) that forms step j+1's coefficients in coef.
/// chunk_done: fused_step_chunks() counters (zeroed per launch).
bool fused_step_eligible(const SellView& A, const SketchDev& S, const VecLayout& lay, const RecLayout& RL, int t,
                         bool distributed);
int64_t fused_step_chunks(const Context& c, int64_t nloc);
void launch_fused_step(Context& c, const SellView& A, const SketchDev& S, const double* y_in, double* y_out, double* V,
                       int64_t ldv, const VecLayout& lay, int j, int nwin, int ngram, int nwin1, double* rec,
                       const RecLayout& RL, double* cvec, double* coef, int64_t row_begin, unsigned* chunk_done);
/// Builds SketchDev::tab / uq (per-row SRDCT constants) once per sketch.
void prepare_srdct_tables(Context& c, SketchDev& S);
/// Deferred folds of the one-GPU step pipeline: K1(j) leaves its window dots
/// as CTA partials; the fused update K2(j) folds them, together with
/// K2(j-1)'s norm / Gram / sketch partials (record row j), in its prologue,
/// forms the MGS coefficients there and leaves its own partials for K2(j+1).
/// No kernel of a step ends in a serial last-CTA fold.
struct StepFold {
  bool fixed_grid = false;  // several ranks: the tile kernel runs one CTA per SM whatever the local size
  const double* k1_partials = nullptr;
  int k1_G = 0;
  const double* prev_partials = nullptr;  // null at j = 0 (row 0 comes from the cycle init)
  int prev_G = 0, prev_nvp = 0, prev_ngram = 0;
  double* out_partials = nullptr;  // this update's partials (update_sketch_partials_size doubles)
  int out_G = 0, out_nvp = 0;      // set by the launch
};
/// out[v] = sum_b partials over G CTAs, fixed order: value-major [nv][G]
/// (K1) or CTA-major [G][nv] (K2). The several-rank pipeline folds locally
/// before its allreduces.
void launch_fold_partials(Context& c, const double* partials, int G, int nv, bool value_major, double* out);
/// The same over two value-major partial arrays (a split K1: [nv][G1] then [nv][G2]), in that order.
void launch_fold_partials2(Context& c, const double* p1, int G1, const double* p2, int G2, int nv, double* out);
bool update_sketch_eligible(const SketchDev& S, const VecLayout& lay, int need, int64_t row_begin, int64_t ldv);
int64_t update_sketch_partials_size(const SketchDev& S, int num_sms);
/// Fused K2 + K3a (update pass and SRDCT of w_{j+1} in one sweep), writing
/// the record's B part (norm, Gram, sketch) — through a fold kernel, or, with
/// sf (deferred pipeline), left as partials for the next step. Returns false
/// when the configuration is not eligible (caller runs K2 and K3 separately).
bool launch_update_sketch(Context& c, const SketchDev& S, const double* y, double* V, int64_t ldv, const VecLayout& lay,
                          int j, int nwin, int ngram, double* rec, const RecLayout& RL, double* cvec,
                          const double* coef_ready, int64_t row_begin, StepFold* sf = nullptr);
/// Split step pipeline (one GPU): K2'(j) = update alone, the SRDCT of w_{j+1}
/// on a side stream overlapping K1(j+1) / K2'(j+1); K2'(j) folds K1(j)'s
/// dots, K2'(j-1)'s norm / Gram (row j) and SRDCT(j-2)'s partials (row j-1).
struct SplitFold {
  const double* k1_partials = nullptr;
  int k1_G = 0;
  const double* prev_ng = nullptr;  // K2'(j-1) norm / Gram partials, null at j = 0
  int prev_ng_G = 0, prev_ngram = 0;
  const double* prev_sk = nullptr;  // SRDCT(j-2) partials, null for j < 2
  int prev_sk_G = 0, prev_sk_ld = 0, sk_row = 0;
  double* out_ng = nullptr;  // this update's norm / Gram partials (update_split_partials_size doubles)
};
bool sketch_partials_eligible(const SketchDev& S, int64_t nloc, int64_t row_begin);
int64_t sketch_partials_size(const SketchDev& S, int num_sms);
int64_t update_split_partials_size(int num_sms);
/// SRDCT CTA partials of x (two tile groups per CTA, no fold); G / ld out.
void launch_sketch_partials(Context& c, const SketchDev& S, const double* x_own, int64_t nloc, int64_t row_begin,
                            double* partials, int* G, int* ld);
/// out[0, s) = the sketch rows folded from launch_sketch_partials' CTA partials.
void launch_sketch_fold_partials(Context& c, const SketchDev& S, const double* partials, int G, int ld, double* out);
/// K2' (update alone) with the deferred prologue; returns its grid size.
int launch_update_split(Context& c, const SketchDev& S, const double* y, double* V, int64_t ldv, const VecLayout& lay,
                        int j, int nwin, int ngram, double* rec, const RecLayout& RL, double* cvec, const SplitFold& sf);
/// Completes rows j (sketch, from ska; may be null) and j+1 (sketch from skb,
/// norm / Gram from ng) at the end of a split cycle.
void launch_split_flush(Context& c, const SketchDev& S, const double* ska, int Ga, int lda, const double* skb, int Gb,
                        int ldb, const double* ng, int Gn, double* rec, const RecLayout& RL, int j, int ngram, int maxt);
/// Folds the partials a deferred K2(j) left (sf.out_*) into record row j+1.
void launch_update_sketch_flush(Context& c, const SketchDev& S, const StepFold& sf, double* rec, const RecLayout& RL,
                                int j, int ngram);

}  // namespace sdr
