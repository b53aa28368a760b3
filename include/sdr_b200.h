/*
 * sdr_b200.h — C-ABI of the B200-native GMRES-SDR hot path.
 *
 * Drop-in boundary for the reference `skrylov` library's data-parallel inner
 * loop (/root/reference/proj/include/skrylov). Plain pointers and sizes only;
 * no C++ or torch types cross this boundary, and no exception escapes it.
 * Every entry point returns an sdr_status; on failure sdr_last_error()
 * returns the message (thread-local), reproducing the reference's exception
 * text where the reference raises one.
 *
 * Pointer arguments documented as "host or device" are classified with
 * cudaPointerGetAttributes: a cudaMalloc'd pointer is used in place, anything
 * else is staged through pinned memory on the context's stream.
 *
 * Reference interface each entry point replaces (file:line under proj/):
 *   sdr_csr_*            SparseMatrix + OperatorRef    sparse.hpp:27-150, operator_ref.hpp:20-56
 *   sdr_sketch_*         SketchOperator                sketch.hpp:93-193
 *   sdr_gaussian_vector  gaussian_vector(n, seed)      rng.hpp:87-96
 *   sdr_qr_*             IncrementalQR                 incremental_qr.hpp:26-162
 *   sdr_harmonic         truncated_svd/fill_pencil/harmonic_pairs  recycle.hpp:98-218
 *   sdr_recycle_*        RecycleSpace, refresh_for_new_matrix       recycle.hpp:31-72,297-318
 *   sdr_krylov_run       init_krylov + arnoldi_step                  arnoldi.hpp:47-119
 *   sdr_solve            solve(A, b, cfg, space, sketch, x0, cb)    solver.hpp:269-365
 *   sdr_solve_sequence   solve_sequence(seq, cfg, sketch, space)     solver.hpp:385-459
 *   sdr_gen_*            gen_convdiff, gen_neumann (+ BASELINE generators)  problems.hpp:38-88
 *   sdr_spmm             the exact refresh's k products              recycle.hpp:309-316
 *   sdr_baseline_*       BaselineConfig, baseline_gmres              baseline.hpp:24-216
 *   sdr_mm_*, sdr_csr_read_matrix_market  read/write_matrix_market   matrix_market.hpp:83-181
 *   sdr_space_file_*, sdr_recycle_save/load_file  SKRYRCY1 dump      recycle.hpp:337-390
 *   sdr_csr_create_complex   complex-fp64 operators (BASELINE C4; no reference counterpart)
 *   sdr_debug_*, sdr_ctx_set_stamps   measurement / test hooks (no reference counterpart)
 */
#ifndef SDR_B200_H
#define SDR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SDR_API __attribute__((visibility("default")))
#else
#define SDR_API
#endif

/* ------------------------------------------------------------- errors -- */
/* Mirrors the reference's exception classes:
 *   std::invalid_argument -> SDR_EINVAL, std::domain_error -> SDR_EDOMAIN,
 *   std::logic_error -> SDR_ELOGIC, std::runtime_error -> SDR_ERUNTIME. */
typedef enum {
  SDR_OK = 0,
  SDR_EINVAL = 1,
  SDR_EDOMAIN = 2,
  SDR_ELOGIC = 3,
  SDR_ERUNTIME = 4,
  SDR_ECUDA = 5,
  SDR_ENCCL = 6,
  SDR_ENOMEM = 7
} sdr_status;

SDR_API const char* sdr_last_error(void);
SDR_API int sdr_version(int* major, int* minor, int* patch);

/* ------------------------------------------------------------ handles -- */
typedef struct sdr_ctx sdr_ctx;         /* one GPU, one stream, optional NCCL rank */
typedef struct sdr_csr sdr_csr;         /* device operator (owns device memory)    */
typedef struct sdr_sketch sdr_sketch;   /* device sketch (owns device memory)      */
typedef struct sdr_recycle sdr_recycle; /* recycle space: U on device, SU/SAU host */
typedef struct sdr_report sdr_report;   /* SolveReport (report.hpp:50-63)          */
typedef struct sdr_qr sdr_qr;           /* host IncrementalQR                      */

/* ------------------------------------------------------------ context -- */
SDR_API int sdr_ctx_create(int device, sdr_ctx** out);
/* Multi-GPU: one process per GPU; rank 0 obtains a 128-byte NCCL unique id
 * with sdr_nccl_unique_id and every rank passes the same bytes. */
SDR_API int sdr_nccl_unique_id(void* out_128_bytes);
SDR_API int sdr_ctx_create_dist(int device, int rank, int world, const void* nccl_id_128, sdr_ctx** out);
/* Host-staged transport: the distributed pipeline (z-slab halos, one
 * allreduce per Arnoldi step) with the caller's collectives instead of NCCL,
 * each one on host memory after the context stream drained. For ranks that
 * cannot run NCCL between them (e.g. several processes sharing one GPU in
 * tests); never a fast path. Callbacks return 0 on success.
 *   allreduce_sum: in-place sum over ranks of n doubles
 *   allgather_i64: out[q * count + i] = rank q's in[i]
 *   exchange:      send nsend doubles to `peer` and receive nrecv from it */
typedef struct {
  int (*allreduce_sum)(double* buf, int64_t n, void* user);
  int (*allgather_i64)(const int64_t* in, int64_t count, int64_t* out, void* user);
  int (*exchange)(int peer, const double* send, int64_t nsend, double* recv, int64_t nrecv, void* user);
  void* user;
} sdr_host_comm;
SDR_API int sdr_ctx_create_hostcomm(int device, int rank, int world, const sdr_host_comm* comm, sdr_ctx** out);
SDR_API int sdr_ctx_destroy(sdr_ctx* ctx);
SDR_API int sdr_ctx_info(const sdr_ctx* ctx, int* device, int* rank, int* world, int* num_sms);
SDR_API int sdr_ctx_stream(const sdr_ctx* ctx, void** cuda_stream);
SDR_API int sdr_ctx_synchronize(sdr_ctx* ctx);
/* Per-kernel CUDA-event timing on the context stream (off by default).
 * names: "spmv_arnoldi", "update", "sketch", "tallskinny", "residual", ... */
SDR_API int sdr_ctx_set_timing(sdr_ctx* ctx, int enable);
SDR_API int sdr_ctx_timing_reset(sdr_ctx* ctx);
SDR_API int sdr_ctx_timing_get(const sdr_ctx* ctx, const char* kernel, int64_t* launches, double* total_ms);
/* Number of kernels this context has launched since creation. */
SDR_API int sdr_ctx_launch_count(const sdr_ctx* ctx, int64_t* launches);

/* ----------------------------------------------------------- operator -- */
/* Validates exactly like SparseMatrix::validate (sparse.hpp:117-143) and
 * copies the CSR into device SELL-32 storage with int32 indices. In a
 * distributed context each rank passes its own contiguous row block
 * [row_begin, row_begin + local_rows) with GLOBAL column indices. */
SDR_API int sdr_csr_create(sdr_ctx* ctx, int64_t rows, int64_t cols, const int64_t* offsets,
                           const int64_t* columns, const double* values, sdr_csr** out);
/* Complex fp64 CSR (values: nnz (re, im) pairs; BASELINE C4 operators): the
 * operator acts on interleaved vectors [re_0, im_0, re_1, im_1, ...] of length
 * 2·rows and is stored as ZSELL (see sdr_csr_storage). Single-rank contexts;
 * validated like sdr_csr_create in complex row / column terms. */
SDR_API int sdr_csr_create_complex(sdr_ctx* ctx, int64_t rows, int64_t cols, const int64_t* offsets,
                                   const int64_t* columns, const double* values, sdr_csr** out);
SDR_API int sdr_csr_create_local(sdr_ctx* ctx, int64_t global_rows, int64_t global_cols, int64_t row_begin,
                                 int64_t local_rows, const int64_t* offsets, const int64_t* columns,
                                 const double* values, sdr_csr** out);
/* Callable operator: OperatorRef(rows, cols, Apply) (operator_ref.hpp:22-25;
 * README: "Anything that applies vectors can be an operator"). apply must
 * enqueue y = A x on `cuda_stream` (or finish it before returning); x and y
 * are device pointers of cols / rows doubles; return 0 on success (nonzero is
 * reported as SDR_ERUNTIME). The handle is non-owning like OperatorRef: user
 * must outlive it. Usable wherever an sdr_csr is (sdr_spmv, sdr_solve,
 * sequences, exact refresh); the solver then runs the product and its
 * epilogues (window dots, residual) as separate launches. Single-rank
 * contexts; sdr_csr_storage reports format 3 and 0 bytes. */
typedef int (*sdr_apply_fn)(const double* x, double* y, void* cuda_stream, void* user);
SDR_API int sdr_operator_create_callback(sdr_ctx* ctx, int64_t rows, int64_t cols, sdr_apply_fn apply, void* user,
                                         sdr_csr** out);
SDR_API int sdr_csr_destroy(sdr_csr* A);
/* rows/cols global; nnz local (stored, before SELL padding); row_begin/local_rows this rank. */
SDR_API int sdr_csr_info(const sdr_csr* A, int64_t* rows, int64_t* cols, int64_t* nnz, int64_t* row_begin,
                         int64_t* local_rows, int64_t* halo_lo, int64_t* halo_hi);
/* NEW: device storage chosen for the block. format 0 = SELL-32 (12 B per stored
 * entry), 1 = SELL-DIA (8 B per stored entry + one int32 offset per slice
 * diagonal), 2 = ZSELL (a one-rank operator whose 2x2 blocks are all
 * [[a, -b], [b, a]]: a complex matrix on interleaved (re, im) vectors, stored
 * as complex entries, 20 B each — the complex-fp64 SpMV of BASELINE C4);
 * diagonals = DIA diagonals per slice (0 otherwise); stored = entries incl.
 * padding (complex entries for ZSELL); bytes = storage bytes one SpMV streams;
 * 3 = callable operator (sdr_operator_create_callback, nothing stored). */
SDR_API int sdr_csr_storage(const sdr_csr* A, int32_t* format, int32_t* diagonals, int64_t* stored, int64_t* bytes);
/* y = A x (OperatorRef::apply, operator_ref.hpp:38-44). x: local_rows entries of this
 * rank's block (halos are exchanged internally); y: local_rows entries. Host or device. */
SDR_API int sdr_spmv(sdr_ctx* ctx, const sdr_csr* A, const double* x, int64_t xlen, double* y);
/* Y(:, q) = A X(:, q) for q < nb (column-major, host or device): the batched
 * product of the exact recycle refresh (recycle.hpp:309-316), one pass over A
 * per 8 columns; each column equals sdr_spmv bit for bit. Single-rank context. */
SDR_API int sdr_spmm(sdr_ctx* ctx, const sdr_csr* A, int64_t nb, const double* X, int64_t ldx, double* Y,
                     int64_t ldy);

/* ------------------------------------------------------------- sketch -- */
typedef enum { SDR_SKETCH_SRDCT = 0, SDR_SKETCH_IDENTITY = 1, SDR_SKETCH_SPARSE_SIGN = 2 } sdr_sketch_kind;
/* SketchOperator::subsampled_dct (sketch.hpp:105-122): n sign draws then
 * s Fisher-Yates row draws from std::mt19937_64(seed), bit-exact. */
SDR_API int sdr_sketch_create_srdct(sdr_ctx* ctx, int64_t n, int64_t s, uint64_t seed, sdr_sketch** out);
SDR_API int sdr_sketch_create_identity(sdr_ctx* ctx, int64_t n, sdr_sketch** out);
/* NEW (not in the reference): sparse sign map, zeta nonzeros per column, block construction. */
SDR_API int sdr_sketch_create_sparse_sign(sdr_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int64_t zeta,
                                          sdr_sketch** out);
SDR_API int sdr_sketch_destroy(sdr_sketch* S);
SDR_API int sdr_sketch_info(const sdr_sketch* S, int* kind, int64_t* n, int64_t* s, uint64_t* seed, int64_t* zeta);
/* Exported generator output for bit-exact checks: rows (s entries, SRDCT only),
 * signs (+1/-1, n entries, SRDCT only). */
SDR_API int sdr_sketch_rows(const sdr_sketch* S, int64_t* rows_out);
SDR_API int sdr_sketch_signs(const sdr_sketch* S, double* signs_out);
/* out = S x. x: this rank's block (host or device); out: s entries on the host,
 * summed over ranks. */
SDR_API int sdr_sketch_apply(sdr_ctx* ctx, const sdr_sketch* S, const double* x, int64_t xlen, double* out);

/* -------------------------------------------------------- host pieces -- */
SDR_API int sdr_gaussian_vector(int64_t n, uint64_t seed, double* out);
/* Rng(seed).uniform() stream (rng.hpp:32): (engine() >> 11) * 2^-53, n draws
 * (the C3 diagonal perturbation of the BASELINE sequence). */
SDR_API int sdr_uniform_stream(int64_t n, uint64_t seed, double* out);
/* Host generator behind sdr_sketch_create_srdct: rows (s, sorted) and signs
 * (+1/-1, n; may be NULL) drawn from std::mt19937_64(seed) in the reference
 * order (sketch.hpp:116-119). Needs no GPU. */
SDR_API int sdr_srdct_indices(int64_t n, int64_t s, uint64_t seed, int64_t* rows, double* signs);
/* Sparse-sign (row, sign) entries of columns [j0, j0+count): rows/signs hold count*zeta. */
SDR_API int sdr_sparse_sign_entries(int64_t s, uint64_t seed, int64_t zeta, int64_t j0, int64_t count,
                                    int64_t* rows, double* signs);

/* IncrementalQR (incremental_qr.hpp:26-162), host, two-pass classical GS. */
SDR_API int sdr_qr_create(int64_t rows, int64_t capacity, double rank_tol, sdr_qr** out);
SDR_API int sdr_qr_destroy(sdr_qr* qr);
SDR_API int sdr_qr_append(sdr_qr* qr, const double* col, int64_t len, int64_t* column, int* rank_deficient);
SDR_API int sdr_qr_exclude(sdr_qr* qr, int64_t column);
SDR_API int sdr_qr_cols(const sdr_qr* qr, int64_t* cols);
/* y: cols() entries; residual evaluated against the raw appended columns. */
SDR_API int sdr_qr_solve(const sdr_qr* qr, const double* rhs, int64_t len, double* y, double* residual_norm);
/* Q (rows x cols) and R (cols x cols), column-major. */
SDR_API int sdr_qr_factors(const sdr_qr* qr, double* Q, double* R);

/* Harmonic pencil + selection (recycle.hpp:98-218). SAW, SW: s x p column-major.
 * coeffs: p x (k+1) buffer, first k_eff columns filled; mu: k+1 entries. */
SDR_API int sdr_harmonic(const double* SAW, const double* SW, int64_t s, int64_t p, int64_t k, double rank_tol,
                         int64_t* rank, int64_t* k_eff, int* pair_extended, int* rank_limited, double* coeffs,
                         double* mu_re, double* mu_im);
/* Same, with via_qr != 0: SAW is first factored by the incremental QR the
 * solver keeps per cycle (two-pass Gram-Schmidt, incremental_qr.hpp:46-93), and
 * the extraction runs on the factors as in the solver (when R is well
 * conditioned the pencil is formed as R^{-1} Q^T SW without an SVD). */
SDR_API int sdr_harmonic_qr(const double* SAW, const double* SW, int64_t s, int64_t p, int64_t k, double rank_tol,
                            int32_t via_qr, int64_t* rank, int64_t* k_eff, int* pair_extended, int* rank_limited,
                            double* coeffs, double* mu_re, double* mu_im);

/* 1-D row partition of a banded operator: given every rank's
 * [row_begin, row_end) and referenced column range [min_col, max_col],
 * returns for `rank` the rows it must receive from / send to each peer.
 * recv_lo/recv_cnt/send_lo/send_cnt: world entries each (global row index, count). */
SDR_API int sdr_partition_halo(int world, int rank, const int64_t* row_begin, const int64_t* row_end,
                               const int64_t* min_col, const int64_t* max_col, int64_t* recv_lo,
                               int64_t* recv_cnt, int64_t* send_lo, int64_t* send_cnt);
/* Balanced contiguous block split (z-slabs when `granule` = plane size). */
SDR_API int sdr_partition_rows(int64_t rows, int world, int64_t granule, int64_t* row_begin, int64_t* row_end);

/* ------------------------------------------------------------ generators */
/* CSR arrays are written by the caller-allocated buffers; call with NULL
 * buffers first to get nnz. convdiff2d(n, bx, by, shift, diag_rel):
 * −Δu + β·∇u on n×n, equals −gen_convdiff(n, −β) when bx == by (problems.hpp:70-88). */
/* gen_neumann (problems.hpp:38-61): shifted five-point grid operator with mirrored
 * boundary neighbours, CSR as SparseMatrix::from_triplets builds it. Two-call:
 * NULL arrays -> *nnz. */
SDR_API int sdr_gen_neumann(int64_t grid_side, double shift, int64_t* nnz, int64_t* offsets, int64_t* columns,
                            double* values);
SDR_API int sdr_gen_convdiff2d(int64_t n, double bx, double by, double shift, const double* diag_rel,
                               int64_t* nnz, int64_t* offsets, int64_t* columns, double* values);
SDR_API int sdr_gen_convdiff3d(int64_t n, double bx, double by, double bz, int64_t z_begin, int64_t z_end,
                               int64_t* nnz, int64_t* offsets, int64_t* columns, double* values);
/* Device-side 3D operator on an nx×ny×nz grid (h_d = 1/(n_d+1)) for the z-slab
 * [z_begin, z_end), built in HBM without a host CSR (C5 scale). */
SDR_API int sdr_csr_create_convdiff3d(sdr_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double bx, double by,
                                      double bz, int64_t z_begin, int64_t z_end, sdr_csr** out);

/* ------------------------------------------------------------- solver -- */
typedef enum { SDR_VARIANT_REUSE = 0, SDR_VARIANT_EXACT = 1, SDR_VARIANT_INEXACT = 2 } sdr_variant;
typedef enum { SDR_CONVERGED = 0, SDR_MAX_RESTARTS = 1, SDR_BREAKDOWN = 2, SDR_DIVERGED = 3 } sdr_solve_status;
typedef enum {
  SDR_PROV_EMPTY = 0, SDR_PROV_FRESH = 1, SDR_PROV_REUSED = 2, SDR_PROV_EXACT_RESKETCH = 3,
  SDR_PROV_INEXACT_CARRYOVER = 4
} sdr_provenance;

/* SolverConfig (solver.hpp:48-79); sdr_config_default fills the reference defaults.
 * Validation is the reference's. Any window t >= 1 is accepted as there:
 * min(t, m) <= 33 runs the fused step kernels (the window lives in
 * registers), longer windows the unfused passes of wide.cu. */
typedef struct {
  int64_t m, t, k, s;
  double tol, safety_init;
  int32_t max_restarts, variant;
  uint64_t sketch_seed;
  double rank_tol, breakdown_tol;
} sdr_config;
SDR_API int sdr_config_default(sdr_config* cfg);
SDR_API int sdr_config_validate(const sdr_config* cfg);

/* IterationEvent / ResidualEvent (solver.hpp:82-104). y points at host memory valid for the call. */
typedef struct {
  int32_t cycle;
  int64_t step, iteration;
  double sres, new_basis_sketch_norm;
  const double* y;
  int64_t y_len, space_dim;
} sdr_iteration_event;
typedef struct {
  int32_t cycle;
  int64_t iteration;
  double sres, true_residual;
} sdr_residual_event;
typedef struct {
  void (*on_iteration)(const sdr_iteration_event* ev, void* user);
  void (*on_residual_check)(const sdr_residual_event* ev, void* user);
  void* user;
} sdr_callbacks;

SDR_API int sdr_recycle_create(sdr_ctx* ctx, sdr_recycle** out);
SDR_API int sdr_recycle_destroy(sdr_recycle* sp);
SDR_API int sdr_recycle_info(const sdr_recycle* sp, int64_t* rows, int64_t* s, int64_t* dim, int* provenance);
/* U: local_rows x dim (normalised, host or device), SU/SAU: s x dim host; column-major. */
SDR_API int sdr_recycle_get(sdr_ctx* ctx, const sdr_recycle* sp, double* U, double* SU, double* SAU);
SDR_API int sdr_recycle_set(sdr_ctx* ctx, sdr_recycle* sp, int64_t rows, int64_t s, int64_t dim, const double* U,
                            const double* SU, const double* SAU, int provenance);
SDR_API int sdr_recycle_drop_columns(sdr_recycle* sp, const int64_t* cols, int64_t ncols);
/* refresh_for_new_matrix (recycle.hpp:297-318): mode 0 exact, 1 inexact.
 * counters (may be NULL): matvecs, inner_products, sketch_applies are incremented. */
SDR_API int sdr_recycle_refresh(sdr_ctx* ctx, sdr_recycle* sp, const sdr_csr* A, const sdr_sketch* S, int mode,
                                int64_t* counters3);

/* init_krylov + up to `steps` arnoldi_step calls (arnoldi.hpp:47-119) through the
 * device pipeline. r0: this rank's block (host or device). Outputs (column-major,
 * each may be NULL): V local_rows x (m+1) normalised basis (host or device),
 * H (m+1) x m, SV s x (m+1), SAV s x m (host). counters3 as in sdr_recycle_refresh. */
SDR_API int sdr_krylov_run(sdr_ctx* ctx, const sdr_csr* A, const sdr_sketch* S, const double* r0, int64_t t, int64_t m,
                           int64_t steps, double breakdown_tol, double* V, double* H, double* SV, double* SAV,
                           int64_t* j_out, int* breakdown, double* r0_norm, int64_t* counters3);

/* Test hook: C = [A1 A2] B (n rows, k1 + k2 inputs, nout <= 24 outputs,
 * column-major) and norms2[q] = ||C(:, q)||^2 through the recycle-product
 * kernels (kernel 0: k_tsgemm, nout <= 24 and even n / leading dims;
 * 1: k_rgemm). Host or device arrays. */
SDR_API int sdr_debug_block_product(sdr_ctx* ctx, int32_t kernel, int64_t n, const double* A1, int64_t lda1,
                                    int32_t k1, const double* A2, int64_t lda2, int32_t k2, const double* B,
                                    int32_t nout, double* C, int64_t ldc, double* norms2);

/* Test hook for the NVLink peer-memory one-shot allreduce (SDR_PEER=1 on
 * several ranks): `world` virtual ranks as CTAs of one cooperative launch on
 * this GPU run `epochs` allreduces of n values back to back through the same
 * device code. vals / out: host [epochs][world][n]; out[e][r] must equal the
 * rank-ordered sum over vals[e][*] for every r. */
SDR_API int sdr_debug_peer_emulate(int32_t world, int32_t n, int32_t epochs, const double* vals, double* out);

/* Measurement: init + `steps` pipelined Arnoldi steps from r0, then the mean
 * CUDA-event duration (microseconds) of `reps` back-to-back relaunches of the
 * last step's K1 (SpMV + window dots) and K2 (fused update + SRDCT) on the
 * library stream. The relaunches are idempotent. One-GPU SRDCT contexts. */
SDR_API int sdr_debug_time_step(sdr_ctx* ctx, const sdr_csr* A, const sdr_sketch* S, const double* r0, int64_t t,
                                int64_t m, int64_t steps, int32_t reps, double* k1_us, double* k2_us);
/* Debugging / measurement: kernel phase trace (SDR_TRACE=1), per-launch CUDA-event
 * timeline and device-clock launch stamps (first CTA start, last CTA end,
 * %globaltimer), written as CSV; stamps are recorded with SDR_TRACE=2 or after
 * sdr_ctx_set_stamps(ctx, 1), and reading them resets the buffer. */
SDR_API int sdr_debug_trace(sdr_ctx* ctx, uint64_t* out, int64_t cap, int64_t* n);
SDR_API int sdr_debug_timeline(sdr_ctx* ctx, const char* path);
SDR_API int sdr_debug_stamps(sdr_ctx* ctx, const char* path);
SDR_API int sdr_ctx_set_stamps(sdr_ctx* ctx, int on);

/* solve (solver.hpp:269-365). b, x0 (may be NULL), x_out: this rank's block,
 * host or device. space (may be NULL) is updated in place. sketch may be NULL
 * (SRDCT from cfg->s, cfg->sketch_seed). report_out may be NULL. */
SDR_API int sdr_solve(sdr_ctx* ctx, const sdr_csr* A, const double* b, const double* x0, const sdr_config* cfg,
                      sdr_recycle* space, const sdr_sketch* sketch, const sdr_callbacks* cb, double* x_out,
                      sdr_report** report_out);
/* solve_sequence (solver.hpp:385-459). mats[i] may repeat (pointer equality
 * = same matrix, solver.hpp:417-418). x0s and tols may be NULL. */
SDR_API int sdr_solve_sequence(sdr_ctx* ctx, int32_t nprob, const sdr_csr* const* mats, const double* const* rhs,
                               const double* const* x0s, const double* tols, int32_t shared_matrix,
                               const sdr_config* cfg, const sdr_sketch* sketch, sdr_recycle* space,
                               double* const* x_outs, sdr_report** reports_out);

/* ---------------------------------------------------------------- files --
 * Matrix Market (matrix_market.hpp:83-181) and the SKRYRCY1 recycle-space dump
 * (recycle.hpp:337-385). Host only except sdr_csr_read_matrix_market /
 * sdr_recycle_save_file / sdr_recycle_load_file. Parse and IO failures return
 * SDR_ERUNTIME with the reference's message text (line numbers included). */
typedef struct sdr_host_csr sdr_host_csr;
SDR_API int sdr_mm_read_file(const char* path, sdr_host_csr** out);
SDR_API int sdr_mm_read_string(const char* text, int64_t len, sdr_host_csr** out);
SDR_API int sdr_host_csr_info(const sdr_host_csr* h, int64_t* rows, int64_t* cols, int64_t* nnz);
SDR_API int sdr_host_csr_arrays(const sdr_host_csr* h, const int64_t** offsets, const int64_t** columns,
                                const double** values);
SDR_API int sdr_host_csr_destroy(sdr_host_csr* h);
/* coordinate / real / general, 17 significant digits. _string: buf NULL -> *len = bytes needed (with NUL). */
SDR_API int sdr_mm_write_file(const char* path, int64_t rows, int64_t cols, const int64_t* offsets,
                              const int64_t* columns, const double* values);
SDR_API int sdr_mm_write_string(int64_t rows, int64_t cols, const int64_t* offsets, const int64_t* columns,
                                const double* values, char* buf, int64_t* len);
/* read_matrix_market_file + upload (single-rank context). */
SDR_API int sdr_csr_read_matrix_market(sdr_ctx* ctx, const char* path, sdr_csr** out);

typedef struct sdr_space_file sdr_space_file;
SDR_API int sdr_space_file_read(const char* path, sdr_space_file** out);
SDR_API int sdr_space_file_read_bytes(const void* data, int64_t len, sdr_space_file** out);
SDR_API int sdr_space_file_info(const sdr_space_file* f, int64_t* n, int64_t* s, int64_t* k, int* provenance);
SDR_API int sdr_space_file_arrays(const sdr_space_file* f, const double** U, const double** SU, const double** SAU);
SDR_API int sdr_space_file_destroy(sdr_space_file* f);
SDR_API int sdr_space_file_write(const char* path, int64_t n, int64_t s, int64_t k, int provenance, const double* U,
                                 const double* SU, const double* SAU);
/* buf NULL -> *len = bytes needed. */
SDR_API int sdr_space_file_write_bytes(int64_t n, int64_t s, int64_t k, int provenance, const double* U,
                                       const double* SU, const double* SAU, void* buf, int64_t* len);
/* save_recycle_space_file / load_recycle_space_file on a device space (this
 * rank's rows: one file per rank in a distributed context). */
SDR_API int sdr_recycle_save_file(sdr_ctx* ctx, const sdr_recycle* sp, const char* path);
SDR_API int sdr_recycle_load_file(sdr_ctx* ctx, sdr_recycle* sp, const char* path);

/* ----------------------------------------------------------- baseline --
 * Classical restarted GMRES, the reference's comparison point
 * (baseline.hpp:24-39 BaselineConfig, :51-216 baseline_gmres): full
 * orthogonalisation against the whole basis every step, Givens rotations,
 * one verification product per cycle. Same statuses / notes / counters
 * (one inner product per MGS dot) as the reference; m <= 255 on the device.
 * b, x0 (may be NULL), x_out: this rank's block, host or device. */
typedef struct {
  int64_t m;
  double tol;
  int32_t max_restarts;
  double breakdown_tol;
} sdr_baseline_config;
SDR_API int sdr_baseline_config_default(sdr_baseline_config* cfg);
SDR_API int sdr_baseline_gmres(sdr_ctx* ctx, const sdr_csr* A, const double* b, const double* x0,
                               const sdr_baseline_config* cfg, double* x_out, sdr_report** report_out);

/* SolveReport accessors (report.hpp:50-63). */
SDR_API int sdr_report_destroy(sdr_report* r);
SDR_API int sdr_report_summary(const sdr_report* r, int* status, int64_t* iterations, int32_t* cycles,
                               double* rhs_norm, double* final_relative_residual, double* seconds);
SDR_API int sdr_report_counters(const sdr_report* r, int64_t* matvecs, int64_t* inner_products,
                                int64_t* sketch_applies);
/* which: 0 sketched residuals, 1 true residuals. Call with NULL to get n. */
SDR_API int sdr_report_samples(const sdr_report* r, int which, int64_t* n, int64_t* iteration, double* value);
/* per cycle: steps, entry_residual, sketched_entry, exit_sres, exit_residual, safety_after, basis_cond, deflation_rank */
SDR_API int sdr_report_cycles(const sdr_report* r, int64_t* n, double* stats8);
SDR_API int sdr_report_notes(const sdr_report* r, int64_t* n);
SDR_API const char* sdr_report_note(const sdr_report* r, int64_t i);
SDR_API const char* sdr_report_error(const sdr_report* r);
/* Device-phase timing of the solve: arnoldi_ms (K1+K2+sketch), host_ms, steps. */
/* Wall-clock phase breakdown (ms): "setup", "cycle_init", "step_wait", "host_step",
 * "check", "drain", "basis_cond", "recycle", "recycle_harmonic". Unknown names give 0. */
SDR_API int sdr_report_phase(const sdr_report* r, const char* name, double* ms);
SDR_API int sdr_report_timing(const sdr_report* r, double* device_ms, double* host_wait_ms, double* total_ms);

#ifdef __cplusplus
}
#endif
#endif /* SDR_B200_H */
