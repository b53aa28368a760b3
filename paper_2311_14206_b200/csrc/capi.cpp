// C-ABI (include/sdr_b200.h): handles, error translation, host/device
// pointer staging. No exception crosses this boundary.
#include "../../include/sdr_b200.h"

#include "baseline.hpp"
#include "context.hpp"
#include "host_linalg.hpp"
#include "io.hpp"
#include "peer.hpp"
#include "operator.hpp"
#include "sketch.hpp"
#include "solver.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <sstream>

using namespace sdr;

namespace sdr {
void nccl_unique_id(void* out);
}

struct sdr_ctx {
  std::unique_ptr<Context> c;
};
struct sdr_csr {
  Context* ctx;
  std::unique_ptr<DeviceOperator> op;
};
struct sdr_sketch {
  Context* ctx;
  std::unique_ptr<SketchDev> S;
};
struct sdr_recycle {
  Context* ctx;
  Recycle sp;
};
struct sdr_report {
  Report r;
};
struct sdr_host_csr {
  HostCsr h;
};
struct sdr_space_file {
  SpaceFile f;
};
struct sdr_qr {
  std::unique_ptr<HostQR> qr;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SDR_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return SDR_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SDR_ERUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw invalid(std::string(what) + " must not be null");
}

Config to_cfg(const sdr_config* c) {
  Config k;
  k.m = c->m;
  k.t = c->t;
  k.k = c->k;
  k.s = c->s;
  k.tol = c->tol;
  k.safety_init = c->safety_init;
  k.max_restarts = c->max_restarts;
  k.variant = c->variant;
  k.sketch_seed = c->sketch_seed;
  k.rank_tol = c->rank_tol;
  k.breakdown_tol = c->breakdown_tol;
  return k;
}

bool host_nonzero(Context& c, const double* x, i64 n) {
  std::vector<double> h;
  const double* p = x;
  if (!x) n = 0;
  if (x && is_device_pointer(x)) {
    h.resize(static_cast<size_t>(n));
    SDR_CUDA(cudaMemcpy(h.data(), x, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost));
    p = h.data();
  }
  i64 nz = 0;
  for (i64 i = 0; i < n && !nz; ++i)
    if (p[i] != 0.0) nz = 1;
  if (c.distributed()) {
    // every rank must take the same branch (the x0 != 0 residual exchanges the
    // halo): x0 counts as nonzero when any rank's slice is
    std::vector<i64> all(static_cast<size_t>(c.world));
    c.allgather_i64(&nz, 1, all.data());
    for (i64 v : all) nz |= v;
  }
  return nz != 0;
}

/// Output staging: device pointers are written directly, host pointers via a
/// device buffer copied back on finish().
struct DeviceOut {
  double* user;
  double* ptr;
  i64 n;
  DeviceBuffer<double> own;
  /// pinned_ok: the callee only copies into the destination (cudaMemcpyAsync),
  /// so page-locked host memory is used in place and the copy-out can overlap
  /// the callee's remaining host work.
  DeviceOut(double* p, i64 nn, bool pinned_ok = false) : user(p), ptr(p), n(nn) {
    if (p && !is_device_pointer(p) && !(pinned_ok && is_pinned_host_pointer(p))) {
      own.resize(std::max<i64>(n, 1));
      ptr = own.get();
    }
  }
  void finish(Context& c) {
    if (user && ptr != user)
      SDR_CUDA(cudaMemcpyAsync(user, ptr, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  }
};

}  // namespace

extern "C" {

const char* sdr_last_error(void) { return g_err.c_str(); }

int sdr_version(int* major, int* minor, int* patch) {
  if (major) *major = 0;
  if (minor) *minor = 1;
  if (patch) *patch = 0;
  return SDR_OK;
}

// ------------------------------------------------------------------ context
int sdr_ctx_create(int device, sdr_ctx** out) {
  return guard([&] {
    need(out, "out");
    auto h = std::make_unique<sdr_ctx>();
    h->c = std::make_unique<Context>(device, 0, 1, nullptr);
    *out = h.release();
  });
}

int sdr_nccl_unique_id(void* out) {
  return guard([&] {
    need(out, "out");
    nccl_unique_id(out);
  });
}

int sdr_ctx_create_dist(int device, int rank, int world, const void* id, sdr_ctx** out) {
  return guard([&] {
    need(out, "out");
    if (world < 1 || rank < 0 || rank >= world) throw invalid("sdr_ctx_create_dist: bad rank/world");
    auto h = std::make_unique<sdr_ctx>();
    h->c = std::make_unique<Context>(device, rank, world, id);
    *out = h.release();
  });
}

int sdr_ctx_create_hostcomm(int device, int rank, int world, const sdr_host_comm* comm, sdr_ctx** out) {
  return guard([&] {
    need(out, "out");
    need(comm, "comm");
    if (world < 1 || rank < 0 || rank >= world) throw invalid("sdr_ctx_create_hostcomm: bad rank/world");
    HostComm hc;
    hc.allreduce_sum = comm->allreduce_sum;
    hc.allgather_i64 = reinterpret_cast<int (*)(const i64*, i64, i64*, void*)>(comm->allgather_i64);
    hc.exchange = comm->exchange;
    hc.user = comm->user;
    auto h = std::make_unique<sdr_ctx>();
    h->c = std::make_unique<Context>(device, rank, world, nullptr, &hc);
    *out = h.release();
  });
}

int sdr_ctx_destroy(sdr_ctx* ctx) {
  return guard([&] { delete ctx; });
}

int sdr_ctx_info(const sdr_ctx* ctx, int* device, int* rank, int* world, int* num_sms) {
  return guard([&] {
    need(ctx, "ctx");
    if (device) *device = ctx->c->device;
    if (rank) *rank = ctx->c->rank;
    if (world) *world = ctx->c->world;
    if (num_sms) *num_sms = ctx->c->num_sms;
  });
}

int sdr_ctx_stream(const sdr_ctx* ctx, void** stream) {
  return guard([&] {
    need(ctx, "ctx");
    need(stream, "stream");
    *stream = ctx->c->stream;
  });
}

int sdr_ctx_synchronize(sdr_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->sync();
  });
}

int sdr_ctx_set_timing(sdr_ctx* ctx, int enable) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->timing_flush();
    ctx->c->timing = enable != 0;
  });
}

int sdr_ctx_timing_reset(sdr_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->timing_reset();
  });
}

int sdr_ctx_timing_get(const sdr_ctx* ctx, const char* kernel, int64_t* launches, double* total_ms) {
  return guard([&] {
    need(ctx, "ctx");
    need(kernel, "kernel");
    ctx->c->timing_flush();
    auto it = ctx->c->timings.find(kernel);
    if (launches) *launches = it == ctx->c->timings.end() ? 0 : it->second.launches;
    if (total_ms) *total_ms = it == ctx->c->timings.end() ? 0.0 : it->second.ms;
  });
}

int sdr_ctx_launch_count(const sdr_ctx* ctx, int64_t* launches) {
  return guard([&] {
    need(ctx, "ctx");
    need(launches, "launches");
    *launches = ctx->c->launches;
  });
}

// ----------------------------------------------------------------- operator
int sdr_csr_create(sdr_ctx* ctx, int64_t rows, int64_t cols, const int64_t* offsets, const int64_t* columns,
                   const double* values, sdr_csr** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    if (ctx->c->distributed()) throw invalid("sdr_csr_create: use sdr_csr_create_local in a distributed context");
    auto h = std::make_unique<sdr_csr>();
    h->ctx = ctx->c.get();
    h->op.reset(create_operator_csr(*ctx->c, rows, cols, 0, rows, offsets, columns, values));
    *out = h.release();
  });
}

int sdr_csr_create_complex(sdr_ctx* ctx, int64_t rows, int64_t cols, const int64_t* offsets, const int64_t* columns,
                           const double* values, sdr_csr** out) {
  return guard([&] {  // complex CSR (values as (re, im) pairs) -> the real-equivalent operator, stored as ZSELL
    need(ctx, "ctx");
    need(out, "out");
    if (ctx->c->distributed()) throw invalid("sdr_csr_create_complex: single-rank contexts only");
    if (rows < 0 || cols < 0) throw invalid("SparseMatrix: negative dimensions");
    need(offsets, "offsets");
    if (offsets[0] != 0) throw invalid("SparseMatrix: offsets must start at 0");
    const int64_t nnz = offsets[rows];
    if (nnz > 0 && (!columns || !values)) throw invalid("SparseMatrix: offsets/columns/values sizes inconsistent");
    std::vector<int64_t> ro(static_cast<size_t>(2 * rows) + 1, 0), rc;
    std::vector<double> rv;
    rc.reserve(static_cast<size_t>(4 * nnz));
    rv.reserve(static_cast<size_t>(4 * nnz));
    for (int64_t r = 0; r < rows; ++r) {
      if (offsets[r + 1] < offsets[r]) throw invalid("SparseMatrix: offsets decrease at row " + std::to_string(r));
      for (int64_t p = offsets[r]; p < offsets[r + 1]; ++p) {
        if (columns[p] < 0 || columns[p] >= cols)
          throw invalid("SparseMatrix: column index " + std::to_string(columns[p]) + " out of range in row " +
                        std::to_string(r));
        if (p > offsets[r] && columns[p - 1] >= columns[p])
          throw invalid("SparseMatrix: column indices not strictly increasing in row " + std::to_string(r));
        if (!std::isfinite(values[2 * p]) || !std::isfinite(values[2 * p + 1]))
          throw invalid("SparseMatrix: non-finite value in row " + std::to_string(r));
      }
      for (int half = 0; half < 2; ++half) {  // real row 2r (re), 2r + 1 (im): [[a, -b], [b, a]]
        for (int64_t p = offsets[r]; p < offsets[r + 1]; ++p) {
          const double a = values[2 * p], b = values[2 * p + 1];
          const double v0 = half == 0 ? a : b, v1 = half == 0 ? -b : a;
          if (v0 != 0.0) {
            rc.push_back(2 * columns[p]);
            rv.push_back(v0);
          }
          if (v1 != 0.0) {
            rc.push_back(2 * columns[p] + 1);
            rv.push_back(v1);
          }
        }
        ro[static_cast<size_t>(2 * r + half) + 1] = static_cast<int64_t>(rc.size());
      }
    }
    auto h = std::make_unique<sdr_csr>();
    h->ctx = ctx->c.get();
    h->op.reset(create_operator_csr(*ctx->c, 2 * rows, 2 * cols, 0, 2 * rows, ro.data(), rc.data(), rv.data()));
    *out = h.release();
  });
}

int sdr_csr_create_local(sdr_ctx* ctx, int64_t grows, int64_t gcols, int64_t row_begin, int64_t local_rows,
                         const int64_t* offsets, const int64_t* columns, const double* values, sdr_csr** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    auto h = std::make_unique<sdr_csr>();
    h->ctx = ctx->c.get();
    h->op.reset(create_operator_csr(*ctx->c, grows, gcols, row_begin, local_rows, offsets, columns, values));
    *out = h.release();
  });
}

int sdr_csr_create_convdiff3d(sdr_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double bx, double by, double bz,
                              int64_t z0, int64_t z1, sdr_csr** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    auto h = std::make_unique<sdr_csr>();
    h->ctx = ctx->c.get();
    h->op.reset(create_operator_convdiff3d(*ctx->c, nx, ny, nz, bx, by, bz, z0, z1));
    *out = h.release();
  });
}

int sdr_operator_create_callback(sdr_ctx* ctx, int64_t rows, int64_t cols, sdr_apply_fn apply, void* user,
                                 sdr_csr** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    if (!apply) throw invalid("OperatorRef: apply function required");
    if (rows < 0 || cols < 0) throw invalid("SparseMatrix: negative dimensions");
    Context& c = *ctx->c;
    if (c.distributed()) throw invalid("OperatorRef: callable operators need a single-rank context");
    auto op = std::make_unique<DeviceOperator>();
    op->rows = rows;
    op->cols = cols;
    op->local_rows = rows;
    op->halo_hi = std::max<int64_t>(0, cols - rows);
    op->reach_hi_begin = rows;
    op->plan.recv_lo.assign(1, 0);
    op->plan.recv_cnt.assign(1, 0);
    op->plan.send_lo.assign(1, 0);
    op->plan.send_cnt.assign(1, 0);
    op->apply = apply;
    op->apply_user = user;
    auto h = std::make_unique<sdr_csr>();
    h->op.reset(op.release());
    h->ctx = &c;
    *out = h.release();
  });
}

int sdr_csr_destroy(sdr_csr* A) {
  return guard([&] { delete A; });
}

int sdr_csr_storage(const sdr_csr* A, int32_t* format, int32_t* diagonals, int64_t* stored, int64_t* bytes) {
  return guard([&] {
    need(A, "A");
    const auto& o = *A->op;
    const int64_t nslices = o.view().nslices;
    if (o.apply) {
      if (format) *format = 3;
      if (diagonals) *diagonals = 0;
      if (stored) *stored = 0;
      if (bytes) *bytes = 0;
      return;
    }
    if (format) *format = o.dia ? 1 : (o.cplx ? 2 : 0);
    if (diagonals) *diagonals = o.dia ? o.dia_d : 0;
    if (stored) *stored = o.stored;
    if (bytes)
      *bytes = o.dia ? 8 * o.stored + 4 * nslices * o.dia_d
                     : (o.cplx ? 20 * o.stored : 12 * o.stored) + 8 * (nslices + 1);
  });
}

int sdr_csr_info(const sdr_csr* A, int64_t* rows, int64_t* cols, int64_t* nnz, int64_t* row_begin, int64_t* local_rows,
                 int64_t* halo_lo, int64_t* halo_hi) {
  return guard([&] {
    need(A, "A");
    const auto& o = *A->op;
    if (rows) *rows = o.rows;
    if (cols) *cols = o.cols;
    if (nnz) *nnz = o.nnz;
    if (row_begin) *row_begin = o.row_begin;
    if (local_rows) *local_rows = o.local_rows;
    if (halo_lo) *halo_lo = o.halo_lo;
    if (halo_hi) *halo_hi = o.halo_hi;
  });
}

int sdr_spmv(sdr_ctx* ctx, const sdr_csr* A, const double* x, int64_t xlen, double* y) {
  return guard([&] {
    need(ctx, "ctx");
    need(A, "A");
    Context& c = *ctx->c;
    const auto& op = *A->op;
    const i64 expect = c.distributed() ? op.local_rows : op.cols;
    if (xlen != expect)
      throw invalid("OperatorRef::apply: operator has " + std::to_string(expect) + " columns but vector has " +
                    std::to_string(xlen) + " entries");
    need(x, "x");
    need(y, "y");
    const VecLayout L = op.layout();
    DeviceBuffer<double> xb(std::max<i64>(L.ld, 1));
    DeviceIn xin(c, x, xlen);
    SDR_CUDA(cudaMemcpyAsync(xb.get() + L.own_off, xin.ptr, sizeof(double) * static_cast<size_t>(xlen),
                             cudaMemcpyDeviceToDevice, c.stream));
    DeviceOut yo(y, op.local_rows);
    operator_apply(c, op, xb.get(), yo.ptr);
    yo.finish(c);
  });
}

int sdr_spmm(sdr_ctx* ctx, const sdr_csr* A, int64_t nb, const double* X, int64_t ldx, double* Y, int64_t ldy) {
  return guard([&] {  // nb products of one operator in ceil(nb / 8) passes over it
    need(ctx, "ctx");
    need(A, "A");
    if (nb < 0) throw invalid("sdr_spmm: negative column count");
    if (nb == 0) return;
    need(X, "X");
    need(Y, "Y");
    Context& c = *ctx->c;
    const auto& op = *A->op;
    if (c.distributed()) throw invalid("sdr_spmm: single-rank contexts only (use sdr_spmv per column)");
    if (ldx < op.cols || ldy < op.local_rows) throw invalid("sdr_spmm: leading dimension smaller than the operator");
    const VecLayout L = op.layout();
    DeviceIn xin(c, X, ldx * (nb - 1) + op.cols);
    DeviceBuffer<double> xb(L.ld * std::min<i64>(nb, kSpmmMax));
    DeviceOut yo(Y, ldy * (nb - 1) + op.local_rows);
    for (i64 q0 = 0; q0 < nb; q0 += kSpmmMax) {
      const int k = static_cast<int>(std::min<i64>(kSpmmMax, nb - q0));
      SpmmCols cols;
      for (int q = 0; q < k; ++q) {  // the operator layout (halo / padding) of each column
        SDR_CUDA(cudaMemcpyAsync(xb.get() + q * L.ld + L.own_off, xin.ptr + (q0 + q) * ldx,
                                 sizeof(double) * static_cast<size_t>(op.cols), cudaMemcpyDeviceToDevice, c.stream));
        cols.x[q] = xb.get() + q * L.ld + L.ext_shift();
      }
      launch_spmm(c, op.view(), cols, k, yo.ptr + q0 * ldy, ldy);
    }
    yo.finish(c);
  });
}

// ------------------------------------------------------------------- sketch
int sdr_sketch_create_srdct(sdr_ctx* ctx, int64_t n, int64_t s, uint64_t seed, sdr_sketch** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    auto h = std::make_unique<sdr_sketch>();
    h->ctx = ctx->c.get();
    h->S.reset(create_sketch(*ctx->c, kSrdct, n, s, seed, 0));
    *out = h.release();
  });
}

int sdr_sketch_create_identity(sdr_ctx* ctx, int64_t n, sdr_sketch** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    auto h = std::make_unique<sdr_sketch>();
    h->ctx = ctx->c.get();
    h->S.reset(create_sketch(*ctx->c, kIdentity, n, n, 0, 0));
    *out = h.release();
  });
}

int sdr_sketch_create_sparse_sign(sdr_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int64_t zeta, sdr_sketch** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    auto h = std::make_unique<sdr_sketch>();
    h->ctx = ctx->c.get();
    h->S.reset(create_sketch(*ctx->c, kSparseSign, n, s, seed, zeta));
    *out = h.release();
  });
}

int sdr_sketch_destroy(sdr_sketch* S) {
  return guard([&] { delete S; });
}

int sdr_sketch_info(const sdr_sketch* S, int* kind, int64_t* n, int64_t* s, uint64_t* seed, int64_t* zeta) {
  return guard([&] {
    need(S, "S");
    if (kind) *kind = S->S->kind;
    if (n) *n = S->S->n;
    if (s) *s = S->S->s;
    if (seed) *seed = S->S->seed;
    if (zeta) *zeta = S->S->zeta;
  });
}

int sdr_sketch_rows(const sdr_sketch* S, int64_t* rows) {
  return guard([&] {
    need(S, "S");
    need(rows, "rows");
    if (S->S->kind != kSrdct) throw invalid("sdr_sketch_rows: only the subsampled DCT sketch has rows");
    std::memcpy(rows, S->S->rows_host.data(), sizeof(int64_t) * S->S->rows_host.size());
  });
}

int sdr_sketch_signs(const sdr_sketch* S, double* signs) {
  return guard([&] {
    need(S, "S");
    need(signs, "signs");
    if (S->S->kind != kSrdct) throw invalid("sdr_sketch_signs: only the subsampled DCT sketch has signs");
    for (i64 i = 0; i < S->S->n; ++i) signs[i] = (S->S->sign_bits_host[static_cast<size_t>(i >> 5)] >> (i & 31)) & 1u ? 1.0 : -1.0;
  });
}

int sdr_sketch_apply(sdr_ctx* ctx, const sdr_sketch* S, const double* x, int64_t xlen, double* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(S, "S");
    need(x, "x");
    need(out, "out");
    Context& c = *ctx->c;
    if (!c.distributed() && xlen != S->S->n)
      throw invalid("SketchOperator::apply: operator takes length " + std::to_string(S->S->n) +
                    " but vector has length " + std::to_string(xlen));
    i64 row_begin = 0;
    if (c.distributed()) {
      std::vector<i64> all(static_cast<size_t>(c.world));
      c.allgather_i64(&xlen, 1, all.data());
      for (int q = 0; q < c.rank; ++q) row_begin += all[static_cast<size_t>(q)];
    }
    DeviceIn xin(c, x, xlen);
    sketch_apply(c, *S->S, xin.ptr, xlen, row_begin, out);
  });
}

// -------------------------------------------------------------- host pieces
int sdr_uniform_stream(int64_t n, uint64_t seed, double* out) {  // rng.hpp:32
  return guard([&] {
    if (n < 0) throw invalid("uniform_stream: n must be nonnegative");
    if (n > 0) need(out, "out");
    std::mt19937_64 eng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
  });
}

int sdr_gaussian_vector(int64_t n, uint64_t seed, double* out) {  // rng.hpp:45-60,87-96
  return guard([&] {
    if (n < 0) throw invalid("gaussian_vector: n must be nonnegative");
    if (n > 0) need(out, "out");
    std::mt19937_64 eng(seed);
    double spare = 0.0;
    bool have = false;
    auto uniform = [&] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
    for (int64_t i = 0; i < n; ++i) {
      if (have) {
        have = false;
        out[i] = spare;
        continue;
      }
      double u1;
      do {
        u1 = uniform();
      } while (u1 <= 0.0);
      const double u2 = uniform();
      const double radius = std::sqrt(-2.0 * std::log(u1));
      const double angle = 2.0 * 3.14159265358979323846 * u2;
      spare = radius * std::sin(angle);
      have = true;
      out[i] = radius * std::cos(angle);
    }
  });
}

int sdr_srdct_indices(int64_t n, int64_t s, uint64_t seed, int64_t* rows, double* signs) {
  return guard([&] {
    if (n < 2 || s < 1 || s >= n)
      throw invalid("SketchOperator: need 1 <= s < n, got s = " + std::to_string(s) + ", n = " + std::to_string(n));
    need(rows, "rows");
    const SrdctHost h = make_srdct_host(n, s, seed);
    std::memcpy(rows, h.rows.data(), sizeof(int64_t) * h.rows.size());
    if (signs)
      for (int64_t i = 0; i < n; ++i) signs[i] = (h.sign_bits[static_cast<size_t>(i >> 5)] >> (i & 31)) & 1u ? 1.0 : -1.0;
  });
}

int sdr_sparse_sign_entries(int64_t s, uint64_t seed, int64_t zeta, int64_t j0, int64_t count, int64_t* rows,
                            double* signs) {
  return guard([&] {
    if (s < 1 || zeta < 1 || zeta > s) throw invalid("sparse_sign: need 1 <= zeta <= s");
    std::mt19937_64 eng(seed);
    const std::uint64_t key = eng();
    for (int64_t j = 0; j < count; ++j)
      for (int64_t l = 0; l < zeta; ++l) {
        int64_t r;
        bool pos;
        sparse_sign_entry(key, s, zeta, j0 + j, l, &r, &pos);
        rows[j * zeta + l] = r;
        signs[j * zeta + l] = pos ? 1.0 : -1.0;
      }
  });
}

int sdr_qr_create(int64_t rows, int64_t capacity, double rank_tol, sdr_qr** out) {
  return guard([&] {
    need(out, "out");
    init_host_blas();
    auto h = std::make_unique<sdr_qr>();
    h->qr = std::make_unique<HostQR>(rows, capacity, rank_tol);
    *out = h.release();
  });
}

int sdr_qr_destroy(sdr_qr* qr) {
  return guard([&] { delete qr; });
}

int sdr_qr_append(sdr_qr* qr, const double* col, int64_t len, int64_t* column, int* rank_deficient) {
  return guard([&] {
    need(qr, "qr");
    need(col, "col");
    const auto info = qr->qr->append(col, len);
    if (column) *column = info.column;
    if (rank_deficient) *rank_deficient = info.rank_deficient ? 1 : 0;
  });
}

int sdr_qr_exclude(sdr_qr* qr, int64_t column) {
  return guard([&] {
    need(qr, "qr");
    qr->qr->exclude(column);
  });
}

int sdr_qr_cols(const sdr_qr* qr, int64_t* cols) {
  return guard([&] {
    need(qr, "qr");
    need(cols, "cols");
    *cols = qr->qr->cols();
  });
}

int sdr_qr_solve(const sdr_qr* qr, const double* rhs, int64_t len, double* y, double* res) {
  return guard([&] {
    need(qr, "qr");
    need(rhs, "rhs");
    std::vector<double> yy(static_cast<size_t>(qr->qr->cols()));
    const double r = qr->qr->solve(rhs, len, yy.data());
    if (y) std::memcpy(y, yy.data(), sizeof(double) * yy.size());
    if (res) *res = r;
  });
}

int sdr_qr_factors(const sdr_qr* qr, double* Q, double* R) {
  return guard([&] {
    need(qr, "qr");
    qr->qr->factors(Q, R);
  });
}

int sdr_harmonic(const double* SAW, const double* SW, int64_t s, int64_t p, int64_t k, double rank_tol, int64_t* rank,
                 int64_t* k_eff, int* pair_extended, int* rank_limited, double* coeffs, double* mu_re, double* mu_im) {
  return sdr_harmonic_qr(SAW, SW, s, p, k, rank_tol, 0, rank, k_eff, pair_extended, rank_limited, coeffs, mu_re, mu_im);
}

int sdr_harmonic_qr(const double* SAW, const double* SW, int64_t s, int64_t p, int64_t k, double rank_tol,
                    int32_t via_qr, int64_t* rank, int64_t* k_eff, int* pair_extended, int* rank_limited,
                    double* coeffs, double* mu_re, double* mu_im) {
  return guard([&] {
    init_host_blas();
    if (s < 0 || p < 0) throw invalid("sdr_harmonic: negative dimensions");
    HMat a(s, p), w(s, p);
    if (s * p > 0) {
      need(SAW, "SAW");
      need(SW, "SW");
      std::memcpy(a.a.data(), SAW, sizeof(double) * static_cast<size_t>(s * p));
      std::memcpy(w.a.data(), SW, sizeof(double) * static_cast<size_t>(s * p));
    }
    Harmonic h;
    HostQR qr(s, std::max<i64>(p, 1), 1e-12);
    bool use_qr = via_qr != 0;
    for (i64 j = 0; use_qr && j < p; ++j) use_qr = !qr.append(a.col(j), s).rank_deficient;
    if (use_qr && qr.clean()) {  // the solver's route: the cycle's least-squares QR of SAW
      HMat Q(s, p), R(p, p);
      qr.factors(Q.a.data(), R.a.data());
      h = harmonic_extract(a, w, k, rank_tol, &Q, &R);
    } else {
      h = harmonic_extract(a, w, k, rank_tol);
    }
    if (rank) *rank = h.rank;
    if (k_eff) *k_eff = h.k_eff;
    if (pair_extended) *pair_extended = h.pair_extended;
    if (rank_limited) *rank_limited = h.rank_limited;
    if (coeffs) std::memcpy(coeffs, h.coeffs.a.data(), sizeof(double) * h.coeffs.a.size());
    for (size_t i = 0; i < h.mu.size(); ++i) {
      if (mu_re) mu_re[i] = h.mu[i].real();
      if (mu_im) mu_im[i] = h.mu[i].imag();
    }
  });
}

int sdr_partition_halo(int world, int rank, const int64_t* rb, const int64_t* re, const int64_t* mnc,
                       const int64_t* mxc, int64_t* recv_lo, int64_t* recv_cnt, int64_t* send_lo, int64_t* send_cnt) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) throw invalid("sdr_partition_halo: bad rank/world");
    partition_halo(world, rank, rb, re, mnc, mxc, recv_lo, recv_cnt, send_lo, send_cnt);
  });
}

int sdr_partition_rows(int64_t rows, int world, int64_t granule, int64_t* rb, int64_t* re) {
  return guard([&] {
    if (world < 1 || granule < 1 || rows < 0 || rows % granule)
      throw invalid("sdr_partition_rows: rows must be a multiple of granule and world >= 1");
    const int64_t G = rows / granule;
    for (int q = 0; q < world; ++q) {
      rb[q] = (G * q / world) * granule;
      re[q] = (G * (q + 1) / world) * granule;
    }
  });
}

// --------------------------------------------------------------- generators
int sdr_gen_convdiff2d(int64_t n, double bx, double by, double shift, const double* diag_rel, int64_t* nnz,
                       int64_t* off, int64_t* col, double* val) {
  return guard([&] {
    if (n < 1) throw invalid("gen_convdiff: n must be positive");
    const double h2 = static_cast<double>((n + 1) * (n + 1));
    const double cx = bx * static_cast<double>(n + 1) / 2.0, cy = by * static_cast<double>(n + 1) / 2.0;
    const double c[4] = {-h2 - cy, -h2 - cx, -h2 + cx, -h2 + cy};  // p-n, p-1, p+1, p+n
    int64_t k = 0;
    if (off) off[0] = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        const int64_t p = i * n + j;
        double d = 4.0 * h2 + shift;
        if (diag_rel) d = d + d * diag_rel[p];
        const bool has[5] = {i > 0, j > 0, true, j + 1 < n, i + 1 < n};
        const int64_t cc[5] = {p - n, p - 1, p, p + 1, p + n};
        const double vv[5] = {c[0], c[1], d, c[2], c[3]};
        for (int e = 0; e < 5; ++e) {
          if (!has[e] || vv[e] == 0.0) continue;  // from_triplets drops exact zeros
          if (col) col[k] = cc[e];
          if (val) val[k] = vv[e];
          ++k;
        }
        if (off) off[p + 1] = k;
      }
    if (nnz) *nnz = k;
  });
}

int sdr_gen_neumann(int64_t g, double shift, int64_t* nnz, int64_t* off, int64_t* col, double* val) {
  return guard([&] {  // gen_neumann (problems.hpp:38-61): mirrored neighbours, duplicates summed, zeros dropped
    if (g < 2) throw invalid("gen_neumann: grid_side must be at least 2");
    auto reflect = [g](int64_t i) { return i < 0 ? -i : (i >= g ? 2 * g - 2 - i : i); };
    int64_t k = 0;
    if (off) off[0] = 0;
    for (int64_t r = 0; r < g; ++r)
      for (int64_t c = 0; c < g; ++c) {
        const int64_t p = r * g + c;
        std::pair<int64_t, double> e[5] = {{p, 4.0 + shift},
                                           {reflect(r - 1) * g + c, -1.0},
                                           {reflect(r + 1) * g + c, -1.0},
                                           {r * g + reflect(c - 1), -1.0},
                                           {r * g + reflect(c + 1), -1.0}};
        std::stable_sort(e, e + 5, [](const auto& a, const auto& b) { return a.first < b.first; });
        for (int i = 0; i < 5;) {
          const int64_t cc = e[i].first;
          double v = 0.0;
          for (; i < 5 && e[i].first == cc; ++i) v += e[i].second;
          if (v == 0.0) continue;
          if (col) col[k] = cc;
          if (val) val[k] = v;
          ++k;
        }
        if (off) off[p + 1] = k;
      }
    if (nnz) *nnz = k;
  });
}

int sdr_gen_convdiff3d(int64_t n, double bx, double by, double bz, int64_t z0, int64_t z1, int64_t* nnz, int64_t* off,
                       int64_t* col, double* val) {
  return guard([&] {
    if (n < 1) throw invalid("gen_convdiff3d: n must be positive");
    if (z0 < 0 || z1 > n || z0 > z1) throw invalid("gen_convdiff3d: bad z-slab");
    const double h2 = static_cast<double>((n + 1) * (n + 1));
    const double cx = bx * static_cast<double>(n + 1) / 2.0, cy = by * static_cast<double>(n + 1) / 2.0,
                 cz = bz * static_cast<double>(n + 1) / 2.0;
    const int64_t n2 = n * n;
    int64_t k = 0;
    if (off) off[0] = 0;
    for (int64_t z = z0; z < z1; ++z)
      for (int64_t y = 0; y < n; ++y)
        for (int64_t x = 0; x < n; ++x) {
          const int64_t p = z * n2 + y * n + x;
          const bool has[7] = {z > 0, y > 0, x > 0, true, x + 1 < n, y + 1 < n, z + 1 < n};
          const int64_t cc[7] = {p - n2, p - n, p - 1, p, p + 1, p + n, p + n2};
          const double vv[7] = {-h2 - cz, -h2 - cy, -h2 - cx, 6.0 * h2, -h2 + cx, -h2 + cy, -h2 + cz};
          for (int e = 0; e < 7; ++e) {
            if (!has[e] || vv[e] == 0.0) continue;
            if (col) col[k] = cc[e];
            if (val) val[k] = vv[e];
            ++k;
          }
          if (off) off[p - z0 * n2 + 1] = k;
        }
    if (nnz) *nnz = k;
  });
}

// ------------------------------------------------------------------- solver
int sdr_config_default(sdr_config* cfg) {
  return guard([&] {
    need(cfg, "cfg");
    Config d;
    cfg->m = d.m;
    cfg->t = d.t;
    cfg->k = d.k;
    cfg->s = d.s;
    cfg->tol = d.tol;
    cfg->safety_init = d.safety_init;
    cfg->max_restarts = d.max_restarts;
    cfg->variant = d.variant;
    cfg->sketch_seed = d.sketch_seed;
    cfg->rank_tol = d.rank_tol;
    cfg->breakdown_tol = d.breakdown_tol;
  });
}

int sdr_config_validate(const sdr_config* cfg) {
  return guard([&] {
    need(cfg, "cfg");
    to_cfg(cfg).validate();
  });
}

int sdr_recycle_create(sdr_ctx* ctx, sdr_recycle** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    auto h = std::make_unique<sdr_recycle>();
    h->ctx = ctx->c.get();
    *out = h.release();
  });
}

int sdr_recycle_destroy(sdr_recycle* sp) {
  return guard([&] { delete sp; });
}

int sdr_recycle_info(const sdr_recycle* sp, int64_t* rows, int64_t* s, int64_t* dim, int* prov) {
  return guard([&] {
    need(sp, "space");
    if (rows) *rows = sp->sp.empty() ? 0 : sp->sp.nloc;
    if (s) *s = sp->sp.s;
    if (dim) *dim = sp->sp.dim();
    if (prov) *prov = sp->sp.provenance;
  });
}

int sdr_recycle_get(sdr_ctx* ctx, const sdr_recycle* sp, double* U, double* SU, double* SAU) {
  return guard([&] {
    need(ctx, "ctx");
    need(sp, "space");
    Context& c = *ctx->c;
    const Recycle& r = sp->sp;
    if (U && r.dim() > 0) {
      DeviceOut uo(U, r.nloc * r.dim());
      for (i64 q = 0; q < r.dim(); ++q) launch_scale_copy(c, r.uscale[static_cast<size_t>(q)], r.col(q), uo.ptr + q * r.nloc, r.nloc);
      uo.finish(c);
    }
    if (SU) std::memcpy(SU, r.SU.a.data(), sizeof(double) * static_cast<size_t>(r.s * r.dim()));
    if (SAU) std::memcpy(SAU, r.SAU.a.data(), sizeof(double) * static_cast<size_t>(r.s * r.dim()));
  });
}

int sdr_recycle_set(sdr_ctx* ctx, sdr_recycle* sp, int64_t rows, int64_t s, int64_t dim, const double* U,
                    const double* SU, const double* SAU, int provenance) {
  return guard([&] {
    need(ctx, "ctx");
    need(sp, "space");
    if (rows < 0 || s < 0 || dim < 0) throw invalid("sdr_recycle_set: negative dimensions");
    Context& c = *ctx->c;
    Recycle& r = sp->sp;
    r.clear();
    r.nloc = 0;
    r.cap = 0;
    r.ld = 0;
    r.s = s;
    i64 grows = rows;
    if (c.distributed()) {
      std::vector<i64> all(static_cast<size_t>(c.world));
      c.allgather_i64(&rows, 1, all.data());
      grows = 0;
      for (i64 v : all) grows += v;
    }
    r.n = grows;
    r.ensure(rows, std::max<i64>(dim, 1));
    if (dim > 0) {
      need(U, "U");
      need(SU, "SU");
      need(SAU, "SAU");
      DeviceIn uin(c, U, rows * dim);
      for (i64 q = 0; q < dim; ++q)
        SDR_CUDA(cudaMemcpyAsync(r.buf[r.cur].get() + q * r.ld, uin.ptr + q * rows, sizeof(double) * static_cast<size_t>(rows),
                                 cudaMemcpyDeviceToDevice, c.stream));
      c.sync();
    }
    r.slot.resize(static_cast<size_t>(dim));
    r.uscale.assign(static_cast<size_t>(dim), 1.0);
    for (i64 q = 0; q < dim; ++q) r.slot[static_cast<size_t>(q)] = static_cast<int>(q);
    r.SU = HMat(s, dim);
    r.SAU = HMat(s, dim);
    if (dim > 0) {
      std::memcpy(r.SU.a.data(), SU, sizeof(double) * static_cast<size_t>(s * dim));
      std::memcpy(r.SAU.a.data(), SAU, sizeof(double) * static_cast<size_t>(s * dim));
    }
    r.provenance = provenance;
  });
}

int sdr_recycle_drop_columns(sdr_recycle* sp, const int64_t* cols, int64_t ncols) {
  return guard([&] {
    need(sp, "space");
    std::vector<i64> v(cols, cols + ncols);
    sp->sp.drop_columns(v);
  });
}

int sdr_recycle_refresh(sdr_ctx* ctx, sdr_recycle* sp, const sdr_csr* A, const sdr_sketch* S, int mode, int64_t* counters3) {
  return guard([&] {
    need(ctx, "ctx");
    need(sp, "space");
    need(A, "A");
    need(S, "S");
    Counters cnt;
    refresh_recycle(*ctx->c, sp->sp, *A->op, *S->S, mode == 0, &cnt);
    if (counters3) {
      counters3[0] += cnt.matvecs;
      counters3[1] += cnt.inner_products;
      counters3[2] += cnt.sketch_applies;
    }
  });
}

int sdr_krylov_run(sdr_ctx* ctx, const sdr_csr* A, const sdr_sketch* S, const double* r0, int64_t t, int64_t m,
                   int64_t steps, double breakdown_tol, double* V, double* H, double* SV, double* SAV, int64_t* j_out,
                   int* breakdown, double* r0_norm, int64_t* counters3) {
  return guard([&] {
    need(ctx, "ctx");
    need(A, "A");
    need(S, "S");
    need(r0, "r0");
    Context& c = *ctx->c;
    DeviceIn rin(c, r0, A->op->local_rows);
    DeviceOut vo(V, A->op->local_rows * (m + 1));
    krylov_run(c, *A->op, *S->S, rin.ptr, t, m, steps, breakdown_tol, vo.ptr, H, SV, SAV, j_out, breakdown, r0_norm,
               counters3);
    vo.finish(c);
  });
}

int sdr_debug_block_product(sdr_ctx* ctx, int32_t kernel, int64_t n, const double* A1, int64_t lda1, int32_t k1,
                            const double* A2, int64_t lda2, int32_t k2, const double* B, int32_t nout, double* C,
                            int64_t ldc, double* norms2) {
  return guard([&] {  // recycle product U_new = [A1 A2] B + norms (test hook; host or device arrays)
    need(ctx, "ctx");
    Context& c = *ctx->c;
    const i64 K = k1 + k2;
    DeviceIn a1(c, A1, lda1 * std::max(k1 - 1, 0) + n), a2(c, A2, k2 > 0 ? lda2 * (k2 - 1) + n : 0), b(c, B, K * nout);
    DeviceOut co(C, ldc * (nout - 1) + n);
    DeviceBuffer<double> nr(std::max(nout, 1)), scratch(tsgemm_scratch_size(c.num_sms));
    if (kernel == 0)
      launch_tsgemm(c, a1.ptr, lda1, k1, a2.ptr ? a2.ptr : a1.ptr, lda2, k2, b.ptr, nout, co.ptr, ldc, n, nr.get(),
                    scratch.get());
    else
      launch_rgemm(c, a1.ptr, lda1, k1, a2.ptr ? a2.ptr : a1.ptr, lda2, k2, b.ptr, nout, co.ptr, ldc, n, nr.get(),
                   scratch.get());
    co.finish(c);
    SDR_CUDA(cudaMemcpy(norms2, nr.get(), sizeof(double) * static_cast<size_t>(nout), cudaMemcpyDeviceToHost));
  });
}

int sdr_debug_peer_emulate(int32_t world, int32_t n, int32_t epochs, const double* vals, double* out) {
  return guard([&] {
    need(vals, "vals");
    need(out, "out");
    peer_emulate(world, n, epochs, vals, out);
  });
}

int sdr_debug_time_step(sdr_ctx* ctx, const sdr_csr* A, const sdr_sketch* S, const double* r0, int64_t t, int64_t m,
                        int64_t steps, int32_t reps, double* k1_us, double* k2_us) {
  return guard([&] {
    need(ctx, "ctx");
    need(A, "A");
    need(S, "S");
    need(r0, "r0");
    need(k1_us, "k1_us");
    need(k2_us, "k2_us");
    Context& c = *ctx->c;
    DeviceIn rin(c, r0, A->op->local_rows);
    time_step_kernels(c, *A->op, *S->S, rin.ptr, t, m, steps, reps, k1_us, k2_us);
  });
}

int sdr_solve(sdr_ctx* ctx, const sdr_csr* A, const double* b, const double* x0, const sdr_config* cfg,
              sdr_recycle* space, const sdr_sketch* sketch, const sdr_callbacks* cb, double* x_out,
              sdr_report** report_out) {
  return guard([&] {
    need(ctx, "ctx");
    need(A, "A");
    need(b, "b");
    need(cfg, "cfg");
    Context& c = *ctx->c;
    const auto& op = *A->op;
    const i64 n = op.local_rows;
    auto rep = std::make_unique<sdr_report>();
    Recycle tmp_space;
    Recycle& sp = space ? space->sp : tmp_space;
    Callbacks cbs;
    if (cb) {
      cbs.on_iteration = reinterpret_cast<void (*)(const void*, void*)>(cb->on_iteration);
      cbs.on_residual = reinterpret_cast<void (*)(const void*, void*)>(cb->on_residual_check);
      cbs.user = cb->user;
    }
    DeviceIn bin(c, b, n);
    DeviceIn x0in(c, x0, n);
    const bool nz = x0 && host_nonzero(c, x0, n);
    DeviceOut xo(x_out, n, true);  // solve() writes x_out by cudaMemcpyAsync only
    solve(c, op, bin.ptr, x0in.ptr, nz, to_cfg(cfg), sp, sketch ? sketch->S.get() : nullptr, cb ? &cbs : nullptr, xo.ptr,
          rep->r);
    xo.finish(c);
    if (report_out) *report_out = rep.release();
  });
}

int sdr_mm_read_file(const char* path, sdr_host_csr** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    auto h = std::make_unique<sdr_host_csr>();
    h->h = mm_read_file(path);
    *out = h.release();
  });
}

int sdr_mm_read_string(const char* text, int64_t len, sdr_host_csr** out) {
  return guard([&] {
    need(text, "text");
    need(out, "out");
    std::istringstream in(std::string(text, static_cast<size_t>(len)));
    auto h = std::make_unique<sdr_host_csr>();
    h->h = mm_read(in);
    *out = h.release();
  });
}

int sdr_host_csr_info(const sdr_host_csr* h, int64_t* rows, int64_t* cols, int64_t* nnz) {
  return guard([&] {
    need(h, "csr");
    if (rows) *rows = h->h.rows;
    if (cols) *cols = h->h.cols;
    if (nnz) *nnz = static_cast<int64_t>(h->h.values.size());
  });
}

int sdr_host_csr_arrays(const sdr_host_csr* h, const int64_t** offsets, const int64_t** columns,
                        const double** values) {
  return guard([&] {
    need(h, "csr");
    if (offsets) *offsets = h->h.offsets.data();
    if (columns) *columns = h->h.columns.data();
    if (values) *values = h->h.values.data();
  });
}

int sdr_host_csr_destroy(sdr_host_csr* h) {
  delete h;
  return SDR_OK;
}

int sdr_mm_write_file(const char* path, int64_t rows, int64_t cols, const int64_t* offsets, const int64_t* columns,
                      const double* values) {
  return guard([&] {
    need(path, "path");
    need(offsets, "offsets");
    mm_write_file(path, rows, cols, offsets, columns, values);
  });
}

int sdr_mm_write_string(int64_t rows, int64_t cols, const int64_t* offsets, const int64_t* columns,
                        const double* values, char* buf, int64_t* len) {
  return guard([&] {
    need(offsets, "offsets");
    need(len, "len");
    std::ostringstream out;
    mm_write(out, rows, cols, offsets, columns, values);
    const std::string t = out.str();
    if (buf) {
      if (*len < static_cast<int64_t>(t.size() + 1)) throw invalid("sdr_mm_write_string: buffer too small");
      std::memcpy(buf, t.c_str(), t.size() + 1);
    }
    *len = static_cast<int64_t>(t.size() + 1);
  });
}

int sdr_csr_read_matrix_market(sdr_ctx* ctx, const char* path, sdr_csr** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(path, "path");
    need(out, "out");
    if (ctx->c->distributed()) throw invalid("sdr_csr_read_matrix_market: use sdr_csr_create_local in a distributed context");
    const HostCsr m = mm_read_file(path);
    auto h = std::make_unique<sdr_csr>();
    h->ctx = ctx->c.get();
    h->op.reset(create_operator_csr(*ctx->c, m.rows, m.cols, 0, m.rows, m.offsets.data(), m.columns.data(),
                                    m.values.data()));
    *out = h.release();
  });
}

int sdr_space_file_read(const char* path, sdr_space_file** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    auto f = std::make_unique<sdr_space_file>();
    f->f = space_read_file(path);
    *out = f.release();
  });
}

int sdr_space_file_read_bytes(const void* data, int64_t len, sdr_space_file** out) {
  return guard([&] {
    need(data, "data");
    need(out, "out");
    std::istringstream in(std::string(static_cast<const char*>(data), static_cast<size_t>(len)), std::ios::binary);
    auto f = std::make_unique<sdr_space_file>();
    f->f = space_read(in);
    *out = f.release();
  });
}

int sdr_space_file_info(const sdr_space_file* f, int64_t* n, int64_t* s, int64_t* k, int* provenance) {
  return guard([&] {
    need(f, "file");
    if (n) *n = f->f.n;
    if (s) *s = f->f.s;
    if (k) *k = f->f.k;
    if (provenance) *provenance = static_cast<int>(f->f.provenance);
  });
}

int sdr_space_file_arrays(const sdr_space_file* f, const double** U, const double** SU, const double** SAU) {
  return guard([&] {
    need(f, "file");
    if (U) *U = f->f.U.data();
    if (SU) *SU = f->f.SU.data();
    if (SAU) *SAU = f->f.SAU.data();
  });
}

int sdr_space_file_destroy(sdr_space_file* f) {
  delete f;
  return SDR_OK;
}

namespace {
SpaceFile space_from(int64_t n, int64_t s, int64_t k, int provenance, const double* U, const double* SU,
                     const double* SAU) {
  if (n < 0 || s < 0 || k < 0 || provenance < 0 || provenance > 4)
    throw invalid("recycle-space save: invalid dimensions or provenance");
  if (k > 0) {
    need(U, "U");
    need(SU, "SU");
    need(SAU, "SAU");
  }
  SpaceFile f;
  f.n = n, f.s = s, f.k = k, f.provenance = provenance;
  f.U.assign(U, U + n * k);
  f.SU.assign(SU, SU + s * k);
  f.SAU.assign(SAU, SAU + s * k);
  return f;
}
}  // namespace

int sdr_space_file_write(const char* path, int64_t n, int64_t s, int64_t k, int provenance, const double* U,
                         const double* SU, const double* SAU) {
  return guard([&] {
    need(path, "path");
    space_write_file(path, space_from(n, s, k, provenance, U, SU, SAU));
  });
}

int sdr_space_file_write_bytes(int64_t n, int64_t s, int64_t k, int provenance, const double* U, const double* SU,
                               const double* SAU, void* buf, int64_t* len) {
  return guard([&] {
    need(len, "len");
    const int64_t bytes = 40 + 8 * (n * k + 2 * s * k);
    if (buf) {
      if (*len < bytes) throw invalid("sdr_space_file_write_bytes: buffer too small");
      std::ostringstream out(std::ios::binary);
      space_write(out, space_from(n, s, k, provenance, U, SU, SAU));
      const std::string t = out.str();
      std::memcpy(buf, t.data(), t.size());
    }
    *len = bytes;
  });
}

int sdr_recycle_save_file(sdr_ctx* ctx, const sdr_recycle* sp, const char* path) {
  return guard([&] {  // save_recycle_space_file (recycle.hpp:380-384)
    need(ctx, "ctx");
    need(sp, "space");
    need(path, "path");
    Context& c = *ctx->c;
    const Recycle& r = sp->sp;
    SpaceFile f;
    f.n = r.dim() > 0 ? r.nloc : 0;
    f.s = r.SU.rows;
    f.k = r.dim();
    f.provenance = r.provenance;
    f.U.resize(static_cast<size_t>(f.n * f.k));
    if (f.k > 0) {
      DeviceBuffer<double> u(f.n * f.k);
      for (i64 q = 0; q < f.k; ++q) launch_scale_copy(c, r.uscale[static_cast<size_t>(q)], r.col(q), u.get() + q * f.n, f.n);
      SDR_CUDA(cudaMemcpyAsync(f.U.data(), u.get(), sizeof(double) * f.U.size(), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
    }
    f.SU.assign(r.SU.a.begin(), r.SU.a.begin() + f.s * f.k);
    f.SAU.assign(r.SAU.a.begin(), r.SAU.a.begin() + f.s * f.k);
    space_write_file(path, f);
  });
}

int sdr_recycle_load_file(sdr_ctx* ctx, sdr_recycle* sp, const char* path) {
  return guard([&] {  // load_recycle_space_file (recycle.hpp:386-390)
    need(ctx, "ctx");
    need(sp, "space");
    need(path, "path");
    const SpaceFile f = space_read_file(path);
    const int rc = sdr_recycle_set(ctx, sp, f.n, f.s, f.k, f.U.data(), f.SU.data(), f.SAU.data(),
                                   static_cast<int>(f.provenance));
    if (rc != SDR_OK) throw Error(rc, g_err);
  });
}

int sdr_baseline_config_default(sdr_baseline_config* cfg) {
  return guard([&] {
    need(cfg, "cfg");
    BaselineConfig d;
    cfg->m = d.m;
    cfg->tol = d.tol;
    cfg->max_restarts = d.max_restarts;
    cfg->breakdown_tol = d.breakdown_tol;
  });
}

int sdr_baseline_gmres(sdr_ctx* ctx, const sdr_csr* A, const double* b, const double* x0,
                       const sdr_baseline_config* cfg, double* x_out, sdr_report** report_out) {
  return guard([&] {  // baseline.hpp:51-216
    need(ctx, "ctx");
    need(A, "A");
    need(b, "b");
    need(cfg, "cfg");
    Context& c = *ctx->c;
    const auto& op = *A->op;
    const i64 n = op.local_rows;
    BaselineConfig bc;
    bc.m = cfg->m;
    bc.tol = cfg->tol;
    bc.max_restarts = cfg->max_restarts;
    bc.breakdown_tol = cfg->breakdown_tol;
    bc.validate();
    auto rep = std::make_unique<sdr_report>();
    DeviceIn bin(c, b, n);
    DeviceIn x0in(c, x0, n);
    const bool nz = x0 && host_nonzero(c, x0, n);
    DeviceOut xo(x_out, n);
    baseline_solve(c, op, bin.ptr, x0in.ptr, nz, bc, xo.ptr, rep->r);
    xo.finish(c);
    if (report_out) *report_out = rep.release();
  });
}

int sdr_solve_sequence(sdr_ctx* ctx, int32_t nprob, const sdr_csr* const* mats, const double* const* rhs,
                       const double* const* x0s, const double* tols, int32_t shared_matrix, const sdr_config* cfg,
                       const sdr_sketch* sketch, sdr_recycle* space, double* const* x_outs, sdr_report** reports_out) {
  return guard([&] {  // solver.hpp:385-459
    need(ctx, "ctx");
    need(cfg, "cfg");
    Context& c = *ctx->c;
    Config base = to_cfg(cfg);
    base.validate();
    if (nprob <= 0) return;
    need(mats, "mats");
    need(rhs, "rhs");
    need(reports_out, "reports_out");
    if (!mats[0]) throw invalid("solve_sequence: problem 0 has no matrix");
    const i64 n = mats[0]->op->rows;
    std::unique_ptr<SketchDev> own;
    const SketchDev* S = sketch ? sketch->S.get() : nullptr;
    if (!S) {
      own.reset(create_sketch(c, kSrdct, n, base.s, base.sketch_seed, 0));
      S = own.get();
    }
    Recycle tmp_space;
    Recycle& sp = space ? space->sp : tmp_space;
    const DeviceOperator* prev = nullptr;
    for (int32_t i = 0; i < nprob; ++i) {
      auto rep = std::make_unique<sdr_report>();
      Config local = base;
      if (tols && tols[i] > 0.0) local.tol = tols[i];
      Counters pre;
      try {
        if (!mats[i]) throw invalid("solve_sequence: problem " + std::to_string(i) + " has no matrix");
        const DeviceOperator& op = *mats[i]->op;
        if (op.rows != n || op.cols != n)
          throw invalid("solve_sequence: problem " + std::to_string(i) + " is " + std::to_string(op.rows) + " x " +
                        std::to_string(op.cols) + " but the sequence runs at size " + std::to_string(n));
        const bool changed = prev != nullptr && prev != &op && !shared_matrix;
        std::string note;
        if (changed && !sp.empty()) {
          if (local.variant == 1) {
            refresh_recycle(c, sp, op, *S, true, &pre);
          } else {
            refresh_recycle(c, sp, op, *S, false, &pre);
            if (local.variant == 0) note = "matrix changed under variant=reuse; sketched image carried unrefreshed";
          }
        } else if (prev != nullptr && !sp.empty()) {
          sp.provenance = 2;
        }
        need(rhs[i], "rhs");
        const i64 nl = op.local_rows;
        DeviceIn bin(c, rhs[i], nl);
        const double* x0 = x0s ? x0s[i] : nullptr;
        DeviceIn x0in(c, x0, nl);
        const bool nz = x0 && host_nonzero(c, x0, nl);
        DeviceOut xo(x_outs ? x_outs[i] : nullptr, nl);
        solve(c, op, bin.ptr, x0in.ptr, nz, local, sp, S, nullptr, xo.ptr, rep->r);
        xo.finish(c);
        rep->r.counters += pre;
        if (!note.empty()) rep->r.notes.push_back(note);
      } catch (const Error& e) {
        if (e.code == SDR_ECUDA || e.code == SDR_ENCCL || e.code == SDR_ENOMEM) throw;
        rep = std::make_unique<sdr_report>();
        rep->r.error = e.what();
        rep->r.counters = pre;
        rep->r.notes.push_back("system " + std::to_string(i) + " aborted: " + e.what());
      }
      reports_out[i] = rep.release();
      prev = mats[i] ? mats[i]->op.get() : nullptr;
    }
  });
}

int sdr_report_destroy(sdr_report* r) {
  return guard([&] { delete r; });
}

int sdr_report_summary(const sdr_report* r, int* status, int64_t* it, int32_t* cycles, double* rhs, double* frr,
                       double* seconds) {
  return guard([&] {
    need(r, "report");
    if (status) *status = r->r.status;
    if (it) *it = r->r.iterations;
    if (cycles) *cycles = r->r.cycles;
    if (rhs) *rhs = r->r.rhs_norm;
    if (frr) *frr = r->r.final_relative_residual;
    if (seconds) *seconds = r->r.seconds;
  });
}

int sdr_report_counters(const sdr_report* r, int64_t* mv, int64_t* ip, int64_t* sk) {
  return guard([&] {
    need(r, "report");
    if (mv) *mv = r->r.counters.matvecs;
    if (ip) *ip = r->r.counters.inner_products;
    if (sk) *sk = r->r.counters.sketch_applies;
  });
}

int sdr_report_samples(const sdr_report* r, int which, int64_t* n, int64_t* it, double* val) {
  return guard([&] {
    need(r, "report");
    const auto& v = which == 0 ? r->r.sketched : r->r.truth;
    if (n) *n = static_cast<int64_t>(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
      if (it) it[i] = v[i].first;
      if (val) val[i] = v[i].second;
    }
  });
}

int sdr_report_cycles(const sdr_report* r, int64_t* n, double* st) {
  return guard([&] {
    need(r, "report");
    if (n) *n = static_cast<int64_t>(r->r.cycle_stats.size());
    if (st)
      for (size_t i = 0; i < r->r.cycle_stats.size(); ++i) {
        const auto& c = r->r.cycle_stats[i];
        double* o = st + 8 * i;
        o[0] = static_cast<double>(c.steps);
        o[1] = c.entry_residual;
        o[2] = c.sketched_entry;
        o[3] = c.exit_sres;
        o[4] = c.exit_residual;
        o[5] = c.safety_after;
        o[6] = c.basis_cond;
        o[7] = static_cast<double>(c.deflation_rank);
      }
  });
}

int sdr_report_notes(const sdr_report* r, int64_t* n) {
  return guard([&] {
    need(r, "report");
    need(n, "n");
    *n = static_cast<int64_t>(r->r.notes.size());
  });
}

const char* sdr_report_note(const sdr_report* r, int64_t i) {
  if (!r || i < 0 || i >= static_cast<int64_t>(r->r.notes.size())) return nullptr;
  return r->r.notes[static_cast<size_t>(i)].c_str();
}

const char* sdr_report_error(const sdr_report* r) { return r ? r->r.error.c_str() : nullptr; }

/* internal diagnostics (not part of the public header): ||x||^2 through the
   copy_norm kernel and sum of y = A x through the plain SpMV. */
SDR_API int sdr_debug_norm2(sdr_ctx* ctx, const double* x, int64_t n, double* out) {
  return guard([&] {
    Context& c = *ctx->c;
    DeviceIn xin(c, x, n);
    DeviceBuffer<double> dst(std::max<int64_t>(n, 1)), nrm(1);
    launch_copy_norm(c, xin.ptr, dst.get(), n, nrm.get());
    SDR_CUDA(cudaMemcpyAsync(out, nrm.get(), sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  });
}

/* internal: kernel phase trace (SDR_TRACE=1); copies min(cap, size) entries, *n = size */
SDR_API int sdr_debug_trace(sdr_ctx* ctx, uint64_t* out, int64_t cap, int64_t* n) {
  return guard([&] {
    const auto v = ctx->c->trace_read();
    if (n) *n = static_cast<int64_t>(v.size());
    for (int64_t i = 0; i < std::min<int64_t>(cap, static_cast<int64_t>(v.size())); ++i) out[i] = v[static_cast<size_t>(i)];
  });
}

/* internal: writes the timed-launch timeline (name,start_us,end_us) as CSV */
SDR_API int sdr_debug_timeline(sdr_ctx* ctx, const char* path) {
  return guard([&] {
    Context& c = *ctx->c;
    c.timing_flush();
    FILE* f = std::fopen(path, "w");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    std::fprintf(f, "name,start_us,end_us\n");
    for (const auto& sp : c.timeline) std::fprintf(f, "%s,%.3f,%.3f\n", sp.name.c_str(), sp.start_us, sp.end_us);
    std::fclose(f);
  });
}

/* internal: device-clock launch timeline (SDR_TRACE=2) as CSV name,start_ns,end_ns */
SDR_API int sdr_ctx_set_stamps(sdr_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->stamps_on = on != 0;
  });
}

SDR_API int sdr_debug_stamps(sdr_ctx* ctx, const char* path) {
  return guard([&] {
    const auto v = ctx->c->launch_stamps_read();
    FILE* f = std::fopen(path, "w");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    std::fprintf(f, "name,start_ns,end_ns\n");
    for (const auto& e : v) std::fprintf(f, "%s,%llu,%llu\n", e.first.c_str(), e.second.first, e.second.second);
    std::fclose(f);
  });
}

int sdr_report_phase(const sdr_report* r, const char* name, double* ms) {
  return guard([&] {
    need(r, "report");
    need(name, "name");
    need(ms, "ms");
    auto it = r->r.phase_ms.find(name);
    *ms = it == r->r.phase_ms.end() ? 0.0 : it->second;
  });
}

int sdr_report_timing(const sdr_report* r, double* device_ms, double* host_wait_ms, double* total_ms) {
  return guard([&] {
    need(r, "report");
    if (device_ms) *device_ms = r->r.device_ms;
    if (host_wait_ms) *host_wait_ms = r->r.host_wait_ms;
    if (total_ms) *total_ms = r->r.seconds * 1e3;
  });
}

}  // extern "C"
