// Operator construction: CSR validation (sparse.hpp:117-143) and SELL-32
// packing, the device-side 3D convection–diffusion generator, and the 1-D
// row-partition halo plan.
#include "operator.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <memory>

namespace sdr {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SDR_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

/// SDR_DIA=0 forces plain SELL storage (A/B and parity checks).
bool zsell_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SDR_ZSELL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

/// Complex structure of a one-rank real operator: every 2x2 block (rows
/// 2p, 2p+1; columns 2q, 2q+1) is [[a, -b], [b, a]] (missing entries = 0),
/// i.e. the operator is a complex matrix acting on interleaved (re, im)
/// vectors. On success ccol / cval / coff hold its complex CSR (value pairs).
bool complex_structure(int64_t rows, const int64_t* off, const int64_t* col, const double* val,
                       std::vector<int64_t>& coff, std::vector<int64_t>& ccol, std::vector<double>& cval) {
  if (rows % 2) return false;
  const int64_t nc = rows / 2;
  coff.assign(static_cast<size_t>(nc) + 1, 0);
  ccol.clear();
  cval.clear();
  for (int64_t pr = 0; pr < nc; ++pr) {
    int64_t i0 = off[2 * pr], i1 = off[2 * pr + 1];          // row 2p (real part)
    int64_t k0 = off[2 * pr + 1], k1 = off[2 * pr + 2];      // row 2p + 1 (imaginary part)
    while (i0 < i1 || k0 < k1) {
      const int64_t q = std::min(i0 < i1 ? col[i0] / 2 : std::numeric_limits<int64_t>::max(), k0 < k1 ? col[k0] / 2 : std::numeric_limits<int64_t>::max());
      double a = 0, mb = 0, b = 0, a2 = 0;
      if (i0 < i1 && col[i0] == 2 * q) a = val[i0++];
      if (i0 < i1 && col[i0] == 2 * q + 1) mb = val[i0++];
      if (k0 < k1 && col[k0] == 2 * q) b = val[k0++];
      if (k0 < k1 && col[k0] == 2 * q + 1) a2 = val[k0++];
      if (a != a2 || mb != -b) return false;
      ccol.push_back(q);
      cval.push_back(a);
      cval.push_back(b);
    }
    coff[static_cast<size_t>(pr) + 1] = static_cast<int64_t>(ccol.size());
  }
  return true;
}

bool dia_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SDR_DIA");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

void partition_halo(int world, int rank, const int64_t* rb, const int64_t* re, const int64_t* mnc, const int64_t* mxc,
                    int64_t* recv_lo, int64_t* recv_cnt, int64_t* send_lo, int64_t* send_cnt) {
  auto halo_of = [&](int p, int64_t* lo0, int64_t* lo1, int64_t* hi0, int64_t* hi1) {
    *lo0 = std::min(mnc[p], rb[p]);
    *lo1 = rb[p];
    *hi0 = re[p];
    *hi1 = std::max(mxc[p] + 1, re[p]);
  };
  auto inter = [](int64_t a0, int64_t a1, int64_t b0, int64_t b1, int64_t* lo, int64_t* cnt) {
    const int64_t l = std::max(a0, b0), h = std::min(a1, b1);
    if (h > l) {
      *lo = l;
      *cnt = h - l;
      return true;
    }
    return false;
  };
  for (int q = 0; q < world; ++q) {
    recv_lo[q] = recv_cnt[q] = send_lo[q] = send_cnt[q] = 0;
    if (q == rank) continue;
    int64_t l0, l1, h0, h1, lo, cnt;
    halo_of(rank, &l0, &l1, &h0, &h1);
    int hits = 0;
    if (inter(l0, l1, rb[q], re[q], &lo, &cnt)) recv_lo[q] = lo, recv_cnt[q] = cnt, ++hits;
    if (inter(h0, h1, rb[q], re[q], &lo, &cnt)) recv_lo[q] = lo, recv_cnt[q] = cnt, ++hits;
    if (hits > 1) throw invalid("partition: rank " + std::to_string(q) + " overlaps both halos of rank " + std::to_string(rank));
    halo_of(q, &l0, &l1, &h0, &h1);
    hits = 0;
    if (inter(l0, l1, rb[rank], re[rank], &lo, &cnt)) send_lo[q] = lo, send_cnt[q] = cnt, ++hits;
    if (inter(h0, h1, rb[rank], re[rank], &lo, &cnt)) send_lo[q] = lo, send_cnt[q] = cnt, ++hits;
    if (hits > 1) throw invalid("partition: rank " + std::to_string(rank) + " overlaps both halos of rank " + std::to_string(q));
  }
}

void finish_partition(Context& c, DeviceOperator& op, int64_t min_col, int64_t max_col) {
  const int64_t row_end = op.row_begin + op.local_rows;
  if (op.local_rows == 0 || max_col < min_col) min_col = op.row_begin, max_col = op.row_begin - 1;
  op.ext_begin = std::min(min_col, op.row_begin);
  op.halo_lo = op.row_begin - op.ext_begin;
  op.halo_hi = std::max(max_col + 1, row_end) - row_end;
  const int W = c.world;
  op.plan.recv_lo.assign(W, 0);
  op.plan.recv_cnt.assign(W, 0);
  op.plan.send_lo.assign(W, 0);
  op.plan.send_cnt.assign(W, 0);
  if (W <= 1) {
    if (op.halo_lo || op.halo_hi) throw invalid("SparseMatrix: column index out of range");
    return;
  }
  const int64_t mine[4] = {op.row_begin, row_end, min_col, max_col};
  std::vector<int64_t> all(4 * static_cast<size_t>(W));
  c.allgather_i64(mine, 4, all.data());
  std::vector<int64_t> rb(W), re(W), mn(W), mx(W);
  for (int q = 0; q < W; ++q) rb[q] = all[4 * q], re[q] = all[4 * q + 1], mn[q] = all[4 * q + 2], mx[q] = all[4 * q + 3];
  partition_halo(W, c.rank, rb.data(), re.data(), mn.data(), mx.data(), op.plan.recv_lo.data(), op.plan.recv_cnt.data(),
                 op.plan.send_lo.data(), op.plan.send_cnt.data());
  int64_t covered = 0;
  for (int q = 0; q < W; ++q) covered += op.plan.recv_cnt[q];
  if (covered != op.halo_lo + op.halo_hi)
    throw invalid("partition: halo rows of rank " + std::to_string(c.rank) + " are not owned by any rank");
}

DeviceOperator* create_operator_csr(Context& c, int64_t rows, int64_t cols, int64_t row_begin, int64_t local_rows,
                                    const int64_t* off, const int64_t* col, const double* val) {
  if (rows < 0 || cols < 0 || local_rows < 0) throw invalid("SparseMatrix: negative dimensions");
  if (row_begin < 0 || row_begin + local_rows > rows) throw invalid("SparseMatrix: row block outside the matrix");
  if (!off) throw invalid("SparseMatrix: offsets size 0 does not match rows + 1 = " + std::to_string(local_rows + 1));
  if (off[0] != 0) throw invalid("SparseMatrix: offsets must start at 0");
  const int64_t nnz = off[local_rows];
  if (nnz > 0 && (!col || !val)) throw invalid("SparseMatrix: offsets/columns/values sizes inconsistent");
  int64_t mnc = std::numeric_limits<int64_t>::max(), mxc = std::numeric_limits<int64_t>::min();
  int64_t reach_lo_end = 0, reach_hi_begin = local_rows;  // see DeviceOperator::reach_lo_end
  const int64_t row_end = row_begin + local_rows;
  for (int64_t r = 0; r < local_rows; ++r) {
    if (off[r + 1] < off[r]) throw invalid("SparseMatrix: offsets decrease at row " + std::to_string(row_begin + r));
    for (int64_t p = off[r]; p < off[r + 1]; ++p) {
      const int64_t cc = col[p];
      if (cc < 0 || cc >= cols)
        throw invalid("SparseMatrix: column index " + std::to_string(cc) + " out of range in row " +
                      std::to_string(row_begin + r));
      if (p > off[r] && col[p - 1] >= cc)
        throw invalid("SparseMatrix: column indices not strictly increasing in row " + std::to_string(row_begin + r));
      if (!std::isfinite(val[p])) throw invalid("SparseMatrix: non-finite value in row " + std::to_string(row_begin + r));
      mnc = std::min(mnc, cc);
      mxc = std::max(mxc, cc);
      if (cc < row_begin) reach_lo_end = r + 1;
      if (cc >= row_end && reach_hi_begin == local_rows) reach_hi_begin = r;
    }
  }
  auto op = std::make_unique<DeviceOperator>();
  op->rows = rows;
  op->cols = cols;
  op->row_begin = row_begin;
  op->local_rows = local_rows;
  op->nnz = nnz;
  op->reach_lo_end = reach_lo_end;
  op->reach_hi_begin = reach_hi_begin;
  if (!c.distributed() && rows != cols) {
    // rectangular operators are accepted (apply checks dims); ext covers all columns
  }
  if (!c.distributed()) {
    op->ext_begin = 0;
    op->halo_lo = 0;
    op->halo_hi = std::max<int64_t>(0, cols - local_rows);
    op->plan.recv_lo.assign(1, 0);
    op->plan.recv_cnt.assign(1, 0);
    op->plan.send_lo.assign(1, 0);
    op->plan.send_cnt.assign(1, 0);
  } else {
    finish_partition(c, *op, mnc, mxc);
  }
  const int64_t ext_len = op->halo_lo + local_rows + op->halo_hi;
  if (ext_len > std::numeric_limits<int32_t>::max())
    throw invalid("SparseMatrix: local extended block of " + std::to_string(ext_len) + " rows exceeds int32 indexing");
  // ZSELL: a complex matrix in real-equivalent form (interleaved vectors)
  // is stored as complex entries — 20 bytes per complex entry instead of four
  // 12-byte real entries (BASELINE C4)
  {
    std::vector<int64_t> coff, ccol;
    std::vector<double> cval;
    if (!c.distributed() && zsell_enabled() && rows == cols && local_rows > 0 &&
        complex_structure(local_rows, off, col, val, coff, ccol, cval)) {
      const int64_t nc = local_rows / 2, ns = (nc + kSlice - 1) / kSlice;
      std::vector<int64_t> zsp(static_cast<size_t>(ns) + 1, 0);
      for (int64_t sl = 0; sl < ns; ++sl) {
        int64_t mx = 0;
        for (int64_t r = sl * kSlice; r < std::min(nc, (sl + 1) * kSlice); ++r)
          mx = std::max(mx, coff[static_cast<size_t>(r) + 1] - coff[static_cast<size_t>(r)]);
        zsp[static_cast<size_t>(sl) + 1] = zsp[static_cast<size_t>(sl)] + mx * kSlice;
      }
      const int64_t total = zsp[static_cast<size_t>(ns)];
      std::vector<int32_t> hc(static_cast<size_t>(total));
      std::vector<double> hv(static_cast<size_t>(2 * total), 0.0);
      for (int64_t sl = 0; sl < ns; ++sl) {
        const int64_t len = (zsp[static_cast<size_t>(sl) + 1] - zsp[static_cast<size_t>(sl)]) / kSlice;
        for (int lane = 0; lane < kSlice; ++lane) {
          const int64_t r = sl * kSlice + lane;
          const int64_t self = std::min(r, nc - 1);
          for (int64_t k = 0; k < len; ++k) {
            const size_t dst = static_cast<size_t>(zsp[static_cast<size_t>(sl)] + k * kSlice + lane);
            const int64_t n_r = r < nc ? coff[static_cast<size_t>(r) + 1] - coff[static_cast<size_t>(r)] : 0;
            if (k < n_r) {
              const size_t src = static_cast<size_t>(coff[static_cast<size_t>(r)] + k);
              hc[dst] = static_cast<int32_t>(ccol[src]);
              hv[2 * dst] = cval[2 * src];
              hv[2 * dst + 1] = cval[2 * src + 1];
            } else {
              hc[dst] = static_cast<int32_t>(self);  // padding: zero value, own column
            }
          }
        }
      }
      op->cplx = true;
      op->stored = total;
      op->slice_ptr.resize(ns + 1);
      op->cols_idx.resize(std::max<int64_t>(total, 1));
      op->vals.resize(std::max<int64_t>(2 * total, 2));
      SDR_CUDA(cudaMemcpyAsync(op->slice_ptr.get(), zsp.data(), sizeof(int64_t) * zsp.size(), cudaMemcpyHostToDevice,
                               c.stream));
      if (total) {
        SDR_CUDA(cudaMemcpyAsync(op->cols_idx.get(), hc.data(), sizeof(int32_t) * hc.size(), cudaMemcpyHostToDevice,
                                 c.stream));
        SDR_CUDA(cudaMemcpyAsync(op->vals.get(), hv.data(), sizeof(double) * hv.size(), cudaMemcpyHostToDevice, c.stream));
      }
      c.sync();
      return op.release();
    }
  }
  const int64_t nslices = (local_rows + kSlice - 1) / kSlice;
  std::vector<int64_t> sp(static_cast<size_t>(nslices) + 1, 0);
  // SELL-DIA when every slice's entries lie on at most kMaxDiag diagonals
  // (offset = column - row); gaps become explicit zeros.
  constexpr size_t kMaxDiag = 16;
  std::vector<std::vector<int64_t>> diag(static_cast<size_t>(nslices));
  bool use_dia = local_rows > 0 && dia_enabled();
  for (int64_t s = 0; s < nslices && use_dia; ++s) {
    auto& d = diag[static_cast<size_t>(s)];
    for (int64_t r = s * kSlice; r < std::min(local_rows, (s + 1) * kSlice) && use_dia; ++r)
      for (int64_t p = off[r]; p < off[r + 1]; ++p) {
        const int64_t o = col[p] - (row_begin + r);
        if (std::find(d.begin(), d.end(), o) == d.end()) {
          d.push_back(o);
          if (d.size() > kMaxDiag) {
            use_dia = false;
            break;
          }
        }
      }
    std::sort(d.begin(), d.end());
  }
  size_t D = 0;
  int64_t used = 0;
  for (const auto& d : diag) {
    D = std::max(D, d.size());
    used += static_cast<int64_t>(d.size());
  }
  // uniform D per slice (no slice_ptr indirection); padding is offset 0 /
  // value 0 and must stay below 1/8 of the stored diagonals
  if (use_dia && static_cast<int64_t>(D) * nslices * 8 > used * 9) use_dia = false;
  if (use_dia) {
    const int64_t total = static_cast<int64_t>(D) * nslices * kSlice;
    for (int64_t s = 0; s <= nslices; ++s) sp[static_cast<size_t>(s)] = s * static_cast<int64_t>(D) * kSlice;
    std::vector<int32_t> hd(static_cast<size_t>(total / kSlice), 0);
    std::vector<double> hv(static_cast<size_t>(total), 0.0);
    for (int64_t s = 0; s < nslices; ++s) {
      const auto& d = diag[static_cast<size_t>(s)];
      const int64_t base = sp[static_cast<size_t>(s)];
      for (size_t k = 0; k < d.size(); ++k) hd[static_cast<size_t>(base / kSlice) + k] = static_cast<int32_t>(d[k]);
      for (int64_t r = s * kSlice; r < std::min(local_rows, (s + 1) * kSlice); ++r)
        for (int64_t p = off[r]; p < off[r + 1]; ++p) {
          const int64_t k = std::lower_bound(d.begin(), d.end(), col[p] - (row_begin + r)) - d.begin();
          hv[static_cast<size_t>(base + k * kSlice + (r - s * kSlice))] = val[p];
        }
    }
    op->dia = true;
    op->dia_d = static_cast<int>(D);
    op->stored = total;
    op->slice_ptr.resize(nslices + 1);
    op->doff.resize(std::max<int64_t>(total / kSlice, 1));
    op->vals.resize(std::max<int64_t>(total, 1));
    SDR_CUDA(cudaMemcpyAsync(op->slice_ptr.get(), sp.data(), sizeof(int64_t) * sp.size(), cudaMemcpyHostToDevice, c.stream));
    if (total) {
      SDR_CUDA(cudaMemcpyAsync(op->doff.get(), hd.data(), sizeof(int32_t) * hd.size(), cudaMemcpyHostToDevice, c.stream));
      SDR_CUDA(cudaMemcpyAsync(op->vals.get(), hv.data(), sizeof(double) * hv.size(), cudaMemcpyHostToDevice, c.stream));
    }
    c.sync();
    return op.release();
  }
  // SELL-32 packing
  for (int64_t s = 0; s < nslices; ++s) {
    int64_t mx = 0;
    for (int64_t r = s * kSlice; r < std::min(local_rows, (s + 1) * kSlice); ++r) mx = std::max(mx, off[r + 1] - off[r]);
    sp[static_cast<size_t>(s) + 1] = sp[static_cast<size_t>(s)] + mx * kSlice;
  }
  const int64_t total = sp[static_cast<size_t>(nslices)];
  op->stored = total;
  std::vector<int32_t> hc(static_cast<size_t>(total));
  std::vector<double> hv(static_cast<size_t>(total));
  for (int64_t s = 0; s < nslices; ++s) {
    const int64_t len = (sp[static_cast<size_t>(s) + 1] - sp[static_cast<size_t>(s)]) / kSlice;
    for (int lane = 0; lane < kSlice; ++lane) {
      const int64_t r = s * kSlice + lane;
      const int64_t self = op->halo_lo + std::min(r, std::max<int64_t>(local_rows - 1, 0));
      for (int64_t k = 0; k < len; ++k) {
        const size_t dst = static_cast<size_t>(sp[static_cast<size_t>(s)] + k * kSlice + lane);
        if (r < local_rows && k < off[r + 1] - off[r]) {
          hc[dst] = static_cast<int32_t>(col[off[r] + k] - op->ext_begin);
          hv[dst] = val[off[r] + k];
        } else {
          hc[dst] = static_cast<int32_t>(std::min<int64_t>(self, std::max<int64_t>(ext_len - 1, 0)));
          hv[dst] = 0.0;
        }
      }
    }
  }
  op->slice_ptr.resize(nslices + 1);
  op->cols_idx.resize(std::max<int64_t>(total, 1));
  op->vals.resize(std::max<int64_t>(total, 1));
  SDR_CUDA(cudaMemcpyAsync(op->slice_ptr.get(), sp.data(), sizeof(int64_t) * sp.size(), cudaMemcpyHostToDevice, c.stream));
  if (total) {
    SDR_CUDA(cudaMemcpyAsync(op->cols_idx.get(), hc.data(), sizeof(int32_t) * hc.size(), cudaMemcpyHostToDevice, c.stream));
    SDR_CUDA(cudaMemcpyAsync(op->vals.get(), hv.data(), sizeof(double) * hv.size(), cudaMemcpyHostToDevice, c.stream));
  }
  c.sync();
  return op.release();
}

namespace {

__global__ void k_gen_convdiff3d(int64_t nx, int64_t ny, int64_t nz, int64_t row_begin, int64_t local_rows,
                                 int64_t ext_begin, double diag, double mx, double px, double my, double py, double mz,
                                 double pz, int32_t* __restrict__ cols, double* __restrict__ vals) {
  const int64_t nslices = (local_rows + kSlice - 1) / kSlice;
  const int64_t total = nslices * kSlice;
  const int64_t n2 = nx * ny;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < total;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = r / kSlice, lane = r % kSlice;
    const int64_t base = s * kSlice * 7 + lane;
    const int64_t rr = r < local_rows ? r : local_rows - 1;
    const int64_t p = row_begin + rr;
    const int64_t z = p / n2, y = (p / nx) % ny, x = p % nx;
    int k = 0;
    auto put = [&](int64_t c, double v) {
      cols[base + k * kSlice] = static_cast<int32_t>(c - ext_begin);
      vals[base + k * kSlice] = r < local_rows ? v : 0.0;
      ++k;
    };
    // CSR order: increasing column (sparse.hpp:136-138)
    if (z > 0) put(p - n2, mz);
    if (y > 0) put(p - nx, my);
    if (x > 0) put(p - 1, mx);
    put(p, diag);
    if (x + 1 < nx) put(p + 1, px);
    if (y + 1 < ny) put(p + nx, py);
    if (z + 1 < nz) put(p + n2, pz);
    while (k < 7) put(p, 0.0);
  }
}

// SELL-DIA form of the same operator: every slice uses the seven offsets
// {-nx*ny, -nx, -1, 0, 1, nx, nx*ny} (increasing column = CSR order); entries
// whose neighbour is outside the grid hold 0 (the column is clamped in K1).
__global__ void k_gen_convdiff3d_dia(int64_t nx, int64_t ny, int64_t nz, int64_t row_begin, int64_t local_rows,
                                     double diag, double mx, double px, double my, double py, double mz, double pz,
                                     double* __restrict__ vals) {
  const int64_t nslices = (local_rows + kSlice - 1) / kSlice;
  const int64_t total = nslices * kSlice;
  const int64_t n2 = nx * ny;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < total;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = r / kSlice, lane = r % kSlice;
    double* v = vals + s * kSlice * 7 + lane;
    const bool live = r < local_rows;
    const int64_t p = row_begin + (live ? r : 0);
    const int64_t z = p / n2, y = (p / nx) % ny, x = p % nx;
    v[0 * kSlice] = live && z > 0 ? mz : 0.0;
    v[1 * kSlice] = live && y > 0 ? my : 0.0;
    v[2 * kSlice] = live && x > 0 ? mx : 0.0;
    v[3 * kSlice] = live ? diag : 0.0;
    v[4 * kSlice] = live && x + 1 < nx ? px : 0.0;
    v[5 * kSlice] = live && y + 1 < ny ? py : 0.0;
    v[6 * kSlice] = live && z + 1 < nz ? pz : 0.0;
  }
}

__global__ void k_fill_doff(int32_t* doff, int64_t nslices, int32_t nx, int32_t n2) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nslices * 7;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % 7);
    const int32_t o[7] = {-n2, -nx, -1, 0, 1, nx, n2};
    doff[i] = o[k];
  }
}

__global__ void k_fill_slice_ptr(int64_t* sp, int64_t nslices, int64_t width) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s <= nslices;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    sp[s] = s * width;
}

}  // namespace

DeviceOperator* create_operator_convdiff3d(Context& c, int64_t nx, int64_t ny, int64_t nz, double bx, double by,
                                           double bz, int64_t z0, int64_t z1) {
  if (nx < 1 || ny < 1 || nz < 1) throw invalid("gen_convdiff3d: grid sides must be positive");
  if (z0 < 0 || z1 > nz || z0 > z1) throw invalid("gen_convdiff3d: bad z-slab [" + std::to_string(z0) + ", " + std::to_string(z1) + ")");
  const int64_t n2 = nx * ny, N = n2 * nz;
  auto op = std::make_unique<DeviceOperator>();
  op->rows = op->cols = N;
  op->row_begin = z0 * n2;
  op->local_rows = (z1 - z0) * n2;
  // coefficients exactly as the host generator (problems.hpp:70-88 convention), h_d = 1/(n_d + 1)
  const double hx = static_cast<double>((nx + 1) * (nx + 1)), hy = static_cast<double>((ny + 1) * (ny + 1)),
               hz = static_cast<double>((nz + 1) * (nz + 1));
  const double cx = bx * static_cast<double>(nx + 1) / 2.0, cy = by * static_cast<double>(ny + 1) / 2.0,
               cz = bz * static_cast<double>(nz + 1) / 2.0;
  const double coef[6] = {-hx - cx, -hx + cx, -hy - cy, -hy + cy, -hz - cz, -hz + cz};
  const double diag = nx == ny && ny == nz ? 6.0 * hx : 2.0 * hx + 2.0 * hy + 2.0 * hz;
  // stored nonzeros (from_triplets drops exact zeros)
  const int64_t zl = z1 - z0;
  const int64_t cnt[6] = {(nx - 1) * ny * zl, (nx - 1) * ny * zl, nx * (ny - 1) * zl, nx * (ny - 1) * zl,
                          zl == 0 ? 0 : (z1 - std::max<int64_t>(z0, 1)) * n2,
                          zl == 0 ? 0 : (std::min<int64_t>(z1, nz - 1) - z0) * n2};
  op->nnz = op->local_rows;
  for (int d = 0; d < 6; ++d)
    if (coef[d] != 0.0) op->nnz += std::max<int64_t>(cnt[d], 0);
  // only the first / last plane of the slab reaches into a neighbour's rows
  op->reach_lo_end = z0 > 0 ? std::min(n2, op->local_rows) : 0;
  op->reach_hi_begin = z1 < nz ? std::max<int64_t>(0, op->local_rows - n2) : op->local_rows;
  const int64_t mnc = z0 > 0 ? op->row_begin - n2 : op->row_begin;
  const int64_t mxc = z1 < nz ? op->row_begin + op->local_rows - 1 + n2 : op->row_begin + op->local_rows - 1;
  if (c.distributed()) {
    finish_partition(c, *op, mnc, mxc);
  } else {
    op->ext_begin = 0;
    op->halo_lo = op->halo_hi = 0;
    if (z0 != 0 || z1 != nz) throw invalid("gen_convdiff3d: a single-GPU context needs the full grid");
    op->plan.recv_lo.assign(1, 0);
    op->plan.recv_cnt.assign(1, 0);
    op->plan.send_lo.assign(1, 0);
    op->plan.send_cnt.assign(1, 0);
  }
  if (op->halo_lo + op->local_rows + op->halo_hi > std::numeric_limits<int32_t>::max())
    throw invalid("gen_convdiff3d: local block exceeds int32 indexing");
  const int64_t nslices = (op->local_rows + kSlice - 1) / kSlice;
  op->dia = dia_enabled() && n2 <= std::numeric_limits<int32_t>::max();
  op->dia_d = op->dia ? 7 : 0;
  op->stored = nslices * kSlice * 7;
  op->slice_ptr.resize(nslices + 1);
  op->vals.resize(std::max<int64_t>(nslices * kSlice * 7, 1));
  if (op->dia)
    op->doff.resize(std::max<int64_t>(nslices * 7, 1));
  else
    op->cols_idx.resize(std::max<int64_t>(nslices * kSlice * 7, 1));
  if (nslices > 0) {
    const int g = static_cast<int>(std::min<int64_t>((nslices * kSlice + 255) / 256, 148 * 16));
    k_fill_slice_ptr<<<g, 256, 0, c.stream>>>(op->slice_ptr.get(), nslices, kSlice * 7);
    SDR_KERNEL_CHECK();
    if (op->dia) {
      k_fill_doff<<<g, 256, 0, c.stream>>>(op->doff.get(), nslices, static_cast<int32_t>(nx), static_cast<int32_t>(n2));
      SDR_KERNEL_CHECK();
      k_gen_convdiff3d_dia<<<g, 256, 0, c.stream>>>(nx, ny, nz, op->row_begin, op->local_rows, diag, coef[0], coef[1],
                                                    coef[2], coef[3], coef[4], coef[5], op->vals.get());
    } else {
      k_gen_convdiff3d<<<g, 256, 0, c.stream>>>(nx, ny, nz, op->row_begin, op->local_rows, op->ext_begin, diag,
                                               coef[0], coef[1], coef[2], coef[3], coef[4], coef[5],
                                               op->cols_idx.get(), op->vals.get());
    }
    SDR_KERNEL_CHECK();
  }
  c.sync();
  return op.release();
}

void operator_apply(Context& c, const DeviceOperator& op, double* x_buf, double* y) {
  const VecLayout L = op.layout();
  c.halo_exchange(op.plan, x_buf + L.ext_shift(), op.ext_begin, x_buf + L.own_off, op.row_begin);
  launch_spmv(c, op.view(), x_buf + L.ext_shift(), y);
}

}  // namespace sdr
