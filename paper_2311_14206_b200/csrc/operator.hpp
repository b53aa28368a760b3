// Device operator: the rank-local row block of A in SELL-32 storage plus
// its halo plan. Replaces SparseMatrix/OperatorRef (sparse.hpp:27-150,
// operator_ref.hpp:20-56) on the device side.
#pragma once

#include "context.hpp"
#include "kernels.hpp"

#include <vector>

namespace sdr {

struct DeviceOperator {
  int64_t rows = 0, cols = 0;            // global
  int64_t row_begin = 0, local_rows = 0;  // this rank's block
  int64_t nnz = 0;                        // stored entries of the block (before padding)
  int64_t ext_begin = 0;                  // global row of extended-vector index 0
  int64_t halo_lo = 0, halo_hi = 0;
  /// Stencil reach of the local rows: rows [0, reach_lo_end) are the only ones
  /// that read a column below row_begin, rows [reach_hi_begin, local_rows) the
  /// only ones that read a column at/after row_begin + local_rows. Rows in
  /// between never touch the halo, so their SpMV may overlap the halo transfer.
  int64_t reach_lo_end = 0, reach_hi_begin = 0;
  DeviceBuffer<int64_t> slice_ptr;
  DeviceBuffer<int32_t> cols_idx;  // SELL
  DeviceBuffer<int32_t> doff;      // SELL-DIA
  DeviceBuffer<double> vals;
  HaloPlan plan;
  bool dia = false;
  bool cplx = false;  // ZSELL (complex-structured real operator, see SellView::cplx)
  int dia_d = 0;  // SELL-DIA diagonals per slice
  // callable operator (sdr_operator_create_callback): no storage
  int (*apply)(const double* x, double* y, void* stream, void* user) = nullptr;
  void* apply_user = nullptr;
  int64_t stored = 0;  // stored entries (incl. padding) — bytes = stored * (dia ? 8 : cplx ? 20 : 12)

  SellView view() const {
    SellView v;
    v.slice_ptr = slice_ptr.get();
    v.cols = dia ? nullptr : cols_idx.get();
    v.doff = dia ? doff.get() : nullptr;
    v.dia_d = dia ? dia_d : 0;
    v.cplx = cplx ? 1 : 0;
    v.vals = vals.get();
    v.nrows = local_rows;
    v.nslices = cplx ? (local_rows / 2 + kSlice - 1) / kSlice : (local_rows + kSlice - 1) / kSlice;
    v.halo_lo = halo_lo;
    v.ext_len = halo_lo + local_rows + halo_hi;
    v.apply = apply;
    v.apply_user = apply_user;
    return v;
  }
  /// Layout for vectors used as SpMV inputs of this operator.
  VecLayout layout() const {
    VecLayout L;
    L.nloc = local_rows;
    L.halo_lo = halo_lo;
    L.halo_hi = halo_hi;
    L.own_off = round_up(halo_lo, 32);
    L.ld = round_up(L.own_off + local_rows + halo_hi, 32);
    return L;
  }
};

/// Validates like SparseMatrix::validate and uploads; offsets/columns/values
/// describe local_rows rows with global column indices.
DeviceOperator* create_operator_csr(Context& c, int64_t rows, int64_t cols, int64_t row_begin, int64_t local_rows,
                                    const int64_t* offsets, const int64_t* columns, const double* values);
/// 7-point −Δ + β·∇ on an nx×ny×nz grid (h_d = 1/(n_d+1)), z-slab [z0, z1), built on the device.
DeviceOperator* create_operator_convdiff3d(Context& c, int64_t nx, int64_t ny, int64_t nz, double bx, double by,
                                           double bz, int64_t z0, int64_t z1);

/// Fills the halo plan and extended range of op from every rank's ranges
/// (allgather over the context's communicator).
void finish_partition(Context& c, DeviceOperator& op, int64_t min_col, int64_t max_col);

/// Host partition logic (exported through the C-ABI for CPU tests).
void partition_halo(int world, int rank, const int64_t* rb, const int64_t* re, const int64_t* mnc, const int64_t* mxc,
                    int64_t* recv_lo, int64_t* recv_cnt, int64_t* send_lo, int64_t* send_cnt);

/// y = A x on one vector held in the layout of op (halo exchanged here).
/// x_buf: buffer in op.layout(), own part filled; y: local_rows entries.
void operator_apply(Context& c, const DeviceOperator& op, double* x_buf, double* y);

}  // namespace sdr
