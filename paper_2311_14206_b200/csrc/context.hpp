// Device context: one GPU, one CUDA stream, optional NCCL rank, reusable
// reduction scratch and per-kernel CUDA-event timing.
#pragma once

#include "common.hpp"

#include <map>
#include <memory>
#include <string>
#include <vector>

namespace sdr {

struct NcclApi;  // dlopen'd NCCL entry points (context.cpp)

/// Halo plan of one operator in a distributed context: which global rows
/// this rank receives from / sends to each peer.
struct HaloPlan {
  std::vector<i64> recv_lo, recv_cnt, send_lo, send_cnt;  // per peer, global rows
  bool empty() const {
    for (i64 c : recv_cnt)
      if (c) return false;
    for (i64 c : send_cnt)
      if (c) return false;
    return true;
  }
};

/// Host-staged collectives (sdr_host_comm in the C-ABI): test transport for
/// ranks without NCCL between them.
struct HostComm {
  int (*allreduce_sum)(double* buf, i64 n, void* user) = nullptr;
  int (*allgather_i64)(const i64* in, i64 count, i64* out, void* user) = nullptr;
  int (*exchange)(int peer, const double* send, i64 nsend, double* recv, i64 nrecv, void* user) = nullptr;
  void* user = nullptr;
};

struct KernelTiming {
  i64 launches = 0;
  double ms = 0.0;
};

class Context {
 public:
  Context(int device, int rank, int world, const void* nccl_id, const HostComm* host_comm = nullptr);
  ~Context();

  int device = 0, rank = 0, world = 1, num_sms = 148;
  cudaStream_t stream = nullptr;
  i64 launches = 0;

  /// Multi-GPU code path: world > 1, or a one-rank NCCL communicator
  /// (sdr_ctx_create_dist with world = 1 and an id) that runs the distributed
  /// pipeline — halo plans, allreduces, fold kernels — on a single GPU.
  bool distributed() const { return world > 1 || comm_ != nullptr || host_comm_; }

  // ---- reductions scratch: per-kernel-class partial buffers and
  // last-block-done counters (zeroed once, reset by the last block).
  double* partials(i64 n) {
    partials_.ensure(n);
    return partials_.get();
  }
  double* partials2(i64 n) {
    partials2_.ensure(n);
    return partials2_.get();
  }
  unsigned* counters() { return counters_.get(); }  // kNumCounters slots
  /// Kernel phase trace buffer (SDR_TRACE=1, debugging only): null when off.
  unsigned long long* trace(i64 n);
  /// Device-clock launch timeline (SDR_TRACE=2, debugging only): a (first CTA
  /// start, last CTA end) %globaltimer pair for this launch, or null.
  unsigned long long* launch_stamp(const char* name);
  bool stamps_on = false;  // launch stamps without SDR_TRACE=2 (sdr_ctx_set_stamps, bench measurements)
  std::vector<std::pair<std::string, std::pair<unsigned long long, unsigned long long>>> launch_stamps_read();
  std::vector<unsigned long long> trace_read();
  static constexpr int kNumCounters = 64;

  // ---- collectives (no-ops on one rank)
  /// Sum over ranks in place: NCCL, or with SDR_PEER=1 (several ranks, n <=
  /// kPeerMaxN) the one-shot NVLink peer-memory kernel (peer.cu).
  void allreduce_sum(double* dev, i64 n);
  void allgather_i64(const i64* host_in, i64 count, i64* host_out);  // host in/out, small
  /// on: the stream the transfers are issued on (default: the context stream).
  void halo_exchange(const HaloPlan& plan, double* x_ext, i64 ext_begin, const double* x_own, i64 row_begin,
                     cudaStream_t on = nullptr);

  // ---- timing
  bool timing = false;
  void time_begin(const char* name);
  void time_end();
  void timing_flush();
  void timing_reset();
  std::map<std::string, KernelTiming> timings;
  struct Span {
    std::string name;
    double start_us, end_us;  // from the first timed launch since timing_reset
  };
  std::vector<Span> timeline;  // debugging (sdr_debug_timeline)

  // ---- staging
  double* stage(i64 n) {
    stage_.ensure(n);
    return stage_.get();
  }
  double* pinned(i64 n) {
    pinned_.ensure(n);
    return pinned_.get();
  }

  void sync() { SDR_CUDA(cudaStreamSynchronize(stream)); }

  /// Auxiliary streams for independent small launches (created once per
  /// context): aux_stream(i) for i < kAuxStreams, each with an event that
  /// aux_join() records and makes the main stream wait on.
  static constexpr int kAuxStreams = 4;
  cudaStream_t aux_stream(int i);
  /// aux streams [0, n) wait for the main stream's work so far
  void aux_fork(int n);
  /// the main stream waits for aux streams [0, n)
  void aux_join(int n);

  /// C (n x nout, ldc) = beta C + A (n x k, lda) B (k x nout, ldb), column-major
  /// fp64 on the context stream through cuBLAS (plain tall-skinny GEMM of the
  /// recycle update; deterministic for a fixed GPU).
  void dgemm_tall(i64 n, i64 nout, i64 k, const double* A, i64 lda, const double* B, i64 ldb, double beta, double* C,
                  i64 ldc);

  /// Solver workspace cached across solves (solver.cpp owns the type).
  std::shared_ptr<void> workspace;

 private:
  DeviceBuffer<double> partials_, partials2_, stage_;
  cudaStream_t aux_[kAuxStreams] = {};
  cudaEvent_t aux_ev_[kAuxStreams] = {}, fork_ev_ = nullptr;
  DeviceBuffer<unsigned> counters_;
  DeviceBuffer<unsigned long long> trace_, stamps_;
  std::vector<std::string> stamp_names_;
  PinnedBuffer<double> pinned_;
  NcclApi* nccl_ = nullptr;
  bool host_comm_ = false;
  HostComm hc_;
  PinnedBuffer<double> hstage_;
  void* blas_ = nullptr;  // cublasHandle_t, created on first use
  void* comm_ = nullptr;
  // peer-memory allreduce (SDR_PEER=1): own symmetric buffer, mapped peers, epoch
  bool peer_tried_ = false, peer_ok_ = false;
  void* peer_own_ = nullptr;                 // cudaMalloc'ed: slots then flags
  std::vector<void*> peer_mapped_;           // IPC-opened peer buffers (null for self)
  DeviceBuffer<double*> peer_slots_;
  DeviceBuffer<uint64_t*> peer_flags_;
  uint64_t peer_epoch_ = 0;

 public:
  /// SDR_PEER=1 on several ranks: the mapped peer buffers are set up (first
  /// call) and allreduces of <= kPeerMaxN values go through peer memory.
  bool peer_setup();
  const double* const* peer_slots() const { return peer_slots_.get(); }
  uint64_t* const* peer_flags() const { return peer_flags_.get(); }
  uint64_t next_peer_epoch() { return ++peer_epoch_; }

 private:
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> free_events_;
  std::string open_name_;
  cudaEvent_t open_start_ = nullptr;
  cudaEvent_t origin_ = nullptr;  // first event since timing_reset (kept)
  cudaEvent_t take_event();
};

/// RAII timing scope around one launch: `TimedLaunch t(ctx, "update");`.
struct TimedLaunch {
  Context& c;
  TimedLaunch(Context& ctx, const char* name) : c(ctx) {
    ++c.launches;
    if (c.timing) c.time_begin(name);
  }
  ~TimedLaunch() {
    if (c.timing) c.time_end();
  }
};

/// Staged view of a user pointer: device pointers are used in place, host
/// pointers are copied through a device buffer.
struct DeviceIn {
  const double* ptr = nullptr;
  DeviceBuffer<double> own;
  DeviceIn(Context& c, const double* p, i64 n) {
    if (!p || n == 0 || is_device_pointer(p)) {
      ptr = p;
      return;
    }
    own.resize(n);
    SDR_CUDA(cudaMemcpyAsync(own.get(), p, sizeof(double) * static_cast<size_t>(n), cudaMemcpyHostToDevice, c.stream));
    ptr = own.get();
  }
};

}  // namespace sdr
