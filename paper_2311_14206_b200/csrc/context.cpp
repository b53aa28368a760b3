// Context implementation: stream, scratch, NCCL (dlopen'd so the library
// shares whatever libnccl.so.2 the host process — e.g. torch — already
// loaded instead of linking a second copy), and event timing.
#include "context.hpp"
#include "peer.hpp"

#include <cublas_v2.h>

#include <cstdlib>

#include <nccl.h>
#include <dlfcn.h>

namespace sdr {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi* load_nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) {
    if (!api.handle) throw Error(6, "NCCL unavailable: libnccl.so.2 could not be loaded");
    return &api;
  }
  tried = true;
  api.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!api.handle) throw Error(6, std::string("NCCL unavailable: ") + dlerror());
#define SDR_SYM(f)                                                                      \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.handle, "nccl" #f));             \
  if (!api.f) {                                                                         \
    api.handle = nullptr;                                                               \
    throw Error(6, "NCCL symbol nccl" #f " missing");                                   \
  }
  SDR_SYM(GetUniqueId)
  SDR_SYM(CommInitRank)
  SDR_SYM(CommDestroy)
  SDR_SYM(AllReduce)
  SDR_SYM(AllGather)
  SDR_SYM(Send)
  SDR_SYM(Recv)
  SDR_SYM(GroupStart)
  SDR_SYM(GroupEnd)
  SDR_SYM(GetErrorString)
#undef SDR_SYM
  return &api;
}

#define SDR_NCCL(call)                                                                        \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) throw Error(6, std::string(#call) + ": " + nccl_->GetErrorString(r_)); \
  } while (0)

void nccl_unique_id(void* out) {
  NcclApi* api = load_nccl();
  ncclUniqueId id;
  ncclResult_t r = api->GetUniqueId(&id);
  if (r != ncclSuccess) throw Error(6, std::string("ncclGetUniqueId: ") + api->GetErrorString(r));
  std::memcpy(out, &id, sizeof(id));
}

Context::Context(int dev, int rk, int ws, const void* nccl_id, const HostComm* host_comm)
    : device(dev), rank(rk), world(ws) {
  int count = 0;
  SDR_CUDA(cudaGetDeviceCount(&count));
  if (dev < 0 || dev >= count) throw invalid("sdr_ctx_create: no CUDA device " + std::to_string(dev));
  SDR_CUDA(cudaSetDevice(dev));
  SDR_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  SDR_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  counters_.resize(kNumCounters);
  SDR_CUDA(cudaMemset(counters_.get(), 0, sizeof(unsigned) * kNumCounters));
  if (host_comm) {
    if (!host_comm->allreduce_sum || !host_comm->allgather_i64 || !host_comm->exchange)
      throw invalid("sdr_ctx_create_hostcomm: every collective callback is required");
    host_comm_ = true;
    hc_ = *host_comm;
  } else if (world > 1 || nccl_id) {
    if (!nccl_id) throw invalid("sdr_ctx_create_dist: NCCL id required for world > 1");
    nccl_ = load_nccl();
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclComm_t c = nullptr;
    SDR_NCCL(nccl_->CommInitRank(&c, world, id, rank));
    comm_ = c;
  }
  SDR_CUDA(cudaDeviceSynchronize());
}

Context::~Context() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  if (blas_) cublasDestroy(static_cast<cublasHandle_t>(blas_));
  if (comm_ && nccl_) nccl_->CommDestroy(static_cast<ncclComm_t>(comm_));
  for (void* m : peer_mapped_)
    if (m) cudaIpcCloseMemHandle(m);
  if (peer_own_) cudaFree(peer_own_);
  for (auto& p : pending_) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : free_events_) cudaEventDestroy(e);
  for (int i = 0; i < kAuxStreams; ++i) {
    if (aux_ev_[i]) cudaEventDestroy(aux_ev_[i]);
    if (aux_[i]) cudaStreamDestroy(aux_[i]);
  }
  if (fork_ev_) cudaEventDestroy(fork_ev_);
  if (open_start_) cudaEventDestroy(open_start_);
  if (stream) cudaStreamDestroy(stream);
}

bool Context::peer_setup() {
  if (peer_tried_) return peer_ok_;
  peer_tried_ = true;
  const char* e = std::getenv("SDR_PEER");
  if (!e || std::atoi(e) == 0 || world < 2) return false;
  const size_t slot_bytes = sizeof(double) * 2 * static_cast<size_t>(world) * kPeerMaxN;
  const size_t bytes = slot_bytes + sizeof(uint64_t) * static_cast<size_t>(world);
  SDR_CUDA(cudaMalloc(&peer_own_, bytes));
  SDR_CUDA(cudaMemset(peer_own_, 0, bytes));
  cudaIpcMemHandle_t h{};
  SDR_CUDA(cudaIpcGetMemHandle(&h, peer_own_));
  static_assert(sizeof(cudaIpcMemHandle_t) % sizeof(i64) == 0, "IPC handle size");
  constexpr i64 kWords = sizeof(cudaIpcMemHandle_t) / sizeof(i64);
  std::vector<i64> mine(kWords), all(static_cast<size_t>(kWords * world));
  std::memcpy(mine.data(), &h, sizeof(h));
  allgather_i64(mine.data(), kWords, all.data());
  peer_mapped_.assign(static_cast<size_t>(world), nullptr);
  std::vector<double*> sl(static_cast<size_t>(world));
  std::vector<uint64_t*> fl(static_cast<size_t>(world));
  for (int q = 0; q < world; ++q) {
    void* base = peer_own_;
    if (q != rank) {
      cudaIpcMemHandle_t hq{};
      std::memcpy(&hq, all.data() + q * kWords, sizeof(hq));
      SDR_CUDA(cudaIpcOpenMemHandle(&base, hq, cudaIpcMemLazyEnablePeerAccess));
      peer_mapped_[static_cast<size_t>(q)] = base;
    }
    sl[static_cast<size_t>(q)] = static_cast<double*>(base);
    fl[static_cast<size_t>(q)] = reinterpret_cast<uint64_t*>(static_cast<char*>(base) + slot_bytes);
  }
  peer_slots_.resize(world);
  peer_flags_.resize(world);
  SDR_CUDA(cudaMemcpy(peer_slots_.get(), sl.data(), sizeof(double*) * sl.size(), cudaMemcpyHostToDevice));
  SDR_CUDA(cudaMemcpy(peer_flags_.get(), fl.data(), sizeof(uint64_t*) * fl.size(), cudaMemcpyHostToDevice));
  peer_ok_ = true;
  return true;
}

void Context::allreduce_sum(double* dev, i64 n) {
  if (host_comm_ && n > 0) {
    ++launches;
    hstage_.ensure(n);
    SDR_CUDA(cudaMemcpyAsync(hstage_.get(), dev, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, stream));
    sync();
    if (hc_.allreduce_sum(hstage_.get(), n, hc_.user) != 0) throw Error(6, "host transport: allreduce failed");
    SDR_CUDA(cudaMemcpyAsync(dev, hstage_.get(), sizeof(double) * static_cast<size_t>(n), cudaMemcpyHostToDevice, stream));
    sync();
    return;
  }
  if (!comm_ || n <= 0) return;
  if (n <= kPeerMaxN && peer_setup()) {
    launch_peer_allreduce(*this, PeerView{peer_slots_.get(), peer_flags_.get(), world, rank}, dev, static_cast<int>(n),
                          next_peer_epoch());
    return;
  }
  ++launches;
  if (timing) time_begin("allreduce");
  SDR_NCCL(nccl_->AllReduce(dev, dev, static_cast<size_t>(n), ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), stream));
  if (timing) time_end();
}

void Context::allgather_i64(const i64* host_in, i64 count, i64* host_out) {
  if (host_comm_) {
    if (hc_.allgather_i64(host_in, count, host_out, hc_.user) != 0) throw Error(6, "host transport: allgather failed");
    return;
  }
  if (!comm_) {
    std::memcpy(host_out, host_in, sizeof(i64) * static_cast<size_t>(count));
    return;
  }
  DeviceBuffer<i64> buf(count * (world + 1));
  SDR_CUDA(cudaMemcpyAsync(buf.get(), host_in, sizeof(i64) * count, cudaMemcpyHostToDevice, stream));
  SDR_NCCL(nccl_->AllGather(buf.get(), buf.get() + count, static_cast<size_t>(count), ncclInt64,
                            static_cast<ncclComm_t>(comm_), stream));
  SDR_CUDA(cudaMemcpyAsync(host_out, buf.get() + count, sizeof(i64) * count * world, cudaMemcpyDeviceToHost, stream));
  sync();
}

void Context::halo_exchange(const HaloPlan& plan, double* x_ext, i64 ext_begin, const double* x_own, i64 row_begin,
                            cudaStream_t on) {
  if (host_comm_ && !plan.empty()) {
    cudaStream_t st = on ? on : this->stream;
    ++launches;
    for (int q = 0; q < world; ++q) {
      if (q == rank || (plan.send_cnt[q] == 0 && plan.recv_cnt[q] == 0)) continue;
      const i64 ns = plan.send_cnt[q], nr = plan.recv_cnt[q];
      std::vector<double> sbuf(static_cast<size_t>(ns)), rbuf(static_cast<size_t>(nr));
      if (ns)
        SDR_CUDA(cudaMemcpyAsync(sbuf.data(), x_own + (plan.send_lo[q] - row_begin), sizeof(double) * static_cast<size_t>(ns),
                                 cudaMemcpyDeviceToHost, st));
      SDR_CUDA(cudaStreamSynchronize(st));
      if (hc_.exchange(q, sbuf.data(), ns, rbuf.data(), nr, hc_.user) != 0) throw Error(6, "host transport: exchange failed");
      if (nr)
        SDR_CUDA(cudaMemcpyAsync(x_ext + (plan.recv_lo[q] - ext_begin), rbuf.data(), sizeof(double) * static_cast<size_t>(nr),
                                 cudaMemcpyHostToDevice, st));
      SDR_CUDA(cudaStreamSynchronize(st));
    }
    return;
  }
  if (!comm_ || plan.empty()) return;
  cudaStream_t stream = on ? on : this->stream;
  const bool timed = timing && stream == this->stream;
  ++launches;
  if (timed) time_begin("halo");
  auto comm = static_cast<ncclComm_t>(comm_);
  SDR_NCCL(nccl_->GroupStart());
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    if (plan.send_cnt[q] > 0)
      SDR_NCCL(nccl_->Send(x_own + (plan.send_lo[q] - row_begin), static_cast<size_t>(plan.send_cnt[q]), ncclDouble, q,
                           comm, stream));
    if (plan.recv_cnt[q] > 0)
      SDR_NCCL(nccl_->Recv(x_ext + (plan.recv_lo[q] - ext_begin), static_cast<size_t>(plan.recv_cnt[q]), ncclDouble, q,
                           comm, stream));
  }
  SDR_NCCL(nccl_->GroupEnd());
  if (timed) time_end();
}

cudaStream_t Context::aux_stream(int i) {
  if (!aux_[i]) {
    SDR_CUDA(cudaStreamCreateWithFlags(&aux_[i], cudaStreamNonBlocking));
    SDR_CUDA(cudaEventCreateWithFlags(&aux_ev_[i], cudaEventDisableTiming));
  }
  return aux_[i];
}

void Context::aux_fork(int n) {
  if (!fork_ev_) SDR_CUDA(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming));
  SDR_CUDA(cudaEventRecord(fork_ev_, stream));
  for (int i = 0; i < n; ++i) SDR_CUDA(cudaStreamWaitEvent(aux_stream(i), fork_ev_, 0));
}

void Context::aux_join(int n) {
  for (int i = 0; i < n; ++i) {
    SDR_CUDA(cudaEventRecord(aux_ev_[i], aux_stream(i)));
    SDR_CUDA(cudaStreamWaitEvent(stream, aux_ev_[i], 0));
  }
}

cudaEvent_t Context::take_event() {
  if (!free_events_.empty()) {
    cudaEvent_t e = free_events_.back();
    free_events_.pop_back();
    return e;
  }
  cudaEvent_t e;
  SDR_CUDA(cudaEventCreate(&e));
  return e;
}

void Context::time_begin(const char* name) {
  open_name_ = name;
  open_start_ = take_event();
  SDR_CUDA(cudaEventRecord(open_start_, stream));
  if (!origin_) {
    SDR_CUDA(cudaEventCreate(&origin_));
    SDR_CUDA(cudaEventRecord(origin_, stream));
  }
}

void Context::time_end() {
  cudaEvent_t b = take_event();
  SDR_CUDA(cudaEventRecord(b, stream));
  pending_.push_back({open_name_, open_start_, b});
  open_start_ = nullptr;
  if (pending_.size() > 4096) timing_flush();
}

void Context::timing_flush() {
  if (pending_.empty()) return;
  sync();
  for (auto& p : pending_) {
    float ms = 0.f;
    SDR_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& t = timings[p.name];
    ++t.launches;
    t.ms += ms;
    if (origin_ && timeline.size() < 100000) {
      float s0 = 0.f, s1 = 0.f;
      SDR_CUDA(cudaEventElapsedTime(&s0, origin_, p.a));
      SDR_CUDA(cudaEventElapsedTime(&s1, origin_, p.b));
      timeline.push_back({p.name, 1e3 * s0, 1e3 * s1});
    }
    free_events_.push_back(p.a);
    free_events_.push_back(p.b);
  }
  pending_.clear();
}

void Context::timing_reset() {
  timing_flush();
  timings.clear();
  timeline.clear();
  if (origin_) {
    SDR_CUDA(cudaEventDestroy(origin_));
    origin_ = nullptr;
  }
}

void Context::dgemm_tall(i64 n, i64 nout, i64 k, const double* A, i64 lda, const double* B, i64 ldb, double beta,
                         double* C, i64 ldc) {
  if (n == 0 || nout == 0) return;
  if (!blas_) {
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw runtime("cublasCreate failed");
    blas_ = h;
  }
  auto h = static_cast<cublasHandle_t>(blas_);
  if (cublasSetStream(h, stream) != CUBLAS_STATUS_SUCCESS) throw runtime("cublasSetStream failed");
  const double one = 1.0;
  ++launches;
  if (timing) time_begin("recycle_gemm");
  const cublasStatus_t st = cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(nout),
                                        static_cast<int>(k), &one, A, static_cast<int>(lda), B, static_cast<int>(ldb),
                                        &beta, C, static_cast<int>(ldc));
  if (timing) time_end();
  if (st != CUBLAS_STATUS_SUCCESS) throw runtime("cublasDgemm failed with status " + std::to_string(static_cast<int>(st)));
}

static int trace_mode() {
  static const int m = [] {
    const char* e = std::getenv("SDR_TRACE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

unsigned long long* Context::trace(i64 n) {
  if (trace_mode() != 1) return nullptr;
  if (trace_.size() < n) {
    trace_.resize(n);
    SDR_CUDA(cudaMemsetAsync(trace_.get(), 0, sizeof(unsigned long long) * static_cast<size_t>(n), stream));
  }
  return trace_.get();
}

unsigned long long* Context::launch_stamp(const char* name) {
  constexpr i64 kCap = 1 << 16;
  if (trace_mode() != 2 && !stamps_on) return nullptr;
  if (stamps_.size() == 0) {
    stamps_.resize(2 * kCap);
    SDR_CUDA(cudaMemsetAsync(stamps_.get(), 0xFF, sizeof(unsigned long long) * kCap, stream));
    SDR_CUDA(cudaMemsetAsync(stamps_.get() + kCap, 0, sizeof(unsigned long long) * kCap, stream));
  }
  const i64 i = static_cast<i64>(stamp_names_.size());
  if (i >= kCap) return nullptr;
  stamp_names_.push_back(name);
  return stamps_.get() + i;  // start at [i], end at [i + kCap]
}

std::vector<std::pair<std::string, std::pair<unsigned long long, unsigned long long>>> Context::launch_stamps_read() {
  constexpr i64 kCap = 1 << 16;
  std::vector<std::pair<std::string, std::pair<unsigned long long, unsigned long long>>> out;
  if (stamps_.size() == 0) return out;
  std::vector<unsigned long long> h(static_cast<size_t>(2 * kCap));
  SDR_CUDA(cudaMemcpyAsync(h.data(), stamps_.get(), sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, stream));
  sync();
  for (size_t i = 0; i < stamp_names_.size(); ++i) out.push_back({stamp_names_[i], {h[i], h[i + kCap]}});
  stamp_names_.clear();
  SDR_CUDA(cudaMemsetAsync(stamps_.get(), 0xFF, sizeof(unsigned long long) * kCap, stream));
  SDR_CUDA(cudaMemsetAsync(stamps_.get() + kCap, 0, sizeof(unsigned long long) * kCap, stream));
  return out;
}

std::vector<unsigned long long> Context::trace_read() {
  std::vector<unsigned long long> out(static_cast<size_t>(trace_.size()));
  if (!out.empty())
    SDR_CUDA(cudaMemcpyAsync(out.data(), trace_.get(), sizeof(unsigned long long) * out.size(), cudaMemcpyDeviceToHost,
                             stream));
  sync();
  return out;
}

}  // namespace sdr
