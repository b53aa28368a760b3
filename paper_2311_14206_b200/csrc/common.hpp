// Shared host-side plumbing: error classes mirroring the reference's
// exception taxonomy, CUDA checks, RAII device / pinned buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

namespace sdr {

using i64 = std::int64_t;

/// Error carrying the C-ABI status code (sdr_status).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
inline Error invalid(const std::string& m) { return Error(1, m); }
inline Error domain(const std::string& m) { return Error(2, m); }
inline Error logic(const std::string& m) { return Error(3, m); }
inline Error runtime(const std::string& m) { return Error(4, m); }

#define SDR_CUDA(call)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      throw ::sdr::Error(e_ == cudaErrorMemoryAllocation ? 7 : 5,                                   \
                         std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                             std::to_string(__LINE__) + ")");                                      \
  } while (0)

#define SDR_KERNEL_CHECK() SDR_CUDA(cudaGetLastError())

/// Process-wide cache of large freed device allocations (keyed by device and
/// exact byte size), so per-solve buffers — the recycle space's U blocks,
/// staging vectors — are recycled instead of going through cudaMalloc /
/// cudaFree (both synchronise the device) on every solve.
struct DeviceCache {
  static constexpr size_t kMinBytes = size_t{8} << 20;
  static constexpr int kPerSize = 4;
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::multimap<std::pair<int, size_t>, void*>& pool() {
    static std::multimap<std::pair<int, size_t>, void*> p;
    return p;
  }
  static void* take(size_t bytes) {
    if (bytes < kMinBytes) return nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu());
    auto it = pool().find({dev, bytes});
    if (it == pool().end()) return nullptr;
    void* p = it->second;
    pool().erase(it);
    return p;
  }
  static bool give(void* p, size_t bytes) {
    if (bytes < kMinBytes) return false;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu());
    if (static_cast<int>(pool().count({dev, bytes})) >= kPerSize) return false;
    pool().insert({{dev, bytes}, p});
    return true;
  }
};

/// Owning device allocation.
template <class T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(i64 n) { resize(n); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_, n_ = o.n_;
      o.p_ = nullptr, o.n_ = 0;
    }
    return *this;
  }
  void resize(i64 n) {
    if (n == n_) return;
    release();
    if (n > 0) {
      const size_t bytes = sizeof(T) * static_cast<size_t>(n);
      p_ = static_cast<T*>(DeviceCache::take(bytes));
      if (!p_) SDR_CUDA(cudaMalloc(&p_, bytes));
    }
    n_ = n;
  }
  void ensure(i64 n) {
    if (n > n_) resize(n);
  }
  void release() {
    if (p_ && !DeviceCache::give(p_, sizeof(T) * static_cast<size_t>(n_))) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  i64 size() const { return n_; }

 private:
  T* p_ = nullptr;
  i64 n_ = 0;
};

/// Page-locked host allocation (for async D2H of step records).
template <class T>
class PinnedBuffer {
 public:
  PinnedBuffer() = default;
  ~PinnedBuffer() { release(); }
  PinnedBuffer(const PinnedBuffer&) = delete;
  PinnedBuffer& operator=(const PinnedBuffer&) = delete;
  void ensure(i64 n) {
    if (n <= n_) return;
    release();
    SDR_CUDA(cudaMallocHost(&p_, sizeof(T) * static_cast<size_t>(n)));
    n_ = n;
  }
  void release() {
    if (p_) cudaFreeHost(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  i64 size() const { return n_; }

 private:
  T* p_ = nullptr;
  i64 n_ = 0;
};

inline bool is_device_pointer(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

inline bool is_pinned_host_pointer(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

inline i64 round_up(i64 v, i64 m) { return (v + m - 1) / m * m; }

#ifdef __CUDACC__
/// Programmatic dependent launch: a kernel launched with programmatic stream
/// serialization may start while its predecessor drains; it must call
/// pdl_wait() before touching the predecessor's output (no-op otherwise).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

/// SDR_TRACE=2 launch timeline: first CTA start / last CTA end (%globaltimer).
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp_begin(unsigned long long* st) {
  if (st && threadIdx.x == 0) atomicMin(st, global_ns());
}
/// Call with the whole CTA (contains a barrier).
__device__ __forceinline__ void stamp_end(unsigned long long* st) {
  if (st) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(st + (1 << 16), global_ns());
  }
}
#endif

/// Launch attribute set for programmatic stream serialization (PDL).
inline cudaLaunchAttribute pdl_attribute() {
  cudaLaunchAttribute a{};
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  return a;
}

}  // namespace sdr
