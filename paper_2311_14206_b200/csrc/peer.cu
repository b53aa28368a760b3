// One-shot allreduce over NVLink peer memory for the per-step folded
// partials (a few hundred doubles; SURVEY.md §8e "one fused small allreduce
// per Arnoldi step"). Each rank owns a symmetric buffer — receive slots
// [2 parities][world][kPeerMaxN] doubles and world 64-bit flags — mapped into
// every peer with CUDA IPC. A single CTA per rank stores its values straight
// into every peer's slot row (st.global on mapped peer addresses), fences at
// system scope and release-stores its epoch into each peer's flag; it then
// acquire-spins on its own flags until every peer reached the epoch and sums
// the rows in rank order. Every rank therefore computes the same sums in the
// same order (deterministic, identical across ranks). Slot rows alternate by
// epoch parity: a peer can publish epoch e + 2 only after its gather of
// e + 1, which needs this rank's publication of e + 1, issued after this
// rank's gather of e — so no row is overwritten before it was read.
//
// Enabled with SDR_PEER=1 (the NCCL allreduce stays the default until it is
// measured on several GPUs). The same device function runs in
// sdr_debug_peer_emulate: all ranks as CTAs of one cooperative launch on one
// GPU (co-resident, so the spins are safe), which is how it is tested here.
#include "kernels.hpp"
#include "peer.hpp"

#include <cooperative_groups.h>

namespace sdr {

namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

/// The CTA's part of one allreduce: vals[0..n) in, out[0..n) = sum over ranks.
__device__ void peer_allreduce_cta(const PeerView& a, const double* vals, int n, uint64_t epoch, double* out) {
  const int par = static_cast<int>(epoch & 1);
  const int64_t row = (static_cast<int64_t>(par) * a.world + a.rank) * kPeerMaxN;
  for (int q = 0; q < a.world; ++q) {  // publish into every rank's slot row `rank` (own included)
    double* dst = a.slots[q] + row;
    for (int v = threadIdx.x; v < n; v += blockDim.x) dst[v] = vals[v];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < a.world) st_release_sys(a.flags[threadIdx.x] + a.rank, epoch);
  // gather: wait for every rank's publication of this epoch in the own buffer
  if (threadIdx.x < a.world)
    while (ld_acquire_sys(a.flags[a.rank] + threadIdx.x) < epoch) {
    }
  __syncthreads();
  const double* mine = a.slots[a.rank] + static_cast<int64_t>(par) * a.world * kPeerMaxN;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < a.world; ++q) s += __ldcg(mine + static_cast<int64_t>(q) * kPeerMaxN + v);
    out[v] = s;
  }
}

__global__ void __launch_bounds__(256) k_peer_allreduce(PeerView a, double* vals, int n, uint64_t epoch) {
  peer_allreduce_cta(a, vals, n, epoch, vals);
}

/// Fold (fixed order: p1's CTAs then p2's) into buf[off ..], then the peer
/// allreduce of buf[0 .. off + nv) — one launch per step on several ranks.
__global__ void __launch_bounds__(256) k_fold_peer_allreduce(PeerView a, const double* __restrict__ p1, int G1,
                                                             const double* __restrict__ p2, int G2, int nv,
                                                             double* buf, int off, uint64_t epoch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = warp; v < nv; v += blockDim.x >> 5) {
    double s = 0.0;
    for (int b = lane; b < G1; b += 32) s += p1[static_cast<int64_t>(v) * G1 + b];
    if (p2)
      for (int b = lane; b < G2; b += 32) s += p2[static_cast<int64_t>(v) * G2 + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) buf[off + v] = s;
  }
  __syncthreads();
  peer_allreduce_cta(a, buf, off + nv, epoch, buf);
}

/// Emulation: CTA r acts as rank r with its own view; vals[r * n ..] in/out.
__global__ void __launch_bounds__(256) k_peer_emulate(const PeerView* views, double* vals, int n, uint64_t epoch) {
  const PeerView a = views[blockIdx.x];
  double* v = vals + static_cast<int64_t>(blockIdx.x) * n;
  peer_allreduce_cta(a, v, n, epoch, v);
}

}  // namespace

void launch_peer_allreduce(Context& c, const PeerView& v, double* dev, int n, uint64_t epoch) {
  if (n > kPeerMaxN) throw invalid("peer allreduce: at most " + std::to_string(kPeerMaxN) + " values");
  TimedLaunch t(c, "peer_allreduce");
  k_peer_allreduce<<<1, 256, 0, c.stream>>>(v, dev, n, epoch);
  SDR_KERNEL_CHECK();
}

void fold_allreduce(Context& c, const double* p1, int G1, const double* p2, int G2, int nv, double* buf, int off) {
  if (off + nv <= kPeerMaxN && c.peer_setup()) {
    const PeerView v{const_cast<double* const*>(c.peer_slots()), c.peer_flags(), c.world, c.rank};
    TimedLaunch t(c, "fold_peer_allreduce");
    k_fold_peer_allreduce<<<1, 256, 0, c.stream>>>(v, p1, G1, p2, G2, nv, buf, off, c.next_peer_epoch());
    SDR_KERNEL_CHECK();
    return;
  }
  if (p2)
    launch_fold_partials2(c, p1, G1, p2, G2, nv, buf + off);
  else
    launch_fold_partials(c, p1, G1, nv, true, buf + off);
  c.allreduce_sum(buf, off + nv);
}

void peer_emulate(int world, int n, int epochs, const double* vals_host, double* out_host) {
  if (world < 1 || world > 64 || n < 1 || n > kPeerMaxN || epochs < 1) throw invalid("peer emulation: bad sizes");
  // one symmetric buffer per virtual rank, all on this GPU
  std::vector<DeviceBuffer<double>> slots(static_cast<size_t>(world));
  std::vector<DeviceBuffer<uint64_t>> flags(static_cast<size_t>(world));
  std::vector<double*> sp(static_cast<size_t>(world));
  std::vector<uint64_t*> fp(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r) {
    slots[static_cast<size_t>(r)].resize(2 * static_cast<int64_t>(world) * kPeerMaxN);
    flags[static_cast<size_t>(r)].resize(world);
    SDR_CUDA(cudaMemset(flags[static_cast<size_t>(r)].get(), 0, sizeof(uint64_t) * static_cast<size_t>(world)));
    sp[static_cast<size_t>(r)] = slots[static_cast<size_t>(r)].get();
    fp[static_cast<size_t>(r)] = flags[static_cast<size_t>(r)].get();
  }
  DeviceBuffer<double*> dsp(world);
  DeviceBuffer<uint64_t*> dfp(world);
  SDR_CUDA(cudaMemcpy(dsp.get(), sp.data(), sizeof(double*) * sp.size(), cudaMemcpyHostToDevice));
  SDR_CUDA(cudaMemcpy(dfp.get(), fp.data(), sizeof(uint64_t*) * fp.size(), cudaMemcpyHostToDevice));
  std::vector<PeerView> hv(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r) hv[static_cast<size_t>(r)] = PeerView{dsp.get(), dfp.get(), world, r};
  DeviceBuffer<PeerView> dv(world);
  SDR_CUDA(cudaMemcpy(dv.get(), hv.data(), sizeof(PeerView) * hv.size(), cudaMemcpyHostToDevice));
  DeviceBuffer<double> vals(static_cast<int64_t>(world) * n);
  int dev = 0, coop = 0;
  SDR_CUDA(cudaGetDevice(&dev));
  SDR_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) throw runtime("peer emulation: cooperative launch unsupported");
  // several epochs back to back: the parity double-buffering is exercised
  for (int e = 1; e <= epochs; ++e) {
    SDR_CUDA(cudaMemcpy(vals.get(), vals_host + static_cast<int64_t>(e - 1) * world * n,
                        sizeof(double) * static_cast<size_t>(world) * n, cudaMemcpyHostToDevice));
    const PeerView* vp = dv.get();
    double* valp = vals.get();
    uint64_t ep = static_cast<uint64_t>(e);
    void* args[] = {&vp, &valp, &n, &ep};
    SDR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_peer_emulate), dim3(world), dim3(256), args, 0,
                                         nullptr));
    SDR_CUDA(cudaDeviceSynchronize());
    SDR_CUDA(cudaMemcpy(out_host + static_cast<int64_t>(e - 1) * world * n, vals.get(),
                        sizeof(double) * static_cast<size_t>(world) * n, cudaMemcpyDeviceToHost));
  }
}

}  // namespace sdr
