// NVLink peer-memory one-shot allreduce (peer.cu).
#pragma once

#include "context.hpp"

#include <vector>

namespace sdr {

constexpr int kPeerMaxN = 1024;  // values per allreduce (the per-step payload is 2s + 2t + 1 <= 1024 for s <= 500)

/// Device view of the symmetric buffers: slots[q] / flags[q] are rank q's
/// receive slots [2][world][kPeerMaxN] and flags [world], mapped in this process.
struct PeerView {
  double* const* slots = nullptr;
  uint64_t* const* flags = nullptr;
  int world = 1, rank = 0;
};

void launch_peer_allreduce(Context& c, const PeerView& v, double* dev, int n, uint64_t epoch);

/// The several-rank step reduction in one go: buf[off + v] = sum over the
/// value-major partials p1 [nv][G1] and p2 [nv][G2] (p2 may be null), then
/// buf[0 .. off + nv) summed over ranks. With SDR_PEER=1 one kernel folds,
/// publishes and gathers; otherwise the fold kernel and the NCCL allreduce.
void fold_allreduce(Context& c, const double* p1, int G1, const double* p2, int G2, int nv, double* buf, int off);

/// Test hook: `world` virtual ranks as CTAs of one cooperative launch on this
/// GPU, `epochs` allreduces back to back. vals_host / out_host: [epochs][world][n].
void peer_emulate(int world, int n, int epochs, const double* vals_host, double* out_host);

}  // namespace sdr
