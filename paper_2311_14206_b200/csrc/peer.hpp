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

/// Test hook: `world` virtual ranks as CTAs of one cooperative launch on this
/// GPU, `epochs` allreduces back to back. vals_host / out_host: [epochs][world][n].
void peer_emulate(int world, int n, int epochs, const double* vals_host, double* out_host);

}  // namespace sdr
