// Sketch operators: host generation (bit-exact with the reference Rng) and
// the device representation the kernels consume.
#pragma once

#include "common.hpp"

#include <algorithm>
#include <cmath>
#include <random>
#include <unordered_map>
#include <vector>

namespace sdr {

enum SketchKind { kSrdct = 0, kIdentity = 1, kSparseSign = 2 };

/// splitmix64 finalizer — counter hash of the sparse-sign map. Must stay
/// identical to oracle/skrylov_oracle.hpp detail::mix64.
__host__ __device__ inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr std::uint64_t kPhi64 = 0x9E3779B97F4A7C15ull;

/// Hashes per column of the sparse-sign map: four 16-bit entry fields each.
__host__ __device__ inline std::int64_t sparse_sign_chunks(std::int64_t zeta) { return (zeta + 3) / 4; }

/// (row, sign) of nonzero l of column j of the sparse-sign map (block
/// construction: one nonzero per row block [l*s/zeta, (l+1)*s/zeta)).
/// Entries 4c..4c+3 of column j share h_c = mix64(key + (j*nc + c + 1)*phi),
/// nc = ceil(zeta/4); entry l uses the 16-bit field f = h_c >> 16*(l mod 4):
/// sign = f & 1 ? +1 : -1, row = b0 + (((f >> 1) & 0x7FFF) * bsize) >> 15.
/// Must stay identical to oracle/skrylov_oracle.hpp SketchOperator::sparse_entry.
__host__ __device__ inline void sparse_sign_entry(std::uint64_t key, std::int64_t s, std::int64_t zeta, std::int64_t j,
                                                  std::int64_t l, std::int64_t* row, bool* positive) {
  const std::uint64_t nc = static_cast<std::uint64_t>(sparse_sign_chunks(zeta));
  const std::uint64_t h = mix64(key + (static_cast<std::uint64_t>(j) * nc + static_cast<std::uint64_t>(l / 4) + 1u) * kPhi64);
  const std::uint32_t f = static_cast<std::uint32_t>(h >> (16 * (l % 4))) & 0xFFFFu;
  const std::int64_t b0 = (l * s) / zeta, b1 = ((l + 1) * s) / zeta;
  *row = b0 + static_cast<std::int64_t>((static_cast<std::uint64_t>((f >> 1) & 0x7FFFu) * static_cast<std::uint64_t>(b1 - b0)) >> 15);
  *positive = (f & 1u) != 0;
}

/// Host-side generator state, reproducing SketchOperator::subsampled_dct
/// (sketch.hpp:105-122): n draws of Rng::sign (low bit of mt19937_64), then
/// Rng::sample_without_replacement(n, s) (rng.hpp:66-78), bit-exact. The
/// partial Fisher–Yates runs over a sparse swap map instead of an n-long
/// iota, so generation needs O(s) memory even at n = 2^27.
struct SrdctHost {
  std::vector<std::uint32_t> sign_bits;  // bit j set <=> sign_j = +1
  std::vector<std::int64_t> rows;        // sorted, s entries
};

inline SrdctHost make_srdct_host(std::int64_t n, std::int64_t s, std::uint64_t seed) {
  SrdctHost h;
  std::mt19937_64 eng(seed);
  h.sign_bits.assign(static_cast<size_t>((n + 31) / 32), 0u);
  for (std::int64_t i = 0; i < n; ++i)
    if (eng() & 1u) h.sign_bits[static_cast<size_t>(i >> 5)] |= (1u << (i & 31));
  std::unordered_map<std::int64_t, std::int64_t> swapped;
  swapped.reserve(static_cast<size_t>(2 * s));
  auto at = [&](std::int64_t i) {
    auto it = swapped.find(i);
    return it == swapped.end() ? i : it->second;
  };
  for (std::int64_t i = 0; i < s; ++i) {
    const std::uint64_t bound = static_cast<std::uint64_t>(n - i);
    const std::uint64_t threshold = (-bound) % bound;  // rng.hpp:37
    std::uint64_t r;
    do {
      r = eng();
    } while (r < threshold);
    const std::int64_t j = i + static_cast<std::int64_t>(r % bound);
    const std::int64_t vi = at(i), vj = at(j);
    swapped[i] = vj;
    swapped[j] = vi;
  }
  h.rows.resize(static_cast<size_t>(s));
  for (std::int64_t i = 0; i < s; ++i) h.rows[static_cast<size_t>(i)] = at(i);
  std::sort(h.rows.begin(), h.rows.end());
  return h;
}

/// Device-side sketch. The SRDCT four-step plan is chosen
/// per launch from (n, local block) in sketch.cu.
struct SketchDev {
  int kind = kSrdct;
  std::int64_t n = 0, s = 0, zeta = 0;
  std::uint64_t seed = 0, key = 0;
  double scale = 1.0;                      // sqrt(n/s)
  DeviceBuffer<std::uint32_t> sign_bits;   // SRDCT
  DeviceBuffer<std::int64_t> rows;         // SRDCT, sorted
  DeviceBuffer<double> row_scale;          // SRDCT: alpha_k * sqrt(n/s)
  DeviceBuffer<double2> tab;               // SRDCT per-row constants (sketch.cu k_srdct_tables)
  DeviceBuffer<int> uq;                    // SRDCT k mod 256
  DeviceBuffer<int> uperm;                 // SRDCT rows ordered by k mod 256 (tile kernels' Horner order)
  std::vector<std::int64_t> rows_host;
  std::vector<std::uint32_t> sign_bits_host;
};

}  // namespace sdr
