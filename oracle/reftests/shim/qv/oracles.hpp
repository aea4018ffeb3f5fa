// qv/oracles.hpp: the Monte-Carlo oracles are outside the north-star path;
// declared for the test binary and throw if called.
#pragma once
#include <optional>

#include "qv/metrics.hpp"

namespace qv {
struct PsgsMcEstimate {
  double mean = 0.0;
  double std_error = 0.0;
  double unique_mean = 0.0;
  std::uint64_t trials = 0;
};
PsgsMcEstimate psgs_oracle_mc(const Graph& g, const SamplingConfig& cfg, NodeId node,
                              std::uint64_t trials, std::uint64_t rng_seed);
struct FapMcResult {
  std::vector<double> mean;
  std::vector<double> std_error;
  std::uint64_t trials = 0;
};
FapMcResult fap_oracle_mc(const Graph& g, std::uint32_t hops, std::uint64_t trials,
                          std::uint64_t rng_seed, std::optional<std::span<const double>> seed_dist = {});
}  // namespace qv
