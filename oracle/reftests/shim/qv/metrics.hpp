// qv/metrics.hpp -> the qv:: drop-in, plus declarations of the metrics the
// drop-in does not carry (PSGS and table summaries are outside the
// north-star path). shim_stubs.cpp defines them for the test binary only.
#pragma once
#include <utility>

#include "qv_b200.hpp"

namespace qv {
struct PsgsTable {
  std::vector<double> values;
  SamplingConfig config;
};
PsgsTable compute_psgs(const TransitionView& t, const SamplingConfig& cfg);
namespace serial {
PsgsTable compute_psgs(const TransitionView& t, const SamplingConfig& cfg);
}
struct TableSummary {
  double min = 0.0;
  double max = 0.0;
  double mean = 0.0;
  std::vector<std::pair<NodeId, double>> hottest;
};
TableSummary summarize_table(std::span<const double> values, std::size_t top_k);
}  // namespace qv
