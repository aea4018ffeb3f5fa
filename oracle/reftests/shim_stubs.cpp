// Out-of-path pieces the reference's test files reference, for the
// reference-test binary only (never the product library):
//  - compute_psgs: the PSGS definition (metrics.hpp:22-29) evaluated by a
//    plain Horner recursion, so the mixed P/FAP/PSGS cases of
//    test_metrics.cpp compile and run; the pure-PSGS cases are filtered out
//    (tests/test_reference_tests_gpu.py), they would test this stand-in;
//  - summarize_table (metrics.hpp:76-82): min / max / mean / top-k;
//  - topology JSON I/O and the Monte-Carlo oracles: throw (filtered out).
#include <algorithm>
#include <numeric>
#include <stdexcept>

#include "qv/metrics.hpp"
#include "qv/oracles.hpp"
#include "qv/topology.hpp"

namespace qv {

PsgsTable compute_psgs(const TransitionView& t, const SamplingConfig& cfg) {
  cfg.validate();
  const Graph& g = *t.graph;
  const std::uint64_t n = g.node_count;
  const std::size_t K = cfg.hops();
  std::vector<double> acc(n, 0.0), next(n);
  for (std::size_t k = K; k >= 1; --k) {  // acc <- m_k + delta * acc
    for (NodeId i = 0; i < n; ++i) {
      double pull = 0.0;
      if (k < K && t.row_sums[i] > 0.0)
        for (EdgeIdx e = g.row_offsets[i]; e < g.row_offsets[i + 1]; ++e)
          pull += t.edge_prob(i, e) * acc[g.col_indices[e]];
      next[i] = static_cast<double>(std::min<std::uint64_t>(t.distinct_out[i], cfg.fanouts[k - 1])) + pull;
    }
    acc.swap(next);
  }
  PsgsTable out;
  out.config = cfg;
  out.values.resize(n);
  for (NodeId i = 0; i < n; ++i) out.values[i] = 1.0 + (K ? acc[i] : 0.0);
  return out;
}

namespace serial {
PsgsTable compute_psgs(const TransitionView& t, const SamplingConfig& cfg) {
  return qv::compute_psgs(t, cfg);
}
}  // namespace serial

TableSummary summarize_table(std::span<const double> values, std::size_t top_k) {
  TableSummary s;
  if (values.empty()) return s;
  s.min = *std::min_element(values.begin(), values.end());
  s.max = *std::max_element(values.begin(), values.end());
  s.mean = std::accumulate(values.begin(), values.end(), 0.0) / static_cast<double>(values.size());
  std::vector<NodeId> ids(values.size());
  std::iota(ids.begin(), ids.end(), 0);
  const std::size_t k = std::min(top_k, ids.size());
  std::partial_sort(ids.begin(), ids.begin() + k, ids.end(), [&](NodeId a, NodeId b) {
    return values[a] > values[b] || (values[a] == values[b] && a < b);
  });
  for (std::size_t i = 0; i < k; ++i) s.hottest.emplace_back(ids[i], values[ids[i]]);
  return s;
}

[[noreturn]] static void out_of_scope(const char* what) {
  throw std::logic_error(std::string(what) + " is outside the north-star path (not in the drop-in)");
}
ClusterTopology load_topology(const std::string&) { out_of_scope("load_topology"); }
ClusterTopology topology_from_json_text(const std::string&, const std::string&) {
  out_of_scope("topology_from_json_text");
}
std::string topology_to_json_text(const ClusterTopology&) { out_of_scope("topology_to_json_text"); }
PsgsMcEstimate psgs_oracle_mc(const Graph&, const SamplingConfig&, NodeId, std::uint64_t, std::uint64_t) {
  out_of_scope("psgs_oracle_mc");
}
FapMcResult fap_oracle_mc(const Graph&, std::uint32_t, std::uint64_t, std::uint64_t,
                          std::optional<std::span<const double>>) {
  out_of_scope("fap_oracle_mc");
}

}  // namespace qv
