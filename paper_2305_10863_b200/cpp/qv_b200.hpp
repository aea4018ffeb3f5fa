// qv_b200.hpp — C++ drop-in for the reference planner's hot-path API
// (namespace qv of /root/reference/proj/include/qv/*.hpp), implemented over
// the qvb C-ABI (include/qvb.h) and its sm_100a kernels.
//
// A reference user switches by including this header instead of
// qv/{graph,metrics,placement,topology,error}.hpp and linking libqvb.so +
// libqv_b200.so. Names, argument meaning, value semantics and exception types
// follow the reference; every compute call runs on the GPU (there is no CPU
// fallback — without a device the calls throw qv::DeviceError).
//
// Reference interface -> this header:
//   graph.hpp:25-48   Graph / Edge / from_edges / validate
//   graph.hpp:72-93   in_adjacency (device transpose) / TransitionView
//   metrics.hpp:32-64 FapTable / AccessProbTable / compute_access_prob_ie
//   sampler.hpp:11-53 SamplingConfig / SampleResult / sample_khop / batch_sample
//   topology.hpp:11-54 LinkClass / LinkSpec / ClusterTopology
//   placement.hpp:14-121 Tier / Location / PlacementPlan / plan_placement /
//                     FeatureLookupTable / build_lookup_table / ReadPlan /
//                     plan_reads / page_transitions / classify_link / fetch_cost
//   error.hpp:10-32   Error hierarchy
// plus FeatureStore, the real gather the reference only models.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

struct qvb_store;
struct qvb_sampler;
struct qvb_graph;

namespace qv {

// ---- errors (error.hpp:10-32) ------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : Error {
  using Error::Error;
};
struct ValidationError : Error {
  using Error::Error;
};
struct ConfigError : Error {
  using Error::Error;
};
struct PlacementError : Error {
  using Error::Error;
};
struct CalibrationError : Error {
  using Error::Error;
};
// Extension: CUDA failure / no device (the reference has no device).
struct DeviceError : Error {
  using Error::Error;
};

// ---- graph (graph.hpp:10-93) -------------------------------------------------
using NodeId = std::uint64_t;
using EdgeIdx = std::uint64_t;

struct Edge {
  NodeId src = 0;
  NodeId dst = 0;
  double weight = 1.0;
};

struct Graph {
  std::uint64_t node_count = 0;
  std::uint64_t edge_count = 0;
  std::vector<EdgeIdx> row_offsets;
  std::vector<NodeId> col_indices;
  std::vector<double> edge_weights;

  static Graph from_edges(std::uint64_t node_count, std::span<const Edge> edges);
  std::uint64_t out_degree(NodeId i) const { return row_offsets[i + 1] - row_offsets[i]; }
  std::span<const NodeId> neighbors(NodeId i) const {
    return {col_indices.data() + row_offsets[i], col_indices.data() + row_offsets[i + 1]};
  }
  std::span<const double> weights(NodeId i) const {
    return {edge_weights.data() + row_offsets[i], edge_weights.data() + row_offsets[i + 1]};
  }
  void validate() const;
};

// Transpose on the device (the reference's in_adjacency, graph.cpp:260-281).
Graph in_adjacency(const Graph& g);

struct TransitionView {
  const Graph* graph = nullptr;
  std::vector<double> row_sums;
  std::vector<std::uint64_t> distinct_out;
  bool has_parallel_edges = false;
  std::uint64_t node_count() const { return graph->node_count; }
  double edge_prob(NodeId i, EdgeIdx e) const {
    return row_sums[i] > 0.0 ? graph->edge_weights[e] / row_sums[i] : 0.0;
  }
  double prob(NodeId i, NodeId j) const;

  // Extension: the device graph transition_view() built on its one upload
  // (qvb_transition_view), which compute_access_prob_ie(g, view, L) reuses
  // when `graph` is still the Graph it was built from (same arrays, sizes).
  std::shared_ptr<qvb_graph> resident;
  const void* resident_key[3] = {nullptr, nullptr, nullptr};
  bool resident_for(const Graph& g) const;
};
// transition_view (graph.cpp:292-318) on the device: row sums, distinct
// out-degrees and has_parallel_edges come from the same upload that builds
// the P(n,j) in-CSR (kept in `resident`).
TransitionView transition_view(const Graph& g);

// ---- metrics (metrics.hpp:32-64) ---------------------------------------------
struct FapTable {
  std::vector<double> values;
  std::uint32_t hops = 0;
  std::vector<double> seed_distribution;
};

struct AccessProbTable {
  std::vector<double> values;
  std::uint32_t layers = 0;
};

// FAP visit mass (metrics.cpp:95-132) on the GPU, bit-identical; seed_dist
// must sum to 1 (1e-12), uniform when absent.
FapTable compute_fap(const TransitionView& t, std::uint32_t hops,
                     std::optional<std::span<const double>> seed_dist = {});

// P(n,j) on the GPU, bit-identical to the reference.
AccessProbTable compute_access_prob_ie(const Graph& g, const TransitionView& t,
                                       std::uint32_t layers);
namespace serial {
AccessProbTable compute_access_prob_ie(const Graph& g, const TransitionView& t,
                                       std::uint32_t layers);
FapTable compute_fap(const TransitionView& t, std::uint32_t hops,
                     std::optional<std::span<const double>> seed_dist = {});
}

// ---- sampler (sampler.hpp:11-53, metrics.hpp:14-19) ----------------------------
struct SamplingConfig {
  std::vector<std::uint32_t> fanouts;
  std::size_t hops() const { return fanouts.size(); }
  void validate() const;  // metrics.cpp:13-18
};

struct SampleResult {
  NodeId seed = 0;
  std::vector<std::vector<NodeId>> frontiers;  // index 0 is {seed}
  std::vector<std::uint64_t> instance_counts;  // per hop
  std::vector<NodeId> unique_nodes;            // sorted, across all hops
  std::uint64_t total_instances() const {
    std::uint64_t n = 0;
    for (std::uint64_t c : instance_counts) n += c;
    return n;
  }
};

struct BatchSampleStats {
  std::uint64_t total_instances = 0;
  std::uint64_t unique_count = 0;
  std::vector<NodeId> unique_nodes;  // sorted union
};

struct BatchSampleResult {
  std::vector<SampleResult> per_seed;
  BatchSampleStats stats;
};

// The device-resident sampling candidates of one graph (qvb_sampler), for
// many batches; the free functions below build one per call.
class Sampler {
 public:
  explicit Sampler(const Graph& g, int device = -1);
  ~Sampler();
  Sampler(const Sampler&) = delete;
  Sampler& operator=(const Sampler&) = delete;
  BatchSampleResult batch_sample(std::span<const NodeId> seeds, const SamplingConfig& cfg,
                                 std::uint64_t rng_seed) const;
  // Only the sorted union (what simulator.cpp:250-254 keeps), no per-seed copy.
  BatchSampleStats batch_stats(std::span<const NodeId> seeds, const SamplingConfig& cfg,
                               std::uint64_t rng_seed) const;

 private:
  qvb_sampler* s_ = nullptr;
};

// sample_khop (sampler.cpp:56-112) / batch_sample (:114-149) on the GPU,
// identical frontiers.
SampleResult sample_khop(const TransitionView& t, NodeId seed, const SamplingConfig& cfg,
                         std::uint64_t rng_seed);
BatchSampleResult batch_sample(const TransitionView& t, std::span<const NodeId> seeds,
                               const SamplingConfig& cfg, std::uint64_t rng_seed);

// ---- topology (topology.hpp:11-54) -------------------------------------------
enum class LinkClass : std::uint8_t { local = 0, nvlink, pcie, upi, infiniband, ethernet, disk };
constexpr std::size_t kLinkClassCount = 7;
const char* link_class_name(LinkClass c);

struct LinkSpec {
  double latency_s = 0.0;
  double bandwidth_Bps = 1.0;
};

struct ClusterTopology {
  std::uint32_t servers = 1;
  std::uint32_t numa_per_server = 1;
  std::uint32_t gpus_per_server = 1;
  std::uint64_t gpu_feature_capacity = 0;
  std::uint64_t host_feature_capacity = 0;
  std::uint64_t disk_feature_capacity = 0;
  bool nvlink_within_numa = false;
  bool infiniband = false;
  std::array<LinkSpec, kLinkClassCount> links{};
  double tlb_miss_penalty_s = 1e-7;
  // Extension (0 == reference): hottest rows replicated on every GPU.
  std::uint64_t gpu_replicated_capacity = 0;

  std::uint32_t gpus_per_numa() const { return gpus_per_server / numa_per_server; }
  const LinkSpec& link(LinkClass c) const { return links[static_cast<std::size_t>(c)]; }
  void validate() const;
  static ClusterTopology with_defaults();
};

// ---- placement (placement.hpp:14-121) ----------------------------------------
enum class Tier : std::uint8_t { gpu = 0, host = 1, disk = 2 };
const char* tier_name(Tier t);

struct Location {
  std::uint32_t server = 0;
  Tier tier = Tier::host;
  std::uint32_t device = 0;
  bool replica = false;
};

std::int64_t encode_location(const ClusterTopology& topo, std::uint32_t server, Tier tier,
                             std::uint32_t device);
Location decode_location(const ClusterTopology& topo, std::int64_t id);

struct PlacementPlan {
  std::uint64_t feature_count = 0;
  std::vector<std::vector<Location>> locations;
  void validate(const ClusterTopology& topo) const;
};

PlacementPlan plan_placement(const FapTable& fap, const ClusterTopology& topo);

struct FeatureLookupTable {
  std::uint32_t home_server = 0;
  std::uint32_t gpus_per_server = 0;
  std::vector<std::int64_t> location_ids;
  std::vector<std::uint64_t> offsets;
};

// Extension: reader_device > 0 builds the per-reader table of that GPU.
FeatureLookupTable build_lookup_table(const PlacementPlan& plan, const ClusterTopology& topo,
                                      std::uint32_t home_server, std::uint32_t reader_device = 0);

struct ReadPlan {
  std::uint32_t home_server = 0;
  std::uint64_t page_size = 8;
  struct LocationReads {
    std::int64_t location_id = 0;
    std::vector<std::uint64_t> offsets;
    std::uint64_t page_transitions = 0;
  };
  std::vector<LocationReads> per_location;
};

ReadPlan plan_reads(const FeatureLookupTable& table, std::span<const NodeId> feature_ids,
                    std::uint64_t page_size = 8);
class FeatureStore;
// Extension: the same plan over a store's resident lookup table (the store's
// reader table; reader 0 is the reference's), with no per-call table upload
// — the per-batch call of the reference's serving loop (simulator.cpp:320).
ReadPlan plan_reads(const FeatureStore& store, std::span<const NodeId> feature_ids,
                    std::uint64_t page_size = 8);
std::uint64_t page_transitions(std::span<const std::uint64_t> offsets, std::uint64_t page_size);

struct DeviceRef {
  std::uint32_t server = 0;
  Tier tier = Tier::gpu;
  std::uint32_t device = 0;
};
struct LinkPath {
  LinkClass first = LinkClass::local;
  std::optional<LinkClass> second;
};
LinkPath classify_link(const ClusterTopology& topo, const DeviceRef& reader,
                       std::int64_t location_id);

struct FetchCost {
  double total_s = 0.0;
  std::vector<std::pair<std::int64_t, double>> per_location_s;
};
// The reference's latency model of a collect (placement.cpp:382-404), kept
// for callers such as its simulator; FeatureStore::gather is the real thing.
FetchCost fetch_cost(const ReadPlan& plan, const ClusterTopology& topo,
                     std::uint64_t feature_bytes, std::optional<DeviceRef> reader = {});

// ---- on-disk formats (graph.cpp:197-258, metrics.cpp:203-250,
//      placement.cpp:406-459), byte-compatible with the reference ------------
enum class GraphFormat { edge_list_text, csr_binary };
Graph load_graph(const std::string& path, GraphFormat format, bool remap_sparse_ids = false);
void save_graph_csr(const Graph& g, const std::string& path);
void save_table_binary(const std::string& path, std::span<const double> values, std::uint64_t k);
struct LoadedTable {
  std::vector<double> values;
  std::uint64_t k = 0;
};
LoadedTable load_table_binary(const std::string& path);
void save_table_csv(const std::string& path, std::span<const double> values);
std::string placement_to_json_text(const PlacementPlan& plan);
void save_placement_csv(const PlacementPlan& plan, const std::string& path);
std::string lookup_to_json_text(const FeatureLookupTable& table);
void save_lookup_csv(const FeatureLookupTable& table, const std::string& path);

// ---- feature store (new: the collect the reference only models) ---------------
class FeatureStore {
 public:
  // Builds reader GPU `reader_device`'s store on CUDA device `cuda_device`
  // from a single-server plan; features: n x dim row-major fp32 (empty =
  // the synthetic SURVEY §8(d) generator).
  FeatureStore(const PlacementPlan& plan, const ClusterTopology& topo, std::uint32_t dim,
               std::uint32_t reader_device, std::span<const float> features = {},
               int cuda_device = -1);
  ~FeatureStore();
  FeatureStore(const FeatureStore&) = delete;
  FeatureStore& operator=(const FeatureStore&) = delete;

  std::array<std::uint8_t, 64> export_handle() const;
  void attach_peer(std::uint32_t peer_device, const std::array<std::uint8_t, 64>& handle);
  // Device pointers, stream-ordered (stream = cudaStream_t as void*).
  void gather(const std::uint64_t* d_ids, std::uint64_t count, float* d_out,
              void* stream = nullptr) const;
  // Host buffers, synchronous: returns count x dim rows.
  std::vector<float> gather(std::span<const NodeId> ids) const;
  std::uint32_t dim() const { return dim_; }
  qvb_store* handle() const { return s_; }

 private:
  qvb_store* s_ = nullptr;
  std::uint32_t dim_ = 0;
};

}  // namespace qv
