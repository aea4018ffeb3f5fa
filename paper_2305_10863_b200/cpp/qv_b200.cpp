// qv_b200.cpp — the qv:: drop-in over the qvb C-ABI (see qv_b200.hpp).
// Host code here only marshals arguments and rebuilds the reference's value
// types; every hot-path computation is a qvb_* call into the sm_100a library.
#include "qv_b200.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <numeric>
#include <sstream>

#include "../../include/qvb.h"

namespace qv {
namespace {

[[noreturn]] void rethrow(int rc) {
  const std::string m = qvb_last_error();
  switch (rc) {
    case QVB_ERR_VALIDATION: throw ValidationError(m);
    case QVB_ERR_PLACEMENT: throw PlacementError(m);
    case QVB_ERR_CUDA: throw DeviceError(m);
    default: throw Error(m);
  }
}
inline void check(int rc) {
  if (rc != QVB_OK) rethrow(rc);
}

int default_device() {
  int d = 0;
  const char* env = std::getenv("QVB_DEVICE");
  if (env) d = std::atoi(env);
  return d;
}

qvb_topology to_c(const ClusterTopology& t) {
  qvb_topology c;
  std::memset(&c, 0, sizeof c);
  c.servers = t.servers;
  c.numa_per_server = t.numa_per_server;
  c.gpus_per_server = t.gpus_per_server;
  c.nvlink_within_numa = t.nvlink_within_numa;
  c.infiniband = t.infiniband;
  c.gpu_feature_capacity = t.gpu_feature_capacity;
  c.host_feature_capacity = t.host_feature_capacity;
  c.disk_feature_capacity = t.disk_feature_capacity;
  for (std::size_t i = 0; i < kLinkClassCount; ++i) {
    c.link_latency_s[i] = t.links[i].latency_s;
    c.link_bandwidth_Bps[i] = t.links[i].bandwidth_Bps;
  }
  c.tlb_miss_penalty_s = t.tlb_miss_penalty_s;
  c.gpu_replicated_capacity = t.gpu_replicated_capacity;
  return c;
}

struct PlanCsr {
  std::vector<std::uint64_t> offsets;
  std::vector<std::int64_t> ids;
};

PlanCsr to_csr(const PlacementPlan& plan, const ClusterTopology& topo) {
  PlanCsr c;
  c.offsets.resize(plan.feature_count + 1, 0);
  for (std::uint64_t f = 0; f < plan.feature_count; ++f) {
    for (const Location& l : plan.locations[f])
      c.ids.push_back(encode_location(topo, l.server, l.tier, l.device));
    c.offsets[f + 1] = c.ids.size();
  }
  return c;
}

}  // namespace

// ---- graph ------------------------------------------------------------------
static_assert(sizeof(Edge) == sizeof(qvb_edge) && offsetof(Edge, dst) == offsetof(qvb_edge, dst) &&
                  offsetof(Edge, weight) == offsetof(qvb_edge, weight),
              "qv::Edge must keep the qvb_edge layout");

Graph Graph::from_edges(std::uint64_t node_count, std::span<const Edge> edges) {
  // build_csr (graph.cpp:16-56) on the device: checks in input order, a
  // stable sort by source, then the validate() the reference ends with
  Graph g;
  g.node_count = node_count;
  g.edge_count = edges.size();
  g.row_offsets.resize(node_count + 1);
  g.col_indices.resize(edges.size());
  g.edge_weights.resize(edges.size());
  check(qvb_build_csr(default_device(), node_count, reinterpret_cast<const qvb_edge*>(edges.data()),
                      edges.size(), g.row_offsets.data(), g.col_indices.data(),
                      g.edge_weights.data()));
  return g;
}

namespace {
// Graph::validate's container-shape checks (graph.cpp:58-70): properties of
// the std::vectors, which the C-ABI (plain pointers) cannot see.
void check_shape(const Graph& g) {
  if (g.node_count == 0) throw ValidationError("empty graph: node count is zero");
  const bool sized = g.row_offsets.size() == g.node_count + 1;
  if (!sized) throw ValidationError("row_offsets size mismatch");
  if (g.row_offsets.front() != 0 || g.row_offsets.back() != g.edge_count)
    throw ValidationError("row_offsets endpoints invalid");
  const bool edges_sized =
      g.col_indices.size() == g.edge_count && g.edge_weights.size() == g.edge_count;
  if (!edges_sized) throw ValidationError("edge array size mismatch");
}
}  // namespace

void Graph::validate() const {
  check_shape(*this);
  // monotone offsets, column range, weight sign, all-zero rows: on the device
  check(qvb_graph_validate(default_device(), node_count, edge_count, row_offsets.data(),
                           col_indices.data(), edge_weights.data()));
}

Graph in_adjacency(const Graph& g) {
  Graph t;
  t.node_count = g.node_count;
  t.edge_count = g.edge_count;
  t.row_offsets.resize(g.node_count + 1);
  t.col_indices.resize(g.edge_count);
  t.edge_weights.resize(g.edge_count);
  check(qvb_in_adjacency(default_device(), g.node_count, g.edge_count, g.row_offsets.data(),
                         g.col_indices.data(), g.edge_weights.data(), t.row_offsets.data(),
                         t.col_indices.data(), t.edge_weights.data()));
  return t;
}

double TransitionView::prob(NodeId i, NodeId j) const {
  // summed weight of i's edges to j over i's row sum (0 for sink rows)
  const double total = row_sums[i];
  if (!(total > 0.0)) return 0.0;
  const auto cols = graph->neighbors(i);
  const auto ws = graph->weights(i);
  double hit = 0.0;
  for (std::size_t k = 0; k < cols.size(); ++k) hit += cols[k] == j ? ws[k] : 0.0;
  return hit / total;
}

bool TransitionView::resident_for(const Graph& g) const {
  return resident && graph == &g && resident_key[0] == g.row_offsets.data() &&
         resident_key[1] == g.col_indices.data() && resident_key[2] == g.edge_weights.data();
}

TransitionView transition_view(const Graph& g) {
  check_shape(g);
  TransitionView t;
  t.graph = &g;
  t.row_sums.resize(g.node_count);
  t.distinct_out.resize(g.node_count);
  int parallel = 0;
  qvb_graph* dg = nullptr;
  check(qvb_transition_view(default_device(), g.node_count, g.edge_count, g.row_offsets.data(),
                            g.col_indices.data(), g.edge_weights.data(), t.row_sums.data(),
                            t.distinct_out.data(), &parallel, &dg));
  t.has_parallel_edges = parallel != 0;
  t.resident = std::shared_ptr<qvb_graph>(dg, [](qvb_graph* p) { qvb_graph_destroy(p); });
  t.resident_key[0] = g.row_offsets.data();
  t.resident_key[1] = g.col_indices.data();
  t.resident_key[2] = g.edge_weights.data();
  return t;
}

// ---- metrics ------------------------------------------------------------------
AccessProbTable compute_access_prob_ie(const Graph& g, const TransitionView& view,
                                       std::uint32_t layers) {
  if (layers < 1) throw ValidationError("access probability needs layers >= 1");
  AccessProbTable t;
  t.layers = layers;
  t.values.resize(g.node_count);
  if (view.resident_for(g)) {  // the graph is on the device since transition_view(g)
    check(qvb_access_prob(view.resident.get(), layers, t.values.data(), 0, nullptr));
    return t;
  }
  check(qvb_compute_access_prob_ie(default_device(), g.node_count, g.edge_count,
                                   g.row_offsets.data(), g.col_indices.data(),
                                   g.edge_weights.data(), layers, t.values.data(), nullptr));
  return t;
}

FapTable compute_fap(const TransitionView& t, std::uint32_t hops,
                     std::optional<std::span<const double>> seed_dist) {
  const Graph& g = *t.graph;
  if (seed_dist && seed_dist->size() != g.node_count)
    throw ValidationError("seed distribution size does not match node count");
  FapTable f;
  f.hops = hops;
  f.values.resize(g.node_count);
  check(qvb_compute_fap(default_device(), g.node_count, g.edge_count, g.row_offsets.data(),
                        g.col_indices.data(), g.edge_weights.data(), hops,
                        seed_dist ? seed_dist->data() : nullptr, f.values.data()));
  if (seed_dist) f.seed_distribution.assign(seed_dist->begin(), seed_dist->end());
  else f.seed_distribution.assign(g.node_count, 1.0 / static_cast<double>(g.node_count));
  return f;
}

namespace serial {
AccessProbTable compute_access_prob_ie(const Graph& g, const TransitionView& t,
                                       std::uint32_t layers) {
  return qv::compute_access_prob_ie(g, t, layers);  // one implementation: bit-identical
}
FapTable compute_fap(const TransitionView& t, std::uint32_t hops,
                     std::optional<std::span<const double>> seed_dist) {
  return qv::compute_fap(t, hops, seed_dist);
}
}  // namespace serial

// ---- sampler ------------------------------------------------------------------
void SamplingConfig::validate() const {
  if (fanouts.empty()) throw ValidationError("sampling config needs >= 1 hop");
  for (std::uint32_t l : fanouts)
    if (l < 1) throw ValidationError("fanouts must be >= 1");
}

namespace {
struct SampleHandle {
  qvb_sample* r = nullptr;
  ~SampleHandle() {
    if (r) qvb_sample_destroy(r);
  }
};

qvb_sample* run_batch(qvb_sampler* s, std::span<const NodeId> seeds, const SamplingConfig& cfg,
                      std::uint64_t rng_seed, SampleHandle& h) {
  cfg.validate();
  check(qvb_batch_sample(s, seeds.data(), seeds.size(), 0, cfg.fanouts.data(),
                         static_cast<std::uint32_t>(cfg.fanouts.size()), rng_seed, nullptr, &h.r));
  return h.r;
}

// splitmix64 (rng.hpp:10-16) inverted: batch_sample runs seed s under
// splitmix64(rng ^ s*gamma), so sample_khop(seed, rs) is the one-seed batch
// with rng = splitmix64^-1(rs) ^ seed*gamma.
std::uint64_t inv_mul(std::uint64_t c) {
  std::uint64_t x = c;  // Newton: x <- x(2 - cx) doubles the correct bits
  for (int i = 0; i < 6; ++i) x *= 2 - c * x;
  return x;
}
std::uint64_t unxorshift(std::uint64_t y, int s) {
  std::uint64_t x = y;
  for (int i = 0; i < 64 / s + 1; ++i) x = y ^ (x >> s);
  return x;
}
std::uint64_t unsplitmix64(std::uint64_t z) {
  z = unxorshift(z, 31);
  z *= inv_mul(0x94d049bb133111ebULL);
  z = unxorshift(z, 27);
  z *= inv_mul(0xbf58476d1ce4e5b9ULL);
  z = unxorshift(z, 30);
  return z - 0x9e3779b97f4a7c15ULL;
}
}  // namespace

Sampler::Sampler(const Graph& g, int device) {
  check(qvb_sampler_create(device >= 0 ? device : default_device(), g.node_count, g.edge_count,
                           g.row_offsets.data(), g.col_indices.data(),
                           g.edge_weights.empty() ? nullptr : g.edge_weights.data(), nullptr, &s_));
}

Sampler::~Sampler() {
  if (s_) qvb_sampler_destroy(s_);
}

BatchSampleStats Sampler::batch_stats(std::span<const NodeId> seeds, const SamplingConfig& cfg,
                                      std::uint64_t rng_seed) const {
  SampleHandle h;
  run_batch(s_, seeds, cfg, rng_seed, h);
  qvb_sample_info info;
  check(qvb_sample_info_get(h.r, &info));
  BatchSampleStats st;
  st.total_instances = info.total_instances;
  st.unique_count = info.unique_count;
  st.unique_nodes.resize(info.unique_count);
  check(qvb_sample_copy(h.r, nullptr, nullptr, st.unique_nodes.data()));
  return st;
}

BatchSampleResult Sampler::batch_sample(std::span<const NodeId> seeds, const SamplingConfig& cfg,
                                        std::uint64_t rng_seed) const {
  SampleHandle h;
  run_batch(s_, seeds, cfg, rng_seed, h);
  qvb_sample_info info;
  check(qvb_sample_info_get(h.r, &info));
  const std::size_t H = cfg.hops();
  std::vector<std::uint64_t> nodes(info.total_instances), counts(seeds.size() * (H + 1));
  BatchSampleResult out;
  out.stats.total_instances = info.total_instances;
  out.stats.unique_count = info.unique_count;
  out.stats.unique_nodes.resize(info.unique_count);
  check(qvb_sample_copy(h.r, nodes.data(), counts.data(), out.stats.unique_nodes.data()));
  out.per_seed.resize(seeds.size());
  std::size_t at = 0;
  for (std::size_t i = 0; i < seeds.size(); ++i) {
    SampleResult& r = out.per_seed[i];
    r.seed = seeds[i];
    r.frontiers.resize(H + 1);
    r.instance_counts.resize(H + 1);
    for (std::size_t k = 0; k <= H; ++k) {
      const std::uint64_t c = counts[i * (H + 1) + k];
      r.instance_counts[k] = c;
      r.frontiers[k].assign(nodes.begin() + at, nodes.begin() + at + c);
      r.unique_nodes.insert(r.unique_nodes.end(), r.frontiers[k].begin(), r.frontiers[k].end());
      at += c;
    }
    std::sort(r.unique_nodes.begin(), r.unique_nodes.end());
    r.unique_nodes.erase(std::unique(r.unique_nodes.begin(), r.unique_nodes.end()),
                         r.unique_nodes.end());
  }
  return out;
}

SampleResult sample_khop(const TransitionView& t, NodeId seed, const SamplingConfig& cfg,
                         std::uint64_t rng_seed) {
  cfg.validate();
  if (seed >= t.node_count())
    throw ValidationError("sample seed " + std::to_string(seed) + " out of range");
  const NodeId one[1] = {seed};
  Sampler s(*t.graph);
  const std::uint64_t rng = unsplitmix64(rng_seed) ^ (seed * 0x9e3779b97f4a7c15ULL);
  return std::move(s.batch_sample(one, cfg, rng).per_seed[0]);
}

BatchSampleResult batch_sample(const TransitionView& t, std::span<const NodeId> seeds,
                               const SamplingConfig& cfg, std::uint64_t rng_seed) {
  cfg.validate();
  Sampler s(*t.graph);
  return s.batch_sample(seeds, cfg, rng_seed);
}

// ---- topology -------------------------------------------------------------------
const char* link_class_name(LinkClass c) {
  static const char* names[] = {"local", "nvlink", "pcie", "upi", "infiniband", "ethernet", "disk"};
  return names[static_cast<int>(c)];
}

ClusterTopology ClusterTopology::with_defaults() {
  qvb_topology c;
  qvb_topology_defaults(&c);
  ClusterTopology t;
  for (std::size_t i = 0; i < kLinkClassCount; ++i)
    t.links[i] = {c.link_latency_s[i], c.link_bandwidth_Bps[i]};
  t.tlb_miss_penalty_s = c.tlb_miss_penalty_s;
  return t;
}

void ClusterTopology::validate() const {
  qvb_topology c = to_c(*this);
  check(qvb_topology_validate(&c));
}

// ---- placement ----------------------------------------------------------------
const char* tier_name(Tier t) {
  switch (t) {
    case Tier::gpu: return "gpu";
    case Tier::host: return "host";
    case Tier::disk: return "disk";
  }
  return "?";
}

std::int64_t encode_location(const ClusterTopology& topo, std::uint32_t server, Tier tier,
                             std::uint32_t device) {
  qvb_topology c = to_c(topo);
  return qvb_encode_location(&c, server, static_cast<uint32_t>(tier), device);
}

Location decode_location(const ClusterTopology& topo, std::int64_t id) {
  qvb_topology c = to_c(topo);
  uint32_t s, t, d;
  check(qvb_decode_location(&c, id, &s, &t, &d));
  Location l;
  l.server = s;
  l.tier = static_cast<Tier>(t);
  l.device = d;
  return l;
}

void PlacementPlan::validate(const ClusterTopology& topo) const {
  // copies per encoded location id (ids are dense, < servers x (G+2)); the
  // first location over its tier's capacity in ascending id order is named
  const std::uint64_t nloc = static_cast<std::uint64_t>(topo.servers) * (topo.gpus_per_server + 2);
  std::vector<std::uint64_t> per_loc(nloc, 0);
  for (std::uint64_t f = 0; f < feature_count; ++f) {
    const auto& copies = locations[f];
    if (copies.empty()) throw Error("feature " + std::to_string(f) + " has no location");
    for (const Location& l : copies) {
      const auto id = static_cast<std::uint64_t>(encode_location(topo, l.server, l.tier, l.device));
      if (id >= per_loc.size()) per_loc.resize(id + 1, 0);
      per_loc[id] += 1;
    }
  }
  for (std::uint64_t id = 0; id < per_loc.size(); ++id) {
    if (per_loc[id] == 0) continue;
    const Location l = decode_location(topo, static_cast<std::int64_t>(id));
    const std::uint64_t caps[3] = {topo.gpu_feature_capacity, topo.host_feature_capacity,
                                   topo.disk_feature_capacity};
    const std::uint64_t cap = caps[static_cast<int>(l.tier)];
    if (per_loc[id] <= cap) continue;
    throw Error(std::string("placement overfills ") + tier_name(l.tier) + " on server " +
                std::to_string(l.server) + ": " + std::to_string(per_loc[id]) + " > " +
                std::to_string(cap));
  }
}

PlacementPlan plan_placement(const FapTable& fap, const ClusterTopology& topo) {
  qvb_topology c = to_c(topo);
  const std::uint64_t n = fap.values.size();
  qvb_plan* h = nullptr;
  check(qvb_plan_placement_create(default_device(), fap.values.data(), n, &c, &h));
  std::uint64_t nn = 0, copies = 0;
  std::vector<std::uint64_t> lo(n + 1);
  std::vector<std::int64_t> ids;
  int rc = qvb_plan_size(h, &nn, &copies);
  if (rc == QVB_OK) {
    ids.resize(copies);
    rc = qvb_plan_copy(h, lo.data(), ids.data());
  }
  qvb_plan_destroy(h);
  check(rc);
  PlacementPlan p;
  p.feature_count = n;
  p.locations.resize(n);
  for (std::uint64_t f = 0; f < n; ++f)
    for (std::uint64_t k = lo[f]; k < lo[f + 1]; ++k) {
      Location l = decode_location(topo, ids[k]);
      l.replica = k > lo[f];
      p.locations[f].push_back(l);
    }
  return p;
}

FeatureLookupTable build_lookup_table(const PlacementPlan& plan, const ClusterTopology& topo,
                                      std::uint32_t home_server, std::uint32_t reader_device) {
  if (home_server >= topo.servers) throw ValidationError("home server out of range");
  qvb_topology c = to_c(topo);
  PlanCsr csr = to_csr(plan, topo);
  FeatureLookupTable t;
  t.home_server = home_server;
  t.gpus_per_server = topo.gpus_per_server;
  t.location_ids.resize(plan.feature_count);
  t.offsets.resize(plan.feature_count);
  check(qvb_build_lookup_table(default_device(), csr.offsets.data(), csr.ids.data(),
                               plan.feature_count, &c, home_server, reader_device,
                               t.location_ids.data(), t.offsets.data()));
  return t;
}

std::uint64_t page_transitions(std::span<const std::uint64_t> offsets, std::uint64_t page_size) {
  std::uint64_t out = 0;
  check(qvb_page_transitions(offsets.data(), offsets.size(), page_size, &out));
  return out;
}

ReadPlan plan_reads(const FeatureLookupTable& table, std::span<const NodeId> feature_ids,
                    std::uint64_t page_size) {
  if (page_size == 0) throw ValidationError("page size must be > 0");
  ReadPlan plan;
  plan.home_server = table.home_server;
  plan.page_size = page_size;
  const std::uint64_t b = feature_ids.size();
  if (b == 0) return plan;
  std::vector<std::int64_t> gl(b);
  std::vector<std::uint64_t> gc(b), gt(b), off(b);
  std::uint64_t ng = 0;
  check(qvb_plan_reads(default_device(), table.location_ids.data(), table.offsets.data(),
                       table.location_ids.size(), feature_ids.data(), b, page_size, gl.data(),
                       gc.data(), gt.data(), &ng, off.data()));
  std::uint64_t at = 0;
  for (std::uint64_t g = 0; g < ng; ++g) {
    ReadPlan::LocationReads r;
    r.location_id = gl[g];
    r.page_transitions = gt[g];
    r.offsets.assign(off.begin() + at, off.begin() + at + gc[g]);
    at += gc[g];
    plan.per_location.push_back(std::move(r));
  }
  return plan;
}

ReadPlan plan_reads(const FeatureStore& store, std::span<const NodeId> feature_ids,
                    std::uint64_t page_size) {
  if (page_size == 0) throw ValidationError("page size must be > 0");
  ReadPlan plan;
  plan.home_server = 0;  // the device store serves one server
  plan.page_size = page_size;
  const std::uint64_t b = feature_ids.size();
  if (b == 0) return plan;
  qvb_store_info info;
  check(qvb_store_info_get(store.handle(), &info));
  const std::uint64_t cap = std::min<std::uint64_t>(b, info.location_count);
  std::vector<std::int64_t> gl(cap);
  std::vector<std::uint64_t> gc(cap), gt(cap), off(b);
  std::uint64_t ng = 0;
  check(qvb_store_plan_reads(store.handle(), feature_ids.data(), b, 0, page_size, gl.data(),
                             gc.data(), gt.data(), &ng, off.data(), nullptr));
  std::uint64_t at = 0;
  plan.per_location.resize(ng);
  for (std::uint64_t g = 0; g < ng; ++g) {
    auto& r = plan.per_location[g];
    r.location_id = gl[g];
    r.page_transitions = gt[g];
    r.offsets.assign(off.begin() + at, off.begin() + at + gc[g]);
    at += gc[g];
  }
  return plan;
}

LinkPath classify_link(const ClusterTopology& topo, const DeviceRef& reader,
                       std::int64_t location_id) {
  qvb_topology c = to_c(topo);
  int first = 0, second = -1;
  check(qvb_classify_link(&c, reader.server, static_cast<std::uint32_t>(reader.tier), reader.device,
                          location_id, &first, &second));
  LinkPath path;
  path.first = static_cast<LinkClass>(first);
  if (second >= 0) path.second = static_cast<LinkClass>(second);
  return path;
}

FetchCost fetch_cost(const ReadPlan& plan, const ClusterTopology& topo,
                     std::uint64_t feature_bytes, std::optional<DeviceRef> reader) {
  qvb_topology c = to_c(topo);
  // default reader: GPU 0 of the plan's home server, the host without GPUs
  const DeviceRef rd = reader.value_or(
      DeviceRef{plan.home_server, topo.gpus_per_server > 0 ? Tier::gpu : Tier::host, 0});
  const std::size_t groups = plan.per_location.size();
  std::vector<std::int64_t> loc(groups);
  std::vector<std::uint64_t> count(groups), trans(groups);
  for (std::size_t g = 0; g < groups; ++g) {
    loc[g] = plan.per_location[g].location_id;
    count[g] = plan.per_location[g].offsets.size();
    trans[g] = plan.per_location[g].page_transitions;
  }
  std::vector<double> per(groups);
  FetchCost cost;
  check(qvb_fetch_cost(&c, rd.server, static_cast<std::uint32_t>(rd.tier), rd.device, groups,
                       loc.data(), count.data(), trans.data(), feature_bytes, per.data(),
                       &cost.total_s));
  cost.per_location_s.reserve(groups);
  for (std::size_t g = 0; g < groups; ++g) cost.per_location_s.emplace_back(loc[g], per[g]);
  return cost;
}

// ---- on-disk formats ----------------------------------------------------------------
namespace {
constexpr char kCsrMagic[6] = {'Q', 'V', 'C', 'S', 'R', '1'};
constexpr char kTabMagic[6] = {'Q', 'V', 'T', 'A', 'B', '1'};

// Binary table files: a 6-byte magic, little-endian u64 header words, raw
// payload arrays (QVCSR1 graph.cpp:197-258, QVTAB1 metrics.cpp:203-250).
class BinFile {
 public:
  BinFile(const std::string& path, bool write) : path_(path), f_(std::fopen(path.c_str(), write ? "wb" : "rb")) {}
  ~BinFile() {
    if (f_) std::fclose(f_);
  }
  BinFile(const BinFile&) = delete;
  BinFile& operator=(const BinFile&) = delete;
  bool open() const { return f_ != nullptr; }
  // reads count items; false when the file ends first
  template <typename T>
  bool get(T* dst, std::size_t count) {
    return std::fread(dst, sizeof(T), count, f_) == count;
  }
  template <typename T>
  bool put(const T* src, std::size_t count) {
    return std::fwrite(src, sizeof(T), count, f_) == count;
  }
  bool close_ok() {
    const bool ok = std::fflush(f_) == 0 && !std::ferror(f_);
    std::fclose(f_);
    f_ = nullptr;
    return ok;
  }

 private:
  std::string path_;
  std::FILE* f_;
};

// Text exports: the whole file is formatted in memory and written once.
void write_text_file(const std::string& path, const std::string& text, const char* kind) {
  BinFile f(path, true);
  if (!f.open()) throw Error(std::string("cannot write ") + kind + " file: " + path);
  if (!f.put(text.data(), text.size()) || !f.close_ok()) throw Error("short write to " + path);
}

// The text edge-list format (graph.cpp:112-188 semantics): "src dst [w]"
// per line, '#' starts a comment, blank lines skipped; numbers extract as
// from a std::istream; errors name "path:line".
struct LineParser {
  const std::string& path;
  std::uint64_t line_no = 0;

  [[noreturn]] void bad(const std::string& what) const {
    throw ParseError(path + ":" + std::to_string(line_no) + ": " + what);
  }

  // false for a line with nothing but whitespace/comment
  bool parse(std::string body, Edge& out) const {
    body.erase(std::min(body.find('#'), body.size()));
    std::istringstream in(body);
    std::uint64_t ends[2];
    for (int k = 0; k < 2; ++k) {
      if (in >> ends[k]) continue;
      std::istringstream probe(body);
      std::string any;
      if (k == 0 && !(probe >> any)) return false;
      bad("malformed edge line: '" + body + "'");
    }
    out = Edge{ends[0], ends[1], 1.0};
    std::string tok;
    if (!(in >> tok)) return true;
    std::size_t used = 0;
    bool ok = true;
    try {
      out.weight = std::stod(tok, &used);
    } catch (const std::exception&) {
      ok = false;
    }
    if (!ok || used != tok.size()) bad("malformed weight '" + tok + "'");
    if (in >> tok) bad("trailing tokens after weight: '" + tok + "'");
    return true;
  }
};

Graph load_edge_list(const std::string& path, bool remap) {
  std::ifstream file(path);
  if (!file) throw ParseError("cannot open graph file: " + path);
  std::vector<Edge> edges;
  LineParser lp{path};
  NodeId top = 0;
  for (std::string text; std::getline(file, text);) {
    ++lp.line_no;
    Edge ed;
    if (!lp.parse(std::move(text), ed)) continue;
    top = std::max({top, ed.src, ed.dst});
    edges.push_back(ed);
  }
  if (edges.empty()) throw ValidationError("empty graph: no edges in " + path);
  // ids used, and their dense rank when some id in 0..top never appears
  std::vector<NodeId> rank(top + 2, 0);
  for (const Edge& ed : edges) rank[ed.src + 1] = rank[ed.dst + 1] = 1;
  std::partial_sum(rank.begin(), rank.end(), rank.begin());
  const NodeId used = rank[top + 1];
  if (used != top + 1) {
    if (!remap)
      throw ValidationError(path + ": node ids are not contiguous 0..N-1 (use id remapping "
                                   "for sparse-id inputs)");
    for (Edge& ed : edges) {  // ascending original id -> 0..used-1
      ed.src = rank[ed.src];
      ed.dst = rank[ed.dst];
    }
  }
  return Graph::from_edges(used, edges);
}

void json_escape_free_write(std::ostringstream& o, int indent) {
  for (int i = 0; i < indent; ++i) o << ' ';
}
}  // namespace

Graph load_graph(const std::string& path, GraphFormat format, bool remap_sparse_ids) {
  if (format == GraphFormat::edge_list_text) return load_edge_list(path, remap_sparse_ids);
  BinFile f(path, false);
  if (!f.open()) throw ParseError("cannot open graph file: " + path);
  const std::string truncated = path + ": truncated csr-binary file";
  char magic[6];
  if (!f.get(magic, 6)) throw ParseError(truncated);
  if (std::memcmp(magic, kCsrMagic, 6) != 0) throw ParseError(path + ": bad magic, not a QVCSR1 file");
  std::uint64_t head[2];  // node count, edge count
  if (!f.get(head, 2)) throw ParseError(truncated);
  if (head[0] == 0) throw ValidationError("empty graph in " + path);
  Graph g;
  g.node_count = head[0];
  g.edge_count = head[1];
  g.row_offsets.resize(head[0] + 1);
  g.col_indices.resize(head[1]);
  g.edge_weights.resize(head[1]);
  const bool whole = f.get(g.row_offsets.data(), g.row_offsets.size()) &&
                     f.get(g.col_indices.data(), g.col_indices.size()) &&
                     f.get(g.edge_weights.data(), g.edge_weights.size());
  if (!whole) throw ParseError(truncated);
  g.validate();  // on the device
  return g;
}

void save_graph_csr(const Graph& g, const std::string& path) {
  BinFile f(path, true);
  if (!f.open()) throw Error("cannot write graph file: " + path);
  const std::uint64_t head[2] = {g.node_count, g.edge_count};
  const bool ok = f.put(kCsrMagic, 6) && f.put(head, 2) &&
                  f.put(g.row_offsets.data(), g.row_offsets.size()) &&
                  f.put(g.col_indices.data(), g.col_indices.size()) &&
                  f.put(g.edge_weights.data(), g.edge_weights.size());
  if (!ok || !f.close_ok()) throw Error("short write to " + path);
}

void save_table_binary(const std::string& path, std::span<const double> values, std::uint64_t k) {
  BinFile f(path, true);
  if (!f.open()) throw Error("cannot write table file: " + path);
  const std::uint64_t head[2] = {values.size(), k};
  if (!(f.put(kTabMagic, 6) && f.put(head, 2) && f.put(values.data(), values.size())) || !f.close_ok())
    throw Error("short write to " + path);
}

LoadedTable load_table_binary(const std::string& path) {
  BinFile f(path, false);
  if (!f.open()) throw ParseError("cannot open table file: " + path);
  char magic[6];
  if (!f.get(magic, 6) || std::memcmp(magic, kTabMagic, 6) != 0)
    throw ParseError(path + ": bad magic, not a QVTAB1 file");
  std::uint64_t head[2];  // value count, k
  if (!f.get(head, 2)) throw ParseError(path + ": truncated table header");
  LoadedTable t;
  t.k = head[1];
  t.values.resize(head[0]);
  if (!f.get(t.values.data(), t.values.size())) throw ParseError(path + ": truncated table values");
  return t;
}

void save_table_csv(const std::string& path, std::span<const double> values) {
  std::string text = "node_id,value\n";
  char buf[64];
  for (std::size_t i = 0; i < values.size(); ++i) {
    const int len = std::snprintf(buf, sizeof buf, "%zu,%.17g\n", i, values[i]);
    text.append(buf, static_cast<std::size_t>(len));
  }
  write_text_file(path, text, "csv");
}

std::string placement_to_json_text(const PlacementPlan& plan) {
  // nlohmann ordered_json::dump(2) layout (placement.cpp:406-422)
  std::ostringstream o;
  o << "{\n  \"feature_count\": " << plan.feature_count << ",\n  \"features\": ";
  if (plan.feature_count == 0) o << "[]";
  else {
    o << "[\n";
    for (std::uint64_t f = 0; f < plan.feature_count; ++f) {
      o << "    {\n      \"id\": " << f << ",\n      \"locations\": ";
      const auto& locs = plan.locations[f];
      if (locs.empty()) o << "[]";
      else {
        o << "[\n";
        for (std::size_t i = 0; i < locs.size(); ++i) {
          const Location& l = locs[i];
          json_escape_free_write(o, 8);
          o << "{\n          \"server\": " << l.server << ",\n          \"tier\": \""
            << tier_name(l.tier) << "\",\n          \"device\": " << l.device
            << ",\n          \"replica\": " << (l.replica ? "true" : "false") << "\n        }"
            << (i + 1 < locs.size() ? ",\n" : "\n");
        }
        o << "      ]";
      }
      o << "\n    }" << (f + 1 < plan.feature_count ? ",\n" : "\n");
    }
    o << "  ]";
  }
  o << "\n}\n";
  return o.str();
}

void save_placement_csv(const PlacementPlan& plan, const std::string& path) {
  std::string text = "feature_id,server,tier,device,replica\n";
  for (std::uint64_t f = 0; f < plan.feature_count; ++f)
    for (const Location& l : plan.locations[f])
      text += std::to_string(f) + ',' + std::to_string(l.server) + ',' + tier_name(l.tier) + ',' +
              std::to_string(l.device) + ',' + (l.replica ? '1' : '0') + '\n';
  write_text_file(path, text, "csv");
}

std::string lookup_to_json_text(const FeatureLookupTable& table) {
  // nlohmann ordered_json::dump(2) layout (placement.cpp:437-449)
  std::ostringstream o;
  o << "{\n  \"home_server\": " << table.home_server << ",\n  \"gpus_per_server\": "
    << table.gpus_per_server << ",\n  \"rows\": ";
  const std::size_t n = table.location_ids.size();
  if (n == 0) o << "[]";
  else {
    o << "[\n";
    for (std::size_t f = 0; f < n; ++f)
      o << "    {\n      \"feature\": " << f << ",\n      \"location\": " << table.location_ids[f]
        << ",\n      \"offset\": " << table.offsets[f] << "\n    }" << (f + 1 < n ? ",\n" : "\n");
    o << "  ]";
  }
  o << "\n}\n";
  return o.str();
}

void save_lookup_csv(const FeatureLookupTable& table, const std::string& path) {
  std::string text = "feature_id,location_id,offset\n";
  for (std::size_t f = 0; f < table.location_ids.size(); ++f)
    text += std::to_string(f) + ',' + std::to_string(table.location_ids[f]) + ',' +
            std::to_string(table.offsets[f]) + '\n';
  write_text_file(path, text, "csv");
}

// ---- feature store ----------------------------------------------------------------
FeatureStore::FeatureStore(const PlacementPlan& plan, const ClusterTopology& topo,
                           std::uint32_t dim, std::uint32_t reader_device,
                           std::span<const float> features, int cuda_device)
    : dim_(dim) {
  qvb_topology c = to_c(topo);
  PlanCsr csr = to_csr(plan, topo);
  if (!features.empty() && features.size() != plan.feature_count * dim)
    throw ValidationError("features must hold feature_count x dim values");
  check(qvb_store_create(cuda_device >= 0 ? cuda_device : static_cast<int>(reader_device),
                         csr.offsets.data(), csr.ids.data(), plan.feature_count, dim, &c,
                         reader_device, features.empty() ? nullptr : features.data(), &s_));
}

FeatureStore::~FeatureStore() {
  if (s_) qvb_store_destroy(s_);
}

std::array<std::uint8_t, 64> FeatureStore::export_handle() const {
  std::array<std::uint8_t, 64> h{};
  check(qvb_store_export_handle(s_, h.data()));
  return h;
}

void FeatureStore::attach_peer(std::uint32_t peer_device, const std::array<std::uint8_t, 64>& handle) {
  check(qvb_store_attach_peer(s_, peer_device, handle.data()));
}

void FeatureStore::gather(const std::uint64_t* d_ids, std::uint64_t count, float* d_out,
                          void* stream) const {
  check(qvb_gather(s_, d_ids, count, d_out, stream));
}

std::vector<float> FeatureStore::gather(std::span<const NodeId> ids) const {
  std::vector<float> out(ids.size() * dim_);
  check(qvb_gather_host(s_, ids.data(), ids.size(), out.data(), nullptr));
  return out;
}

}  // namespace qv
