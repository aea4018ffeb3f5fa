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
Graph Graph::from_edges(std::uint64_t node_count, std::span<const Edge> edges) {
  // build_csr semantics (graph.cpp:16-56): counting sort by source, input
  // order kept inside a row; input construction, not the hot path.
  if (node_count == 0) throw ValidationError("empty graph: node count is zero");
  Graph g;
  g.node_count = node_count;
  g.edge_count = edges.size();
  g.row_offsets.assign(node_count + 1, 0);
  for (const Edge& e : edges) {
    if (e.src >= node_count || e.dst >= node_count)
      throw ValidationError("edge endpoint " + std::to_string(std::max(e.src, e.dst)) +
                            " out of range for node count " + std::to_string(node_count));
    if (!(e.weight >= 0.0))
      throw ValidationError("negative or NaN edge weight on edge " + std::to_string(e.src) +
                            " -> " + std::to_string(e.dst));
    ++g.row_offsets[e.src + 1];
  }
  std::partial_sum(g.row_offsets.begin(), g.row_offsets.end(), g.row_offsets.begin());
  g.col_indices.resize(g.edge_count);
  g.edge_weights.resize(g.edge_count);
  std::vector<EdgeIdx> cursor(g.row_offsets.begin(), g.row_offsets.end() - 1);
  for (const Edge& e : edges) {
    const EdgeIdx at = cursor[e.src]++;
    g.col_indices[at] = e.dst;
    g.edge_weights[at] = e.weight;
  }
  g.validate();
  return g;
}

void Graph::validate() const {
  // the device validates on upload with the reference's messages
  // (graph.cpp:58-93); host-side size checks come first, as there
  if (node_count == 0) throw ValidationError("empty graph: node count is zero");
  if (row_offsets.size() != node_count + 1) throw ValidationError("row_offsets size mismatch");
  if (row_offsets.front() != 0 || row_offsets.back() != edge_count)
    throw ValidationError("row_offsets endpoints invalid");
  if (col_indices.size() != edge_count || edge_weights.size() != edge_count)
    throw ValidationError("edge array size mismatch");
  for (std::uint64_t i = 0; i < node_count; ++i)
    if (row_offsets[i + 1] < row_offsets[i])
      throw ValidationError("row_offsets not non-decreasing at node " + std::to_string(i));
  for (std::uint64_t i = 0; i < node_count; ++i) {
    bool any_positive = out_degree(i) == 0;
    for (EdgeIdx e = row_offsets[i]; e < row_offsets[i + 1]; ++e) {
      if (col_indices[e] >= node_count)
        throw ValidationError("column index out of range at node " + std::to_string(i));
      if (!(edge_weights[e] >= 0.0))
        throw ValidationError("negative or NaN edge weight at node " + std::to_string(i));
      if (edge_weights[e] > 0.0) any_positive = true;
    }
    if (!any_positive)
      throw ValidationError("node " + std::to_string(i) + " has out-edges but all weights are zero");
  }
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
  if (row_sums[i] <= 0.0) return 0.0;
  double w = 0.0;
  for (EdgeIdx e = graph->row_offsets[i]; e < graph->row_offsets[i + 1]; ++e)
    if (graph->col_indices[e] == j) w += graph->edge_weights[e];
  return w / row_sums[i];
}

TransitionView transition_view(const Graph& g) {
  g.validate();
  TransitionView t;
  t.graph = &g;
  t.row_sums.assign(g.node_count, 0.0);
  t.distinct_out.assign(g.node_count, 0);
  std::vector<std::uint64_t> stamp(g.node_count, ~0ULL);
  for (NodeId i = 0; i < g.node_count; ++i) {
    double sum = 0.0;
    std::uint64_t distinct = 0;
    for (EdgeIdx e = g.row_offsets[i]; e < g.row_offsets[i + 1]; ++e) {
      sum += g.edge_weights[e];
      const NodeId j = g.col_indices[e];
      if (stamp[j] != i) {
        stamp[j] = i;
        ++distinct;
      } else {
        t.has_parallel_edges = true;
      }
    }
    t.row_sums[i] = sum;
    t.distinct_out[i] = distinct;
  }
  return t;
}

// ---- metrics ------------------------------------------------------------------
AccessProbTable compute_access_prob_ie(const Graph& g, const TransitionView&,
                                       std::uint32_t layers) {
  if (layers < 1) throw ValidationError("access probability needs layers >= 1");
  AccessProbTable t;
  t.layers = layers;
  t.values.resize(g.node_count);
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
  std::map<std::int64_t, std::uint64_t> counts;
  for (std::uint64_t f = 0; f < feature_count; ++f) {
    if (locations[f].empty()) throw Error("feature " + std::to_string(f) + " has no location");
    for (const Location& l : locations[f]) ++counts[encode_location(topo, l.server, l.tier, l.device)];
  }
  for (const auto& [id, count] : counts) {
    const Location l = decode_location(topo, id);
    const std::uint64_t cap = l.tier == Tier::gpu    ? topo.gpu_feature_capacity
                              : l.tier == Tier::host ? topo.host_feature_capacity
                                                     : topo.disk_feature_capacity;
    if (count > cap)
      throw Error(std::string("placement overfills ") + tier_name(l.tier) + " on server " +
                  std::to_string(l.server) + ": " + std::to_string(count) + " > " +
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

LinkPath classify_link(const ClusterTopology& topo, const DeviceRef& reader,
                       std::int64_t location_id) {
  // placement.cpp:228-267 (host arithmetic of the cost model)
  const Location loc = decode_location(topo, location_id);
  LinkPath path;
  if (loc.server == reader.server) {
    switch (loc.tier) {
      case Tier::gpu:
        if (reader.tier == Tier::gpu) {
          if (reader.device == loc.device) path.first = LinkClass::local;
          else if (topo.gpus_per_numa() > 0 &&
                   reader.device / topo.gpus_per_numa() == loc.device / topo.gpus_per_numa())
            path.first = topo.nvlink_within_numa ? LinkClass::nvlink : LinkClass::pcie;
          else path.first = LinkClass::upi;
        } else {
          path.first = LinkClass::pcie;
        }
        break;
      case Tier::host:
        path.first = reader.tier == Tier::host ? LinkClass::local : LinkClass::pcie;
        break;
      case Tier::disk: path.first = LinkClass::disk; break;
    }
  } else {
    const LinkClass net = topo.infiniband ? LinkClass::infiniband : LinkClass::ethernet;
    if (loc.tier == Tier::disk) {
      path.first = LinkClass::disk;
      path.second = net;
    } else {
      path.first = net;
    }
  }
  return path;
}

FetchCost fetch_cost(const ReadPlan& plan, const ClusterTopology& topo,
                     std::uint64_t feature_bytes, std::optional<DeviceRef> reader) {
  // placement.cpp:382-404 — the reference's model, unchanged in meaning
  auto translated = [](LinkClass c) {
    return c == LinkClass::pcie || c == LinkClass::upi || c == LinkClass::infiniband ||
           c == LinkClass::ethernet;
  };
  DeviceRef rd = reader ? *reader
                        : (topo.gpus_per_server > 0 ? DeviceRef{plan.home_server, Tier::gpu, 0}
                                                    : DeviceRef{plan.home_server, Tier::host, 0});
  FetchCost cost;
  const std::int64_t max_loc =
      static_cast<std::int64_t>(topo.servers) * static_cast<std::int64_t>(topo.gpus_per_server + 2);
  for (const auto& lr : plan.per_location) {
    if (lr.location_id < 0 || lr.location_id >= max_loc)
      throw ValidationError("unknown location id " + std::to_string(lr.location_id));
    const LinkPath p = classify_link(topo, rd, lr.location_id);
    double setup = topo.link(p.first).latency_s;
    double bw = topo.link(p.first).bandwidth_Bps;
    if (p.second) {
      setup += topo.link(*p.second).latency_s;
      bw = std::min(bw, topo.link(*p.second).bandwidth_Bps);
    }
    const double bytes = static_cast<double>(feature_bytes) * static_cast<double>(lr.offsets.size());
    double lat = setup + bytes / bw;
    if (translated(p.first) || (p.second && translated(*p.second)))
      lat += topo.tlb_miss_penalty_s * static_cast<double>(lr.page_transitions);
    cost.per_location_s.emplace_back(lr.location_id, lat);
    cost.total_s = std::max(cost.total_s, lat);
  }
  return cost;
}

// ---- on-disk formats ----------------------------------------------------------------
namespace {
constexpr char kCsrMagic[6] = {'Q', 'V', 'C', 'S', 'R', '1'};
constexpr char kTabMagic[6] = {'Q', 'V', 'T', 'A', 'B', '1'};

template <typename T>
void read_pod(std::ifstream& in, T* p, std::size_t n, const std::string& path, const char* what) {
  in.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(sizeof(T) * n));
  if (!in) throw ParseError(path + what);
}

Graph load_edge_list(const std::string& path, bool remap) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open graph file: " + path);
  std::vector<Edge> edges;
  std::string line;
  std::uint64_t line_no = 0;
  NodeId max_id = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    std::istringstream ls(line);
    std::uint64_t src, dst;
    if (!(ls >> src)) {
      std::string left;
      std::istringstream probe(line);
      if (probe >> left)
        throw ParseError(path + ":" + std::to_string(line_no) + ": malformed edge line: '" + line + "'");
      continue;
    }
    if (!(ls >> dst))
      throw ParseError(path + ":" + std::to_string(line_no) + ": malformed edge line: '" + line + "'");
    double w = 1.0;
    std::string rest;
    if (ls >> rest) {
      try {
        std::size_t used = 0;
        w = std::stod(rest, &used);
        if (used != rest.size()) throw std::invalid_argument(rest);
      } catch (const std::exception&) {
        throw ParseError(path + ":" + std::to_string(line_no) + ": malformed weight '" + rest + "'");
      }
      std::string extra;
      if (ls >> extra)
        throw ParseError(path + ":" + std::to_string(line_no) +
                         ": trailing tokens after weight: '" + extra + "'");
    }
    edges.push_back({src, dst, w});
    max_id = std::max(max_id, std::max(src, dst));
  }
  if (edges.empty()) throw ValidationError("empty graph: no edges in " + path);
  std::uint64_t n = max_id + 1;
  std::vector<bool> present(n, false);
  for (const Edge& e : edges) present[e.src] = present[e.dst] = true;
  if (!std::all_of(present.begin(), present.end(), [](bool b) { return b; })) {
    if (!remap)
      throw ValidationError(path + ": node ids are not contiguous 0..N-1 (use id remapping "
                                   "for sparse-id inputs)");
    std::vector<NodeId> map(n, 0);
    NodeId next = 0;
    for (NodeId i = 0; i < n; ++i)
      if (present[i]) map[i] = next++;
    for (Edge& e : edges) {
      e.src = map[e.src];
      e.dst = map[e.dst];
    }
    n = next;
  }
  return Graph::from_edges(n, edges);
}

void json_escape_free_write(std::ostringstream& o, int indent) {
  for (int i = 0; i < indent; ++i) o << ' ';
}
}  // namespace

Graph load_graph(const std::string& path, GraphFormat format, bool remap_sparse_ids) {
  if (format == GraphFormat::edge_list_text) return load_edge_list(path, remap_sparse_ids);
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open graph file: " + path);
  char magic[6];
  read_pod(in, magic, 6, path, ": truncated csr-binary file");
  if (std::memcmp(magic, kCsrMagic, 6) != 0) throw ParseError(path + ": bad magic, not a QVCSR1 file");
  Graph g;
  read_pod(in, &g.node_count, 1, path, ": truncated csr-binary file");
  read_pod(in, &g.edge_count, 1, path, ": truncated csr-binary file");
  if (g.node_count == 0) throw ValidationError("empty graph in " + path);
  g.row_offsets.resize(g.node_count + 1);
  g.col_indices.resize(g.edge_count);
  g.edge_weights.resize(g.edge_count);
  read_pod(in, g.row_offsets.data(), g.row_offsets.size(), path, ": truncated csr-binary file");
  read_pod(in, g.col_indices.data(), g.col_indices.size(), path, ": truncated csr-binary file");
  read_pod(in, g.edge_weights.data(), g.edge_weights.size(), path, ": truncated csr-binary file");
  g.validate();
  return g;
}

void save_graph_csr(const Graph& g, const std::string& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw Error("cannot write graph file: " + path);
  out.write(kCsrMagic, 6);
  out.write(reinterpret_cast<const char*>(&g.node_count), 8);
  out.write(reinterpret_cast<const char*>(&g.edge_count), 8);
  out.write(reinterpret_cast<const char*>(g.row_offsets.data()), g.row_offsets.size() * 8);
  out.write(reinterpret_cast<const char*>(g.col_indices.data()), g.col_indices.size() * 8);
  out.write(reinterpret_cast<const char*>(g.edge_weights.data()), g.edge_weights.size() * 8);
  if (!out) throw Error("short write to " + path);
}

void save_table_binary(const std::string& path, std::span<const double> values, std::uint64_t k) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw Error("cannot write table file: " + path);
  const std::uint64_t n = values.size();
  out.write(kTabMagic, 6);
  out.write(reinterpret_cast<const char*>(&n), 8);
  out.write(reinterpret_cast<const char*>(&k), 8);
  out.write(reinterpret_cast<const char*>(values.data()), n * 8);
  if (!out) throw Error("short write to " + path);
}

LoadedTable load_table_binary(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open table file: " + path);
  char magic[6];
  in.read(magic, 6);
  if (!in || std::memcmp(magic, kTabMagic, 6) != 0) throw ParseError(path + ": bad magic, not a QVTAB1 file");
  std::uint64_t n = 0;
  LoadedTable t;
  in.read(reinterpret_cast<char*>(&n), 8);
  in.read(reinterpret_cast<char*>(&t.k), 8);
  if (!in) throw ParseError(path + ": truncated table header");
  t.values.resize(n);
  in.read(reinterpret_cast<char*>(t.values.data()), n * 8);
  if (!in) throw ParseError(path + ": truncated table values");
  return t;
}

void save_table_csv(const std::string& path, std::span<const double> values) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw Error("cannot write csv file: " + path);
  out << "node_id,value\n";
  char buf[64];
  for (std::size_t i = 0; i < values.size(); ++i) {
    std::snprintf(buf, sizeof buf, "%zu,%.17g\n", i, values[i]);
    out << buf;
  }
  if (!out) throw Error("short write to " + path);
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
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw Error("cannot write csv file: " + path);
  out << "feature_id,server,tier,device,replica\n";
  for (std::uint64_t f = 0; f < plan.feature_count; ++f)
    for (const Location& l : plan.locations[f])
      out << f << ',' << l.server << ',' << tier_name(l.tier) << ',' << l.device << ','
          << (l.replica ? 1 : 0) << '\n';
  if (!out) throw Error("short write to " + path);
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
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw Error("cannot write csv file: " + path);
  out << "feature_id,location_id,offset\n";
  for (std::size_t f = 0; f < table.location_ids.size(); ++f)
    out << f << ',' << table.location_ids[f] << ',' << table.offsets[f] << '\n';
  if (!out) throw Error("short write to " + path);
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
