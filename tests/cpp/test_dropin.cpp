// test_dropin.cpp — the reference's own hot-path test cases, restated against
// the qv:: drop-in (paper_2305_10863_b200/cpp/qv_b200.hpp) — the C++ API a
// reference user links. Cases follow tests/test_metrics.cpp:136-235 and
// tests/test_placement.cpp:72-465 of /root/reference/proj; expected values
// come from those tests, from tests/golden (reference outputs) and from the
// C oracle (liboracle.so). Built and run by tests/test_cpp_dropin_gpu.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <set>
#include <string>
#include <vector>

#include "../../oracle/oracle.h"
#include "../../paper_2305_10863_b200/cpp/qv_b200.hpp"

using namespace qv;

static int g_checks = 0, g_fail = 0;
static const char* g_outdir = nullptr;
#define CHECK(x)                                                            \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(x)) {                                                             \
      ++g_fail;                                                             \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #x); \
    }                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, T, substr)                                    \
  do {                                                                      \
    ++g_checks;                                                             \
    bool ok = false;                                                        \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const T& e) {                                                  \
      ok = std::string(e.what()).find(substr) != std::string::npos;         \
    } catch (...) {                                                         \
    }                                                                       \
    if (!ok) {                                                              \
      ++g_fail;                                                             \
      std::fprintf(stderr, "%s:%d: expected %s(%s) from %s\n", __FILE__, __LINE__, #T, substr, #expr); \
    }                                                                       \
  } while (0)

namespace {

uint64_t g_state;
uint64_t next_u() {
  g_state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = g_state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
double uniform() { return static_cast<double>(next_u() >> 11) * 0x1.0p-53; }
uint64_t below(uint64_t n) { return (uint64_t)(((unsigned __int128)next_u() * n) >> 64); }

Graph random_graph(uint64_t max_nodes, uint64_t max_edges, bool weighted) {  // testutil.hpp:43-55
  uint64_t n = 2 + below(max_nodes - 1);
  uint64_t m = 1 + below(max_edges);
  std::vector<Edge> edges;
  for (uint64_t e = 0; e < m; ++e) {
    const uint64_t s = below(n), d = below(n);
    edges.push_back({s, d, weighted ? 0.25 + uniform() : 1.0});
  }
  return Graph::from_edges(n, edges);
}

Graph fig8_graph() {  // testutil.hpp:32-36
  std::vector<Edge> e = {{0, 3, 1.0}, {0, 5, 1.0}, {1, 3, 1.0}, {3, 2, 1.0}, {4, 0, 1.0}};
  return Graph::from_edges(6, e);
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 8) == 0;
}

std::vector<double> oracle_p(const Graph& g, uint32_t L) {
  std::vector<double> out(g.node_count);
  qvo_access_prob(g.node_count, g.edge_count, g.row_offsets.data(), g.col_indices.data(),
                  g.edge_weights.data(), L, out.data());
  return out;
}

FapTable five_features() {  // test_placement.cpp:18-24
  FapTable f;
  f.values = {0.5, 0.4, 0.3, 0.2, 0.1};
  f.hops = 2;
  f.seed_distribution.assign(5, 0.2);
  return f;
}

std::set<std::pair<uint32_t, uint32_t>> gpu_copies(const PlacementPlan& p, NodeId f) {
  std::set<std::pair<uint32_t, uint32_t>> out;
  for (const Location& l : p.locations[f])
    if (l.tier == Tier::gpu) out.insert({l.server, l.device});
  return out;
}

ClusterTopology one_server_2numa_4gpu(bool nvlink) {
  ClusterTopology t = ClusterTopology::with_defaults();
  t.numa_per_server = 2;
  t.gpus_per_server = 4;
  t.gpu_feature_capacity = 1;
  t.host_feature_capacity = 4;
  t.disk_feature_capacity = 8;
  t.nvlink_within_numa = nvlink;
  return t;
}

ClusterTopology two_servers(bool ib) {
  ClusterTopology t = ClusterTopology::with_defaults();
  t.servers = 2;
  t.gpus_per_server = 1;
  t.gpu_feature_capacity = 1;
  t.host_feature_capacity = 1;
  t.disk_feature_capacity = 3;
  t.infiniband = ib;
  return t;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1) g_outdir = argv[1];
  // --- P(n,j): test_metrics.cpp:136-235 --------------------------------------
  {
    Graph g = fig8_graph();
    TransitionView t = transition_view(g);
    AccessProbTable a1 = compute_access_prob_ie(g, t, 1);
    for (double v : a1.values) CHECK(std::abs(v - 1.0 / 6) < 1e-14);
    const std::vector<double> p2 = {0.30555555555555552, 0.16666666666666666, 0.30555555555555552,
                                    0.36342592592592593, 0.16666666666666666, 0.23611111111111113};
    const std::vector<double> p3 = {0.42129629629629622, 0.16666666666666666, 0.55793467078189296,
                                    0.55056691529492463, 0.16666666666666666, 0.35281635802469136};
    CHECK(same_bits(compute_access_prob_ie(g, t, 2).values, p2));
    CHECK(same_bits(compute_access_prob_ie(g, t, 3).values, p3));
    CHECK_THROWS_AS(compute_access_prob_ie(g, t, 0), ValidationError, "layers");
  }
  {
    Graph g = Graph::from_edges(3, std::vector<Edge>{{1, 0, 1.0}, {1, 2, 1.0}});
    AccessProbTable a = compute_access_prob_ie(g, transition_view(g), 2);
    const double base = 1.0 / 3.0;
    CHECK(std::abs(a.values[0] - (base + (1.0 - base) * (base * 0.5))) < 1e-14);
  }
  g_state = 0x1234;
  for (int it = 0; it < 30; ++it) {
    Graph g = random_graph(40, 250, it % 2 == 0);
    TransitionView t = transition_view(g);
    for (uint32_t L = 1; L <= 4; ++L) {
      CHECK(same_bits(compute_access_prob_ie(g, t, L).values, oracle_p(g, L)));
      CHECK(same_bits(serial::compute_access_prob_ie(g, t, L).values, oracle_p(g, L)));
    }
    Graph tg = in_adjacency(g);
    std::vector<uint64_t> tro(g.node_count + 1), tcol(g.edge_count);
    std::vector<double> tw(g.edge_count);
    qvo_in_adjacency(g.node_count, g.edge_count, g.row_offsets.data(), g.col_indices.data(),
                     g.edge_weights.data(), tro.data(), tcol.data(), tw.data());
    CHECK(tg.row_offsets == tro && tg.col_indices == tcol && same_bits(tg.edge_weights, tw));
  }
  {  // FAP (test_metrics.cpp): the worked example's node 3 has visit mass 1/2 at K=2
    Graph g = fig8_graph();
    TransitionView t = transition_view(g);
    FapTable f = compute_fap(t, 2);
    CHECK(std::abs(f.values[3] - 0.5) < 1e-12);
    std::vector<double> exp(g.node_count);
    qvo_compute_fap(g.node_count, g.edge_count, g.row_offsets.data(), g.col_indices.data(),
                    g.edge_weights.data(), 2, nullptr, exp.data());
    CHECK(same_bits(f.values, exp));
    std::vector<double> bad(g.node_count, 1.0);
    CHECK_THROWS_AS(compute_fap(t, 2, std::span<const double>(bad)), ValidationError,
                    "does not sum to 1");
  }
  {
    Graph g = fig8_graph();
    g.edge_weights[3] = -1.0;
    CHECK_THROWS_AS(compute_access_prob_ie(g, TransitionView{}, 2), ValidationError,
                    "negative or NaN edge weight at node 3");
  }

  // --- placement: test_placement.cpp:72-145 -----------------------------------
  {
    ClusterTopology topo = one_server_2numa_4gpu(false);
    PlacementPlan plan = plan_placement(five_features(), topo);
    plan.validate(topo);
    CHECK((gpu_copies(plan, 0) == std::set<std::pair<uint32_t, uint32_t>>{{0, 0}, {0, 1}, {0, 2}, {0, 3}}));
    for (NodeId f = 1; f < 5; ++f)
      CHECK(plan.locations[f].size() == 1 && plan.locations[f][0].tier == Tier::host);
  }
  {
    ClusterTopology topo = one_server_2numa_4gpu(true);
    PlacementPlan plan = plan_placement(five_features(), topo);
    CHECK((gpu_copies(plan, 0) == std::set<std::pair<uint32_t, uint32_t>>{{0, 0}, {0, 2}}));
    CHECK((gpu_copies(plan, 1) == std::set<std::pair<uint32_t, uint32_t>>{{0, 1}, {0, 3}}));
    CHECK(plan.locations[0][0].replica == false && plan.locations[0][1].replica == true);
    FeatureLookupTable table = build_lookup_table(plan, topo, 0);
    DeviceRef gpu0{0, Tier::gpu, 0};
    CHECK(classify_link(topo, gpu0, table.location_ids[0]).first == LinkClass::local);
    CHECK(classify_link(topo, gpu0, table.location_ids[1]).first == LinkClass::nvlink);
    // SURVEY §8(c) golden: f0(0,0) f1(1,0) f2(4,0) f3(4,1) f4(4,2)
    CHECK((table.location_ids == std::vector<int64_t>{0, 1, 4, 4, 4}));
    CHECK((table.offsets == std::vector<uint64_t>{0, 0, 0, 1, 2}));
    if (g_outdir) {  // reference-format exports, compared with golden texts by the test
      const std::string d = g_outdir;
      std::ofstream(d + "/placement_b.json") << placement_to_json_text(plan);
      save_placement_csv(plan, d + "/placement_b.csv");
      std::ofstream(d + "/lookup_b.json") << lookup_to_json_text(table);
      save_lookup_csv(table, d + "/lookup_b.csv");
      Graph f8 = fig8_graph();
      save_graph_csr(f8, d + "/fig8.qvcsr");
      Graph back = load_graph(d + "/fig8.qvcsr", GraphFormat::csr_binary);
      CHECK(back.row_offsets == f8.row_offsets && back.col_indices == f8.col_indices);
      std::vector<double> tab = {0.5, 1.0 / 3.0, 1e-300, 12345.678};
      save_table_binary(d + "/table.qvtab", tab, 2);
      save_table_csv(d + "/table.csv", tab);
      LoadedTable lt = load_table_binary(d + "/table.qvtab");
      CHECK(lt.k == 2 && same_bits(lt.values, tab));
      CHECK_THROWS_AS(load_graph(d + "/table.qvtab", GraphFormat::csr_binary), ParseError, "bad magic");
    }
    std::vector<NodeId> ids = {4, 1, 0, 3, 1};
    ReadPlan rp = plan_reads(table, ids, 2);
    CHECK(rp.per_location.size() == 3);
    CHECK(rp.per_location[1].location_id == 1 && rp.per_location[1].offsets.size() == 2);
    CHECK(rp.per_location[2].page_transitions == 2);
  }
  {
    ClusterTopology topo = two_servers(true);
    PlacementPlan plan = plan_placement(five_features(), topo);
    for (NodeId f = 0; f < 4; ++f) {
      CHECK(plan.locations[f].size() == 1);
      CHECK(plan.locations[f][0].server == (f < 2 ? 0u : 1u));
    }
    CHECK(plan.locations[4][0].tier == Tier::disk);
    FeatureLookupTable table = build_lookup_table(plan, topo, 0);
    CHECK_THROWS_AS(plan_reads(table, std::vector<NodeId>{0, 99}, 4), ValidationError,
                    "feature id 99 outside lookup table");
    CHECK_THROWS_AS(plan_reads(table, std::vector<NodeId>{0}, 0), ValidationError, "page size");
  }
  {
    ClusterTopology topo = two_servers(false);
    topo.disk_feature_capacity = 0;
    topo.host_feature_capacity = 1;
    CHECK_THROWS_AS(plan_placement(five_features(), topo), PlacementError, "short by 3");
  }
  {
    std::vector<uint64_t> u = {2, 10, 3, 11}, s = {2, 3, 10, 11};
    CHECK(page_transitions(u, 2) == 4 && page_transitions(s, 2) == 2);
  }
  {  // fetch_cost tail rule (test_placement.cpp:332-372)
    ClusterTopology topo = ClusterTopology::with_defaults();
    ReadPlan empty;
    CHECK(fetch_cost(empty, topo, 1024).total_s == 0.0);
    ClusterTopology fast = topo;
    fast.links[static_cast<std::size_t>(LinkClass::pcie)] = {0.0, 16e9};
    fast.tlb_miss_penalty_s = 0.0;
    ReadPlan one;
    ReadPlan::LocationReads lr;
    lr.location_id = encode_location(fast, 0, Tier::host, 0);
    lr.offsets = {0};
    lr.page_transitions = 1;
    one.per_location.push_back(lr);
    CHECK(std::abs(fetch_cost(one, fast, 1000000000).total_s - 0.0625) < 1e-12);
  }

  // --- feature store: the real collect ------------------------------------------
  {
    const uint64_t n = 5000;
    const uint32_t dim = 100;
    ClusterTopology topo = ClusterTopology::with_defaults();
    topo.gpu_feature_capacity = n / 2;
    topo.host_feature_capacity = n;
    FapTable fap;
    for (uint64_t i = 0; i < n; ++i) fap.values.push_back(uniform());
    PlacementPlan plan = plan_placement(fap, topo);
    std::vector<float> x(n * dim);
    qvo_features(0, n, dim, x.data());
    FeatureStore store(plan, topo, dim, 0);
    std::vector<NodeId> ids(777);
    for (auto& i : ids) i = below(n);
    std::vector<float> got = store.gather(ids);
    bool ok = true;
    for (size_t r = 0; r < ids.size(); ++r)
      ok &= std::memcmp(got.data() + r * dim, x.data() + ids[r] * dim, dim * 4) == 0;
    CHECK(ok);
    CHECK_THROWS_AS(store.gather(std::vector<NodeId>{n}), ValidationError, "outside lookup table");
    // the per-batch read plan over the store's resident table == the table's
    FeatureLookupTable table = build_lookup_table(plan, topo, 0);
    for (uint64_t page : {1, 3, 8}) {
      ReadPlan a = plan_reads(table, ids, page), b = plan_reads(store, ids, page);
      bool same = a.per_location.size() == b.per_location.size();
      for (size_t k = 0; same && k < a.per_location.size(); ++k)
        same = a.per_location[k].location_id == b.per_location[k].location_id &&
               a.per_location[k].offsets == b.per_location[k].offsets &&
               a.per_location[k].page_transitions == b.per_location[k].page_transitions;
      CHECK(same);
    }
    CHECK_THROWS_AS(plan_reads(store, std::vector<NodeId>{0, n}, 8), ValidationError, "outside lookup table");
  }
  {  // transition_view keeps the device graph; a view of another graph falls back to an upload
    Graph g = random_graph(60, 400, true);
    Graph h = random_graph(60, 400, false);
    TransitionView tg = transition_view(g);
    CHECK(tg.resident_for(g) && !tg.resident_for(h));
    for (uint32_t L = 1; L <= 3; ++L) {
      CHECK(same_bits(compute_access_prob_ie(g, tg, L).values, oracle_p(g, L)));
      CHECK(same_bits(compute_access_prob_ie(h, tg, L).values, oracle_p(h, L)));
    }
    Graph g2 = g;  // a copy owns new arrays: no stale device graph is used for it
    g2.edge_weights[0] *= 2.0;
    CHECK(!tg.resident_for(g2));
    CHECK(same_bits(compute_access_prob_ie(g2, transition_view(g2), 3).values, oracle_p(g2, 3)));
  }

  // --- sampler: test_sampler.cpp:15-150, vs the oracle restatement ------------
  {
    Graph g = fig8_graph();
    TransitionView t = transition_view(g);
    SampleResult r = sample_khop(t, 4, SamplingConfig{{10, 10}}, 1);
    CHECK(r.frontiers[0] == std::vector<NodeId>{4});
    CHECK(r.frontiers[1] == std::vector<NodeId>{0});
    CHECK((std::set<NodeId>(r.frontiers[2].begin(), r.frontiers[2].end()) == std::set<NodeId>{3, 5}));
    CHECK(r.total_instances() == 4);
    Graph c3 = Graph::from_edges(3, std::vector<Edge>{{0, 1, 1.0}, {1, 2, 1.0}});
    SampleResult c = sample_khop(transition_view(c3), 0, SamplingConfig{{1, 1}}, 99);
    CHECK(c.frontiers[2] == std::vector<NodeId>{2});
    CHECK_THROWS_AS(sample_khop(transition_view(c3), 3, SamplingConfig{{1}}, 1), ValidationError,
                    "out of range");
    std::vector<NodeId> bad = {0, 7};
    CHECK_THROWS_AS(batch_sample(transition_view(c3), bad, SamplingConfig{{1}}, 1), ValidationError,
                    "position 1");
    CHECK_THROWS_AS(batch_sample(t, bad, SamplingConfig{{}}, 1), ValidationError, ">= 1 hop");
    std::vector<NodeId> none;
    BatchSampleResult e = batch_sample(t, none, SamplingConfig{{2, 2}}, 5);
    CHECK(e.per_seed.empty() && e.stats.total_instances == 0 && e.stats.unique_count == 0);
    std::vector<NodeId> dup = {0, 0, 3, 0};
    BatchSampleResult d = batch_sample(t, dup, SamplingConfig{{2, 2}}, 7);
    CHECK(d.per_seed[0].frontiers == d.per_seed[1].frontiers);
    CHECK(d.per_seed[0].frontiers == d.per_seed[3].frontiers);
  }
  g_state = 0x5A4D;
  for (int it = 0; it < 20; ++it) {
    Graph g = random_graph(50, 400, it % 2 == 0);
    TransitionView t = transition_view(g);
    SamplingConfig cfg{{static_cast<uint32_t>(1 + below(4)), static_cast<uint32_t>(1 + below(4))}};
    std::vector<NodeId> seeds(30);
    for (auto& s : seeds) s = below(g.node_count);
    const uint64_t rng = 1000 + it;
    Sampler smp(g);
    BatchSampleResult r = smp.batch_sample(seeds, cfg, rng);
    uint64_t total = 0, uc = 0;
    qvo_batch_sample(g.node_count, g.edge_count, g.row_offsets.data(), g.col_indices.data(),
                     g.edge_weights.data(), seeds.data(), seeds.size(), cfg.fanouts.data(), 2, rng,
                     &total, &uc, nullptr, nullptr, nullptr);
    std::vector<uint64_t> nodes(total), counts(seeds.size() * 3), uniq(uc);
    qvo_batch_sample(g.node_count, g.edge_count, g.row_offsets.data(), g.col_indices.data(),
                     g.edge_weights.data(), seeds.data(), seeds.size(), cfg.fanouts.data(), 2, rng,
                     &total, &uc, nodes.data(), counts.data(), uniq.data());
    std::vector<uint64_t> flat;
    for (const SampleResult& sr : r.per_seed)
      for (const auto& f : sr.frontiers) flat.insert(flat.end(), f.begin(), f.end());
    CHECK(flat == nodes);
    CHECK(r.stats.unique_nodes == uniq);
    CHECK(smp.batch_stats(seeds, cfg, rng).unique_nodes == uniq);
    // sample_khop(seed, rs) == the seed's part of a batch run under rng
    const NodeId s0 = seeds[0];
    const uint64_t rs = qvo_splitmix64(rng ^ (s0 * 0x9e3779b97f4a7c15ULL));
    CHECK(sample_khop(t, s0, cfg, rs).frontiers == r.per_seed[0].frontiers);
  }

  std::printf("test_dropin: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
