// ref_shim.cpp — extern "C" wrappers around the UNMODIFIED reference library.
// TEST INFRASTRUCTURE ONLY: compiled by oracle/Makefile together with the
// reference's own sources (/root/reference/proj/src/{graph,metrics,
// placement,topology}.cpp) into oracle/_ref/libqvref.so. Used to pin the C
// restatement (oracle.c), to generate tests/golden fixtures, and as the
// timed CPU baseline (bench.py cpu_baseline kind "reference").
// Nothing here re-implements reference logic; it only marshals arguments.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <span>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "qv/error.hpp"
#include "qv/graph.hpp"
#include "qv/metrics.hpp"
#include "qv/placement.hpp"
#include "qv/sampler.hpp"
#include "qv/topology.hpp"
#include "../include/qvb.h"

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const qv::PlacementError& e) {
    g_err = e.what();
    return QVB_ERR_PLACEMENT;
  } catch (const qv::ValidationError& e) {
    g_err = e.what();
    return QVB_ERR_VALIDATION;
  } catch (const qv::ParseError& e) {
    g_err = e.what();
    return QVB_ERR_VALIDATION;
  } catch (const qv::ConfigError& e) {
    g_err = e.what();
    return QVB_ERR_VALIDATION;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QVB_ERR_GENERIC;
  }
}

qv::Graph make_graph(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                     const double* w) {
  qv::Graph g;
  g.node_count = n;
  g.edge_count = e;
  g.row_offsets.assign(ro, ro + n + 1);
  g.col_indices.assign(col, col + e);
  if (w) g.edge_weights.assign(w, w + e);
  else g.edge_weights.assign(e, 1.0);
  return g;
}

qv::ClusterTopology make_topo(const qvb_topology* t) {
  qv::ClusterTopology c;
  c.servers = t->servers;
  c.numa_per_server = t->numa_per_server;
  c.gpus_per_server = t->gpus_per_server;
  c.gpu_feature_capacity = t->gpu_feature_capacity;
  c.host_feature_capacity = t->host_feature_capacity;
  c.disk_feature_capacity = t->disk_feature_capacity;
  c.nvlink_within_numa = t->nvlink_within_numa != 0;
  c.infiniband = t->infiniband != 0;
  for (std::size_t i = 0; i < qv::kLinkClassCount; ++i) {
    c.links[i].latency_s = t->link_latency_s[i];
    c.links[i].bandwidth_Bps = t->link_bandwidth_Bps[i];
  }
  c.tlb_miss_penalty_s = t->tlb_miss_penalty_s;
  if (t->gpu_replicated_capacity != 0)
    throw qv::ValidationError("reference has no gpu_replicated_capacity extension");
  return c;
}

qv::PlacementPlan make_plan(const uint64_t* lo, const int64_t* ids, uint64_t n,
                            const qv::ClusterTopology& topo) {
  qv::PlacementPlan p;
  p.feature_count = n;
  p.locations.resize(n);
  for (uint64_t f = 0; f < n; ++f) {
    for (uint64_t k = lo[f]; k < lo[f + 1]; ++k) {
      qv::Location l = qv::decode_location(topo, ids[k]);
      l.replica = k > lo[f];
      p.locations[f].push_back(l);
    }
  }
  return p;
}
}  // namespace

extern "C" {

const char* qvr_last_error(void) { return g_err.c_str(); }

int qvr_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void qvr_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

void qvr_topology_defaults(qvb_topology* t) {
  qv::ClusterTopology c = qv::ClusterTopology::with_defaults();
  std::memset(t, 0, sizeof *t);
  t->servers = c.servers;
  t->numa_per_server = c.numa_per_server;
  t->gpus_per_server = c.gpus_per_server;
  t->gpu_feature_capacity = c.gpu_feature_capacity;
  t->host_feature_capacity = c.host_feature_capacity;
  t->disk_feature_capacity = c.disk_feature_capacity;
  t->nvlink_within_numa = c.nvlink_within_numa;
  t->infiniband = c.infiniband;
  for (std::size_t i = 0; i < qv::kLinkClassCount; ++i) {
    t->link_latency_s[i] = c.links[i].latency_s;
    t->link_bandwidth_Bps[i] = c.links[i].bandwidth_Bps;
  }
  t->tlb_miss_penalty_s = c.tlb_miss_penalty_s;
}

// qv::compute_access_prob_ie / qv::serial::compute_access_prob_ie; ms_out
// (nullable) receives the wall time of the call alone (graph marshalling
// excluded).
int qvr_access_prob(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                    const double* w, uint32_t layers, int parallel, double* out, double* ms_out) {
  return guard([&] {
    qv::Graph g = make_graph(n, e, ro, col, w);
    qv::TransitionView t = qv::transition_view(g);
    auto t0 = std::chrono::steady_clock::now();
    qv::AccessProbTable a = parallel ? qv::compute_access_prob_ie(g, t, layers)
                                     : qv::serial::compute_access_prob_ie(g, t, layers);
    auto t1 = std::chrono::steady_clock::now();
    if (ms_out) *ms_out = std::chrono::duration<double, std::milli>(t1 - t0).count();
    std::memcpy(out, a.values.data(), n * sizeof(double));
  });
}

int qvr_compute_fap(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                    const double* w, uint32_t hops, int parallel, const double* seed,
                    double* values) {
  return guard([&] {
    qv::Graph g = make_graph(n, e, ro, col, w);
    qv::TransitionView t = qv::transition_view(g);
    std::optional<std::span<const double>> sd;
    if (seed) sd = std::span<const double>(seed, n);
    qv::FapTable f = parallel ? qv::compute_fap(t, hops, sd) : qv::serial::compute_fap(t, hops, sd);
    std::memcpy(values, f.values.data(), n * sizeof(double));
  });
}

int qvr_in_adjacency(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                     const double* w, uint64_t* tro, uint64_t* tcol, double* tw) {
  return guard([&] {
    qv::Graph g = make_graph(n, e, ro, col, w);
    qv::Graph t = qv::in_adjacency(g);
    std::memcpy(tro, t.row_offsets.data(), (n + 1) * sizeof(uint64_t));
    std::memcpy(tcol, t.col_indices.data(), e * sizeof(uint64_t));
    std::memcpy(tw, t.edge_weights.data(), e * sizeof(double));
  });
}

int qvr_row_sums(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col, const double* w,
                 double* rs) {
  return guard([&] {
    qv::Graph g = make_graph(n, e, ro, col, w);
    qv::TransitionView t = qv::transition_view(g);
    std::memcpy(rs, t.row_sums.data(), n * sizeof(double));
  });
}

int qvr_transition_view(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                        const double* w, double* rs, uint64_t* distinct, int* parallel) {
  return guard([&] {
    qv::Graph g = make_graph(n, e, ro, col, w);
    qv::TransitionView t = qv::transition_view(g);
    std::memcpy(rs, t.row_sums.data(), n * sizeof(double));
    std::memcpy(distinct, t.distinct_out.data(), n * sizeof(uint64_t));
    *parallel = t.has_parallel_edges ? 1 : 0;
  });
}

/* Graph::from_edges over struct-of-arrays edges (the shim only marshals) */
int qvr_from_edges(uint64_t n, uint64_t e, const uint64_t* src, const uint64_t* dst, const double* w,
                   uint64_t* ro, uint64_t* col, double* wo) {
  return guard([&] {
    std::vector<qv::Edge> edges(e);
    for (uint64_t i = 0; i < e; ++i) edges[i] = qv::Edge{src[i], dst[i], w[i]};
    qv::Graph g = qv::Graph::from_edges(n, edges);
    std::memcpy(ro, g.row_offsets.data(), (n + 1) * sizeof(uint64_t));
    std::memcpy(col, g.col_indices.data(), e * sizeof(uint64_t));
    std::memcpy(wo, g.edge_weights.data(), e * sizeof(double));
  });
}

int qvr_validate(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col, const double* w) {
  return guard([&] { make_graph(n, e, ro, col, w).validate(); });
}

int qvr_classify_link(const qvb_topology* topo, uint32_t rs, uint32_t rtier, uint32_t rdev,
                      int64_t id, int* first, int* second) {
  return guard([&] {
    qv::ClusterTopology t = make_topo(topo);
    qv::DeviceRef r{rs, static_cast<qv::Tier>(rtier), rdev};
    qv::LinkPath p = qv::classify_link(t, r, id);
    *first = static_cast<int>(p.first);
    *second = p.second ? static_cast<int>(*p.second) : -1;
  });
}

/* fetch_cost over a flattened plan: the groups' offsets are only counted, so
 * each group gets count zero offsets */
int qvr_fetch_cost(const qvb_topology* topo, uint32_t rs, uint32_t rtier, uint32_t rdev, uint64_t groups,
                   const int64_t* gl, const uint64_t* gc, const uint64_t* gt, uint64_t feature_bytes,
                   double* per, double* total) {
  return guard([&] {
    qv::ClusterTopology t = make_topo(topo);
    qv::ReadPlan plan;
    plan.home_server = rs;
    for (uint64_t g = 0; g < groups; ++g) {
      qv::ReadPlan::LocationReads r;
      r.location_id = gl[g];
      r.offsets.assign(gc[g], 0);
      r.page_transitions = gt[g];
      plan.per_location.push_back(std::move(r));
    }
    qv::FetchCost c = qv::fetch_cost(plan, t, feature_bytes, qv::DeviceRef{rs, static_cast<qv::Tier>(rtier), rdev});
    for (uint64_t g = 0; g < groups; ++g) per[g] = c.per_location_s[g].second;
    *total = c.total_s;
  });
}

int qvr_plan_placement(const double* v, uint64_t n, const qvb_topology* topo,
                       uint64_t* loc_offsets, int64_t* loc_ids, uint64_t cap, uint64_t* copies,
                       double* ms_out) {
  return guard([&] {
    qv::ClusterTopology t = make_topo(topo);
    qv::FapTable fap;
    fap.values.assign(v, v + n);
    auto t0 = std::chrono::steady_clock::now();
    qv::PlacementPlan p = qv::plan_placement(fap, t);
    auto t1 = std::chrono::steady_clock::now();
    if (ms_out) *ms_out = std::chrono::duration<double, std::milli>(t1 - t0).count();
    uint64_t total = 0;
    for (const auto& l : p.locations) total += l.size();
    *copies = total;
    if (total > cap) throw qv::ValidationError("loc_capacity too small");
    uint64_t at = 0;
    for (uint64_t f = 0; f < n; ++f) {
      loc_offsets[f] = at;
      for (const auto& l : p.locations[f])
        loc_ids[at++] = qv::encode_location(t, l.server, l.tier, l.device);
    }
    loc_offsets[n] = at;
  });
}

int qvr_build_lookup_table(const uint64_t* lo, const int64_t* ids, uint64_t n,
                           const qvb_topology* topo, uint32_t home, int64_t* location_ids,
                           uint64_t* offsets, double* ms_out) {
  return guard([&] {
    qv::ClusterTopology t = make_topo(topo);
    qv::PlacementPlan p = make_plan(lo, ids, n, t);
    auto t0 = std::chrono::steady_clock::now();
    qv::FeatureLookupTable lut = qv::build_lookup_table(p, t, home);
    auto t1 = std::chrono::steady_clock::now();
    if (ms_out) *ms_out = std::chrono::duration<double, std::milli>(t1 - t0).count();
    std::memcpy(location_ids, lut.location_ids.data(), n * sizeof(int64_t));
    std::memcpy(offsets, lut.offsets.data(), n * sizeof(uint64_t));
  });
}

int qvr_page_transitions(const uint64_t* o, uint64_t count, uint64_t page, uint64_t* out) {
  return guard([&] { *out = qv::page_transitions(std::span<const uint64_t>(o, count), page); });
}

int qvr_plan_reads(const int64_t* location_ids, const uint64_t* offsets, uint64_t table_n,
                   const uint64_t* ids, uint64_t b, uint64_t page, int64_t* group_loc,
                   uint64_t* group_count, uint64_t* group_transitions, uint64_t* n_groups,
                   uint64_t* offsets_out, double* ms_out) {
  return guard([&] {
    qv::FeatureLookupTable lut;
    lut.location_ids.assign(location_ids, location_ids + table_n);
    lut.offsets.assign(offsets, offsets + table_n);
    auto t0 = std::chrono::steady_clock::now();
    qv::ReadPlan rp = qv::plan_reads(lut, std::span<const qv::NodeId>(ids, b), page);
    auto t1 = std::chrono::steady_clock::now();
    if (ms_out) *ms_out = std::chrono::duration<double, std::milli>(t1 - t0).count();
    uint64_t g = 0, at = 0;
    for (const auto& lr : rp.per_location) {
      group_loc[g] = lr.location_id;
      group_count[g] = lr.offsets.size();
      group_transitions[g] = lr.page_transitions;
      ++g;
      for (uint64_t o : lr.offsets) offsets_out[at++] = o;
    }
    *n_groups = g;
  });
}

// qv::batch_sample, flattened like qvo_batch_sample (two calls: sizes, fill).
int qvr_batch_sample(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                     const double* w, const uint64_t* seeds, uint64_t nseeds,
                     const uint32_t* fanouts, uint32_t hops, uint64_t rng_seed, uint64_t* total,
                     uint64_t* unique_count, uint64_t* nodes_out, uint64_t* counts_out,
                     uint64_t* unique_out, double* ms_out) {
  return guard([&] {
    qv::Graph g = make_graph(n, e, ro, col, w);
    qv::TransitionView t = qv::transition_view(g);
    qv::SamplingConfig cfg;
    cfg.fanouts.assign(fanouts, fanouts + hops);
    auto t0 = std::chrono::steady_clock::now();
    qv::BatchSampleResult r =
        qv::batch_sample(t, std::span<const qv::NodeId>(seeds, nseeds), cfg, rng_seed);
    auto t1 = std::chrono::steady_clock::now();
    if (ms_out) *ms_out = std::chrono::duration<double, std::milli>(t1 - t0).count();
    *total = r.stats.total_instances;
    *unique_count = r.stats.unique_count;
    if (!nodes_out) return;
    uint64_t at = 0;
    for (std::size_t i = 0; i < r.per_seed.size(); ++i) {
      for (std::size_t k = 0; k < r.per_seed[i].frontiers.size(); ++k) {
        counts_out[i * (hops + 1) + k] = r.per_seed[i].frontiers[k].size();
        for (qv::NodeId v : r.per_seed[i].frontiers[k]) nodes_out[at++] = v;
      }
    }
    std::copy(r.stats.unique_nodes.begin(), r.stats.unique_nodes.end(), unique_out);
  });
}

// ---- file formats (graph.cpp:197-258, metrics.cpp:203-250, placement.cpp:406-459)
int qvr_save_graph_csr(uint64_t n, uint64_t e, const uint64_t* ro, const uint64_t* col,
                       const double* w, const char* path) {
  return guard([&] { qv::save_graph_csr(make_graph(n, e, ro, col, w), path); });
}

// Two calls: sizes (ro/col/w null), then fill.
int qvr_load_graph(const char* path, int csr_binary, int remap, uint64_t* n, uint64_t* e,
                   uint64_t* ro, uint64_t* col, double* w) {
  return guard([&] {
    qv::Graph g = qv::load_graph(path, csr_binary ? qv::GraphFormat::csr_binary
                                                  : qv::GraphFormat::edge_list_text,
                                 remap != 0);
    *n = g.node_count;
    *e = g.edge_count;
    if (ro) {
      std::memcpy(ro, g.row_offsets.data(), (g.node_count + 1) * 8);
      std::memcpy(col, g.col_indices.data(), g.edge_count * 8);
      std::memcpy(w, g.edge_weights.data(), g.edge_count * 8);
    }
  });
}

int qvr_save_table_binary(const char* path, const double* v, uint64_t n, uint64_t k) {
  return guard([&] { qv::save_table_binary(path, std::span<const double>(v, n), k); });
}

int qvr_save_table_csv(const char* path, const double* v, uint64_t n) {
  return guard([&] { qv::save_table_csv(path, std::span<const double>(v, n)); });
}

int qvr_placement_exports(const uint64_t* lo, const int64_t* ids, uint64_t n,
                          const qvb_topology* topo, const char* json_path, const char* csv_path) {
  return guard([&] {
    qv::ClusterTopology t = make_topo(topo);
    qv::PlacementPlan p = make_plan(lo, ids, n, t);
    std::ofstream(json_path) << qv::placement_to_json_text(p);
    qv::save_placement_csv(p, csv_path);
  });
}

int qvr_lookup_exports(const int64_t* loc, const uint64_t* off, uint64_t n, uint32_t home,
                       uint32_t gps, const char* json_path, const char* csv_path) {
  return guard([&] {
    qv::FeatureLookupTable t;
    t.home_server = home;
    t.gpus_per_server = gps;
    t.location_ids.assign(loc, loc + n);
    t.offsets.assign(off, off + n);
    std::ofstream(json_path) << qv::lookup_to_json_text(t);
    qv::save_lookup_csv(t, csv_path);
  });
}

}  // extern "C"
