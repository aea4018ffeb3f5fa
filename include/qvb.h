/*
 * qvb.h — C-ABI of the B200-native Quiver feature-store hot path.
 *
 * This is the drop-in boundary. Every entry point replaces one function of the
 * reference planner `qvserve` (namespace qv, /root/reference/proj) on the
 * north-star path  P(n,j) -> placement -> lookup table -> collect/gather.
 * The reference interface each entry replaces is cited as file:line.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes; no C++ or torch types.
 *  - Every function returns a status code (qvb_status). On failure the
 *    thread-local message is available from qvb_last_error(). Codes mirror the
 *    reference exception hierarchy (include/qv/error.hpp:10-32) and the exit
 *    codes its CLI maps them to (tools/qvserve.cpp:347-367).
 *  - Host output buffers are caller-allocated. Device objects (qvb_graph,
 *    qvb_store) are library-owned opaque handles, immutable after build, so
 *    concurrent read-only calls on different streams are safe.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - There is no CPU fallback: on a machine without a usable sm_100 device
 *    every compute entry point fails with QVB_ERR_CUDA.
 */
#ifndef QVB_H
#define QVB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (error.hpp:10-32; qvserve.cpp:347-367) ---------------- */
typedef enum {
  QVB_OK = 0,
  QVB_ERR_GENERIC = 1,     /* qv::Error                                    */
  QVB_ERR_VALIDATION = 2,  /* qv::ValidationError / ParseError / ConfigError */
  QVB_ERR_PLACEMENT = 3,   /* qv::PlacementError                           */
  QVB_ERR_CUDA = 10,       /* CUDA runtime failure or no usable device      */
  QVB_ERR_UNSUPPORTED = 11 /* valid input outside the device path's limits  */
} qvb_status;

/* Message of the last failing call on this thread ("" if none). */
const char* qvb_last_error(void);
/* Library version string. */
const char* qvb_version(void);

/* ---- topology (include/qv/topology.hpp:11-54) --------------------------- */
/* Link classes, same order as qv::LinkClass (topology.hpp:11-20). */
enum {
  QVB_LINK_LOCAL = 0,
  QVB_LINK_NVLINK = 1,
  QVB_LINK_PCIE = 2,
  QVB_LINK_UPI = 3,
  QVB_LINK_INFINIBAND = 4,
  QVB_LINK_ETHERNET = 5,
  QVB_LINK_DISK = 6,
  QVB_LINK_COUNT = 7
};
/* Tier, same values as qv::Tier (placement.hpp:14). */
enum { QVB_TIER_GPU = 0, QVB_TIER_HOST = 1, QVB_TIER_DISK = 2 };

/* Mirrors qv::ClusterTopology (topology.hpp:32-54) field for field, plus one
 * extension: gpu_replicated_capacity (see qvb_plan_placement). */
typedef struct qvb_topology {
  uint32_t servers;
  uint32_t numa_per_server;
  uint32_t gpus_per_server;
  uint32_t nvlink_within_numa; /* bool */
  uint32_t infiniband;         /* bool */
  uint32_t _pad0;
  uint64_t gpu_feature_capacity;
  uint64_t host_feature_capacity;
  uint64_t disk_feature_capacity;
  double link_latency_s[QVB_LINK_COUNT];
  double link_bandwidth_Bps[QVB_LINK_COUNT];
  double tlb_miss_penalty_s;
  /* Extension (0 reproduces the reference exactly): per-GPU slots of the GPU
   * capacity that hold the hottest features replicated on EVERY GPU of the
   * server; the next range is then partitioned by the reference NVLink rule.
   * Must be <= gpu_feature_capacity. */
  uint64_t gpu_replicated_capacity;
} qvb_topology;

/* ClusterTopology::with_defaults (topology.cpp:27-40). */
void qvb_topology_defaults(qvb_topology* t);
/* ClusterTopology::validate (topology.cpp:42-64). */
int qvb_topology_validate(const qvb_topology* t);
/* encode_location / decode_location (placement.cpp:25-51). */
int64_t qvb_encode_location(const qvb_topology* t, uint32_t server, uint32_t tier,
                            uint32_t device);
int qvb_decode_location(const qvb_topology* t, int64_t id, uint32_t* server,
                        uint32_t* tier, uint32_t* device);

/* classify_link (placement.cpp:228-267): the link path from a reader
 * (server, tier QVB_TIER_GPU/HOST, device) to a location id; *second = -1
 * for a one-link path. */
int qvb_classify_link(const qvb_topology* t, uint32_t reader_server, uint32_t reader_tier,
                      uint32_t reader_device, int64_t location_id, int* first, int* second);
/* fetch_cost (placement.cpp:382-404), the reference's latency model of one
 * collect, over a flattened read plan (groups as qvb_plan_reads returns them):
 * per group setup + count*feature_bytes/bandwidth (+ tlb penalty per page
 * transition on translated links) into per_location_s[groups]; *total_s =
 * their max. A location id outside the topology is a ValidationError. */
int qvb_fetch_cost(const qvb_topology* t, uint32_t reader_server, uint32_t reader_tier,
                   uint32_t reader_device, uint64_t groups, const int64_t* group_loc,
                   const uint64_t* group_count, const uint64_t* group_transitions,
                   uint64_t feature_bytes, double* per_location_s, double* total_s);

/* ---- device info ------------------------------------------------------- */
/* Number of usable devices (fails with QVB_ERR_CUDA when there are none). */
int qvb_device_count(int* count);

/* ---- graph: in_adjacency + transition_view on device --------------------- */
/* Device-resident in-CSR with coalesced parallel edges, per-source
 * reciprocal row sums and per-edge transition factors. Replaces the transpose
 * rebuilt inside every compute_access_prob_ie call (metrics.cpp:145 ->
 * graph.cpp:260-281) and transition_view's row sums (graph.cpp:292-318). */
typedef struct qvb_graph qvb_graph;

typedef struct qvb_graph_info {
  uint64_t node_count;
  uint64_t edge_count;         /* as uploaded (parallel edges counted)      */
  uint64_t unique_edge_count;  /* coalesced (source, destination) pairs     */
  uint64_t exception_count;    /* unique edges whose factor != 1/row_sum(s) */
  uint32_t layout;             /* 0 = compact (col + per-source y), 1 = weighted (col + R per edge) */
  uint32_t device;
  uint64_t device_bytes;       /* HBM held by the graph                     */
  double build_ms;             /* device time of the in-CSR build           */
  uint32_t classes;            /* first-sweep out-degree classes (0: the first sweep gathers) */
  uint32_t segments;           /* source segments (passes) of the later sweeps */
  uint64_t first_slots;        /* padded slots of the first sweep's class stream */
  uint64_t segment_columns;    /* columns of the node-major segmented layout (0: sliced) */
} qvb_graph_info;

/* Upload an out-CSR (qv::Graph layout, graph.hpp:25-48): row_offsets[n+1],
 * col[e], weights[e] (NULL = all 1.0). Validates like Graph::validate
 * (graph.cpp:58-93) and throws the same conditions as ValidationError.
 * Limits of the device path: n < 2^31, e < 2^32. */
int qvb_graph_upload(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                     const uint64_t* col, const double* weights, void* stream,
                     qvb_graph** out);
/* Build the graph of tools/bench.cpp:22-34 (seeded SplitMix64 stream
 * derive_stream(seed, 0xBE9C4)) directly on the device, bit-identical to the
 * host generator. weighted=0 uses weight 1.0 (the draw is still consumed);
 * transposed=1 swaps source and destination (skewed in-degree variant). */
int qvb_graph_synthetic(int device, uint64_t n, uint64_t e, uint64_t seed, int weighted,
                        int transposed, void* stream, qvb_graph** out);
/* qv::in_adjacency (graph.cpp:260-281) on the device: the transposed graph
 * (parallel edges kept, each row in ascending source order, weights carried)
 * into host buffers t_row_offsets[n+1], t_col[e], t_weights[e]. Validates
 * like Graph::validate. */
int qvb_in_adjacency(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                     const uint64_t* col, const double* weights, uint64_t* t_row_offsets,
                     uint64_t* t_col, double* t_weights);
/* The same generator's out-CSR copied to host buffers in the qv::Graph
 * layout (row_offsets[n+1], col[e], weights[e]) — the host-side input of the
 * end-to-end compute_access_prob_ie path. */
int qvb_synthetic_csr(int device, uint64_t n, uint64_t e, uint64_t seed, int weighted,
                      int transposed, uint64_t* row_offsets, uint64_t* col, double* weights);
int qvb_graph_info_get(const qvb_graph* g, qvb_graph_info* info);

/* qv::Edge (graph.hpp:12-16): 24 bytes, the layout of std::vector<qv::Edge>. */
typedef struct qvb_edge {
  uint64_t src;
  uint64_t dst;
  double weight;
} qvb_edge;
/* Graph::from_edges / build_csr (graph.cpp:16-56) on the device: the first
 * edge (input order) with an endpoint >= n or a negative/NaN weight is a
 * ValidationError with the reference's message; rows keep input order
 * (stable sort by source). Outputs: row_offsets[n+1], col[e], weights[e]
 * (host), then validated like Graph::validate. */
int qvb_build_csr(int device, uint64_t n, const qvb_edge* edges, uint64_t e,
                  uint64_t* row_offsets, uint64_t* col, double* weights);
/* Graph::validate (graph.cpp:58-93) on the device: same checks, same order,
 * same messages (weights NULL = all 1.0). */
int qvb_graph_validate(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                       const uint64_t* col, const double* weights);
/* transition_view (graph.cpp:292-318) on the device: row_sums[n] (each row's
 * weights summed sequentially in CSR order), distinct_out[n] (distinct
 * out-neighbours per node) and *has_parallel_edges, from one upload that also
 * builds the P(n,j) in-CSR. keep (nullable) receives that device graph, ready
 * for qvb_access_prob, so compute_access_prob_ie(g, transition_view(g), L)
 * uploads the graph once; NULL discards it. */
int qvb_transition_view(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                        const uint64_t* col, const double* weights, double* row_sums,
                        uint64_t* distinct_out, int* has_parallel_edges, qvb_graph** keep);
/* Device time (ms, CUDA events on the call's stream) of the P sweeps of the
 * last qvb_access_prob on g. */
int qvb_graph_last_sweep_ms(const qvb_graph* g, double* ms);
/* Per-phase device time (ms) of the last qvb_access_prob on g: ms[0] first
 * sweep over the class stream, ms[1] code gathers, ms[2] ordered products,
 * ms[3] other sweep kernels; *launches (nullable) = kernels launched. */
int qvb_graph_phase_ms(const qvb_graph* g, double* ms, uint32_t* launches);
/* Diagnostics / size-independent parity: the coalesced in-row of each listed
 * node as the sweeps multiply it — sources ascending, R = w_sum / row_sum(s)
 * (metrics.cpp:157-166). Fills row_ptr[count+1]; src and R receive
 * row_ptr[count] entries unless NULL (call once with NULL to size them).
 * Node-major (segmented) graphs only. */
int qvb_graph_in_rows(const qvb_graph* g, const uint64_t* nodes, uint64_t count,
                      uint64_t* row_ptr, uint32_t* src, double* R);
int qvb_graph_destroy(qvb_graph* g);

/* ---- K1: access probability P(n,j) (metrics.cpp:134-173) ---------------- */
/* P(n,1) = 1/|V|; P(n,j) = P(n,j-1) + (1-P(n,j-1)) * (1 - prod_{s in in(n)}
 * (1 - P(s,j-1) * R(s,n))) with the reference's per-node factor order, so the
 * result is bit-identical to qv::compute_access_prob_ie. `out` holds n doubles
 * on the host (out_on_device=0) or the device (1). layers >= 1. */
int qvb_access_prob(qvb_graph* g, uint32_t layers, double* out, int out_on_device,
                    void* stream);
/* Row-sharded P over `world` ranks (one exchange step per
 * layer), each rank holding the same graph on its own device. Rank r
 * computes nodes [r*chunk, min(n, (r+1)*chunk)), chunk = ceil(n/world/32)*32;
 * after every sweep j the library calls exchange(ctx, j, p, codes,
 * chunk, stream): p (double) and codes (uint32, NULL when the next sweep
 * needs none) each hold world*chunk entries, this rank's chunk written; the
 * callback must all-gather the chunks in place (e.g. ncclAllGather with
 * sendbuff = p + rank*chunk) ordered on `stream`, and return 0. Per-node
 * arithmetic is unchanged: the result is bit-identical to qvb_access_prob.
 * Graphs whose layout does not split by node ranges compute every node on
 * every rank without calling exchange; *sharded (nullable) reports which. */
typedef int (*qvb_exchange_fn)(void* ctx, uint32_t layer, void* p, void* codes,
                               uint64_t chunk_nodes, void* stream);
int qvb_access_prob_sharded(qvb_graph* g, uint32_t layers, uint32_t rank, uint32_t world,
                            qvb_exchange_fn exchange, void* ctx, double* out, int out_on_device,
                            void* stream, int* sharded);
/* The whole reference call from host CSR to host table:
 * qv::compute_access_prob_ie(g, transition_view(g), layers)
 * (metrics.hpp:53-54). Uploads, builds the in-CSR, runs the sweeps and copies
 * P back; ms_out (nullable) receives [upload+build, sweeps, download] ms. */
int qvb_compute_access_prob_ie(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                               const uint64_t* col, const double* weights, uint32_t layers,
                               double* out, double* ms_out);

/* ---- FAP estimator (metrics.cpp:95-132) -------- */
/* qv::compute_fap(transition_view(g), hops, seed): values[i] = sum over
 * k = 0..hops of the k-hop visit mass of a walk started from `seed`
 * (NULL = uniform 1/|V|), each step a Neumaier-compensated pull in the
 * reference's edge order — bit-identical to the reference. Seed errors are
 * ValidationErrors with the reference's messages. */
int qvb_compute_fap(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                    const uint64_t* col, const double* weights, uint32_t hops,
                    const double* seed, double* values);

/* ---- K2: ranking (placement.cpp:79-87) ----------------------------------- */
/* ranks[i] = feature id of rank i: value descending, id ascending on ties
 * (std::stable_sort order). values/ranks are host (on_device=0) or device. */
int qvb_rank_desc(int device, const double* values, uint64_t n, uint64_t* ranks,
                  int on_device, void* stream);

/* ---- placement manager (placement.cpp:138-226) -------------------------- */
/* qv::plan_placement(FapTable{values}, topo). The ranking runs on the GPU;
 * the greedy balance is the reference's sequential rule, on the host.
 * Output: canonical plan in CSR form — feature f's copies are
 * loc_ids[loc_offsets[f] .. loc_offsets[f+1]) as encoded location ids,
 * ascending (== canonical (server, tier, device) order; replica = index > 0).
 * loc_capacity is the size of loc_ids; *copies_out receives the total.
 * Errors: ValidationError for n == 0 / bad topology, PlacementError naming
 * the shortfall, Error for an overfilled device — as the reference. */
int qvb_plan_placement(int device, const double* values, uint64_t n, const qvb_topology* topo,
                       uint64_t* loc_offsets, int64_t* loc_ids, uint64_t loc_capacity,
                       uint64_t* copies_out);

/* The same plan held by the library (no caller-side upper bound on the copy
 * count, which is n x servers x (G+1) in the worst case): create, read its
 * size, copy it into exactly-sized buffers, destroy. */
typedef struct qvb_plan qvb_plan;
int qvb_plan_placement_create(int device, const double* values, uint64_t n,
                              const qvb_topology* topo, qvb_plan** out);
int qvb_plan_size(const qvb_plan* plan, uint64_t* n, uint64_t* copies);
int qvb_plan_copy(const qvb_plan* plan, uint64_t* loc_offsets, int64_t* loc_ids);
int qvb_plan_destroy(qvb_plan* plan);

/* ---- K3: feature lookup table (placement.cpp:306-342) ------------------- */
/* qv::build_lookup_table(plan, topo, home_server). Reader = GPU
 * `reader_device` of home_server (0 reproduces the reference's
 * reference_reader, placement.cpp:292-295; >0 is the per-reader extension).
 * Output: location_ids[n], offsets[n] (host). Any number of locations
 * (servers x (G+2)); a feature without copies gets (-1, 0), as the reference. */
int qvb_build_lookup_table(int device, const uint64_t* loc_offsets, const int64_t* loc_ids,
                           uint64_t n, const qvb_topology* topo, uint32_t home_server,
                           uint32_t reader_device, int64_t* location_ids, uint64_t* offsets);

/* ---- K4: read planner (placement.cpp:344-380) --------------------------- */
/* qv::page_transitions (host arithmetic, tiny). */
int qvb_page_transitions(const uint64_t* offsets, uint64_t count, uint64_t page_size,
                         uint64_t* out);
/* qv::plan_reads(table, ids, page_size) flattened: groups i in
 * [0, *n_groups) have location group_loc[i], group_count[i] offsets and
 * group_transitions[i] page transitions; their offsets are concatenated in
 * offsets_out (size b). group_* arrays need room for every distinct location
 * (at most b). Throws ValidationError for page_size 0 or an id >= table_n. */
int qvb_plan_reads(int device, const int64_t* location_ids, const uint64_t* offsets,
                   uint64_t table_n, const uint64_t* ids, uint64_t b, uint64_t page_size,
                   int64_t* group_loc, uint64_t* group_count, uint64_t* group_transitions,
                   uint64_t* n_groups, uint64_t* offsets_out);

/* The same plan from a lookup table already resident on the device (DEVICE
 * pointers location_ids/offsets[table_n] and ids[b]; outputs are host
 * buffers as above). Stream-ordered on `stream`, returns when the plan is on
 * the host. The per-batch call of the reference's serving loop
 * (simulator.cpp:320-321) without re-uploading the table it builds once. */
int qvb_plan_reads_device(int device, const int64_t* location_ids, const uint64_t* offsets,
                          uint64_t table_n, const uint64_t* ids, uint64_t b, uint64_t page_size,
                          int64_t* group_loc, uint64_t* group_count, uint64_t* group_transitions,
                          uint64_t* n_groups, uint64_t* offsets_out, void* stream);

/* ---- K5: feature store + gather (new; fetch_cost placement.cpp:382-404
 *          only models this transfer) ------------------------------------- */
/* One store per (process, device). It owns this device's shard, an optional
 * host (zero-copy, pinned + mapped) shard, the reader's lookup table in HBM
 * and a table of base pointers for every location (peers are attached with
 * IPC handles). Row layout: dim fp32 values per feature, padded internally to
 * a 16-byte stride. */
typedef struct qvb_store qvb_store;

typedef struct qvb_store_info {
  uint64_t feature_count;
  uint32_t dim;
  uint32_t reader_device;   /* this store's GPU index within the server */
  uint64_t row_stride_bytes;
  uint64_t local_rows;      /* rows in this device's shard              */
  uint64_t host_rows;       /* rows in the host shard                   */
  uint64_t lut_bytes;
  uint32_t location_count;  /* G + 2                                    */
  uint32_t _pad;
} qvb_store_info;

/* Build the store for reader GPU `reader_device` on CUDA device `device`
 * from a single-server plan (CSR of encoded location ids, as produced by
 * qvb_plan_placement). The lookup table is qvb_build_lookup_table for this
 * reader. Features come from `features` (host, n x dim fp32, row-major) or,
 * when features == NULL, from the synthetic generator
 * X[f][k] = float(splitmix64(f*dim+k) >> 40) * 2^-24. Rows of the host tier
 * are kept in pinned mapped host memory when this reader's table uses them. */
int qvb_store_create(int device, const uint64_t* loc_offsets, const int64_t* loc_ids,
                     uint64_t n, uint32_t dim, const qvb_topology* topo,
                     uint32_t reader_device, const float* features, qvb_store** out);
int qvb_store_info_get(const qvb_store* s, qvb_store_info* info);
/* cudaIpcMemHandle_t (64 bytes) of this device's shard, for peers. */
int qvb_store_export_handle(const qvb_store* s, uint8_t handle[64]);
/* Map peer GPU `peer_device`'s shard (from its exported handle). */
int qvb_store_attach_peer(qvb_store* s, uint32_t peer_device, const uint8_t handle[64]);
/* Same-process variant: map the shard of `peer` (a store of this process,
 * reader GPU `peer_device`) directly — P2P access is enabled when the two
 * stores live on different CUDA devices. */
int qvb_store_attach_local_peer(qvb_store* s, uint32_t peer_device, const qvb_store* peer);
int qvb_store_destroy(qvb_store* s);

/* out[i][0:dim] = X[ids[i]][0:dim] for i < b; ids and out are DEVICE
 * pointers. Reads one-sided from local HBM, peer HBM (NVLink P2P) or host
 * pinned memory (zero-copy) per lookup-table entry. Ids >= n are a
 * ValidationError (checked on device; reported at the next synchronising
 * call or by qvb_store_check_error). */
int qvb_gather(qvb_store* s, const uint64_t* ids, uint64_t b, float* out, void* stream);
/* K4-order variant: requests are first sorted by (location, shard offset),
 * the plan_reads order, and the rows are copied in that order. Faster than
 * qvb_gather only when a large host tier is read with big batches (ascending
 * host offsets walk the pinned pages in order: 1.46x on a 14 GB host tier at
 * 1M ids); slower elsewhere (profiles/r01m_gather_sweep.md). */
int qvb_gather_planned(qvb_store* s, const uint64_t* ids, uint64_t b, float* out, void* stream);
/* End-to-end collect from HOST buffers: copies ids host->device, gathers,
 * copies rows device->host, and synchronises. Calls on one store from several
 * threads are serialised (they share the store's staging buffers). */
int qvb_gather_host(qvb_store* s, const uint64_t* ids, uint64_t b, float* out, void* stream);
/* qv::plan_reads over this store's resident lookup table (the reader's
 * table: reader 0 of the server is the reference's build_lookup_table), for
 * ids on the host (ids_on_device=0) or the device. Outputs as
 * qvb_plan_reads. No per-call table upload. */
int qvb_store_plan_reads(qvb_store* s, const uint64_t* ids, uint64_t b, int ids_on_device,
                         uint64_t page_size, int64_t* group_loc, uint64_t* group_count,
                         uint64_t* group_transitions, uint64_t* n_groups, uint64_t* offsets_out,
                         void* stream);
/* Reports (and clears) a device-side id range error of earlier gathers. */
int qvb_store_check_error(qvb_store* s);

/* ---- synthetic request streams ---------------------------- */
/* ids[k] = derive_stream(seed, 0x5EED, batch).below(n) draw k, on device. */
int qvb_request_ids_synthetic(int device, uint64_t seed, uint64_t batch, uint64_t n,
                              uint64_t* ids, uint64_t b, void* stream);

/* ---- K0: k-hop neighbour sampler (include/qv/sampler.hpp:11-53) --------- */
/* The request-ID producer upstream of the collect call
 * (simulator.cpp:250-254 -> :320). A qvb_sampler holds the out-CSR's
 * sampling candidates on the device: one per edge, or — when the graph has
 * parallel edges (transition_view's has_parallel_edges, graph.cpp:299-313) —
 * one per distinct neighbour in first-occurrence order with the weights summed
 * in CSR order (sampler.cpp:75-90). Built once, reused by every batch. */
typedef struct qvb_sampler qvb_sampler;
typedef struct qvb_sample qvb_sample;
typedef struct {
  uint64_t node_count, edge_count;
  uint64_t candidates;        /* coalesced candidate count (== edges without parallel edges) */
  int32_t parallel_edges;     /* 1 when neighbours were coalesced */
  int32_t unit_weights;       /* 1 when every candidate weight is 1.0 */
  uint64_t max_candidates;    /* longest candidate row */
  uint64_t device_bytes;
  double build_ms;
} qvb_sampler_info;
typedef struct {
  uint64_t seeds;
  uint32_t hops;
  uint32_t reserved;
  uint64_t total_instances;   /* BatchSampleStats::total_instances */
  uint64_t unique_count;      /* BatchSampleStats::unique_count */
  double device_ms;           /* CUDA-event time of the sampling kernels */
} qvb_sample_info;

/* From a host out-CSR (qv::Graph layout; weights NULL = 1.0), validated like
 * Graph::validate (graph.cpp:58-93). */
int qvb_sampler_create(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                       const uint64_t* col, const double* weights, void* stream,
                       qvb_sampler** out);
/* From the tools/bench.cpp:22-34 generator, built on the device. */
int qvb_sampler_synthetic(int device, uint64_t n, uint64_t e, uint64_t seed, int weighted,
                          int transposed, void* stream, qvb_sampler** out);
int qvb_sampler_info_get(const qvb_sampler* s, qvb_sampler_info* info);
int qvb_sampler_destroy(qvb_sampler* s);

/* qv::batch_sample (sampler.cpp:114-149) with sample_khop (:56-112) and
 * draw_without_replacement (:21-52): per seed, hop k draws
 * min(#positive candidates, fanouts[k-1]) distinct neighbours of every
 * frontier instance with exponential keys Exp(1)/w from
 * derive_stream(splitmix64(rng_seed ^ seed*gamma), k, idx, parent) — the
 * same streams, keys (glibc log1p reproduced bit-exactly) and tie order as
 * the reference, so every frontier is identical. `seeds` are host
 * (seeds_on_device=0) or device pointers; seeds >= n and an empty fanout list
 * are ValidationErrors with the reference's messages. The result lives on the
 * device until qvb_sample_destroy. */
int qvb_batch_sample(qvb_sampler* s, const uint64_t* seeds, uint64_t nseeds, int seeds_on_device,
                     const uint32_t* fanouts, uint32_t hops, uint64_t rng_seed, void* stream,
                     qvb_sample** out);
int qvb_sample_info_get(const qvb_sample* r, qvb_sample_info* info);
/* Copies to host buffers (each may be NULL): nodes[total_instances] = every
 * per-seed frontier flattened seed-major then hop-major (SampleResult::
 * frontiers), counts[seeds*(hops+1)] = instance_counts, unique[unique_count]
 * = BatchSampleStats::unique_nodes (sorted). Synchronises. */
int qvb_sample_copy(const qvb_sample* r, uint64_t* nodes, uint64_t* counts, uint64_t* unique);
/* Device pointers of the same arrays (owned by r), e.g. to feed
 * qvb_gather(store, unique, unique_count, ...) without a host round trip. */
int qvb_sample_device(const qvb_sample* r, const uint64_t** nodes, const uint64_t** counts,
                      const uint64_t** unique);
int qvb_sample_destroy(qvb_sample* r);

#ifdef __cplusplus
}
#endif
#endif /* QVB_H */
