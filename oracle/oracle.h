/*
 * oracle.h — CPU restatement of the reference hot path. TEST INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline — never as part of the product path.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...). Parity pin: tests/test_oracle.py checks this
 * restatement against golden vectors produced by the unmodified reference
 * (oracle/_ref, built from the reference sources by oracle/Makefile).
 */
#ifndef QV_ORACLE_H
#define QV_ORACLE_H

#include <stdint.h>

#include "../include/qvb.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* qvo_last_error(void);

/* include/qv/rng.hpp:10-57 */
uint64_t qvo_splitmix64(uint64_t x);
uint64_t qvo_derive_state(uint64_t master, uint64_t a, uint64_t b, uint64_t c);

/* tools/bench.cpp:22-34 edge stream (input order) and Graph::from_edges /
 * build_csr (graph.cpp:16-56): out-CSR with row order = input order. */
int qvo_synthetic_edges(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                        uint64_t* src, uint64_t* dst, double* w);
int qvo_build_csr(uint64_t n, uint64_t e, const uint64_t* src, const uint64_t* dst,
                  const double* w, uint64_t* row_offsets, uint64_t* col, double* w_out);
int qvo_synthetic_graph_mt(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                           int threads, uint64_t* ro, uint64_t* col, double* w);
int qvo_synthetic_graph(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                        uint64_t* row_offsets, uint64_t* col, double* w);

/* Graph::validate (graph.cpp:58-93) */
int qvo_validate(uint64_t n, uint64_t e, const uint64_t* row_offsets, const uint64_t* col,
                 const double* w);
/* in_adjacency (graph.cpp:260-281) */
int qvo_in_adjacency(uint64_t n, uint64_t e, const uint64_t* row_offsets, const uint64_t* col,
                     const double* w, uint64_t* t_row_offsets, uint64_t* t_col, double* t_w);
/* transition_view row sums (graph.cpp:292-318) */
int qvo_row_sums(uint64_t n, const uint64_t* row_offsets, const double* w, double* row_sums);
/* compute_access_prob_ie (metrics.cpp:134-173), serial twin. */
int qvo_access_prob(uint64_t n, uint64_t e, const uint64_t* row_offsets, const uint64_t* col,
                    const double* w, uint32_t layers, double* out);
/* One sweep j-1 -> j on a prepared transpose (metrics.cpp:151-170), for
 * sampled layer-wise verification at sizes the full oracle cannot hold. */
int qvo_access_prob_sweep_nodes(uint64_t n, const uint64_t* t_row_offsets, const uint64_t* t_col,
                                const double* t_w, const double* row_sums, const double* prev,
                                const uint64_t* nodes, uint64_t count, double* out);

/* compute_fap (metrics.cpp:95-132) with distribution_step (:42-58); seed
 * NULL = uniform. values[n]. */
int qvo_compute_fap(uint64_t n, uint64_t e, const uint64_t* row_offsets, const uint64_t* col,
                    const double* w, uint32_t hops, const double* seed, double* values);

/* batch_sample / sample_khop (sampler.cpp:21-149): frontiers flattened
 * seed-major then hop-major (counts_out[s*(hops+1)+k]) and the sorted union.
 * Call with nodes_out == NULL first to size the outputs. */
int qvo_batch_sample(uint64_t n, uint64_t e, const uint64_t* row_offsets, const uint64_t* col,
                     const double* w, const uint64_t* seeds, uint64_t nseeds,
                     const uint32_t* fanouts, uint32_t hops, uint64_t rng_seed, uint64_t* total,
                     uint64_t* unique_count, uint64_t* nodes_out, uint64_t* counts_out,
                     uint64_t* unique_out);

/* fap_ranking (placement.cpp:79-87) */
int qvo_rank_desc(const double* values, uint64_t n, uint64_t* ranks);
/* plan_placement (placement.cpp:94-226) + the gpu_replicated_capacity
 * extension (0 = reference). Output in canonical CSR form (see qvb.h). */
int qvo_plan_placement(const double* values, uint64_t n, const qvb_topology* topo,
                       uint64_t* loc_offsets, int64_t* loc_ids, uint64_t loc_capacity,
                       uint64_t* copies_out);
/* build_lookup_table (placement.cpp:306-342) with reader GPU reader_device. */
int qvo_build_lookup_table(const uint64_t* loc_offsets, const int64_t* loc_ids, uint64_t n,
                           const qvb_topology* topo, uint32_t home_server, uint32_t reader_device,
                           int64_t* location_ids, uint64_t* offsets);
/* page_transitions (placement.cpp:344-353) */
int qvo_page_transitions(const uint64_t* offsets, uint64_t count, uint64_t page_size,
                         uint64_t* out);
/* plan_reads (placement.cpp:355-380), flattened as in qvb.h */
int qvo_plan_reads(const int64_t* location_ids, const uint64_t* offsets, uint64_t table_n,
                   const uint64_t* ids, uint64_t b, uint64_t page_size, int64_t* group_loc,
                   uint64_t* group_count, uint64_t* group_transitions, uint64_t* n_groups,
                   uint64_t* offsets_out);

/* Synthetic inputs of SURVEY §8(d). */
void qvo_features(uint64_t first, uint64_t count, uint32_t dim, float* x);
void qvo_feature_rows(const uint64_t* ids, uint64_t b, uint32_t dim, float* out, int threads);
void qvo_features_mt(uint64_t first, uint64_t count, uint32_t dim, float* x, int threads);
void qvo_request_ids(uint64_t seed, uint64_t batch, uint64_t n, uint64_t* ids, uint64_t b);
/* Row gather restatement: out[i] = X[ids[i]] with `threads` pthreads. */
int qvo_gather(const float* x, uint64_t n, uint32_t dim, const uint64_t* ids, uint64_t b,
               float* out, int threads);

#ifdef __cplusplus
}
#endif
#endif
