// graph.cuh — the device-resident in-CSR that replaces the transpose the
// reference rebuilds inside every compute_access_prob_ie call
// (metrics.cpp:145 -> in_adjacency, graph.cpp:260-281) plus the row sums of
// transition_view (graph.cpp:292-318).
//
// HBM layout (N nodes, E_u coalesced in-edges):
//   uptr   u64[N+1]   in-row pointers over coalesced edges, rows by destination
//   col    u32[E_u]   source of each coalesced in-edge, ascending within a row
//                     (the reference's factor order). Compact layout: bit 31
//                     set => index into the exception table instead.
//   R      f64[E_u]   weighted layout only: R = w_sum / row_sum(s)
//   exc_*             compact layout only: (source, R) of the few edges whose
//                     R differs bitwise from 1/row_sum(s) (parallel edges,
//                     non-unit weights)
//   inv    f64[N]     1/row_sum(s) (0 for sinks)
//   p[2], y[2] f64[N] ping-pong P_{j-1}/P_j and y = P * inv (compact layout)
#pragma once

#include "common.cuh"

struct qvb_graph {
  int device = 0;
  uint64_t n = 0, e = 0, eu = 0, nexc = 0;
  uint32_t layout = 0;  // 0 compact, 1 weighted
  uint64_t* uptr = nullptr;
  uint32_t* col = nullptr;
  double* R = nullptr;
  uint32_t* exc_src = nullptr;
  double* exc_R = nullptr;
  double* inv = nullptr;
  double* p[2] = {nullptr, nullptr};
  double* y[2] = {nullptr, nullptr};
  uint64_t bytes = 0;
  double build_ms = 0.0;
  cudaEvent_t ev[2] = {nullptr, nullptr};  // bracket the sweeps of the last run
  ~qvb_graph();
};

namespace qvb {

constexpr uint32_t kExcFlag = 0x80000000u;
constexpr uint64_t kMaxNodes = (1ull << 31) - 1;
constexpr uint64_t kMaxEdges = 0xFFFFFFFFull;

// Builds the in-CSR from a device out-CSR. d_w == nullptr means unit weights.
// d_src (nullable): source of every out-CSR edge if already known.
void build_in_csr(qvb_graph& g, const uint64_t* d_ro, const uint32_t* d_col, const double* d_w,
                  const uint32_t* d_src, cudaStream_t s);

// Runs layers-1 sweeps; returns the device buffer holding P_layers.
const double* run_access_prob(qvb_graph& g, uint32_t layers, cudaStream_t s);

}  // namespace qvb
