// placement.cuh — K2 ranking, the placement planner and K3 lookup-table
// construction, shared with the feature store.
#pragma once

#include <vector>

#include "common.cuh"
#include "topology.cuh"

namespace qvb {

constexpr int kMaxLocations = 64;     // one server: G + 2 <= 64
constexpr int kOffsetBits = 48;       // packed device LUT: loc << 48 | offset
constexpr uint64_t kOffsetMask = (1ull << kOffsetBits) - 1;

// K2: stable descending rank on the device (placement.cpp:79-87).
void rank_desc_device(const double* d_values, uint64_t n, uint64_t* d_ranks, cudaStream_t s);

// Host CSR plan (canonical: ids ascending per feature).
struct HostPlan {
  std::vector<uint64_t> offsets;  // n + 1
  std::vector<int64_t> ids;
};

// plan_placement (placement.cpp:138-226) given, from the device ranking, the
// values in rank order (vr) and each feature's rank position (pos).
HostPlan plan_from_ranks(const double* vr, const uint64_t* pos, uint64_t n,
                         const qvb_topology& t);

// Device -> pageable host copy through pinned slots (graph.cu).
void copy_to_host(void* dst, const void* src, uint64_t bytes, cudaStream_t s);

// Device-side result of K3 for one reader.
struct DeviceLut {
  uint64_t n = 0;
  int nloc = 0;
  DevBuf<uint64_t> masks;      // per-feature location bitmask
  DevBuf<uint64_t> tile_off;   // [nloc][ntiles] exclusive per-location tile prefix
  std::vector<uint64_t> location_rows;  // rows held by each location
  uint64_t ntiles = 0;
};

// Builds masks + per-location tile prefixes from a device CSR plan.
void lut_prepare(DeviceLut& L, const uint64_t* d_lo, const int64_t* d_ids, uint64_t n, int nloc,
                 cudaStream_t s);
// Per-feature (location, offset) chosen for `order` (locations by ascending
// (cost, id)); writes unpacked and/or packed outputs (each nullable).
// Returns the bitmask of locations chosen by at least one feature;
// *first_missing (nullable) = lowest feature with no copy, or ~0.
uint64_t lut_choose(const DeviceLut& L, const std::vector<int>& order, int64_t* d_loc,
                    uint64_t* d_off, uint64_t* d_packed, cudaStream_t s,
                    uint64_t* first_missing = nullptr);
// feat_of_row[r] = feature id stored at row r of location `loc`.
void lut_rows_of_location(const DeviceLut& L, int loc, uint64_t* d_feat_of_row, cudaStream_t s);

// Locations ordered by the reference's replica preference from GPU `reader`
// of `home` (placement.cpp:323-337): ascending (nominal cost, id).
std::vector<int> replica_order(const qvb_topology& t, uint32_t home, uint32_t reader);

}  // namespace qvb
