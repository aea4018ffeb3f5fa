// reads.cuh — K4 device read plan (plan_reads, placement.cpp:355-380).
#pragma once

#include "common.cuh"

namespace qvb {

constexpr int kPackedOffsetBits = 48;  // store tables: loc << 48 | offset (placement.cuh)

struct DeviceReadPlan {
  uint64_t b = 0;
  uint32_t groups = 0;
  int ob = 0;                // offset bits of the keys
  DevBuf<uint64_t> keys;     // sorted location << ob | offset
  DevBuf<uint32_t> order;    // request index of each sorted key
  DevBuf<uint64_t> offsets;  // sorted offsets (the flattened ReadPlan)
  DevBuf<int64_t> gloc;      // per group: location id (ascending)
  DevBuf<uint64_t> gcount;   // per group: offsets in the group
  DevBuf<uint64_t> gtrans;   // per group: page transitions
};

// The lookup table on the device, reference layout (d_loc, d_off) or packed
// (d_packed, loc << 48 | offset; then d_loc/d_off are unused); d_ids: b
// request ids (device, or host-mapped).
void plan_reads_device(const int64_t* d_loc, const uint64_t* d_off, const uint64_t* d_packed,
                       uint64_t table_n, const uint64_t* d_ids, uint64_t b, uint64_t page,
                       DeviceReadPlan& out, cudaStream_t s);
void copy_read_plan(const DeviceReadPlan& rp, int64_t* group_loc, uint64_t* group_count,
                    uint64_t* group_transitions, uint64_t* n_groups, uint64_t* offsets_out,
                    cudaStream_t s);
// Device -> pageable host copy through pinned slots (graph.cu).
void copy_to_host(void* dst, const void* src, uint64_t bytes, cudaStream_t s);

}  // namespace qvb
