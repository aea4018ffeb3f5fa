// reads.cuh — K4 device read plan (plan_reads, placement.cpp:355-380).
#pragma once

#include "common.cuh"

namespace qvb {

struct DeviceReadPlan {
  uint64_t b = 0;
  uint32_t groups = 0;
  DevBuf<uint64_t> keys;     // sorted location << 40 | offset
  DevBuf<uint32_t> order;    // request index of each sorted key
  DevBuf<uint64_t> offsets;  // sorted offsets (the flattened ReadPlan)
  DevBuf<int64_t> gloc;      // per group: location id (ascending)
  DevBuf<uint64_t> gstart;   // per group: first sorted position (+ sentinel b)
  DevBuf<uint64_t> gtrans;   // per group: exclusive prefix of transitions (+ total)
};

// d_loc/d_off: the lookup table (unpacked) on device; d_ids: b request ids.
void plan_reads_device(const int64_t* d_loc, const uint64_t* d_off, uint64_t table_n,
                       const uint64_t* d_ids, uint64_t b, uint64_t page, DeviceReadPlan& out,
                       cudaStream_t s);

}  // namespace qvb
