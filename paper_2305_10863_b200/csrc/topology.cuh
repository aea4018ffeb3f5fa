// topology.cuh — host-side topology arithmetic shared by placement, the
// lookup table and the store: ClusterTopology::validate (topology.cpp:42-64),
// encode/decode_location (placement.cpp:25-51), classify_link
// (placement.cpp:228-267) and the nominal 1 MiB replica cost
// (placement.cpp:276-302). All double arithmetic matches the reference
// expression by expression, so cost comparisons tie and order identically.
#pragma once

#include <string>

#include "common.cuh"

namespace qvb {

inline uint32_t gpus_per_numa(const qvb_topology& t) { return t.gpus_per_server / t.numa_per_server; }

inline void topology_validate(const qvb_topology& t) {
  static const char* names[QVB_LINK_COUNT] = {"local", "nvlink", "pcie", "upi",
                                               "infiniband", "ethernet", "disk"};
  if (t.servers < 1) fail(QVB_ERR_VALIDATION, "topology: servers must be >= 1");
  if (t.numa_per_server < 1) fail(QVB_ERR_VALIDATION, "topology: numa_per_server must be >= 1");
  if (t.gpus_per_server % t.numa_per_server != 0)
    fail(QVB_ERR_VALIDATION, "topology: gpus_per_server must be divisible by numa_per_server");
  for (int i = 0; i < QVB_LINK_COUNT; ++i) {
    if (!(t.link_bandwidth_Bps[i] > 0.0))
      fail(QVB_ERR_VALIDATION, std::string("topology: non-positive bandwidth for ") + names[i]);
    if (t.link_latency_s[i] < 0.0)
      fail(QVB_ERR_VALIDATION, std::string("topology: negative latency for ") + names[i]);
  }
  if (t.tlb_miss_penalty_s < 0.0) fail(QVB_ERR_VALIDATION, "topology: negative tlb_miss_penalty_s");
  if (t.gpu_replicated_capacity > t.gpu_feature_capacity)
    fail(QVB_ERR_VALIDATION, "topology: gpu_replicated_capacity exceeds gpu_feature_capacity");
}

inline int64_t encode_location(const qvb_topology& t, uint32_t server, uint32_t tier,
                               uint32_t device) {
  const int64_t stride = static_cast<int64_t>(t.gpus_per_server) + 2;
  const int64_t base = static_cast<int64_t>(server) * stride;
  if (tier == QVB_TIER_GPU) return base + device;
  if (tier == QVB_TIER_HOST) return base + t.gpus_per_server;
  return base + t.gpus_per_server + 1;
}

inline void decode_location(const qvb_topology& t, int64_t id, uint32_t* server, uint32_t* tier,
                            uint32_t* device) {
  const int64_t stride = static_cast<int64_t>(t.gpus_per_server) + 2;
  *server = static_cast<uint32_t>(id / stride);
  const int64_t slot = id % stride;
  if (slot < static_cast<int64_t>(t.gpus_per_server)) {
    *tier = QVB_TIER_GPU;
    *device = static_cast<uint32_t>(slot);
  } else {
    *tier = slot == static_cast<int64_t>(t.gpus_per_server) ? QVB_TIER_HOST : QVB_TIER_DISK;
    *device = 0;
  }
}

// classify_link (placement.cpp:228-267) for a reader on server `rs` of tier
// `rtier` (QVB_TIER_*; GPU `rdev` when a GPU). Returns the first link;
// *second = -1 when the path has one link.
inline int classify_link_from(const qvb_topology& t, uint32_t rs, uint32_t rtier, uint32_t rdev,
                              int64_t id, int* second) {
  const bool reader_gpu = rtier == QVB_TIER_GPU;
  uint32_t server, tier, dev;
  decode_location(t, id, &server, &tier, &dev);
  *second = -1;
  if (server != rs) {  // another server: over the network (disk: network, then disk)
    const int net = t.infiniband ? QVB_LINK_INFINIBAND : QVB_LINK_ETHERNET;
    if (tier != QVB_TIER_DISK) return net;
    *second = net;
    return QVB_LINK_DISK;
  }
  switch (tier) {
    case QVB_TIER_HOST: return rtier == QVB_TIER_HOST ? QVB_LINK_LOCAL : QVB_LINK_PCIE;
    case QVB_TIER_DISK: return QVB_LINK_DISK;
    default: break;
  }
  if (!reader_gpu) return QVB_LINK_PCIE;  // a non-GPU reader of a GPU copy
  if (rdev == dev) return QVB_LINK_LOCAL;
  const uint32_t gpn = gpus_per_numa(t);
  const bool same_numa = gpn > 0 && rdev / gpn == dev / gpn;
  if (!same_numa) return QVB_LINK_UPI;
  return t.nvlink_within_numa ? QVB_LINK_NVLINK : QVB_LINK_PCIE;
}

// The reference reader (placement.cpp:292-295): GPU `rdev` of server `rs`,
// or the host when the server has no GPUs.
inline int classify_link(const qvb_topology& t, uint32_t rs, uint32_t rdev, int64_t id,
                         int* second) {
  return classify_link_from(t, rs, t.gpus_per_server > 0 ? QVB_TIER_GPU : QVB_TIER_HOST, rdev, id,
                            second);
}

// nominal_read_cost (placement.cpp:298-302): setup + 1 MiB / bandwidth.
inline double nominal_read_cost(const qvb_topology& t, uint32_t rs, uint32_t rdev, int64_t id) {
  int second;
  const int first = classify_link(t, rs, rdev, id, &second);
  double setup = t.link_latency_s[first];
  double bw = t.link_bandwidth_Bps[first];
  if (second >= 0) {
    setup += t.link_latency_s[second];
    if (t.link_bandwidth_Bps[second] < bw) bw = t.link_bandwidth_Bps[second];
  }
  return setup + 1048576.0 / bw;
}

}  // namespace qvb
