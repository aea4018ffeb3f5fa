// capi.cu — C-ABI plumbing: error strings, version, device query and the
// topology helpers (reference topology.cpp:27-64, placement.cpp:25-51).
#include <atomic>
#include <cstring>
#include <string>

#include "common.cuh"
#include "topology.cuh"

namespace qvb {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& m) { g_last_error = m; }

void retain_pool(int device) {
  static std::atomic<uint64_t> done{0};  // bit per device (< 64)
  const uint64_t bit = device < 64 ? 1ull << device : 0;
  if (!bit || (done.load(std::memory_order_acquire) & bit)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done.fetch_or(bit, std::memory_order_acq_rel);
}
}  // namespace qvb

using namespace qvb;

extern "C" const char* qvb_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* qvb_version(void) { return "qvb 0.1 (sm_100a)"; }

extern "C" int qvb_device_count(int* count) {
  return guarded([&] {
    if (!count) fail(QVB_ERR_VALIDATION, "null argument");
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess || *count == 0) {
      cudaGetLastError();
      *count = 0;
      fail(QVB_ERR_CUDA, "no CUDA device available (the qvb library has no CPU fallback)");
    }
  });
}

extern "C" void qvb_topology_defaults(qvb_topology* t) {
  if (!t) return;
  std::memset(t, 0, sizeof *t);
  t->servers = 1;
  t->numa_per_server = 1;
  t->gpus_per_server = 1;
  const double lat[QVB_LINK_COUNT] = {0.0, 2e-6, 1e-5, 5e-6, 2e-6, 5e-5, 1e-4};
  const double bw[QVB_LINK_COUNT] = {1e12, 300e9, 16e9, 20e9, 12.5e9, 1.25e9, 0.5e9};
  for (int i = 0; i < QVB_LINK_COUNT; ++i) {
    t->link_latency_s[i] = lat[i];
    t->link_bandwidth_Bps[i] = bw[i];
  }
  t->tlb_miss_penalty_s = 1e-7;
}

extern "C" int qvb_topology_validate(const qvb_topology* t) {
  return guarded([&] {
    if (!t) fail(QVB_ERR_VALIDATION, "null topology");
    topology_validate(*t);
  });
}

extern "C" int64_t qvb_encode_location(const qvb_topology* t, uint32_t server, uint32_t tier,
                                       uint32_t device) {
  if (!t) return -1;
  return encode_location(*t, server, tier, device);
}

extern "C" int qvb_decode_location(const qvb_topology* t, int64_t id, uint32_t* server,
                                   uint32_t* tier, uint32_t* device) {
  return guarded([&] {
    if (!t || !server || !tier || !device) fail(QVB_ERR_VALIDATION, "null argument");
    decode_location(*t, id, server, tier, device);
  });
}
