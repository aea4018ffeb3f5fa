// reads.cu — K4, the read planner of the collect call (plan_reads +
// page_transitions, reference placement.cpp:344-380).
//
// The reference groups the requested ids by location through a std::map
// (ascending location id) and sorts each group's offsets ascending,
// duplicates kept. On the device: look up (location, offset) per request,
// pack key = location << 40 | offset, stable radix sort with the request
// index as payload (the payload is what the planned gather consumes), then
// mark group heads and page changes and compact them with two scans.
#include <string>
#include <vector>

#include "reads.cuh"

namespace qvb {
namespace {

constexpr int kKeyOffsetBits = 40;

__global__ void k_plan_keys(const int64_t* __restrict__ loc, const uint64_t* __restrict__ off,
                            uint64_t table_n, const uint64_t* __restrict__ ids, uint64_t b,
                            uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                            unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = ids[i];
    uint64_t k = 0;
    if (f >= table_n) {
      atomicMin(bad, (unsigned long long)(i << 1));
    } else {
      const int64_t l = loc[f];
      const uint64_t o = off[f];
      if (l < 0 || l >= (1ll << (64 - kKeyOffsetBits)) || o >= (1ull << kKeyOffsetBits))
        atomicMin(bad, (unsigned long long)((i << 1) | 1));
      else
        k = ((uint64_t)l << kKeyOffsetBits) | o;
    }
    keys[i] = k;
    idx[i] = static_cast<uint32_t>(i);
  }
}

// head: first of a location group; trans: counts toward the group's page
// transitions (1 + adjacent page changes, placement.cpp:344-353).
__global__ void k_plan_marks(const uint64_t* __restrict__ keys, uint64_t b, uint64_t page,
                             uint8_t* __restrict__ head, uint8_t* __restrict__ trans,
                             uint64_t* __restrict__ offsets_out) {
  const uint64_t mask = (1ull << kKeyOffsetBits) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const uint64_t o = k & mask;
    bool h = i == 0, t = i == 0;
    if (i > 0) {
      const uint64_t kp = keys[i - 1];
      h = (kp >> kKeyOffsetBits) != (k >> kKeyOffsetBits);
      t = h || (kp & mask) / page != o / page;
    }
    head[i] = h;
    trans[i] = t;
    if (offsets_out) offsets_out[i] = o;
  }
}

__global__ void k_plan_groups(const uint64_t* __restrict__ keys, const uint8_t* __restrict__ head,
                              const uint32_t* __restrict__ gidx, const uint32_t* __restrict__ tscan,
                              const uint8_t* __restrict__ trans, uint64_t b, uint32_t ngroups,
                              int64_t* __restrict__ gloc, uint64_t* __restrict__ gstart,
                              uint64_t* __restrict__ gtrans_start) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (head[i]) {
      const uint32_t g = gidx[i];
      gloc[g] = static_cast<int64_t>(keys[i] >> kKeyOffsetBits);
      gstart[g] = i;
      gtrans_start[g] = tscan[i];
    }
    if (i == b - 1) {
      gstart[ngroups] = b;
      gtrans_start[ngroups] = (uint64_t)tscan[i] + trans[i];
    }
  }
}

}  // namespace

void plan_reads_device(const int64_t* d_loc, const uint64_t* d_off, uint64_t table_n,
                       const uint64_t* d_ids, uint64_t b, uint64_t page, DeviceReadPlan& out,
                       cudaStream_t s) {
  if (page == 0) fail(QVB_ERR_VALIDATION, "page size must be > 0");
  if (b >= (1ull << 32)) fail(QVB_ERR_UNSUPPORTED, "batch exceeds 2^32 ids");
  out.b = b;
  out.groups = 0;
  if (b == 0) return;
  DevBuf<uint64_t> keys(b, s);
  DevBuf<uint32_t> idx(b, s);
  DevBuf<unsigned long long> bad(1, s);
  QVB_CUDA(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
  k_plan_keys<<<grid_for(b, 256), 256, 0, s>>>(d_loc, d_off, table_n, d_ids, b, keys.p, idx.p, bad.p);
  QVB_LAUNCH_CHECK();
  const unsigned long long bd = read_scalar(bad.p, s);
  if (bd != ~0ull) {
    uint64_t fid = 0;
    QVB_CUDA(cudaMemcpy(&fid, d_ids + (bd >> 1), 8, cudaMemcpyDeviceToHost));
    if (bd & 1) fail(QVB_ERR_UNSUPPORTED, "lookup entry of feature " + std::to_string(fid) +
                                              " outside the device key range");
    fail(QVB_ERR_VALIDATION, "feature id " + std::to_string(fid) + " outside lookup table");
  }
  out.keys.alloc(b, s);
  out.order.alloc(b, s);
  sort_pairs_u64_u32(keys.p, out.keys.p, idx.p, out.order.p, b, 0, 64, s);
  DevBuf<uint8_t> head(b, s), trans(b, s);
  out.offsets.alloc(b, s);
  k_plan_marks<<<grid_for(b, 256), 256, 0, s>>>(out.keys.p, b, page, head.p, trans.p, out.offsets.p);
  QVB_LAUNCH_CHECK();
  DevBuf<uint32_t> gidx(b, s), tscan(b, s);
  exclusive_sum_u8_u32(head.p, gidx.p, b, s);
  exclusive_sum_u8_u32(trans.p, tscan.p, b, s);
  const uint32_t ng = read_scalar(gidx.p + (b - 1), s) + read_scalar(head.p + (b - 1), s);
  out.groups = ng;
  out.gloc.alloc(ng, s);
  out.gstart.alloc(ng + 1, s);
  out.gtrans.alloc(ng + 1, s);
  k_plan_groups<<<grid_for(b, 256), 256, 0, s>>>(out.keys.p, head.p, gidx.p, tscan.p, trans.p, b,
                                                 ng, out.gloc.p, out.gstart.p, out.gtrans.p);
  QVB_LAUNCH_CHECK();
}

}  // namespace qvb

using namespace qvb;

extern "C" int qvb_page_transitions(const uint64_t* offsets, uint64_t count, uint64_t page_size,
                                    uint64_t* out) {
  return guarded([&] {
    if (!out) fail(QVB_ERR_VALIDATION, "null argument");
    // placement.cpp:344-353 (host arithmetic: a handful of integer ops)
    if (count == 0) {
      *out = 0;
      return;
    }
    if (page_size == 0) fail(QVB_ERR_VALIDATION, "page size must be > 0");
    uint64_t t = 1;
    for (uint64_t i = 1; i < count; ++i)
      if (offsets[i] / page_size != offsets[i - 1] / page_size) ++t;
    *out = t;
  });
}

extern "C" int qvb_plan_reads(int device, const int64_t* location_ids, const uint64_t* offsets,
                              uint64_t table_n, const uint64_t* ids, uint64_t b,
                              uint64_t page_size, int64_t* group_loc, uint64_t* group_count,
                              uint64_t* group_transitions, uint64_t* n_groups,
                              uint64_t* offsets_out) {
  return guarded([&] {
    if (page_size == 0) fail(QVB_ERR_VALIDATION, "page size must be > 0");
    if (!n_groups) fail(QVB_ERR_VALIDATION, "null argument");
    *n_groups = 0;
    if (b == 0) return;
    if (!location_ids || !offsets || !ids || !group_loc || !group_count || !group_transitions ||
        !offsets_out)
      fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<int64_t> dloc(table_n ? table_n : 1, s);
    DevBuf<uint64_t> doff(table_n ? table_n : 1, s), dids(b, s);
    if (table_n) {
      QVB_CUDA(cudaMemcpyAsync(dloc.p, location_ids, table_n * 8, cudaMemcpyHostToDevice, s));
      QVB_CUDA(cudaMemcpyAsync(doff.p, offsets, table_n * 8, cudaMemcpyHostToDevice, s));
    }
    QVB_CUDA(cudaMemcpyAsync(dids.p, ids, b * 8, cudaMemcpyHostToDevice, s));
    DeviceReadPlan rp;
    plan_reads_device(dloc.p, doff.p, table_n, dids.p, b, page_size, rp, s);
    const uint32_t ng = rp.groups;
    std::vector<uint64_t> start(ng + 1), tr(ng + 1);
    QVB_CUDA(cudaMemcpyAsync(group_loc, rp.gloc.p, ng * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaMemcpyAsync(start.data(), rp.gstart.p, (ng + 1) * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaMemcpyAsync(tr.data(), rp.gtrans.p, (ng + 1) * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaMemcpyAsync(offsets_out, rp.offsets.p, b * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
    for (uint32_t g = 0; g < ng; ++g) {
      group_count[g] = start[g + 1] - start[g];
      group_transitions[g] = tr[g + 1] - tr[g];
    }
    *n_groups = ng;
  });
}
