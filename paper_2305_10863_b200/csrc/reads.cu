// reads.cu — K4, the read planner of the collect call (plan_reads +
// page_transitions, reference placement.cpp:344-380).
//
// The reference groups the requested ids by location through a std::map
// (ascending location id) and sorts each group's offsets ascending,
// duplicates kept. On the device: look up (location, offset) per request,
// pack key = location << 40 | offset, stable radix sort with the request
// index as payload (the payload is what the planned gather consumes), then
// mark group heads and page changes and compact them with two scans.
#include <algorithm>
#include <string>
#include <vector>

#include "reads.cuh"

namespace qvb {
namespace {

// A request's (location, offset): from the reference-layout table (loc[],
// off[]) or from a store's packed one (loc << 48 | offset, ~0 = no copy).
struct TableView {
  const int64_t* loc;
  const uint64_t* off;
  const uint64_t* packed;
  __device__ __forceinline__ void get(uint64_t f, int64_t& l, uint64_t& o) const {
    if (packed) {
      const uint64_t p = packed[f];
      l = p == ~0ull ? -1 : static_cast<int64_t>(p >> kPackedOffsetBits);
      o = p & ((1ull << kPackedOffsetBits) - 1);
    } else {
      l = loc[f];
      o = off[f];
    }
  }
};

// key = location << ob | offset (ob = bits of the largest possible offset,
// table_n - 1: a location's offsets are dense ranks of its features);
// flags[0] = first bad request (2i: id outside the table, 2i+1: entry outside
// the key range), flags[1] = largest location id (sizes the sort)
__global__ void k_plan_keys(TableView t, uint64_t table_n, int ob, const uint64_t* __restrict__ ids,
                            uint64_t b, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                            unsigned long long* flags) {
  unsigned long long maxloc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = ids[i];
    uint64_t k = 0;
    if (f >= table_n) {
      atomicMin(flags, (unsigned long long)(i << 1));
    } else {
      int64_t l;
      uint64_t o;
      t.get(f, l, o);
      if (l < 0 || (ob < 64 && (uint64_t)l >= (1ull << (64 - ob))) || o >= (1ull << ob)) {
        atomicMin(flags, (unsigned long long)((i << 1) | 1));
      } else {
        k = ((uint64_t)l << ob) | o;
        maxloc = maxloc > (unsigned long long)l ? maxloc : (unsigned long long)l;
      }
    }
    keys[i] = k;
    idx[i] = static_cast<uint32_t>(i);
  }
  maxloc = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(maxloc));
  if ((threadIdx.x & 31) == 0 && maxloc) atomicMax(flags + 1, maxloc);
}

// head: first of a location group; trans: counts toward the group's page
// transitions (1 + adjacent page changes, placement.cpp:344-353).
__global__ void k_plan_marks(const uint64_t* __restrict__ keys, uint64_t b, int ob, uint64_t page,
                             uint8_t* __restrict__ head, uint8_t* __restrict__ trans,
                             uint64_t* __restrict__ offsets_out) {
  const uint64_t mask = (1ull << ob) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const uint64_t o = k & mask;
    bool h = i == 0, t = i == 0;
    if (i > 0) {
      const uint64_t kp = keys[i - 1];
      h = (kp >> ob) != (k >> ob);
      t = h || (kp & mask) / page != o / page;
    }
    head[i] = h;
    trans[i] = t;
    if (offsets_out) offsets_out[i] = o;
  }
}

__global__ void k_plan_groups(const uint64_t* __restrict__ keys, int ob, const uint8_t* __restrict__ head,
                              const uint32_t* __restrict__ gidx, const uint32_t* __restrict__ tscan,
                              const uint8_t* __restrict__ trans, uint64_t b, uint32_t ngroups,
                              int64_t* __restrict__ gloc, uint64_t* __restrict__ gcount,
                              uint64_t* __restrict__ gtr) {
  // gcount/gtr first hold each group's start and transition prefix; the
  // differences are taken by k_plan_counts
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (head[i]) {
      const uint32_t g = gidx[i];
      gloc[g] = static_cast<int64_t>(keys[i] >> ob);
      gcount[g] = i;
      gtr[g] = tscan[i];
    }
    if (i == b - 1) {
      gcount[ngroups] = b;
      gtr[ngroups] = (uint64_t)tscan[i] + trans[i];
    }
  }
}

__global__ void k_plan_counts(uint32_t ngroups, uint64_t* __restrict__ gcount, uint64_t* __restrict__ gtr) {
  // one thread: ngroups is the number of distinct locations (small)
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint32_t g = 0; g < ngroups; ++g) {
      gcount[g] = gcount[g + 1] - gcount[g];
      gtr[g] = gtr[g + 1] - gtr[g];
    }
}

}  // namespace

void plan_reads_device(const int64_t* d_loc, const uint64_t* d_off, const uint64_t* d_packed,
                       uint64_t table_n, const uint64_t* d_ids, uint64_t b, uint64_t page,
                       DeviceReadPlan& out, cudaStream_t s) {
  if (page == 0) fail(QVB_ERR_VALIDATION, "page size must be > 0");
  if (b >= (1ull << 32)) fail(QVB_ERR_UNSUPPORTED, "batch exceeds 2^32 ids");
  out.b = b;
  out.groups = 0;
  if (b == 0) return;
  const int ob = table_n > 1 ? bits_for(table_n - 1) : 1;
  out.ob = ob;
  DevBuf<uint64_t> keys(b, s);
  DevBuf<uint32_t> idx(b, s);
  DevBuf<unsigned long long> flags(2, s);
  QVB_CUDA(cudaMemsetAsync(flags.p, 0xFF, sizeof(unsigned long long), s));
  QVB_CUDA(cudaMemsetAsync(flags.p + 1, 0, sizeof(unsigned long long), s));
  k_plan_keys<<<grid_for(b, 256), 256, 0, s>>>(TableView{d_loc, d_off, d_packed}, table_n, ob, d_ids, b,
                                               keys.p, idx.p, flags.p);
  QVB_LAUNCH_CHECK();
  unsigned long long fl[2];
  QVB_CUDA(cudaMemcpyAsync(fl, flags.p, sizeof fl, cudaMemcpyDeviceToHost, s));
  QVB_CUDA(cudaStreamSynchronize(s));
  if (fl[0] != ~0ull) {
    uint64_t fid = 0;
    QVB_CUDA(cudaMemcpy(&fid, d_ids + (fl[0] >> 1), 8, cudaMemcpyDefault));
    if (fl[0] & 1) fail(QVB_ERR_UNSUPPORTED, "lookup entry of feature " + std::to_string(fid) +
                                                  " outside the device key range");
    fail(QVB_ERR_VALIDATION, "feature id " + std::to_string(fid) + " outside lookup table");
  }
  // sort only the key bits in use: ob offset bits + the largest location's
  // (C4 at one GPU: 27 + 2 bits, 4 passes of 8 instead of 8)
  const int end_bit = std::min(64, ob + bits_for(fl[1]));
  out.keys.alloc(b, s);
  out.order.alloc(b, s);
  sort_pairs_u64_u32(keys.p, out.keys.p, idx.p, out.order.p, b, 0, end_bit, s);
  DevBuf<uint8_t> head(b, s), trans(b, s);
  out.offsets.alloc(b, s);
  k_plan_marks<<<grid_for(b, 256), 256, 0, s>>>(out.keys.p, b, ob, page, head.p, trans.p, out.offsets.p);
  QVB_LAUNCH_CHECK();
  DevBuf<uint32_t> gidx(b, s), tscan(b, s);
  exclusive_sum_u8_u32(head.p, gidx.p, b, s);
  exclusive_sum_u8_u32(trans.p, tscan.p, b, s);
  const uint32_t ng = read_scalar(gidx.p + (b - 1), s) + read_scalar(head.p + (b - 1), s);
  out.groups = ng;
  out.gloc.alloc(ng, s);
  out.gcount.alloc(ng + 1, s);
  out.gtrans.alloc(ng + 1, s);
  k_plan_groups<<<grid_for(b, 256), 256, 0, s>>>(out.keys.p, ob, head.p, gidx.p, tscan.p, trans.p, b,
                                                 ng, out.gloc.p, out.gcount.p, out.gtrans.p);
  QVB_LAUNCH_CHECK();
  k_plan_counts<<<1, 32, 0, s>>>(ng, out.gcount.p, out.gtrans.p);
  QVB_LAUNCH_CHECK();
}

// The flattened ReadPlan into host buffers (group arrays need room for every
// distinct location; offsets_out for b offsets).
void copy_read_plan(const DeviceReadPlan& rp, int64_t* group_loc, uint64_t* group_count,
                    uint64_t* group_transitions, uint64_t* n_groups, uint64_t* offsets_out,
                    cudaStream_t s) {
  const uint32_t ng = rp.groups;
  if (ng) {
    QVB_CUDA(cudaMemcpyAsync(group_loc, rp.gloc.p, ng * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaMemcpyAsync(group_count, rp.gcount.p, ng * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaMemcpyAsync(group_transitions, rp.gtrans.p, ng * 8, cudaMemcpyDeviceToHost, s));
    copy_to_host(offsets_out, rp.offsets.p, rp.b * 8, s);
  }
  QVB_CUDA(cudaStreamSynchronize(s));
  *n_groups = ng;
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
    plan_reads_device(dloc.p, doff.p, nullptr, table_n, dids.p, b, page_size, rp, s);
    copy_read_plan(rp, group_loc, group_count, group_transitions, n_groups, offsets_out, s);
  });
}

extern "C" int qvb_plan_reads_device(int device, const int64_t* location_ids, const uint64_t* offsets,
                                     uint64_t table_n, const uint64_t* ids, uint64_t b,
                                     uint64_t page_size, int64_t* group_loc, uint64_t* group_count,
                                     uint64_t* group_transitions, uint64_t* n_groups,
                                     uint64_t* offsets_out, void* stream) {
  return guarded([&] {
    if (page_size == 0) fail(QVB_ERR_VALIDATION, "page size must be > 0");
    if (!n_groups) fail(QVB_ERR_VALIDATION, "null argument");
    *n_groups = 0;
    if (b == 0) return;
    if (!location_ids || !offsets || !ids || !group_loc || !group_count || !group_transitions ||
        !offsets_out)
      fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceReadPlan rp;
    plan_reads_device(location_ids, offsets, nullptr, table_n, ids, b, page_size, rp, s);
    copy_read_plan(rp, group_loc, group_count, group_transitions, n_groups, offsets_out, s);
  });
}
