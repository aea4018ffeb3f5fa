// store.cu — K5, the feature collection the reference only models
// (fetch_cost, placement.cpp:382-404, called per batch from
// simulator.cpp:320-326): a real one-sided gather
//   out[i][0:dim] = X[ids[i]][0:dim]
// from local HBM, peer HBM (CUDA IPC mapping over NVLink/NVSwitch) or host
// pinned memory (zero-copy UVA), chosen per lookup-table entry.
//
// HBM layout of one store (reader GPU d):
//   lut    u64[n]  packed loc << 48 | offset (this reader's per-reader table)
//   local  shard of location d: rows of the features holding a copy at d,
//          ascending feature id (== the reference's cursor offsets),
//          stride = dim*4 rounded up to 64 bytes (16 for rows < 64 B)
//   host   pinned + mapped shard of the host location, same layout
//   base[] one base pointer per location (peers attached via IPC handles)
//
// Gather kernel: the batch is a flat array of VEC-byte chunks (VEC = 16 when
// rows are 16-byte aligned, else 8 or 4); consecutive lanes take consecutive
// chunks (coalesced row reads and writes), every thread keeps U independent
// chunk loads in flight, loads use ld.global.nc.L1::no_allocate (the source
// is read-only for the store's lifetime). The id and lookup-table reads of a
// row are shared by its lanes (same address, one transaction).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "placement.cuh"
#include "reads.cuh"

namespace qvb {
namespace {

struct Bases {
  const char* p[kMaxLocations];
};

template <int VEC>
struct Vec;
// Row reads and writes are a stream (each row moves once per gather): L2
// evict_first, so they do not push out the lookup table, whose lines are
// reused by several requests of a batch (C2: 8 entries per 64-byte line,
// 1M lookups into 2.4M entries).
template <>
struct Vec<16> {
  using T = uint4;
  static __device__ __forceinline__ T load(const char* p, uint64_t pol) {
    T r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
  }
  static __device__ __forceinline__ void store(char* p, const T& v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
  }
};
template <>
struct Vec<8> {
  using T = uint2;
  static __device__ __forceinline__ T load(const char* p, uint64_t pol) {
    T r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p), "l"(pol));
    return r;
  }
  static __device__ __forceinline__ void store(char* p, const T& v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;" ::"l"(p), "r"(v.x), "r"(v.y),
                 "l"(pol)
                 : "memory");
  }
};
template <>
struct Vec<4> {
  using T = uint32_t;
  static __device__ __forceinline__ T load(const char* p, uint64_t pol) {
    T r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(r)
                 : "l"(p), "l"(pol));
    return r;
  }
  static __device__ __forceinline__ void store(char* p, const T& v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
  }
};

constexpr int kGatherBlock = 256;
constexpr int kUnroll = 8;

// Direct gather over request order. rows < 2^32 / cpr per launch.
template <int VEC>
__global__ void __launch_bounds__(kGatherBlock)
    k_gather(const uint64_t* __restrict__ ids, uint32_t rows, const uint64_t* __restrict__ lut,
             Bases bases, uint64_t stride, uint32_t cpr, uint32_t row_bytes, uint64_t n,
             char* __restrict__ out, uint64_t row_base, unsigned long long* err) {
  using V = Vec<VEC>;
  const uint64_t pol = policy_evict_first();  // rows: a stream
  const uint32_t total = rows * cpr;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  for (uint32_t c0 = blockIdx.x * blockDim.x + threadIdx.x; c0 < total; c0 += nthreads * kUnroll) {
    typename V::T v[kUnroll];
    uint64_t dst[kUnroll];
    bool ok[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t c = c0 + u * nthreads;
      ok[u] = c < total;
      if (ok[u]) {
        const uint32_t i = c / cpr;
        const uint32_t k = c - i * cpr;
        const uint64_t f = __ldg(ids + i);
        if (f >= n) {
          atomicMin(err, (unsigned long long)(row_base + i));
          ok[u] = false;
        } else {
          const uint64_t e = __ldg(lut + f);
          const char* src = bases.p[e >> kOffsetBits] + (e & kOffsetMask) * stride + k * VEC;
          v[u] = V::load(src, pol);
          dst[u] = (uint64_t)i * row_bytes + (uint64_t)k * VEC;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (ok[u]) V::store(out + dst[u], v[u], pol);
  }
}

// Row-group gather (v3): a warp serves 32 consecutive requests at a time.
// Lane l resolves request l of the group (id -> lookup entry -> source row
// address) once; the group's 32 rows are then copied as one flat run of
// VEC-byte chunks — chunk c of the group lands at out + c*VEC because the
// output rows are contiguous, and its source is the row address shuffled
// from lane c/cpr plus (c%cpr)*VEC, with (row, offset) advanced
// incrementally. Ids and lookup entries of the next groups are fetched one
// and two groups ahead so the dependent id -> entry -> row chain overlaps the
// current copy.
template <int VEC, int kU, int kMinBlocks>
__global__ void __launch_bounds__(kGatherBlock, kMinBlocks)
    k_gather_rows(const uint64_t* __restrict__ ids, uint64_t rows,
                  const uint64_t* __restrict__ lut, Bases bases, uint64_t stride, uint32_t cpr,
                  uint32_t row_bytes, uint64_t n, char* __restrict__ out,
                  unsigned long long* err, int lut_keep) {
  using V = Vec<VEC>;
  const uint64_t pol = policy_evict_first();  // rows: a stream
  // a lookup table that fits L2 comfortably is kept there across the batch
  const uint64_t lpol = lut_keep ? policy_evict_last() : policy_evict_normal();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t groups = (rows + 31) / 32;
  const uint32_t q32 = 32 / cpr, r32 = 32 % cpr;
  const uint32_t row0 = lane / cpr, k0 = lane - row0 * cpr;

  auto load_id = [&](uint64_t g) -> uint64_t {
    const uint64_t r = g * 32 + lane;
    return (g < groups && r < rows) ? __ldg(ids + r) : ~0ull;
  };
  auto resolve = [&](uint64_t g, uint64_t f) -> uint64_t {  // source row address or 0
    const uint64_t r = g * 32 + lane;
    if (g >= groups || r >= rows) return 0;
    if (f >= n) {
      atomicMin(err, (unsigned long long)r);
      return 0;
    }
    const uint64_t e = ld_hint(lut + f, lpol);
    return reinterpret_cast<uint64_t>(bases.p[e >> kOffsetBits]) + (e & kOffsetMask) * stride;
  };

  uint64_t g = warp;
  uint64_t src = resolve(g, load_id(g));
  uint64_t id_next = load_id(g + nwarps);
  for (; g < groups; g += nwarps) {
    const uint64_t src_next = resolve(g + nwarps, id_next);  // one group ahead
    id_next = load_id(g + 2 * nwarps);                      // two groups ahead
    const uint32_t nr = static_cast<uint32_t>(rows - g * 32 < 32 ? rows - g * 32 : 32);
    const uint32_t tot = nr * cpr;
    char* dst0 = out + g * 32 * (uint64_t)row_bytes;
    uint32_t row = row0, k = k0;
    for (uint32_t cb = 0; cb < tot; cb += 32 * kU) {  // warp-uniform trip count
      const uint32_t c0 = cb + lane;
      typename V::T v[kU];
      bool ok[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t c = c0 + u * 32;
        const uint64_t s = __shfl_sync(0xffffffffu, src, row < 32 ? row : 31);
        ok[u] = c < tot && s != 0;
        if (ok[u]) v[u] = V::load(reinterpret_cast<const char*>(s) + (uint64_t)k * VEC, pol);
        row += q32;
        k += r32;
        if (k >= cpr) {
          k -= cpr;
          ++row;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ok[u]) V::store(dst0 + (uint64_t)(c0 + u * 32) * VEC, v[u], pol);
    }
    src = src_next;
  }
}

// Row-group gather for 512-byte rows (D = 128 fp32): lane l owns the 16-byte
// column l of every row, so a round of kU loads covers kU whole rows with no
// per-chunk (row, offset) bookkeeping. Lookup entries are fetched two groups
// ahead and ids three, so the dependent id -> entry -> row chain (the table
// does not fit L2 at papers scale) stays off the copy's critical path.
template <int kU, int kMinBlocks>
__global__ void __launch_bounds__(kGatherBlock, kMinBlocks)
    k_gather_rows512(const uint64_t* __restrict__ ids, uint64_t rows,
                     const uint64_t* __restrict__ lut, Bases bases, uint64_t stride,
                     uint64_t n, char* __restrict__ out, unsigned long long* err, int lut_keep) {
  using V = Vec<16>;
  const uint64_t pol = policy_evict_first();  // rows: a stream
  const uint64_t lpol = lut_keep ? policy_evict_last() : policy_evict_normal();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t groups = (rows + 31) / 32;
  auto load_id = [&](uint64_t g) -> uint64_t {
    const uint64_t r = g * 32 + lane;
    return (g < groups && r < rows) ? __ldg(ids + r) : ~0ull;
  };
  auto resolve = [&](uint64_t g, uint64_t f) -> uint64_t {  // source row address or 0
    const uint64_t r = g * 32 + lane;
    if (g >= groups || r >= rows) return 0;
    if (f >= n) {
      atomicMin(err, (unsigned long long)r);
      return 0;
    }
    const uint64_t e = ld_hint(lut + f, lpol);
    return reinterpret_cast<uint64_t>(bases.p[e >> kOffsetBits]) + (e & kOffsetMask) * stride;
  };
  uint64_t g = warp;
  uint64_t src = resolve(g, load_id(g));
  uint64_t src1 = resolve(g + nwarps, load_id(g + nwarps));
  uint64_t id2 = load_id(g + 2 * nwarps);
  for (; g < groups; g += nwarps) {
    const uint64_t src2 = resolve(g + 2 * nwarps, id2);  // two groups ahead
    id2 = load_id(g + 3 * nwarps);                      // three groups ahead
    const uint32_t nr = static_cast<uint32_t>(rows - g * 32 < 32 ? rows - g * 32 : 32);
    char* dst0 = out + g * 32 * 512ull + lane * 16;
    for (uint32_t r0 = 0; r0 < nr; r0 += kU) {  // warp-uniform
      typename V::T v[kU];
      uint32_t ok = 0;  // rows of this round that were loaded (one bit each)
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t sr = __shfl_sync(0xffffffffu, src, (r0 + u) & 31);
        if (r0 + u < nr && sr) {
          v[u] = V::load(reinterpret_cast<const char*>(sr) + lane * 16, pol);
          ok |= 1u << u;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ok >> u & 1) V::store(dst0 + (uint64_t)(r0 + u) * 512, v[u], pol);
    }
    src = src1;
    src1 = src2;
  }
}

// Rows that are 8-byte but not 16-byte multiples (e.g. 602 fp32 = 2408 B):
// the shard stride is 64-byte aligned, so the source side still moves 16-byte
// vectors; the destination rows are only 8-byte aligned, so every 16-byte
// chunk is stored as two 8-byte halves (the row's last chunk keeps one).
template <int kU, int kMinBlocks>
__global__ void __launch_bounds__(kGatherBlock, kMinBlocks)
    k_gather_rows_w(const uint64_t* __restrict__ ids, uint64_t rows,
                    const uint64_t* __restrict__ lut, Bases bases, uint64_t stride, uint32_t cpr,
                    uint32_t row_bytes, uint64_t n, char* __restrict__ out,
                    unsigned long long* err) {
  using V = Vec<16>;
  const uint64_t pol = policy_evict_first();  // rows: a stream
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t groups = (rows + 31) / 32;
  const uint32_t q32 = 32 / cpr, r32 = 32 % cpr;
  const uint32_t row0 = lane / cpr, k0 = lane - row0 * cpr;
  auto load_id = [&](uint64_t g) -> uint64_t {
    const uint64_t r = g * 32 + lane;
    return (g < groups && r < rows) ? __ldg(ids + r) : ~0ull;
  };
  auto resolve = [&](uint64_t g, uint64_t f) -> uint64_t {
    const uint64_t r = g * 32 + lane;
    if (g >= groups || r >= rows) return 0;
    if (f >= n) {
      atomicMin(err, (unsigned long long)r);
      return 0;
    }
    const uint64_t e = __ldg(lut + f);
    return reinterpret_cast<uint64_t>(bases.p[e >> kOffsetBits]) + (e & kOffsetMask) * stride;
  };
  uint64_t g = warp;
  uint64_t src = resolve(g, load_id(g));
  uint64_t id_next = load_id(g + nwarps);
  for (; g < groups; g += nwarps) {
    const uint64_t src_next = resolve(g + nwarps, id_next);
    id_next = load_id(g + 2 * nwarps);
    const uint32_t nr = static_cast<uint32_t>(rows - g * 32 < 32 ? rows - g * 32 : 32);
    const uint32_t tot = nr * cpr;
    char* out0 = out + g * 32 * (uint64_t)row_bytes;
    uint32_t row = row0, k = k0;
    for (uint32_t cb = 0; cb < tot; cb += 32 * kU) {
      typename V::T v[kU];
      uint64_t dst[kU];
      bool ok[kU], half[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t c = cb + lane + u * 32;
        const uint64_t s = __shfl_sync(0xffffffffu, src, row < 32 ? row : 31);
        ok[u] = c < tot && s != 0;
        half[u] = (k + 1) * 16 > row_bytes;
        dst[u] = (uint64_t)row * row_bytes + (uint64_t)k * 16;
        if (ok[u]) v[u] = V::load(reinterpret_cast<const char*>(s) + (uint64_t)k * 16, pol);
        row += q32;
        k += r32;
        if (k >= cpr) {
          k -= cpr;
          ++row;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (!ok[u]) continue;
        uint2* d = reinterpret_cast<uint2*>(out0 + dst[u]);
        d[0] = make_uint2(v[u].x, v[u].y);
        if (!half[u]) d[1] = make_uint2(v[u].z, v[u].w);
      }
    }
    src = src_next;
  }
}

// TMA bulk-copy gather (rows that are 16-byte multiples, device-resident
// sources): each lane owns one request of a 32-row group; it issues one
// cp.async.bulk global->shared copy of its row (completion counted on the
// group's mbarrier) and, once the group has landed, one cp.async.bulk
// shared->global copy to the output row. Two row buffers per warp let the
// next group's loads overlap the previous group's stores; no row data ever
// passes through registers, so every SM keeps hundreds of rows in flight.
// cp.async (LDGSTS) row-group gather for rows of <= 512 B in 16-byte chunks:
// the loads of group j+1 land in shared memory (no registers held) while
// group j is written out, so each SM keeps ~100 KB of rows in flight. Every
// lane reads back only the slots it filled itself (layout [buffer][m][lane]),
// so no cross-lane synchronisation is needed.
__global__ void __launch_bounds__(256)
    k_gather_cp(const uint64_t* __restrict__ ids, uint64_t rows, const uint64_t* __restrict__ lut,
                Bases bases, uint64_t stride, uint32_t cpr, uint32_t row_bytes, uint64_t n,
                char* __restrict__ out, unsigned long long* err) {
  extern __shared__ __align__(128) uint4 slots[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint4* mine = slots + (uint64_t)wid * 2 * cpr * 32;  // [2][cpr][32]
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t groups = (rows + 31) / 32;
  const uint32_t q32 = 32 / cpr, r32 = 32 % cpr;
  const uint32_t row0 = lane / cpr, k0 = lane - row0 * cpr;
  auto resolve = [&](uint64_t g) -> uint64_t {
    const uint64_t r = g * 32 + lane;
    if (g >= groups || r >= rows) return 0;
    const uint64_t f = __ldg(ids + r);
    if (f >= n) {
      atomicMin(err, (unsigned long long)r);
      return 0;
    }
    const uint64_t e = __ldg(lut + f);
    return reinterpret_cast<uint64_t>(bases.p[e >> kOffsetBits]) + (e & kOffsetMask) * stride;
  };
  // issue this lane's chunks of group g into buffer b
  auto issue = [&](uint64_t g, uint64_t src, int b) {
    if (g >= groups) return;
    const uint32_t nr = static_cast<uint32_t>(rows - g * 32 < 32 ? rows - g * 32 : 32);
    const uint32_t tot = nr * cpr;
    uint32_t row = row0, k = k0;
    for (uint32_t m = 0; m < cpr; ++m) {
      const uint32_t c = lane + 32 * m;
      const uint64_t s = __shfl_sync(0xffffffffu, src, row < 32 ? row : 31);
      if (c < tot && s) {
        const uint32_t dst = static_cast<uint32_t>(
            __cvta_generic_to_shared(mine + ((uint64_t)b * cpr + m) * 32 + lane));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                     "l"(s + (uint64_t)k * 16)
                     : "memory");
      }
      row += q32;
      k += r32;
      if (k >= cpr) {
        k -= cpr;
        ++row;
      }
    }
  };
  uint64_t g = warp;
  uint64_t src = resolve(g);
  issue(g, src, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  int b = 0;
  for (; g < groups; g += nwarps, b ^= 1) {
    const uint64_t gn = g + nwarps;
    const uint64_t sn = resolve(gn);
    issue(gn, sn, b ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // group g has landed
    const uint32_t nr = static_cast<uint32_t>(rows - g * 32 < 32 ? rows - g * 32 : 32);
    const uint32_t tot = nr * cpr;
    const bool ok_row = true;
    uint4* dst0 = reinterpret_cast<uint4*>(out + g * 32 * (uint64_t)row_bytes);
    uint32_t row = row0;
    uint32_t k = k0;
    for (uint32_t m = 0; m < cpr; ++m) {
      const uint32_t c = lane + 32 * m;
      const uint64_t s = __shfl_sync(0xffffffffu, src, row < 32 ? row : 31);
      if (c < tot && s && ok_row) dst0[c] = mine[((uint64_t)b * cpr + m) * 32 + lane];
      row += q32;
      k += r32;
      if (k >= cpr) {
        k -= cpr;
        ++row;
      }
    }
    src = sn;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

constexpr int kTmaBuffers = 3;  // per warp: 2 groups of loads + 1 of stores in flight

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256)
    k_gather_tma(const uint64_t* __restrict__ ids, uint64_t rows, const uint64_t* __restrict__ lut,
                 Bases bases, uint64_t stride, uint32_t row_bytes, uint64_t n,
                 char* __restrict__ out, unsigned long long* err) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NB = kTmaBuffers;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t warps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // NB per warp
  unsigned char* buf = smem + 8 * NB * warps + (128 - (8 * NB * warps) % 128) % 128;
  if (lane == 0) {
    for (int i = 0; i < NB; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[NB * wid + i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t groups = (rows + 31) / 32;
  uint32_t phases = 0;  // bit i: parity to wait for on buffer i
  // group j of this warp is global group warp + j*nwarps, buffer j % NB
  auto resolve = [&](uint64_t j) -> uint64_t {
    const uint64_t g = warp + j * nwarps;
    const uint64_t r = g * 32 + lane;
    if (g >= groups || r >= rows) return 0;
    const uint64_t f = __ldg(ids + r);
    if (f >= n) {
      atomicMin(err, (unsigned long long)r);
      return 0;
    }
    const uint64_t e = __ldg(lut + f);
    return reinterpret_cast<uint64_t>(bases.p[e >> kOffsetBits]) + (e & kOffsetMask) * stride;
  };
  auto issue_loads = [&](uint64_t j, uint64_t src) {
    const int bi = static_cast<int>(j % NB);
    const uint32_t bar = smem_addr(&bars[NB * wid + bi]);
    const uint32_t valid = __popc(__ballot_sync(0xffffffffu, src != 0));
    if (valid == 0) return;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(valid * row_bytes)
                   : "memory");
    __syncwarp();
    if (src) {
      const uint32_t slot = smem_addr(buf + ((uint64_t)(NB * wid + bi) * 32 + lane) * row_bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              slot),
          "l"(src), "r"(row_bytes), "r"(bar)
          : "memory");
    }
  };
  const uint64_t mine = warp < groups ? (groups - warp + nwarps - 1) / nwarps : 0;
  uint64_t srcs[NB];
  for (int j = 0; j < NB - 1; ++j) {  // prologue: NB-1 groups of loads in flight
    srcs[j] = resolve(j);
    issue_loads(j, srcs[j]);
  }
  for (uint64_t j = 0; j < mine; ++j) {
    const int bi = static_cast<int>(j % NB);
    const uint64_t src = srcs[bi];
    const uint32_t valid = __popc(__ballot_sync(0xffffffffu, src != 0));
    if (valid) {
      asm volatile(
          "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra W_%=;\n}" ::"r"(smem_addr(&bars[NB * wid + bi])),
          "r"((phases >> bi) & 1u)
          : "memory");
      phases ^= 1u << bi;
      if (src) {
        const uint64_t r = (warp + j * nwarps) * 32 + lane;
        const uint32_t slot = smem_addr(buf + ((uint64_t)(NB * wid + bi) * 32 + lane) * row_bytes);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         out + r * (uint64_t)row_bytes),
                     "r"(slot), "r"(row_bytes)
                     : "memory");
      }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the next loads reuse the buffer whose stores were committed NB-1 groups ago
    const uint64_t jn = j + NB - 1;
    const uint64_t s_next = resolve(jn);
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 2) : "memory");
    __syncwarp();
    srcs[jn % NB] = s_next;
    issue_loads(jn, s_next);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Planned gather: sorted (location, offset) keys with the request index as
// payload (K4 order); no lookup-table read in the copy loop. A key is
// loc << ob | offset: the packed lookup entry (ob = 48), or its 32-bit
// repacking when offsets and locations fit (fewer radix passes).
template <int VEC, typename K>
__global__ void __launch_bounds__(kGatherBlock)
    k_gather_sorted(const K* __restrict__ keys, const uint32_t* __restrict__ order,
                    uint32_t rows, Bases bases, uint64_t stride, uint32_t cpr, uint32_t row_bytes,
                    char* __restrict__ out, int ob) {
  const uint64_t omask = (1ull << ob) - 1;
  using V = Vec<VEC>;
  const uint64_t pol = policy_evict_first();  // rows: a stream
  const uint32_t total = rows * cpr;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  for (uint32_t c0 = blockIdx.x * blockDim.x + threadIdx.x; c0 < total; c0 += nthreads * kUnroll) {
    typename V::T v[kUnroll];
    uint64_t dst[kUnroll];
    bool ok[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t c = c0 + u * nthreads;
      ok[u] = c < total;
      if (ok[u]) {
        const uint32_t j = c / cpr;
        const uint32_t k = c - j * cpr;
        const uint64_t e = __ldg(keys + j);
        const uint32_t i = __ldg(order + j);
        v[u] = V::load(bases.p[e >> ob] + (e & omask) * stride + k * VEC, pol);
        dst[u] = (uint64_t)i * row_bytes + (uint64_t)k * VEC;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (ok[u]) V::store(out + dst[u], v[u], pol);
  }
}

// 32-bit planned keys: loc << ob | offset, from the packed lookup entry.
__global__ void k_plan_keys32(const uint64_t* __restrict__ ids, uint64_t b,
                              const uint64_t* __restrict__ lut, uint64_t n, int ob,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ idx,
                              unsigned long long* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = ids[i];
    uint64_t e = 0;
    if (f >= n) atomicMin(err, (unsigned long long)i);
    else e = lut[f];
    keys[i] = static_cast<uint32_t>(((e >> kOffsetBits) << ob) | (e & kOffsetMask));
    idx[i] = static_cast<uint32_t>(i);
  }
}

__global__ void k_plan_keys_packed(const uint64_t* __restrict__ ids, uint64_t b,
                                   const uint64_t* __restrict__ lut, uint64_t n,
                                   uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                                   unsigned long long* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = ids[i];
    uint64_t k = 0;
    if (f >= n) atomicMin(err, (unsigned long long)i);
    else k = lut[f];
    keys[i] = k;
    idx[i] = static_cast<uint32_t>(i);
  }
}

// ---- tier-isolated gather (requests bucketed by location class) -------------
// The reference groups a batch by location before reading (plan_reads,
// placement.cpp:363-379) and models each location's reads as concurrent
// streams (fetch_cost, :388-402). Here: one pass sorts the requests into
// three lists — local HBM, peer HBM (NVLink), host (PCIe) — and the copy
// kernel's warps take 32-row groups from the lists through atomic cursors,
// each warp starting on its own class, so PCIe rows never sit in the same
// load round as HBM rows (a mixed round waits for its slowest row).
constexpr int kClasses = 3;  // 0 local, 1 peer, 2 host

struct ClassLists {
  uint32_t* req[kClasses];             // request index
  unsigned long long* src[kClasses];   // source row address
  unsigned int* count;                 // [kClasses] list lengths
  unsigned int* cursor;                // [kClasses] next 32-row group to take
  unsigned int* hist;                  // host rows per offset bucket (null: unordered)
  unsigned long long* cur;             // bucket cursors: exclusive prefix of hist
  int hshift;                          // host offset >> hshift = bucket
};

// Host-tier requests in ascending offset buckets (a counting sort of the host
// list on kHostBuckets offset ranges): pinned host pages are then walked in
// address order, which keeps the GPU's page-table walks for system memory
// local — random rows from a 14 GB host tier read at 38 GB/s, rows in offset
// order well above (profiles/r01k_host_tier.txt, r01m_gather_sweep.md).
constexpr int kHostBucketBits = 18;  // upper bound of QVB_HOST_BUCKET_BITS
constexpr int kHostBuckets = 1 << kHostBucketBits;

// One id per thread; list positions are reserved with ONE atomic per class
// per block-iteration (warp ballots -> per-warp counts in shared memory ->
// block prefix), not one per warp: 1M ids with per-warp atomics queued ~65K
// atomics on the three list counters and took 0.11-0.13 ms (ncu, C4 h = 0.1),
// a tenth of the whole gather.
constexpr int kSplitBlock = 256;
__global__ void __launch_bounds__(kSplitBlock)
    k_split_classes(const uint64_t* __restrict__ ids, uint64_t b, const uint64_t* __restrict__ lut,
                    Bases bases, uint64_t stride, uint64_t n, int local_loc, int host_loc,
                    ClassLists L, unsigned long long* err) {
  constexpr int kWarps = kSplitBlock / 32;
  __shared__ unsigned int wpre[kWarps][kClasses];  // per-warp counts -> exclusive block prefix
  __shared__ unsigned int bbase[kClasses];         // the block's reserved list starts
  const uint64_t host_base = reinterpret_cast<uint64_t>(bases.p[host_loc]);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t stride_all = (uint64_t)gridDim.x * blockDim.x;
  // block-uniform trip count: every thread reaches the barriers
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < b; i0 += stride_all) {
    const uint64_t i = i0 + threadIdx.x;
    int cls = -1;
    uint64_t src = 0;
    if (i < b) {
      const uint64_t f = __ldg(ids + i);
      if (f >= n) {
        atomicMin(err, (unsigned long long)i);
      } else {
        const uint64_t e = __ldg(lut + f);
        const int loc = static_cast<int>(e >> kOffsetBits);
        cls = loc == local_loc ? 0 : (loc == host_loc ? 2 : 1);
        src = reinterpret_cast<uint64_t>(bases.p[loc]) + (e & kOffsetMask) * stride;
      }
    }
    unsigned int mine = 0;  // ballot of this lane's class
#pragma unroll
    for (int c = 0; c < kClasses; ++c) {
      const unsigned int m = __ballot_sync(0xffffffffu, cls == c);
      if (cls == c) mine = m;
      if (lane == 0) wpre[warp][c] = __popc(m);
    }
    __syncthreads();
    if (threadIdx.x < kClasses) {
      const int c = threadIdx.x;
      unsigned int run = 0;
      for (int w = 0; w < kWarps; ++w) {
        const unsigned int t = wpre[w][c];
        wpre[w][c] = run;
        run += t;
      }
      bbase[c] = run ? atomicAdd(L.count + c, run) : 0u;
    }
    __syncthreads();
    if (cls >= 0) {
      const unsigned int pos = bbase[cls] + wpre[warp][cls] + __popc(mine & lt);
      L.req[cls][pos] = static_cast<uint32_t>(i);
      L.src[cls][pos] = src;
      if (cls == 2 && L.hist) atomicAdd(L.hist + ((src - host_base) / stride >> L.hshift), 1u);
    }
    __syncthreads();  // wpre / bbase are rewritten by the next iteration
  }
}

// host list -> bucket order (order inside a bucket is arbitrary; every row
// still lands at its request's output position)
__global__ void k_bucket_scatter(ClassLists L, const uint32_t* __restrict__ in_req,
                                 const unsigned long long* __restrict__ in_src, uint64_t host_base,
                                 uint64_t stride, uint64_t cap) {
  const unsigned int cnt = __ldcg(L.count + 2);
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < cap && j < cnt;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long src = in_src[j];
    const unsigned long long pos = atomicAdd(L.cur + ((src - host_base) / stride >> L.hshift), 1ull);
    L.req[2][pos] = in_req[j];
    L.src[2][pos] = src;
  }
}

template <int VEC, int kU, bool kR512>
__global__ void __launch_bounds__(kGatherBlock, 4)
    k_gather_classes(ClassLists L, uint32_t cpr, uint32_t row_bytes, char* __restrict__ out,
                     int host_every, uint32_t host_group) {
  using V = Vec<VEC>;
  const uint64_t pol = policy_evict_first();  // rows: a stream
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t q32 = 32 / cpr, r32 = 32 % cpr;
  const uint32_t row0 = lane / cpr, k0 = lane - row0 * cpr;
  // class order of this warp: one warp in `host_every` starts on the host
  // list (enough PCIe reads in flight), the others on local then peer rows;
  // a warp whose list runs dry moves on to the next class
  int order[kClasses] = {0, 1, 2};
  if (warp % host_every == 0) {
    order[0] = 2;
    order[1] = 0;
    order[2] = 1;
  }
  unsigned int cnt[kClasses];
#pragma unroll
  for (int c = 0; c < kClasses; ++c) cnt[c] = __ldcg(L.count + c);
  int oi = 0;
  // rows per group: 32 for HBM / NVLink rows; host rows in groups of
  // host_group, so the rows in flight across the GPU form one narrow window
  // of the offset-ordered host list (with 32-row groups the ~4.7K resident
  // warps spread their reads over half of a 262K-row list, and the GPU's
  // page walks over system memory lose their locality)
  auto gsz = [&](int c) -> uint32_t { return c == 2 ? host_group : 32u; };
  // next (class, group) for this warp, or class -1 when every list is done
  auto take = [&](int& cls, unsigned int& g) {
    cls = -1;
    while (oi < kClasses) {
      const int c = order[oi];
      unsigned int t = 0;
      if (lane == 0) t = cnt[c] ? atomicAdd(L.cursor + c, 1u) : 0xFFFFFFFFu;
      t = __shfl_sync(0xffffffffu, t, 0);
      if (cnt[c] && (uint64_t)t * gsz(c) < cnt[c]) {
        cls = c;
        g = t;
        return;
      }
      ++oi;
    }
  };
  auto fetch = [&](int cls, unsigned int g, uint64_t& src, uint64_t& dst) {
    src = 0;
    dst = 0;
    if (cls < 0) return;
    const uint64_t j = (uint64_t)g * gsz(cls) + lane;
    if (lane < gsz(cls) && j < cnt[cls]) {
      src = L.src[cls][j];
      dst = reinterpret_cast<uint64_t>(out) + (uint64_t)L.req[cls][j] * row_bytes;
    }
  };
  int cls;
  unsigned int g;
  take(cls, g);
  uint64_t src, dst;
  fetch(cls, g, src, dst);
  while (cls >= 0) {
    int ncls;
    unsigned int ng;
    take(ncls, ng);  // the next group's rows resolve while this one copies
    uint64_t nsrc, ndst;
    fetch(ncls, ng, nsrc, ndst);
    const uint64_t left = cnt[cls] - (uint64_t)g * gsz(cls);
    const uint32_t nr = static_cast<uint32_t>(left < gsz(cls) ? left : gsz(cls));
    if (kR512) {  // rows of 512·m bytes: lane = 16-byte column (k_gather_rows512's loop)
      const uint32_t m = row_bytes / 512;
      for (uint32_t rc = 0; rc < nr * m; rc += kU) {
        typename V::T v[kU];
        uint32_t ok = 0;  // warp-uniform: which (row, column) pairs of the round exist
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t r = (rc + u) / m, c = (rc + u) - r * m;
          const uint64_t s = __shfl_sync(0xffffffffu, src, r & 31);
          if (r < nr) {
            v[u] = V::load(reinterpret_cast<const char*>(s) + c * 512 + lane * 16, pol);
            ok |= 1u << u;
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (!(ok >> u & 1)) continue;
          const uint32_t r = (rc + u) / m, c = (rc + u) - r * m;
          const uint64_t d = __shfl_sync(0xffffffffu, dst, r & 31) + c * 512 + lane * 16;
          V::store(reinterpret_cast<char*>(d), v[u], pol);
        }
      }
      cls = ncls;
      g = ng;
      src = nsrc;
      dst = ndst;
      continue;
    }
    const uint32_t tot = nr * cpr;
    uint32_t row = row0, k = k0;
    for (uint32_t cb = 0; cb < tot; cb += 32 * kU) {  // warp-uniform trip count
      typename V::T v[kU];
      uint64_t d[kU];
      bool ok[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t c = cb + lane + u * 32;
        const uint32_t rr = row < 32 ? row : 31;
        const uint64_t s = __shfl_sync(0xffffffffu, src, rr);
        d[u] = __shfl_sync(0xffffffffu, dst, rr) + (uint64_t)k * VEC;
        ok[u] = c < tot;
        if (ok[u]) v[u] = V::load(reinterpret_cast<const char*>(s) + (uint64_t)k * VEC, pol);
        row += q32;
        k += r32;
        if (k >= cpr) {
          k -= cpr;
          ++row;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ok[u]) V::store(reinterpret_cast<char*>(d[u]), v[u], pol);
    }
    cls = ncls;
    g = ng;
    src = nsrc;
    dst = ndst;
  }
}

__global__ void k_fill_synthetic(const uint64_t* __restrict__ feat_of_row, uint64_t rows,
                                 uint32_t dim, uint64_t stride, char* __restrict__ shard) {
  const uint64_t total = rows * dim;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = t / dim;
    const uint32_t k = static_cast<uint32_t>(t - r * dim);
    reinterpret_cast<float*>(shard + r * stride)[k] = feature_value(feat_of_row[r], dim, k);
  }
}

__global__ void k_restride(const char* __restrict__ in, uint64_t rows, uint32_t row_bytes,
                           uint64_t stride, char* __restrict__ out) {
  const uint64_t words = row_bytes / 4;
  const uint64_t total = rows * words;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = t / words, w = t - r * words;
    reinterpret_cast<uint32_t*>(out + r * stride)[w] =
        reinterpret_cast<const uint32_t*>(in + r * row_bytes)[w];
  }
}

__global__ void k_request_ids(uint64_t state, uint64_t n, uint64_t* __restrict__ ids, uint64_t b) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < b;
       k += (uint64_t)gridDim.x * blockDim.x)
    ids[k] = to_below(stream_draw(state, k), n);
}


}  // namespace
}  // namespace qvb

using namespace qvb;

struct qvb_store {
  int device = 0;
  uint64_t n = 0;
  uint32_t dim = 0;
  uint32_t reader = 0;
  int nloc = 0;
  uint32_t row_bytes = 0;
  uint64_t stride = 0;
  uint64_t* lut = nullptr;
  char* local = nullptr;
  uint64_t local_rows = 0;
  char* host = nullptr;
  char* host_dev = nullptr;
  uint64_t host_rows = 0;
  Bases bases{};
  void* peer[kMaxLocations] = {};
  uint64_t used_mask = 0;
  unsigned long long* err = nullptr;       // qvb_gather / qvb_gather_planned
  unsigned long long* err_host = nullptr;  // qvb_gather_host's own slot (under host_mu)
  // e2e scratch; host_mu serialises qvb_gather_host calls on one store (the
  // scratch and the error slot are shared), device-side qvb_gather calls on
  // different streams stay concurrent
  std::mutex host_mu;
  uint64_t* d_ids = nullptr;
  char* d_out = nullptr;
  uint64_t cap_b = 0;

  cudaStream_t hs[2] = {nullptr, nullptr};  // qvb_gather_host chunk streams
  cudaEvent_t hev[3] = {nullptr, nullptr, nullptr};
  void ensure_host_streams() {
    if (hs[0]) return;
    for (int q = 0; q < 2; ++q) QVB_CUDA(cudaStreamCreateWithFlags(&hs[q], cudaStreamNonBlocking));
    for (int q = 0; q < 3; ++q) QVB_CUDA(cudaEventCreateWithFlags(&hev[q], cudaEventDisableTiming));
  }

  void ensure_scratch(uint64_t b) {
    if (b <= cap_b) return;
    cudaFree(d_ids);
    cudaFree(d_out);
    d_ids = nullptr;
    d_out = nullptr;
    QVB_CUDA(cudaMalloc(&d_ids, b * 8));
    QVB_CUDA(cudaMalloc(&d_out, b * (uint64_t)row_bytes));
    cap_b = b;
  }

  void check_attached() const {
    for (int l = 0; l < nloc; ++l)
      if (((used_mask >> l) & 1) && !bases.p[l])
        fail(QVB_ERR_VALIDATION, "location " + std::to_string(l) +
                                     " is read by this store's lookup table but its shard is not "
                                     "attached (qvb_store_attach_peer)");
  }

  int vec() const { return row_bytes % 16 == 0 ? 16 : (row_bytes % 8 == 0 ? 8 : 4); }
  // keep the lookup table in L2 (evict_last) while it is at most a quarter of it
  int lut_keep_flag() const {
    const char* m = std::getenv("QVB_LUT_KEEP");
    if (m) return std::atoi(m);
    return n * 8 <= (32ull << 20) ? 1 : 0;
  }

  void launch_gather(const uint64_t* ids, uint64_t b, char* out, cudaStream_t s, unsigned long long* err) {
    check_attached();
    if (reinterpret_cast<uintptr_t>(out) % vec() != 0)
      fail(QVB_ERR_VALIDATION, "output buffer is not aligned to the row vector width");
    const int V = vec();
    const uint32_t cpr = row_bytes / V;
    static const int kind = [] {  // 0 rows (default), 1 flat, 2 tma
      const char* k = std::getenv("QVB_GATHER_KERNEL");
      if (!k) return 0;
      const std::string v(k);
      return v == "flat" ? 1 : (v == "tma" ? 2 : (v == "cp" ? 3 : 0));
    }();
    const bool host_used = (used_mask >> (nloc - 2)) & 1;
    if (kind == 3 && row_bytes % 16 == 0 && row_bytes <= 512) {
      launch_cp(ids, b, out, s, err);
      return;
    }
    if (kind == 2 && row_bytes % 16 == 0 && !host_used) {
      launch_tma(ids, b, out, s, err);
      return;
    }
    // Small batches: the row-group kernels give each warp 32 requests, so a
    // batch of a few hundred groups leaves most of the GPU idle behind a chain
    // of sequential copy rounds; the flat kernel spreads (request, chunk)
    // pairs over every thread, one id -> entry -> row chain deep
    // (1K ids: 9.9 -> 7.5 us at 400-byte rows, 44.6 -> 7.6 us at 2408-byte
    // rows; ~40K ids: 11.4 -> 9.8 and 62.6 -> 52.0 us; at 64K ids the row-group
    // kernel is ahead again — profiles/r01m_gather_sweep.md). With a host tier
    // the flat kernel also stays ahead of the class split while the batch
    // holds few host rows: the split's fixed cost (lookups, bucket scan,
    // scatter) is not repaid on a short host list. C4: 64K ids 51 / 113 / 296
    // us against 99-111 / 161-173 / 344-354 at h = 0.05 / 0.10 / 0.25; 256K
    // ids at h = 0.05 206 against 216 us, at h = 0.10 445 against 414
    // (profiles/r02/r02w_host_knobs.txt, r02x_host_knobs.txt). So batches up
    // to 256K ids whose expected host rows (uniform ids: B x host share) are
    // at most 16K take the flat kernel. QVB_GATHER_SMALL overrides the
    // request-count threshold.
    const char* sm = std::getenv("QVB_GATHER_SMALL");
    uint64_t small_rows = sm ? std::strtoull(sm, nullptr, 10) : 49152ull;
    if (!sm && host_used && b <= 262144 && b * host_rows <= 16384ull * n) small_rows = b;
    // rows from more than this GPU's shard (peers over NVLink, the host tier
    // over PCIe): bucket by location class first so the links do not share
    // load rounds (QVB_GATHER_SPLIT=0 keeps the mixed row-group kernel)
    const bool mixed = (used_mask & ~(1ull << reader)) != 0;
    const char* split_e = std::getenv("QVB_GATHER_SPLIT");  // per call (tests flip it)
    const int split_env = split_e ? std::atoi(split_e) : 1;
    if (kind != 1 && b > small_rows && mixed && split_env && b < (1ull << 32) && (V == 16 || V == 4 || V == 8)) {
      launch_split(ids, b, cpr, out, s, err);
      return;
    }
    if (kind != 1 && b > small_rows) {
      if (V == 16) launch_rows<16>(ids, b, cpr, out, s, err);
      else if (V == 8 && stride % 16 == 0) launch_rows_wide(ids, b, out, s, err);
      else if (V == 8) launch_rows<8>(ids, b, cpr, out, s, err);
      else launch_rows<4>(ids, b, cpr, out, s, err);
      return;
    }
    const uint64_t max_rows = std::max<uint64_t>(1, (0xFFFFFFFFull / cpr) / 2);
    for (uint64_t r0 = 0; r0 < b; r0 += max_rows) {
      const uint32_t rows = static_cast<uint32_t>(std::min(max_rows, b - r0));
      char* o = out + r0 * row_bytes;
      if (V == 16) launch_direct<16>(ids + r0, rows, cpr, o, r0, s, err);
      else if (V == 8) launch_direct<8>(ids + r0, rows, cpr, o, r0, s, err);
      else launch_direct<4>(ids + r0, rows, cpr, o, r0, s, err);
    }
  }

  void launch_split(const uint64_t* ids, uint64_t b, uint32_t cpr, char* out, cudaStream_t s,
                    unsigned long long* err) {
    const int host_loc = nloc - 2;
    // host requests in offset order once the host tier outgrows the reach of
    // the translation over system memory (random rows: 51 GB/s up to 2 GB,
    // 41 at 8 GB, 38 at 14 GB; in offset order 52-57, profiles/r02/
    // r02op_host_tier_and_lookup.md). C4 h = 0.05 (a 2.8 GB tier), 1M ids:
    // 886 -> 658 us ordered (r02w_host_knobs.txt); C2's 0.3 GB tier: no gain
    // (profiles/r02/r02d_host_order.md), so tiers below 1 GB stay unordered.
    const char* so = std::getenv("QVB_HOST_SORT");  // per call: tests and A/B flip it
    const bool big_tier = host_rows * stride >= (1ull << 30);
    const bool order_host = host_rows > 0 && (used_mask >> host_loc & 1) &&
                            (so ? *so == '1' : big_tier);
    DevBuf<uint32_t> req(b * (kClasses + (order_host ? 1 : 0)), s);
    DevBuf<unsigned long long> srcs(b * (kClasses + (order_host ? 1 : 0)), s);
    const char* bb = std::getenv("QVB_HOST_BUCKET_BITS");  // A/B knob: 10..18
    // buckets: ~64 requests of the batch per bucket, 2^10..2^16 (the bucket
    // scan's cost follows the bucket count; 2^12 vs 2^16 at 64K-256K ids:
    // -5..-12 us, equal at 1M, r02w_host_knobs.txt)
    int lgb = 0;
    while ((2ull << lgb) <= b) ++lgb;  // floor(log2 b)
    const int bbits = bb ? std::max(10, std::min(kHostBucketBits, std::atoi(bb))) : std::max(10, std::min(16, lgb - 6));
    const int nbuckets = 1 << bbits;
    DevBuf<unsigned int> ctr(2 * kClasses + (order_host ? nbuckets : 0), s);
    QVB_CUDA(cudaMemsetAsync(ctr.p, 0, (2 * kClasses + (order_host ? nbuckets : 0)) * sizeof(unsigned int), s));
    ClassLists L;
    for (int c = 0; c < kClasses; ++c) {
      L.req[c] = req.p + c * b;
      L.src[c] = srcs.p + c * b;
    }
    L.count = ctr.p;
    L.cursor = ctr.p + kClasses;
    L.hist = order_host ? ctr.p + 2 * kClasses : nullptr;
    L.cur = nullptr;
    const int hb = bits_for(host_rows > 1 ? host_rows - 1 : 1);
    L.hshift = hb > bbits ? hb - bbits : 0;
    const unsigned sgrid = resident_grid_cached(k_split_classes, kSplitBlock, 0);
    k_split_classes<<<std::min<uint64_t>(sgrid, (b + kSplitBlock - 1) / kSplitBlock), kSplitBlock, 0, s>>>(
        ids, b, lut, bases, stride, n, static_cast<int>(reader), host_loc, L, err);
    QVB_LAUNCH_CHECK();
    if (order_host) {
      DevBuf<unsigned long long> cur(nbuckets, s);  // bucket starts (device scan primitive)
      exclusive_sum_u32_u64(L.hist, reinterpret_cast<uint64_t*>(cur.p), nbuckets, s);
      L.cur = cur.p;
      ClassLists sorted = L;  // the gather reads the bucket-ordered host list
      sorted.req[2] = req.p + kClasses * b;
      sorted.src[2] = srcs.p + kClasses * b;
      const unsigned bgrid = resident_grid_cached(k_bucket_scatter, 256, 0);
      k_bucket_scatter<<<std::min<uint64_t>(bgrid, (b + 255) / 256), 256, 0, s>>>(
          sorted, L.req[2], L.src[2], reinterpret_cast<uint64_t>(bases.p[host_loc]), stride, b);
      QVB_LAUNCH_CHECK();
      L = sorted;
    }
    static const int host_every = [] {
      const char* e = std::getenv("QVB_HOST_EVERY");
      return e ? std::max(1, std::atoi(e)) : 2;  // C4 h = 0.1: 1.198 ms with 8, 1.148 with 2 (r02t)
    }();
    const int V = vec();
    if (V == 16) launch_classes<16>(L, cpr, out, host_every, s);
    else if (V == 8) launch_classes<8>(L, cpr, out, host_every, s);
    else launch_classes<4>(L, cpr, out, host_every, s);
  }

  template <int V>
  void launch_classes(const ClassLists& L, uint32_t cpr, char* out, int host_every, cudaStream_t s) {
    // host rows per group: 1 when the host list is offset-ordered (C4 uniform
    // ids at h = 0.25: 3.73 ms with 32-row groups, 3.15 with 4, 2.80 with 2,
    // 2.81 with 1 — profiles/r02/r02op_*; P-weighted ids, whose host rows are
    // sparser, at h = 0.05 / 0.10: 497 -> 443 us and 861 -> 831 us from 2 to 1,
    // r02ag_host_knobs_pw.txt), 32 for an unordered list (no locality to keep,
    // fewer cursor atomics); QVB_HOST_GROUP (1..32) overrides
    const char* hg = std::getenv("QVB_HOST_GROUP");
    const uint32_t host_group =
        hg ? static_cast<uint32_t>(std::max(1, std::min(32, std::atoi(hg)))) : (L.hist ? 1u : 32u);
    const char* r5 = std::getenv("QVB_CLASS_R512");  // A/B knob (default on)
    if (V == 16 && row_bytes % 512 == 0 && !(r5 && *r5 == '0')) {
      const unsigned grid = resident_grid_cached(k_gather_classes<16, 4, true>, kGatherBlock, 0);
      k_gather_classes<16, 4, true><<<grid, kGatherBlock, 0, s>>>(L, cpr, row_bytes, out, host_every, host_group);
    } else {
      const unsigned grid = resident_grid_cached(k_gather_classes<V, 4, false>, kGatherBlock, 0);
      k_gather_classes<V, 4, false><<<grid, kGatherBlock, 0, s>>>(L, cpr, row_bytes, out, host_every, host_group);
    }
    QVB_LAUNCH_CHECK();
  }

  static uint64_t work_blocks(uint64_t chunks) {
    const uint64_t per_block = (uint64_t)kGatherBlock * kUnroll;
    return (chunks + per_block - 1) / per_block;
  }

  template <int V>
  void launch_direct(const uint64_t* ids, uint32_t rows, uint32_t cpr, char* o, uint64_t r0,
                     cudaStream_t s, unsigned long long* err) {
    const unsigned full = resident_grid_cached(k_gather<V>, kGatherBlock, 0);  // one resident wave
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(full, work_blocks((uint64_t)rows * cpr)));
    k_gather<V><<<grid, kGatherBlock, 0, s>>>(ids, rows, lut, bases, stride, cpr, row_bytes, n, o,
                                              r0, err);
    QVB_LAUNCH_CHECK();
  }

  template <int V>
  void launch_rows(const uint64_t* ids, uint64_t rows, uint32_t cpr, char* o, cudaStream_t s, unsigned long long* err) {
    static const int variant = [] {
      const char* u = std::getenv("QVB_GATHER_U");
      return u ? std::atoi(u) : 0;
    }();
    // the lean 512-byte-row kernel measured level with this one (r02g/r02h:
    // 0.205-0.240 ms vs 0.207 per 1M C4 ids): opt-in, QVB_GATHER_U=5/6/7/9
    if (V == 16 && row_bytes == 512 && (variant == 5 || variant == 6 || variant == 7 || variant == 9)) {
      launch_rows512(ids, rows, o, s, err, variant);
      return;
    }
    if (variant == 84) launch_rows_u<V, 8, 4>(ids, rows, cpr, o, s, err);
    else if (variant == 46) launch_rows_u<V, 4, 6>(ids, rows, cpr, o, s, err);
    else if (variant == 85) launch_rows_u<V, 8, 3>(ids, rows, cpr, o, s, err);
    else if (variant == 8) launch_rows_u<V, 8, 1>(ids, rows, cpr, o, s, err);
    else if (variant == 4) launch_rows_u<V, 4, 4>(ids, rows, cpr, o, s, err);
    else if (variant == 2) launch_rows_u<V, 2, 6>(ids, rows, cpr, o, s, err);
    else launch_rows_u<V, 4, 4>(ids, rows, cpr, o, s, err);
  }

  void launch_rows512(const uint64_t* ids, uint64_t rows, char* o, cudaStream_t s,
                      unsigned long long* err, int variant) {
    const int lut_keep = lut_keep_flag();
    const uint64_t warps_needed = (rows + 31) / 32;
    const uint64_t blocks = (warps_needed + kGatherBlock / 32 - 1) / (kGatherBlock / 32);
#define QVB_R512(U, MB)                                                                          \
    do {                                                                                         \
      const unsigned full = resident_grid_cached(k_gather_rows512<U, MB>, kGatherBlock, 0);      \
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(full, blocks));             \
      k_gather_rows512<U, MB><<<grid, kGatherBlock, 0, s>>>(ids, rows, lut, bases, stride, n, o, \
                                                            err, lut_keep);                      \
    } while (0)
    if (variant == 5) QVB_R512(2, 6);
    else if (variant == 6) QVB_R512(8, 4);
    else if (variant == 7) QVB_R512(16, 2);
    else QVB_R512(4, 4);  // 9
#undef QVB_R512
    QVB_LAUNCH_CHECK();
  }

  void launch_cp(const uint64_t* ids, uint64_t rows, char* o, cudaStream_t s, unsigned long long* err) {
    const uint32_t cpr = row_bytes / 16;
    const uint64_t per_warp = 2ull * cpr * 32 * 16;
    const uint32_t warps = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>(8, (200u << 10) / per_warp)));
    const size_t smem = warps * per_warp;
    // per call: the attribute is per device, and stores may live on several
    QVB_CUDA(cudaFuncSetAttribute(k_gather_cp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    int per_sm = 0, dev = 0, sms = 0;
    QVB_CUDA(cudaGetDevice(&dev));
    QVB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    QVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_cp, warps * 32, smem));
    const uint64_t groups = (rows + 31) / 32;
    const uint64_t blocks = std::min<uint64_t>((uint64_t)std::max(per_sm, 1) * sms,
                                               (groups + warps - 1) / warps);
    k_gather_cp<<<static_cast<unsigned>(blocks), warps * 32, smem, s>>>(ids, rows, lut, bases, stride,
                                                                       cpr, row_bytes, n, o, err);
    QVB_LAUNCH_CHECK();
  }

  void launch_tma(const uint64_t* ids, uint64_t rows, char* o, cudaStream_t s, unsigned long long* err) {
    const uint64_t per_warp = (uint64_t)kTmaBuffers * 32 * row_bytes;
    const uint32_t warps = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>(8, (200u << 10) / per_warp)));
    const size_t smem = 8 * kTmaBuffers * warps + 128 + (size_t)warps * per_warp;
    if (smem > (227u << 10)) fail(QVB_ERR_UNSUPPORTED, "row too large for the TMA gather");
    QVB_CUDA(cudaFuncSetAttribute(k_gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    int per_sm = 0, dev = 0, sms = 0;
    QVB_CUDA(cudaGetDevice(&dev));
    QVB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    QVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_tma, warps * 32, smem));
    const uint64_t groups = (rows + 31) / 32;
    const uint64_t blocks = std::min<uint64_t>((uint64_t)std::max(per_sm, 1) * sms,
                                               (groups + warps - 1) / warps);
    k_gather_tma<<<static_cast<unsigned>(blocks), warps * 32, smem, s>>>(ids, rows, lut, bases,
                                                                        stride, row_bytes, n, o, err);
    QVB_LAUNCH_CHECK();
  }

  void launch_rows_wide(const uint64_t* ids, uint64_t rows, char* o, cudaStream_t s, unsigned long long* err) {
    const unsigned full = resident_grid_cached(k_gather_rows_w<4, 4>, kGatherBlock, 0);  // one resident wave
    const uint32_t cpr16 = (row_bytes + 15) / 16;
    const uint64_t warps_needed = (rows + 31) / 32;
    const uint64_t blocks = (warps_needed + kGatherBlock / 32 - 1) / (kGatherBlock / 32);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(full, blocks));
    k_gather_rows_w<4, 4><<<grid, kGatherBlock, 0, s>>>(ids, rows, lut, bases, stride, cpr16,
                                                         row_bytes, n, o, err);
    QVB_LAUNCH_CHECK();
  }

  template <int V, int U, int MB>
  void launch_rows_u(const uint64_t* ids, uint64_t rows, uint32_t cpr, char* o, cudaStream_t s, unsigned long long* err) {
    const int lut_keep = lut_keep_flag();
    const unsigned full = resident_grid_cached(k_gather_rows<V, U, MB>, kGatherBlock, 0);  // one resident wave
    const uint64_t warps_needed = (rows + 31) / 32;
    const uint64_t blocks = (warps_needed + kGatherBlock / 32 - 1) / (kGatherBlock / 32);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(full, blocks));
    k_gather_rows<V, U, MB><<<grid, kGatherBlock, 0, s>>>(ids, rows, lut, bases, stride, cpr,
                                                          row_bytes, n, o, err, lut_keep);
    QVB_LAUNCH_CHECK();
  }

  template <int V, typename K>
  void launch_sorted(const K* keys, const uint32_t* order, uint32_t rows, uint32_t cpr, char* o,
                     int ob, cudaStream_t s, unsigned long long* err) {
    const unsigned full = resident_grid_cached(k_gather_sorted<V, K>, kGatherBlock, 0);  // one resident wave
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(full, work_blocks((uint64_t)rows * cpr)));
    k_gather_sorted<V, K><<<grid, kGatherBlock, 0, s>>>(keys, order, rows, bases, stride, cpr,
                                                        row_bytes, o, ob);
    QVB_LAUNCH_CHECK();
  }

  void launch_planned(const uint64_t* ids, uint64_t b, char* out, cudaStream_t s, unsigned long long* err) {
    check_attached();
    if (b >= (1ull << 32)) fail(QVB_ERR_UNSUPPORTED, "batch exceeds 2^32 ids");
    const int V = vec();
    const uint32_t cpr = row_bytes / V;
    if ((uint64_t)b * cpr >= 0xFFFFFFFFull) fail(QVB_ERR_UNSUPPORTED, "planned batch too large");
    DevBuf<uint32_t> idx(b, s), order(b, s);
    const int loc_bits = bits_for(static_cast<uint64_t>(nloc - 1));
    const int ob = bits_for(n);  // every shard offset is below n
    const uint32_t rows = static_cast<uint32_t>(b);
    if (ob + loc_bits <= 32) {  // 32-bit keys: ob + loc_bits radix bits, half the key bytes
      DevBuf<uint32_t> keys(b, s), skeys(b, s);
      k_plan_keys32<<<grid_for(b, 256), 256, 0, s>>>(ids, b, lut, n, ob, keys.p, idx.p, err);
      QVB_LAUNCH_CHECK();
      sort_pairs_u32_u32(keys.p, skeys.p, idx.p, order.p, b, 0, ob + loc_bits, s);
      if (V == 16) launch_sorted<16>(skeys.p, order.p, rows, cpr, out, ob, s, err);
      else if (V == 8) launch_sorted<8>(skeys.p, order.p, rows, cpr, out, ob, s, err);
      else launch_sorted<4>(skeys.p, order.p, rows, cpr, out, ob, s, err);
      return;
    }
    DevBuf<uint64_t> keys(b, s), skeys(b, s);
    k_plan_keys_packed<<<grid_for(b, 256), 256, 0, s>>>(ids, b, lut, n, keys.p, idx.p, err);
    QVB_LAUNCH_CHECK();
    sort_pairs_u64_u32(keys.p, skeys.p, idx.p, order.p, b, 0, kOffsetBits + loc_bits, s);
    if (V == 16) launch_sorted<16>(skeys.p, order.p, rows, cpr, out, kOffsetBits, s, err);
    else if (V == 8) launch_sorted<8>(skeys.p, order.p, rows, cpr, out, kOffsetBits, s, err);
    else launch_sorted<4>(skeys.p, order.p, rows, cpr, out, kOffsetBits, s, err);
  }

  ~qvb_store() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (auto& p : peer)
      if (p) cudaIpcCloseMemHandle(p);
    cudaFree(lut);
    cudaFree(local);
    if (host) cudaFreeHost(host);
    cudaFree(err);
    cudaFree(err_host);
    cudaFree(d_ids);
    cudaFree(d_out);
    for (auto q : hs)
      if (q) cudaStreamDestroy(q);
    for (auto e : hev)
      if (e) cudaEventDestroy(e);
    if (prev >= 0) cudaSetDevice(prev);
  }
};

namespace {

void fill_rows(qvb_store& st, int loc, const DeviceLut& L, const float* features, char* dst_dev,
               char* dst_host, uint64_t rows, cudaStream_t s) {
  if (rows == 0) return;
  DevBuf<uint64_t> fr(rows, s);
  lut_rows_of_location(L, loc, fr.p, s);
  if (!features) {
    k_fill_synthetic<<<grid_for(rows * st.dim, 256), 256, 0, s>>>(fr.p, rows, st.dim, st.stride,
                                                                  dst_dev);
    QVB_LAUNCH_CHECK();
    return;
  }
  std::vector<uint64_t> feat(rows);
  QVB_CUDA(cudaMemcpyAsync(feat.data(), fr.p, rows * 8, cudaMemcpyDeviceToHost, s));
  QVB_CUDA(cudaStreamSynchronize(s));
  if (dst_host) {  // host tier: plain CPU copy into the pinned shard
    for (uint64_t r = 0; r < rows; ++r)
      std::memcpy(dst_host + r * st.stride, features + feat[r] * st.dim, st.row_bytes);
    return;
  }
  const uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / st.row_bytes);
  char* pin = nullptr;
  QVB_CUDA(cudaMallocHost(&pin, std::min(chunk, rows) * st.row_bytes));
  DevBuf<char> stage(std::min(chunk, rows) * st.row_bytes, s);
  for (uint64_t r0 = 0; r0 < rows; r0 += chunk) {
    const uint64_t c = std::min(chunk, rows - r0);
    QVB_CUDA(cudaStreamSynchronize(s));
    for (uint64_t r = 0; r < c; ++r)
      std::memcpy(pin + r * st.row_bytes, features + feat[r0 + r] * st.dim, st.row_bytes);
    QVB_CUDA(cudaMemcpyAsync(stage.p, pin, c * st.row_bytes, cudaMemcpyHostToDevice, s));
    k_restride<<<grid_for(c * st.row_bytes / 4, 256), 256, 0, s>>>(stage.p, c, st.row_bytes,
                                                                   st.stride, dst_dev + r0 * st.stride);
    QVB_LAUNCH_CHECK();
  }
  QVB_CUDA(cudaStreamSynchronize(s));
  cudaFreeHost(pin);
}

}  // namespace

extern "C" int qvb_store_create(int device, const uint64_t* loc_offsets, const int64_t* loc_ids,
                                uint64_t n, uint32_t dim, const qvb_topology* topo,
                                uint32_t reader_device, const float* features, qvb_store** out) {
  return guarded([&] {
    if (!out) fail(QVB_ERR_VALIDATION, "out is null");
    *out = nullptr;
    if (!topo || !loc_offsets || (loc_offsets[n] && !loc_ids)) fail(QVB_ERR_VALIDATION, "null argument");
    if (n == 0 || dim == 0) fail(QVB_ERR_VALIDATION, "store needs features and dim > 0");
    topology_validate(*topo);
    if (topo->servers != 1)
      fail(QVB_ERR_UNSUPPORTED, "the device store serves one server (cross-server reads are out of scope)");
    if (reader_device >= topo->gpus_per_server) fail(QVB_ERR_VALIDATION, "reader_device out of range");
    if (n > kOffsetMask) fail(QVB_ERR_UNSUPPORTED, "too many features");
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    auto st = std::make_unique<qvb_store>();
    st->device = device;
    st->n = n;
    st->dim = dim;
    st->reader = reader_device;
    st->nloc = static_cast<int>(topo->gpus_per_server + 2);
    st->row_bytes = dim * 4u;
    // HBM is read in 64-byte bursts: rows of >= 64 B start on a 64-B boundary
    // so a row costs ceil(row/64) bursts instead of one more on average.
    const uint64_t align = st->row_bytes >= 64 ? 64 : 16;
    st->stride = (st->row_bytes + align - 1) / align * align;
    QVB_CUDA(cudaMalloc(&st->err, sizeof(unsigned long long)));
    QVB_CUDA(cudaMemset(st->err, 0xFF, sizeof(unsigned long long)));
    QVB_CUDA(cudaMalloc(&st->err_host, sizeof(unsigned long long)));
    QVB_CUDA(cudaMemset(st->err_host, 0xFF, sizeof(unsigned long long)));

    const uint64_t copies = loc_offsets[n];
    DevBuf<uint64_t> dlo(n + 1, s);
    DevBuf<int64_t> dids(copies ? copies : 1, s);
    QVB_CUDA(cudaMemcpyAsync(dlo.p, loc_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
    if (copies) QVB_CUDA(cudaMemcpyAsync(dids.p, loc_ids, copies * 8, cudaMemcpyHostToDevice, s));
    DeviceLut L;
    lut_prepare(L, dlo.p, dids.p, n, st->nloc, s);
    QVB_CUDA(cudaMalloc(&st->lut, n * 8));
    uint64_t missing = ~0ull;
    st->used_mask = lut_choose(L, replica_order(*topo, 0, reader_device), nullptr, nullptr,
                               st->lut, s, &missing);
    if (missing != ~0ull)
      fail(QVB_ERR_VALIDATION, "feature " + std::to_string(missing) + " has no location");
    const int host_loc = static_cast<int>(topo->gpus_per_server);
    if ((st->used_mask >> (host_loc + 1)) & 1)
      fail(QVB_ERR_UNSUPPORTED, "the lookup table reads the disk tier, which the device store does not serve");

    st->local_rows = L.location_rows[reader_device];
    QVB_CUDA(cudaMalloc(&st->local, std::max<uint64_t>(1, st->local_rows) * st->stride));
    fill_rows(*st, static_cast<int>(reader_device), L, features, st->local, nullptr, st->local_rows, s);
    st->bases.p[reader_device] = st->local;
    if ((st->used_mask >> host_loc) & 1) {
      st->host_rows = L.location_rows[host_loc];
      QVB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&st->host),
                             std::max<uint64_t>(1, st->host_rows) * st->stride,
                             cudaHostAllocMapped | cudaHostAllocPortable));
      QVB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&st->host_dev), st->host, 0));
      fill_rows(*st, host_loc, L, features, st->host_dev, features ? st->host : nullptr,
                st->host_rows, s);
      st->bases.p[host_loc] = st->host_dev;
    }
    QVB_CUDA(cudaStreamSynchronize(s));
    *out = st.release();
  });
}

extern "C" int qvb_store_info_get(const qvb_store* s, qvb_store_info* info) {
  return guarded([&] {
    if (!s || !info) fail(QVB_ERR_VALIDATION, "null argument");
    std::memset(info, 0, sizeof *info);
    info->feature_count = s->n;
    info->dim = s->dim;
    info->reader_device = s->reader;
    info->row_stride_bytes = s->stride;
    info->local_rows = s->local_rows;
    info->host_rows = s->host_rows;
    info->lut_bytes = s->n * 8;
    info->location_count = static_cast<uint32_t>(s->nloc);
  });
}

extern "C" int qvb_store_export_handle(const qvb_store* s, uint8_t handle[64]) {
  return guarded([&] {
    if (!s || !handle) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(s->device);
    cudaIpcMemHandle_t h;
    QVB_CUDA(cudaIpcGetMemHandle(&h, s->local));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
  });
}

extern "C" int qvb_store_attach_peer(qvb_store* s, uint32_t peer_device, const uint8_t handle[64]) {
  return guarded([&] {
    if (!s || !handle) fail(QVB_ERR_VALIDATION, "null argument");
    if (peer_device == s->reader || (int)peer_device >= s->nloc - 2)
      fail(QVB_ERR_VALIDATION, "peer_device must be another GPU of the server");
    DeviceGuard dg(s->device);
    if (s->peer[peer_device]) {
      cudaIpcCloseMemHandle(s->peer[peer_device]);
      s->peer[peer_device] = nullptr;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* p = nullptr;
    QVB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    s->peer[peer_device] = p;
    s->bases.p[peer_device] = static_cast<const char*>(p);
  });
}

extern "C" int qvb_store_attach_local_peer(qvb_store* s, uint32_t peer_device,
                                           const qvb_store* peer) {
  return guarded([&] {
    if (!s || !peer) fail(QVB_ERR_VALIDATION, "null argument");
    if (peer_device == s->reader || (int)peer_device >= s->nloc - 2)
      fail(QVB_ERR_VALIDATION, "peer_device must be another GPU of the server");
    if (peer->reader != peer_device || peer->n != s->n || peer->dim != s->dim)
      fail(QVB_ERR_VALIDATION, "peer store does not hold that device's shard of this table");
    DeviceGuard dg(s->device);
    if (peer->device != s->device) {
      int can = 0;
      QVB_CUDA(cudaDeviceCanAccessPeer(&can, s->device, peer->device));
      if (!can) fail(QVB_ERR_CUDA, "no P2P access between the two devices");
      cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else QVB_CUDA(e);
    }
    s->bases.p[peer_device] = peer->local;
  });
}

extern "C" int qvb_store_destroy(qvb_store* s) {
  return guarded([&] { delete s; });
}

extern "C" int qvb_gather(qvb_store* s, const uint64_t* ids, uint64_t b, float* out, void* stream) {
  return guarded([&] {
    if (!s) fail(QVB_ERR_VALIDATION, "null store");
    if (b == 0) return;
    if (!ids || !out) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(s->device);
    s->launch_gather(ids, b, reinterpret_cast<char*>(out), static_cast<cudaStream_t>(stream), s->err);
  });
}

extern "C" int qvb_gather_planned(qvb_store* s, const uint64_t* ids, uint64_t b, float* out,
                                  void* stream) {
  return guarded([&] {
    if (!s) fail(QVB_ERR_VALIDATION, "null store");
    if (b == 0) return;
    if (!ids || !out) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(s->device);
    s->launch_planned(ids, b, reinterpret_cast<char*>(out), static_cast<cudaStream_t>(stream), s->err);
  });
}

extern "C" int qvb_store_check_error(qvb_store* s) {
  return guarded([&] {
    if (!s) fail(QVB_ERR_VALIDATION, "null store");
    DeviceGuard dg(s->device);
    unsigned long long e = 0;
    QVB_CUDA(cudaMemcpy(&e, s->err, sizeof e, cudaMemcpyDeviceToHost));
    if (e != ~0ull) {
      QVB_CUDA(cudaMemset(s->err, 0xFF, sizeof(unsigned long long)));
      fail(QVB_ERR_VALIDATION, "request " + std::to_string(e) + ": feature id outside lookup table");
    }
  });
}

extern "C" int qvb_gather_host(qvb_store* s, const uint64_t* ids, uint64_t b, float* out,
                               void* stream) {
  return guarded([&] {
    if (!s) fail(QVB_ERR_VALIDATION, "null store");
    if (b == 0) return;
    if (!ids || !out) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(s->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(s->host_mu);
    s->ensure_scratch(b);
    const uint64_t rb = s->row_bytes;
    // Large batches go in chunks alternating over two internal streams, so
    // one chunk's rows travel device->host while the next chunk is gathered
    // (the copy engines and the SMs overlap; the D2H of the rows bounds it).
    const char* ce = std::getenv("QVB_HOST_CHUNKS");
    const uint64_t want = ce ? std::max<uint64_t>(1, std::strtoull(ce, nullptr, 10)) : 8;
    const uint64_t chunks = b >= want * 16384 ? want : 1;
    if (chunks == 1) {
      QVB_CUDA(cudaMemcpyAsync(s->d_ids, ids, b * 8, cudaMemcpyHostToDevice, st));
      s->launch_gather(s->d_ids, b, s->d_out, st, s->err_host);
      QVB_CUDA(cudaMemcpyAsync(out, s->d_out, b * rb, cudaMemcpyDeviceToHost, st));
    } else {
      s->ensure_host_streams();
      QVB_CUDA(cudaEventRecord(s->hev[2], st));
      for (int q = 0; q < 2; ++q) QVB_CUDA(cudaStreamWaitEvent(s->hs[q], s->hev[2], 0));
      const uint64_t per = (b + chunks - 1) / chunks;
      for (uint64_t c = 0; c < chunks; ++c) {
        const uint64_t a = c * per, len = std::min(per, b - a);
        if (a >= b) break;
        cudaStream_t q = s->hs[c & 1];
        QVB_CUDA(cudaMemcpyAsync(s->d_ids + a, ids + a, len * 8, cudaMemcpyHostToDevice, q));
        s->launch_gather(s->d_ids + a, len, s->d_out + a * rb, q, s->err_host);
        QVB_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(out) + a * rb, s->d_out + a * rb, len * rb,
                                 cudaMemcpyDeviceToHost, q));
      }
      for (int q = 0; q < 2; ++q) {
        QVB_CUDA(cudaEventRecord(s->hev[q], s->hs[q]));
        QVB_CUDA(cudaStreamWaitEvent(st, s->hev[q], 0));
      }
    }
    QVB_CUDA(cudaStreamSynchronize(st));
    unsigned long long e = 0;
    QVB_CUDA(cudaMemcpy(&e, s->err_host, sizeof e, cudaMemcpyDeviceToHost));
    if (e != ~0ull) {
      QVB_CUDA(cudaMemset(s->err_host, 0xFF, sizeof(unsigned long long)));
      // chunked launches report chunk-relative indices: name the first bad id
      uint64_t i = 0;
      while (i < b && ids[i] < s->n) ++i;
      if (i < b) fail(QVB_ERR_VALIDATION, "feature id " + std::to_string(ids[i]) + " outside lookup table");
      fail(QVB_ERR_VALIDATION, "feature id outside lookup table");
    }
  });
}

extern "C" int qvb_store_plan_reads(qvb_store* s, const uint64_t* ids, uint64_t b, int ids_on_device,
                                    uint64_t page_size, int64_t* group_loc, uint64_t* group_count,
                                    uint64_t* group_transitions, uint64_t* n_groups,
                                    uint64_t* offsets_out, void* stream) {
  return guarded([&] {
    if (!s) fail(QVB_ERR_VALIDATION, "null store");
    if (page_size == 0) fail(QVB_ERR_VALIDATION, "page size must be > 0");
    if (!n_groups) fail(QVB_ERR_VALIDATION, "null argument");
    *n_groups = 0;
    if (b == 0) return;
    if (!ids || !group_loc || !group_count || !group_transitions || !offsets_out)
      fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(s->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t* d_ids = ids;
    DevBuf<uint64_t> staged;
    if (!ids_on_device) {  // only the batch travels; the table is resident
      staged.alloc(b, st);
      QVB_CUDA(cudaMemcpyAsync(staged.p, ids, b * 8, cudaMemcpyHostToDevice, st));
      d_ids = staged.p;
    }
    DeviceReadPlan rp;
    plan_reads_device(nullptr, nullptr, s->lut, s->n, d_ids, b, page_size, rp, st);
    copy_read_plan(rp, group_loc, group_count, group_transitions, n_groups, offsets_out, st);
  });
}

extern "C" int qvb_request_ids_synthetic(int device, uint64_t seed, uint64_t batch, uint64_t n,
                                         uint64_t* ids, uint64_t b, void* stream) {
  return guarded([&] {
    if (b == 0) return;
    if (!ids || n == 0) fail(QVB_ERR_VALIDATION, "null ids or n == 0");
    DeviceGuard dg(device);
    const uint64_t state = derive_state(seed, 0x5EEDULL, batch);
    k_request_ids<<<grid_for(b, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(state, n, ids, b);
    QVB_LAUNCH_CHECK();
  });
}
