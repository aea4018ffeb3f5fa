// primitives.cu — hand-written sort / scan / reduce for sm_100a, used by the
// one-time in-CSR build, the ranking (K2) and the read planner (K4).
//
// Scan: reduce-then-scan. Tiles of 4096 items (256 threads x 16); pass 1
// writes per-tile sums, the tile sums are scanned recursively, pass 2 scans
// each tile (warp shuffles + one smem step) and adds the tile offset.
//
// Radix sort: stable LSD, 8-bit digits, three kernels per digit:
//   upsweep   per-tile digit histogram (smem atomics) -> counts[digit][tile]
//   scan      exclusive scan of the digit-major counts (the scan above) gives
//             every (digit, tile) its global output base
//   scatter   each warp walks its 256 items round by round in input order;
//             __match_any_sync groups lanes with equal digits, so an item's
//             rank = items of its digit in earlier rounds of the warp +
//             lower lanes of this round; warp totals are then prefixed in
//             warp order. base + warp prefix + rank is the stable position.
// Keys/values ping-pong between the caller's output buffers and one scratch
// pair; only the digits covering [begin_bit, end_bit) are processed.
#include <cstring>
#include <vector>

#include "common.cuh"

namespace qvb {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanIpt = 16;
constexpr uint64_t kScanTile = kScanThreads * kScanIpt;

template <typename T>
__device__ __forceinline__ T warp_inclusive(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the prefix and
// writes the block total.
template <typename T>
__device__ __forceinline__ T block_exclusive(T v, T* total) {
  __shared__ T warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_inclusive(v);
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kScanThreads / 32 ? warp_sums[lane] : T(0);
    w = warp_inclusive(w);
    if (lane < kScanThreads / 32) warp_sums[lane] = w;
  }
  __syncthreads();
  const T before = warp == 0 ? T(0) : warp_sums[warp - 1];
  *total = warp_sums[kScanThreads / 32 - 1];
  __syncthreads();
  return before + inc - v;
}

template <typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_reduce(const In* __restrict__ in, uint64_t n, Out* __restrict__ tile_sums) {
  const uint64_t base = blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanIpt;
  Out s = 0;
#pragma unroll
  for (int i = 0; i < kScanIpt; ++i)
    if (base + i < n) s += static_cast<Out>(in[base + i]);
  Out total;
  block_exclusive<Out>(s, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

template <typename In, typename Out, bool kInclusive>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_down(const In* __restrict__ in, uint64_t n, const Out* __restrict__ tile_off,
                Out* __restrict__ out) {
  const uint64_t base = blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanIpt;
  Out v[kScanIpt];
  Out s = 0;
#pragma unroll
  for (int i = 0; i < kScanIpt; ++i) {
    v[i] = base + i < n ? static_cast<Out>(in[base + i]) : Out(0);
    s += v[i];
  }
  Out total;
  Out run = block_exclusive<Out>(s, &total) + (tile_off ? tile_off[blockIdx.x] : Out(0));
#pragma unroll
  for (int i = 0; i < kScanIpt; ++i) {
    if (kInclusive) run += v[i];
    if (base + i < n) out[base + i] = run;
    if (!kInclusive) run += v[i];
  }
}

template <typename In, typename Out, bool kInclusive>
void scan(const In* in, Out* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    k_scan_down<In, Out, kInclusive><<<1, kScanThreads, 0, s>>>(in, n, nullptr, out);
    QVB_LAUNCH_CHECK();
    return;
  }
  DevBuf<Out> sums(tiles, s), offs(tiles, s);
  k_scan_reduce<In, Out><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, sums.p);
  QVB_LAUNCH_CHECK();
  scan<Out, Out, false>(sums.p, offs.p, tiles, s);
  k_scan_down<In, Out, kInclusive><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, offs.p, out);
  QVB_LAUNCH_CHECK();
}

// ---- radix sort ---------------------------------------------------------------
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortRounds = 8;  // items per thread
constexpr uint64_t kSortTile = kSortThreads * kSortRounds;
constexpr int kRadix = 256;

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
    k_radix_upsweep(const K* __restrict__ keys, uint64_t n, int shift, uint64_t tiles,
                    uint32_t* __restrict__ counts) {
  __shared__ uint32_t hist[kRadix];
  hist[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = blockIdx.x * kSortTile;
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&hist[(keys[i] >> shift) & 0xFF], 1u);
  }
  __syncthreads();
  counts[(uint64_t)threadIdx.x * tiles + blockIdx.x] = hist[threadIdx.x];
}

template <typename K, typename V>
__global__ void __launch_bounds__(kSortThreads)
    k_radix_scatter(const K* __restrict__ kin, const V* __restrict__ vin, uint64_t n, int shift,
                    uint64_t tiles, const uint64_t* __restrict__ digit_base, K* __restrict__ kout,
                    V* __restrict__ vout) {
  __shared__ uint32_t whist[kSortWarps][kRadix];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < kRadix; d += 32) whist[warp][d] = 0;
  __syncwarp();
  // warp w owns items [tile + w*256, tile + (w+1)*256), round r = 32 of them
  const uint64_t wbase = blockIdx.x * kSortTile + (uint64_t)warp * 32 * kSortRounds;
  K k[kSortRounds];
  V v[kSortRounds];
  uint32_t rank[kSortRounds];
  uint32_t dig[kSortRounds];
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t i = wbase + r * 32 + lane;
    const bool in = i < n;
    if (in) {
      k[r] = kin[i];
      v[r] = vin[i];
    }
    const uint32_t d = in ? static_cast<uint32_t>((k[r] >> shift) & 0xFF) : 0x100u;  // 256: none
    dig[r] = d;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = __popc(peers & lt);
    const int leader = __ffs(peers) - 1;
    uint32_t run = 0;
    if (in) run = whist[warp][d];
    rank[r] = run + before;
    __syncwarp();
    if (in && lane == leader) whist[warp][d] = run + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // prefix of the warp counts over warps (warp order == input order), and
  // the digit's start inside the tile (exclusive over digits)
  __shared__ uint32_t dstart[kRadix];
  __shared__ uint64_t gbase[kRadix];
  uint32_t total = 0;
  {
    const int d = threadIdx.x;  // kSortThreads == kRadix
    uint32_t acc = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = whist[w][d];
      whist[w][d] = acc;
      acc += c;
    }
    total = acc;
    gbase[d] = digit_base[(uint64_t)d * tiles + blockIdx.x];
  }
  // exclusive scan of the digit totals across the block
  {
    __shared__ uint32_t wsum[kSortWarps];
    uint32_t inc = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    dstart[threadIdx.x] = before + inc - total;
  }
  __syncthreads();
  // stage the tile in digit order, then write each digit's run contiguously
  __shared__ K sk[kSortTile];
  __shared__ V sv[kSortTile];
  __shared__ uint8_t sd[kSortTile];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint32_t d = dig[r];
    if (d < kRadix) {
      const uint32_t at = dstart[d] + whist[warp][d] + rank[r];
      sk[at] = k[r];
      sv[at] = v[r];
      sd[at] = static_cast<uint8_t>(d);
    }
  }
  __syncthreads();
  const uint64_t tile_n = n - blockIdx.x * kSortTile < kSortTile ? n - blockIdx.x * kSortTile : kSortTile;
  for (uint32_t i = threadIdx.x; i < tile_n; i += kSortThreads) {
    const uint32_t d = sd[i];
    const uint64_t pos = gbase[d] + (i - dstart[d]);
    kout[pos] = sk[i];
    vout[pos] = sv[i];
  }
}

template <typename K, typename V>
void radix_sort(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int begin_bit,
                int end_bit, cudaStream_t s) {
  if (n == 0) return;
  if (end_bit <= begin_bit) {
    QVB_CUDA(cudaMemcpyAsync(kout, kin, n * sizeof(K), cudaMemcpyDeviceToDevice, s));
    QVB_CUDA(cudaMemcpyAsync(vout, vin, n * sizeof(V), cudaMemcpyDeviceToDevice, s));
    return;
  }
  const int passes = (end_bit - begin_bit + 7) / 8;
  const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
  DevBuf<uint32_t> counts(tiles * kRadix, s);
  DevBuf<uint64_t> base(tiles * kRadix, s);
  DevBuf<K> ktmp(n, s);
  DevBuf<V> vtmp(n, s);
  // ping-pong so that the last pass lands in (kout, vout)
  const K* ksrc = kin;
  const V* vsrc = vin;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    K* kdst = to_out ? kout : ktmp.p;
    V* vdst = to_out ? vout : vtmp.p;
    const int shift = begin_bit + 8 * p;
    k_radix_upsweep<K><<<static_cast<unsigned>(tiles), kSortThreads, 0, s>>>(ksrc, n, shift, tiles,
                                                                             counts.p);
    QVB_LAUNCH_CHECK();
    scan<uint32_t, uint64_t, false>(counts.p, base.p, tiles * kRadix, s);
    k_radix_scatter<K, V><<<static_cast<unsigned>(tiles), kSortThreads, 0, s>>>(
        ksrc, vsrc, n, shift, tiles, base.p, kdst, vdst);
    QVB_LAUNCH_CHECK();
    ksrc = kdst;
    vsrc = vdst;
  }
}

__global__ void k_reduce_u8(const uint8_t* __restrict__ in, uint64_t n,
                            unsigned long long* __restrict__ out) {
  uint64_t s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    s += in[i];
  s = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(s));
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, (unsigned long long)s);
}

}  // namespace

void sort_pairs_u32_u32(const uint32_t* kin, uint32_t* kout, const uint32_t* vin, uint32_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s) {
  radix_sort(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void sort_pairs_u64_u64(const uint64_t* kin, uint64_t* kout, const uint64_t* vin, uint64_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s) {
  radix_sort(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void sort_pairs_u64_u32(const uint64_t* kin, uint64_t* kout, const uint32_t* vin, uint32_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s) {
  radix_sort(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void exclusive_sum_u32_u64(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  scan<uint32_t, uint64_t, false>(in, out, n, s);
}
void exclusive_sum_u8_u32(const uint8_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  scan<uint8_t, uint32_t, false>(in, out, n, s);
}
void inclusive_sum_u32_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  scan<uint32_t, uint32_t, true>(in, out, n, s);
}
void sum_u8_u64(const uint8_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  QVB_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), s));
  if (n == 0) return;
  k_reduce_u8<<<grid_for(n, 256, 148u * 8u), 256, 0, s>>>(in, n,
                                                          reinterpret_cast<unsigned long long*>(out));
  QVB_LAUNCH_CHECK();
}

}  // namespace qvb

// ---- test entry points (include/qvb_test.h) ------------------------------------
using namespace qvb;

extern "C" int qvb_test_sort_pairs_u64(int device, const uint64_t* keys, const uint64_t* vals,
                                       uint64_t n, int begin_bit, int end_bit, uint64_t* keys_out,
                                       uint64_t* vals_out) {
  return guarded([&] {
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> k(n, s), v(n, s), ko(n, s), vo(n, s);
    QVB_CUDA(cudaMemcpyAsync(k.p, keys, n * 8, cudaMemcpyHostToDevice, s));
    QVB_CUDA(cudaMemcpyAsync(v.p, vals, n * 8, cudaMemcpyHostToDevice, s));
    sort_pairs_u64_u64(k.p, ko.p, v.p, vo.p, n, begin_bit, end_bit, s);
    QVB_CUDA(cudaMemcpyAsync(keys_out, ko.p, n * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaMemcpyAsync(vals_out, vo.p, n * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}

namespace qvb {
namespace {
__global__ void k_test_keys(uint64_t* k, uint64_t* v, uint64_t n, uint64_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    k[i] = splitmix64(i) & mask;
    v[i] = i;
  }
}
}  // namespace
}  // namespace qvb

extern "C" int qvb_test_sort_bench(int device, uint64_t n, int bits, int reps, double* ms) {
  return guarded([&] {
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> k(n, s), v(n, s), ko(n, s), vo(n, s);
    k_test_keys<<<grid_for(n, 256), 256, 0, s>>>(k.p, v.p, n, bits >= 64 ? ~0ull : ((1ull << bits) - 1));
    QVB_LAUNCH_CHECK();
    sort_pairs_u64_u64(k.p, ko.p, v.p, vo.p, n, 0, bits, s);  // warm the pool
    cudaEvent_t a, b;
    QVB_CUDA(cudaEventCreate(&a));
    QVB_CUDA(cudaEventCreate(&b));
    QVB_CUDA(cudaEventRecord(a, s));
    for (int r = 0; r < reps; ++r) sort_pairs_u64_u64(k.p, ko.p, v.p, vo.p, n, 0, bits, s);
    QVB_CUDA(cudaEventRecord(b, s));
    QVB_CUDA(cudaEventSynchronize(b));
    float f = 0;
    QVB_CUDA(cudaEventElapsedTime(&f, a, b));
    *ms = f / reps;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

extern "C" int qvb_test_scan_u32(int device, const uint32_t* in, uint64_t n, int inclusive,
                                 uint64_t* out) {
  return guarded([&] {
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint32_t> a(n, s);
    DevBuf<uint64_t> o(n, s);
    QVB_CUDA(cudaMemcpyAsync(a.p, in, n * 4, cudaMemcpyHostToDevice, s));
    if (inclusive) {
      DevBuf<uint32_t> o32(n, s);
      inclusive_sum_u32_u32(a.p, o32.p, n, s);
      std::vector<uint32_t> h(n);
      QVB_CUDA(cudaMemcpyAsync(h.data(), o32.p, n * 4, cudaMemcpyDeviceToHost, s));
      QVB_CUDA(cudaStreamSynchronize(s));
      for (uint64_t i = 0; i < n; ++i) out[i] = h[i];
      return;
    }
    exclusive_sum_u32_u64(a.p, o.p, n, s);
    QVB_CUDA(cudaMemcpyAsync(out, o.p, n * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}
