// rowgather.cu — practical ceiling of random 512-byte row gathers from a
// 57 GB HBM table (the C4 feature table) on one B200: how close can any
// kernel get to the copy bandwidth, by rows in flight per warp (U), warps
// per SM, with and without writing the rows out?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rowgather rowgather.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t err_ = (x);                                                            \
    if (err_ != cudaSuccess) {                                                         \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// one warp = U rows in flight, 16 B per lane per row (512 B rows)
// the same rows through a lookup table: row = lut[hash] (random 8-byte
// reads from a table of nrows entries, as the store's packed table)
template <int U>
__global__ void k_rows_lut(const uint4* __restrict__ tab, const uint64_t* __restrict__ lut, uint64_t nrows,
                           uint64_t b, uint4* __restrict__ out, uint64_t seed) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r0 = w * U; r0 < b; r0 += nw * U) {
    uint64_t row[U];
#pragma unroll
    for (int u = 0; u < U; ++u) row[u] = __ldg(lut + __umul64hi(mix(seed + r0 + u), nrows));
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(tab + row[u] * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out + (r0 + u) * 32 + lane, v[u]);
  }
}

template <int U, bool WRITE>
__global__ void k_rows(const uint4* __restrict__ tab, uint64_t nrows, uint64_t b, uint4* __restrict__ out,
                       uint64_t seed, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned acc = 0;
  for (uint64_t r0 = w * U; r0 < b; r0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t row = __umul64hi(mix(seed + r0 + u), nrows);
      v[u] = ldnc(tab + row * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (WRITE) __stcs(out + (r0 + u) * 32 + lane, v[u]);
      else acc ^= v[u].x ^ v[u].w;
    }
  }
  if (!WRITE && acc == 0x12345678u) atomicAdd(sink, 1u);
}

template <int U, bool WRITE>
void run(const uint4* tab, uint64_t nrows, uint64_t b, uint4* out, unsigned* sink, int blocks_per_sm,
         int threads) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = sms * blocks_per_sm;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_rows<U, WRITE><<<grid, threads>>>(tab, nrows, b, out, 1, sink);
  CK(cudaEventRecord(e0));
  for (int r = 0; r < 5; ++r) k_rows<U, WRITE><<<grid, threads>>>(tab, nrows, b, out, 100 + r * b, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double bytes = 5.0 * b * 512 * (WRITE ? 2 : 1);
  std::printf("U=%d %-5s warps/SM %3d: %.3f ms/launch, HBM %.0f GB/s\n", U, WRITE ? "r+w" : "read",
              blocks_per_sm * threads / 32, ms / 5, bytes / (ms / 1e3) / 1e9);
}

int main() {
  const uint64_t nrows = 111000000ull, b = 1 << 20;
  uint4 *tab, *out;
  unsigned* sink;
  CK(cudaMalloc(&tab, nrows * 512));
  CK(cudaMemset(tab, 1, nrows * 512));
  CK(cudaMalloc(&out, b * 512));
  CK(cudaMalloc(&sink, 4));
  for (int bps : {4, 8}) {
    run<1, true>(tab, nrows, b, out, sink, bps, 256);
    run<2, true>(tab, nrows, b, out, sink, bps, 256);
    run<4, true>(tab, nrows, b, out, sink, bps, 256);
    run<8, true>(tab, nrows, b, out, sink, bps, 256);
    run<4, false>(tab, nrows, b, out, sink, bps, 256);
    run<8, false>(tab, nrows, b, out, sink, bps, 256);
  }
  uint64_t* lut;
  CK(cudaMalloc(&lut, nrows * 8));
  {
    std::vector<uint64_t> h(nrows);
    for (uint64_t i = 0; i < nrows; ++i) h[i] = (i * 2654435761ull) % nrows;
    CK(cudaMemcpy(lut, h.data(), nrows * 8, cudaMemcpyHostToDevice));
  }
  for (int bps : {4, 8}) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, z;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&z));
    k_rows_lut<4><<<sms * bps, 256>>>(tab, lut, nrows, b, out, 1);
    CK(cudaEventRecord(a));
    for (int r = 0; r < 5; ++r) k_rows_lut<4><<<sms * bps, 256>>>(tab, lut, nrows, b, out, 100 + r * b);
    CK(cudaEventRecord(z));
    CK(cudaEventSynchronize(z));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, z));
    std::printf("U=4 r+w via 8-byte lookup, warps/SM %3d: %.3f ms/launch, HBM %.0f GB/s (rows only)\n", bps * 8,
                ms / 5, 5.0 * b * 1024 / (ms / 1e3) / 1e9);
  }
  // the same table size, sequential copy of the same bytes (the copy peak)
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaMemcpy(out, tab, b * 512, cudaMemcpyDeviceToDevice));
  CK(cudaEventRecord(e0));
  for (int r = 0; r < 5; ++r) CK(cudaMemcpyAsync(out, tab + (uint64_t)r * b * 32, b * 512, cudaMemcpyDeviceToDevice));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  std::printf("cudaMemcpy D2D 512 MB: %.3f ms, %.0f GB/s (read+write)\n", ms / 5, 5.0 * 2 * b * 512 / (ms / 1e3) / 1e9);
  return 0;
}
