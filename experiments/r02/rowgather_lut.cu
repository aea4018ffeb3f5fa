// rowgather_lut.cu — what does the lookup in front of a random row gather
// cost, and does it stop costing when the lookup structure fits in L2?
// 1M random 512-byte rows from a 57 GB table (C4), ids read from HBM, the row
// found through a lookup of L entries (8 bytes each) at a random index:
//   L = 111M (888 MB, the store's packed table today), 16M (128 MB),
//   8M (64 MB: fits the 126 MB L2), 1M (8 MB), and no lookup at all;
// fused (lookup then row, U rows in flight per warp) and two-phase (resolve
// every id first, then gather by resolved row).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rowgather_lut rowgather_lut.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t err_ = (x);                                                            \
    if (err_ != cudaSuccess) {                                                         \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {
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

// ids[i] = a random feature id; lut[j] = a row; entry used: lut[id % L]
// (id itself when L == 0), row = (entry + id) % nrows keeps rows uniform.
__global__ void k_ids(uint64_t* ids, uint64_t b, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b; i += (uint64_t)gridDim.x * blockDim.x)
    ids[i] = __umul64hi(mix(seed + i), n);
}
__global__ void k_lut(uint64_t* lut, uint64_t L, uint64_t nrows) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < L; i += (uint64_t)gridDim.x * blockDim.x)
    lut[i] = mix(i * 7 + 3) % nrows;
}

__device__ __forceinline__ uint64_t resolve(const uint64_t* __restrict__ lut, uint64_t L, uint64_t id,
                                            uint64_t nrows) {
  if (L == 0) return id;
  const uint64_t e = __ldg(lut + id % L);
  return (e + id) % nrows;
}

template <int U>
__global__ void __launch_bounds__(256) k_fused(const uint4* __restrict__ tab, const uint64_t* __restrict__ lut,
                                               uint64_t L, uint64_t nrows, const uint64_t* __restrict__ ids,
                                               uint64_t b, uint4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r0 = w * U; r0 < b; r0 += nw * U) {
    uint64_t row[U];
#pragma unroll
    for (int u = 0; u < U; ++u) row[u] = resolve(lut, L, __ldg(ids + r0 + u), nrows);
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(tab + row[u] * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out + (r0 + u) * 32 + lane, v[u]);
  }
}

// lookups spread over lanes: lane k of the warp resolves row r0+k, then the
// warp walks the 32 resolved rows (shuffled) U at a time
template <int U>
__global__ void __launch_bounds__(256) k_lanes(const uint4* __restrict__ tab, const uint64_t* __restrict__ lut,
                                               uint64_t L, uint64_t nrows, const uint64_t* __restrict__ ids,
                                               uint64_t b, uint4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g0 = w * 32; g0 < b; g0 += nw * 32) {
    const uint64_t mine = resolve(lut, L, __ldg(ids + g0 + lane), nrows);
#pragma unroll
    for (int k = 0; k < 32; k += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldnc(tab + __shfl_sync(~0u, mine, k + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs(out + (g0 + k + u) * 32 + lane, v[u]);
    }
  }
}

__global__ void k_resolve(const uint64_t* __restrict__ lut, uint64_t L, uint64_t nrows,
                          const uint64_t* __restrict__ ids, uint64_t b, uint64_t* __restrict__ rows) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b; i += (uint64_t)gridDim.x * blockDim.x)
    rows[i] = resolve(lut, L, ids[i], nrows);
}

template <typename F>
float time5(F f) {
  cudaEvent_t a, z;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&z));
  f(0);
  CK(cudaEventRecord(a));
  for (int r = 1; r <= 5; ++r) f(r);
  CK(cudaEventRecord(z));
  CK(cudaEventSynchronize(z));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, a, z));
  return ms / 5;
}

int main() {
  const uint64_t nrows = 111000000ull, b = 1 << 20;
  const int sms = 148;
  uint4 *tab, *out;
  uint64_t *lut, *ids, *rows;
  CK(cudaMalloc(&tab, nrows * 512));
  CK(cudaMemset(tab, 1, nrows * 512));
  CK(cudaMalloc(&out, b * 512));
  CK(cudaMalloc(&lut, nrows * 8));
  CK(cudaMalloc(&ids, 6 * b * 8));
  CK(cudaMalloc(&rows, b * 8));
  k_lut<<<sms * 8, 256>>>(lut, nrows, nrows);
  k_ids<<<sms * 8, 256>>>(ids, 6 * b, nrows, 99);
  CK(cudaDeviceSynchronize());
  const double gb = b * 1024.0 / 1e9;  // rows in + out
  for (uint64_t L : {111000000ull, 16777216ull, 8388608ull, 1048576ull, 0ull}) {
    for (int bps : {4, 8}) {
      const float f2 = time5([&](int r) {
        k_fused<2><<<sms * bps, 256>>>(tab, lut, L, nrows, ids + r * b, b, out);
      });
      const float f4 = time5([&](int r) {
        k_fused<4><<<sms * bps, 256>>>(tab, lut, L, nrows, ids + r * b, b, out);
      });
      const float l4 = time5([&](int r) {
        k_lanes<4><<<sms * bps, 256>>>(tab, lut, L, nrows, ids + r * b, b, out);
      });
      const float l8 = time5([&](int r) {
        k_lanes<8><<<sms * bps, 256>>>(tab, lut, L, nrows, ids + r * b, b, out);
      });
      const float rs = time5([&](int r) { k_resolve<<<sms * 8, 256>>>(lut, L, nrows, ids + r * b, b, rows); });
      const float tp = time5([&](int r) {
        k_resolve<<<sms * 8, 256>>>(lut, L, nrows, ids + r * b, b, rows);
        k_fused<2><<<sms * bps, 256>>>(tab, nullptr, 0, nrows, rows, b, out);
      });
      std::printf(
          "L=%9llu warps/SM %2d: fused U2 %.4f ms (%.0f GB/s) U4 %.4f (%.0f) | lanes U4 %.4f (%.0f) U8 %.4f (%.0f) | "
          "resolve %.4f, two-phase %.4f (%.0f)\n",
          (unsigned long long)L, bps * 8, f2, gb / f2 * 1e3, f4, gb / f4 * 1e3, l4, gb / l4 * 1e3, l8,
          gb / l8 * 1e3, rs, tp, gb / tp * 1e3);
    }
  }
  return 0;
}
