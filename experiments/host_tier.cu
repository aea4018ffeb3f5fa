// host_tier.cu — random row reads from the pinned host tier over PCIe: does
// the read rate depend on the host table size (GPU TLB reach over system
// memory), and do transparent huge pages behind cudaHostRegister help?
// One warp per 512-byte row (32 lanes x 16 B), 1M uniformly random rows per
// launch, rows written to device memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_tier host_tier.cu
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

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

template <int U>
__global__ void __launch_bounds__(256) k_rows(const uint4* __restrict__ host, uint64_t nrows, uint64_t b,
                                              uint4* __restrict__ out, uint64_t seed) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r0 = w * U; r0 < b; r0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t r = r0 + u;
      const uint64_t row = __umul64hi(mix(seed + r), nrows);
      if (r < b) v[u] = __ldcs(host + row * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < b) __stcs(out + (r0 + u) * 32 + lane, v[u]);
  }
}

int main(int argc, char** argv) {
  const uint64_t b = 1 << 20;
  uint4* out;
  CK(cudaMalloc(&out, b * 512));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (uint64_t mb : {256ull, 2048ull, 14336ull}) {
    const uint64_t bytes = mb << 20;
    for (int mode = 0; mode < 2; ++mode) {
      void* h = nullptr;
      if (mode == 0) {
        CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
      } else {
        h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (h == MAP_FAILED) { std::printf("mmap failed\n"); return 1; }
        madvise(h, bytes, MADV_HUGEPAGE);
      }
      std::memset(h, 1, bytes);
      if (mode == 1) CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
      void* d = nullptr;
      CK(cudaHostGetDevicePointer(&d, h, 0));
      for (int grid : {148 * 8, 148 * 16}) {
        k_rows<4><<<grid, 256>>>(static_cast<const uint4*>(d), bytes / 512, b, out, 1);
        CK(cudaEventRecord(e0));
        for (int r = 0; r < 5; ++r) k_rows<4><<<grid, 256>>>(static_cast<const uint4*>(d), bytes / 512, b, out, r + 2);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::printf("%6llu MB %-22s grid %5d: %.1f GB/s\n", (unsigned long long)mb,
                    mode ? "mmap+THP+HostRegister" : "cudaHostAlloc", grid, 5.0 * b * 512 / (ms / 1e3) / 1e9);
      }
      if (mode == 0) {
        CK(cudaFreeHost(h));
      } else {
        CK(cudaHostUnregister(h));
        munmap(h, bytes);
      }
    }
  }
  return 0;
}
