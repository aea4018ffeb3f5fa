// host_vmm.cu — why do random 512-byte row reads from a 14 GB pinned host
// tier run at 38 GB/s when a 2 GB tier gives 51 GB/s? Candidates: the GPU's
// translation reach over system memory (page size of the sysmem mapping) or
// the host side (NUMA placement of the pinned pages). This compares
//   - cudaHostAlloc (the store's host tier today),
//   - cuMemCreate on CU_MEM_LOCATION_TYPE_HOST_NUMA at the recommended
//     granularity (the GPU maps it with the allocation's page size),
// over tier sizes 2..14 GB, with rows drawn from the whole tier or from its
// first 2 GB (same allocation, smaller touched range), unsorted and sorted.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_vmm host_vmm.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t err_ = (x);                                                            \
    if (err_ != cudaSuccess) {                                                         \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)
#define CU(x)                                                             \
  do {                                                                    \
    CUresult r_ = (x);                                                    \
    if (r_ != CUDA_SUCCESS) {                                             \
      const char* s_ = nullptr;                                           \
      cuGetErrorString(r_, &s_);                                          \
      std::printf("CU %s at %s:%d\n", s_ ? s_ : "?", __FILE__, __LINE__); \
      return false;                                                       \
    }                                                                     \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// rows[] given (sorted or not); one warp per row, U rows in flight
template <int U>
__global__ void __launch_bounds__(256) k_rows(const uint4* __restrict__ host, const uint64_t* __restrict__ rows,
                                              uint64_t b, uint4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r0 = w * U; r0 < b; r0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < b) v[u] = __ldcs(host + rows[r0 + u] * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < b) __stcs(out + (r0 + u) * 32 + lane, v[u]);
  }
}

struct Tier {
  void* host = nullptr;  // CPU address
  void* dev = nullptr;   // GPU address
  size_t bytes = 0;
  int mode = 0;
  CUmemGenericAllocationHandle h{};
  CUdeviceptr va = 0;
};

bool make_vmm(Tier& t, size_t bytes, int numa, bool recommended) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  prop.location.id = numa;
  size_t gran = 0;
  CU(cuMemGetAllocationGranularity(&gran, &prop,
                                   recommended ? CU_MEM_ALLOC_GRANULARITY_RECOMMENDED
                                               : CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  bytes = (bytes + gran - 1) / gran * gran;
  CU(cuMemCreate(&t.h, bytes, &prop, 0));
  CU(cuMemAddressReserve(&t.va, bytes, gran, 0, 0));
  CU(cuMemMap(t.va, bytes, 0, t.h, 0));
  CUmemAccessDesc acc[2]{};
  acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc[0].location.id = 0;
  acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  acc[1].location.id = numa;
  acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (cuMemSetAccess(t.va, bytes, acc, 2) != CUDA_SUCCESS) {
    CU(cuMemSetAccess(t.va, bytes, acc, 1));
    t.host = nullptr;  // GPU-only mapping: filled with cudaMemset
    std::printf("  (no CPU mapping)\n");
  } else {
    t.host = reinterpret_cast<void*>(t.va);
  }
  t.dev = reinterpret_cast<void*>(t.va);
  t.bytes = bytes;
  std::printf("  vmm granularity %zu KB\n", gran >> 10);
  return true;
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaFree(nullptr));
  int numa = -1;
  if (cudaDeviceGetAttribute(&numa, cudaDevAttrHostNumaId, 0) != cudaSuccess) numa = 0;
  if (numa < 0) numa = 0;
  std::printf("device host NUMA id %d\n", numa);
  const uint64_t b = 1 << 20;  // 1M rows = 512 MB per launch (beyond L2)
  uint4* out;
  uint64_t* drows;
  CK(cudaMalloc(&out, b * 512));
  CK(cudaMalloc(&drows, b * 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<uint64_t> rows(b);
  for (uint64_t gb : {2ull, 4ull, 8ull, 14ull}) {
    const size_t bytes = gb << 30;
    for (int mode = 0; mode < 3; ++mode) {
      Tier t;
      t.mode = mode;
      if (mode == 0) {
        CK(cudaHostAlloc(&t.host, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        CK(cudaHostGetDevicePointer(&t.dev, t.host, 0));
        t.bytes = bytes;
      } else if (!make_vmm(t, bytes, numa, mode == 2)) {
        std::printf("%2llu GB mode %d: vmm unavailable\n", (unsigned long long)gb, mode);
        continue;
      }
      if (t.host) std::memset(t.host, 1, t.bytes);
      else CK(cudaMemset(t.dev, 1, t.bytes));
      const char* name = mode == 0 ? "cudaHostAlloc" : mode == 1 ? "vmm host_numa min" : "vmm host_numa rec";
      for (int span = 0; span < 2; ++span) {
        const uint64_t nrows = span ? (2ull << 30) / 512 : bytes / 512;
        for (int sorted = 0; sorted < 2; ++sorted) {
          uint64_t z = 12345 + gb;
          for (auto& r : rows) {
            z += 0x9E3779B97F4A7C15ull;
            uint64_t x = z;
            x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
            x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
            x ^= x >> 31;
            r = x % nrows;
          }
          if (sorted) std::sort(rows.begin(), rows.end());
          CK(cudaMemcpy(drows, rows.data(), b * 8, cudaMemcpyHostToDevice));
          const int grid = 148 * 8;
          k_rows<4><<<grid, 256>>>(static_cast<const uint4*>(t.dev), drows, b, out);
          CK(cudaEventRecord(e0));
          for (int r = 0; r < 5; ++r) k_rows<4><<<grid, 256>>>(static_cast<const uint4*>(t.dev), drows, b, out);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          CK(cudaGetLastError());
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          std::printf("%2llu GB %-18s rows over %-6s %-8s: %.1f GB/s\n", (unsigned long long)gb, name,
                      span ? "2 GB" : "tier", sorted ? "sorted" : "random", 5.0 * b * 512 / (ms / 1e3) / 1e9);
        }
      }
      if (mode == 0) {
        CK(cudaFreeHost(t.host));
      } else {
        cuMemUnmap(t.va, t.bytes);
        cuMemAddressFree(t.va, t.bytes);
        cuMemRelease(t.h);
      }
    }
  }
  return 0;
}
