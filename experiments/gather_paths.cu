// gather_paths.cu — which load path gives the highest rate of random 4-byte
// gathers from an L2-resident vector on B200?  K1's sweep is bound by this
// rate (one L1 wavefront per random LDG), so any path with a cheaper tag
// stage (texture pipe, L1-bypassing loads) would raise K1's ceiling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_paths gather_paths.cu
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

__global__ void k_idx(uint32_t* idx, uint64_t e, uint64_t n, uint64_t seed, uint32_t share) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (i / share + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    // share > 1: groups of `share` consecutive lanes read the same 32-byte sector
    idx[i] = (uint32_t)__umul64hi(z, n) / 8 * 8 + (uint32_t)(i % share);
  }
}

template <int MODE>
__device__ __forceinline__ uint32_t gather(const uint32_t* __restrict__ v, cudaTextureObject_t t, uint32_t c) {
  if constexpr (MODE == 0) return __ldg(v + c);
  if constexpr (MODE == 1) {
    uint32_t r;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(v + c));
    return r;
  }
  if constexpr (MODE == 2) return tex1Dfetch<uint32_t>(t, static_cast<int>(c));
  if constexpr (MODE == 3) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(v + c));
    return r;
  }
  return 0;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ v, cudaTextureObject_t t,
                                                const uint32_t* __restrict__ idx, uint64_t e, uint32_t* out) {
  uint32_t acc = 0;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < e; b += nt * 8) {
    uint32_t c[8], x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = b + u * nt < e ? __ldg(idx + b + u * nt) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = gather<MODE>(v, t, c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += x[u];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// shared-memory reference: the same stream gathered from a 48 KB smem table
__global__ void __launch_bounds__(256) k_smem(const uint32_t* __restrict__ idx, uint64_t e, uint32_t* out) {
  __shared__ uint32_t tab[12288];
  for (int i = threadIdx.x; i < 12288; i += blockDim.x) tab[i] = i * 7u;
  __syncthreads();
  uint32_t acc = 0;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < e; b += nt * 8) {
    uint32_t c[8], x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = b + u * nt < e ? __ldg(idx + b + u * nt) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = tab[c[u] % 12288u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += x[u];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename F>
double rate(F launch, uint64_t e) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();
  CK(cudaEventRecord(a));
  for (int r = 0; r < 5; ++r) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return 5.0 * e / (ms / 1e3) / 1e9;
}

int main() {
  const uint64_t e = 400u << 20;
  uint32_t *idx, *v, *out;
  CK(cudaMalloc(&idx, e * 4));
  CK(cudaMalloc(&out, 4));
  const uint64_t maxn = (64ull << 20) / 4;
  CK(cudaMalloc(&v, maxn * 4));
  CK(cudaMemset(v, 1, maxn * 4));
  const int blocks = 148 * 8, threads = 256;
  for (uint64_t mb : {16, 48}) {
    const uint64_t n = (mb << 20) / 4;
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = v;
    rd.res.linear.desc = cudaCreateChannelDesc<uint32_t>();
    rd.res.linear.sizeInBytes = n * 4;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t = 0;
    CK(cudaCreateTextureObject(&t, &rd, &td, nullptr));
    for (uint32_t share : {1u, 2u, 4u, 8u}) {
      k_idx<<<1184, 256>>>(idx, e, n, 12345, share);
      CK(cudaDeviceSynchronize());
      const double r0 = rate([&] { k_gather<0><<<blocks, threads>>>(v, t, idx, e, out); }, e);
      const double r1 = rate([&] { k_gather<1><<<blocks, threads>>>(v, t, idx, e, out); }, e);
      const double r2 = rate([&] { k_gather<2><<<blocks, threads>>>(v, t, idx, e, out); }, e);
      const double r3 = rate([&] { k_gather<3><<<blocks, threads>>>(v, t, idx, e, out); }, e);
      const double r4 = rate([&] { k_smem<<<blocks, threads>>>(idx, e, out); }, e);
      std::printf("%3llu MB share %u: ldg %.1f  cg %.1f  tex %.1f  nc.noalloc %.1f  smem %.1f  G gathers/s\n",
                  (unsigned long long)mb, share, r0, r1, r2, r3, r4);
    }
    CK(cudaDestroyTextureObject(t));
  }
  CK(cudaGetLastError());
  return 0;
}
