// Random 4-byte gather throughput vs working-set size: where does the
// B200's L2 stop holding a randomly gathered vector?  nvcc -O3 -arch=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void k_gather(const uint32_t* __restrict__ v, uint64_t n, uint64_t per, uint32_t* out, uint64_t seed) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  uint64_t st = mix(t ^ seed);
  for (uint64_t i = 0; i < per; i += 8) {
    uint32_t x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { st = mix(st + 0x9e3779b97f4a7c15ULL); x[u] = __ldg(v + (st % n)); }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += x[u];
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const uint64_t maxmb = 256;
  uint32_t* v; uint32_t* out;
  cudaMalloc(&v, maxmb << 20); cudaMalloc(&out, 4);
  cudaMemset(v, 1, maxmb << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 8, threads = 256; const uint64_t per = 512;
  for (uint64_t mb : {4, 16, 32, 48, 56, 64, 72, 80, 96, 112, 128, 192, 256}) {
    const uint64_t n = (mb << 20) / 4;
    k_gather<<<blocks, threads>>>(v, n, per, out, 1);  // warm
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_gather<<<blocks, threads>>>(v, n, per, out, r + 2);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double g = 5.0 * blocks * threads * per / (ms / 1e3) / 1e9;
    printf("%4llu MB: %7.1f G gathers/s\n", (unsigned long long)mb, g);
  }
  return 0;
}
