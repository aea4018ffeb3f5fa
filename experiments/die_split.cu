// die_split.cu — does splitting a randomly gathered vector between the two
// B200 dies raise the L2 capacity it sees?
//
// 1. Classify SMs into two groups by their L2 hit latency to one 2 KB
//    granule (near-die ~234 cycles vs far-die ~262 on B300-class parts).
// 2. Random 4-byte gathers over S MB: (a) every SM over all of it, (b) group g
//    only over half g. If each die's L2 caches what its own SMs read, (b)
//    holds twice the vector before it starts missing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o die_split die_split.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// chase: p[i] = next index; measures cycles per dependent L2 hit (ld.cg)
__global__ void k_probe(const uint32_t* __restrict__ chain, int steps, uint32_t* lat_by_sm) {
  if (threadIdx.x != 0) return;
  uint32_t i = 0;
  for (int s = 0; s < 8; ++s) {  // warm
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(chain + i));
    i = v;
  }
  i = 0;
  const long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(chain + i));
    i = v;
  }
  const long long t1 = clock64();
  lat_by_sm[smid()] = static_cast<uint32_t>((t1 - t0) / steps) + (i == 0xFFFFFFFF);
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void k_gather(const uint32_t* __restrict__ v, uint64_t n, const uint8_t* __restrict__ group,
                         int split, uint64_t per, uint32_t* out, uint64_t seed) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t lo = 0, span = n;
  if (split) {
    const int g = group[smid()];
    span = n / 2;
    lo = g ? n / 2 : 0;
  }
  uint32_t acc = 0;
  uint64_t st = mix(t ^ seed);
  for (uint64_t i = 0; i < per; i += 8) {
    uint32_t x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      st = mix(st + 0x9e3779b97f4a7c15ULL);
      x[u] = __ldg(v + lo + __umul64hi(st, span));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += x[u];
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // chain inside one 2 KB granule: 512 words, stride 37 (a cycle through all)
  std::vector<uint32_t> h(512);
  for (int i = 0; i < 512; ++i) h[i] = (i + 37) % 512;
  uint32_t *chain, *lat;
  cudaMalloc(&chain, 4 << 20);
  cudaMemcpy(chain, h.data(), 2048, cudaMemcpyHostToDevice);
  cudaMalloc(&lat, 4 * 1024);
  cudaMemset(lat, 0, 4 * 1024);
  std::vector<uint32_t> best(sms, 0xFFFFFFFF);
  for (int rep = 0; rep < 6; ++rep) {  // one thread per CTA, many CTAs: every SM sampled
    k_probe<<<sms * 8, 32>>>(chain, 2000, lat);
    std::vector<uint32_t> l(sms);
    cudaMemcpy(l.data(), lat, 4 * sms, cudaMemcpyDeviceToHost);
    for (int i = 0; i < sms; ++i)
      if (l[i]) best[i] = std::min(best[i], l[i]);
  }
  std::vector<uint32_t> sorted = best;
  std::sort(sorted.begin(), sorted.end());
  const uint32_t mid = (sorted.front() + sorted.back()) / 2;
  std::vector<uint8_t> grp(sms);
  int n0 = 0;
  for (int i = 0; i < sms; ++i) {
    grp[i] = best[i] > mid;
    n0 += !grp[i];
  }
  std::printf("latency min %u max %u split at %u: group0 %d SMs, group1 %d SMs\n", sorted.front(),
              sorted.back(), mid, n0, sms - n0);
  std::printf("per-SM latency:");
  for (int i = 0; i < sms; ++i) std::printf(" %u", best[i]);
  std::printf("\n");
  uint8_t* dgrp;
  cudaMalloc(&dgrp, sms);
  cudaMemcpy(dgrp, grp.data(), sms, cudaMemcpyHostToDevice);

  const uint64_t maxmb = 256;
  uint32_t *v, *out;
  cudaMalloc(&v, maxmb << 20);
  cudaMalloc(&out, 4);
  cudaMemset(v, 1, maxmb << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  const uint64_t per = 512;
  for (uint64_t mb : {32, 48, 64, 80, 96, 112, 128, 160, 192}) {
    const uint64_t n = (mb << 20) / 4;
    double r[2];
    for (int split = 0; split < 2; ++split) {
      k_gather<<<blocks, threads>>>(v, n, dgrp, split, per, out, 1);
      cudaEventRecord(a);
      for (int rr = 0; rr < 5; ++rr) k_gather<<<blocks, threads>>>(v, n, dgrp, split, per, out, rr + 2);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      r[split] = 5.0 * blocks * threads * per / (ms / 1e3) / 1e9;
    }
    std::printf("%4llu MB: all SMs over all %7.1f G/s | groups over halves %7.1f G/s\n",
                (unsigned long long)mb, r[0], r[1]);
  }
  return 0;
}
