// gather4_bench.cu — micro-experiment: random 8-byte gathers y[idx[e]] via
// (a) per-lane LDG (the K1 sweep's pattern) and (b) TMA tile::gather4
// (sm_100a: one instruction fetches 4 arbitrary 16-byte rows into shared
// memory, bypassing the L1 tag pipeline). Prints G gathers/s for an
// L2-resident and an HBM-resident operand vector.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_bench gather4_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t err_ = (x);                                                            \
    if (err_ != cudaSuccess) {                                                       \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

__global__ void k_fill(double* y, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    y[i] = (double)(i % 1000003) * 1e-7;
}
__global__ void k_idx(uint32_t* idx, uint64_t e, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    idx[i] = (uint32_t)__umul64hi(z, n);
  }
}

// (a) LDG: each lane gathers 8 independent operands per step
__global__ void __launch_bounds__(256) k_ldg(const double* __restrict__ y, const uint32_t* __restrict__ idx,
                                             uint64_t e, double* out) {
  double acc = 0;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < e; b += nt * 8) {
    uint32_t c[8];
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = b + u * nt < e ? __ldg(idx + b + u * nt) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(y + c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

// (b) TMA gather4: per warp, S stages of 32 operands (8 gather4 x 4 rows of 16 B)
constexpr int S = 4;
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256) k_tma(const __grid_constant__ CUtensorMap tmap,
                                             const uint32_t* __restrict__ idx, uint64_t e, double* out) {
  __shared__ alignas(128) double buf[8][S][8][16];  // per warp: S stages x 8 gather4 (64 B used of a 128-B aligned slot)
  __shared__ alignas(8) uint64_t bar[8][S];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t batches = (e + 31) / 32;
  double acc = 0;
  uint32_t phase[S] = {0, 0, 0, 0};
  uint32_t myidx[S];
  auto issue = [&](uint64_t batch, int s) {
    const uint64_t i = batch * 32 + lane;
    const uint32_t c = i < e ? idx[i] : 0;
    myidx[s] = c;
    const uint32_t row = c >> 1;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][s])),
                   "r"(32 * 16));
    for (int q = 0; q < 8; ++q) {
      const uint32_t r0 = __shfl_sync(0xffffffffu, row, 4 * q + 0);
      const uint32_t r1 = __shfl_sync(0xffffffffu, row, 4 * q + 1);
      const uint32_t r2 = __shfl_sync(0xffffffffu, row, 4 * q + 2);
      const uint32_t r3 = __shfl_sync(0xffffffffu, row, 4 * q + 3);
      if (lane == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&buf[w][s][q][0])),
            "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar[w][s]))
            : "memory");
      }
    }
  };
  uint64_t b = gw;
  for (int s = 0; s < S; ++s)
    if (b + s * nwarps < batches) issue(b + s * nwarps, s);
  for (; b < batches; b += S * nwarps) {
    for (int s = 0; s < S; ++s) {
      const uint64_t cur = b + s * nwarps;
      if (cur >= batches) break;
      // wait
      asm volatile(
          "{\n .reg .pred p;\n WAIT_%=:\n"
          " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&bar[w][s])),
          "r"(phase[s]));
      phase[s] ^= 1;
      acc += buf[w][s][lane >> 2][(lane & 3) * 2 + (myidx[s] & 1)];
      __syncwarp();
      const uint64_t nxt = cur + S * nwarps;
      if (nxt < batches) issue(nxt, s);
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn encode = (EncodeFn)fn;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (uint64_t n : {2400000ull, 111000000ull}) {
    const uint64_t e = 400000000ull;
    double* y;
    uint32_t* idx;
    double* out;
    CK(cudaMalloc(&y, n * 8));
    CK(cudaMalloc(&idx, e * 4));
    CK(cudaMalloc(&out, 8));
    k_fill<<<1184, 256>>>(y, n);
    k_idx<<<1184, 256>>>(idx, e, n, 7);
    CUtensorMap tmap;
    cuuint64_t dims[2] = {2, n / 2};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, y, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) std::printf("encode failed %d\n", (int)r);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int blocks_per_sm : {4, 8}) {
      const int grid = sms * blocks_per_sm;
      k_ldg<<<grid, 256>>>(y, idx, e, out);
      cudaEventRecord(a);
      k_ldg<<<grid, 256>>>(y, idx, e, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      std::printf("n=%llu LDG  grid=%d: %.3f ms  %.1f G gathers/s\n", (unsigned long long)n, grid, ms, e / ms / 1e6);
      k_tma<<<grid, 256>>>(tmap, idx, e, out);
      CK(cudaGetLastError());
      cudaEventRecord(a);
      k_tma<<<grid, 256>>>(tmap, idx, e, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      std::printf("n=%llu TMA4 grid=%d: %.3f ms  %.1f G gathers/s\n", (unsigned long long)n, grid, ms, e / ms / 1e6);
    }
    cudaFree(y);
    cudaFree(idx);
    cudaFree(out);
  }
  return 0;
}
