// common.cuh — shared plumbing of the qvb library: status/error propagation
// across the C-ABI, device guards, RAII device buffers, and the SplitMix64
// stream (reference include/qv/rng.hpp:10-57) as device code.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <stdexcept>
#include <tuple>
#include <string>
#include <utility>

#include "../../include/qvb.h"

namespace qvb {

// Internal exception; converted to a qvb_status at the C-ABI boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error in %s (%s:%d): %s", what, file, line,
                  cudaGetErrorString(e));
    throw Error(QVB_ERR_CUDA, buf);
  }
}
#define QVB_CUDA(x) ::qvb::cuda_check((x), #x, __FILE__, __LINE__)
#define QVB_LAUNCH_CHECK() ::qvb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

void set_last_error(const std::string& m);
// Keeps the device's stream-ordered pool (cudaMallocAsync) from returning
// memory to the driver at every synchronisation, so per-call scratch is
// recycled instead of re-mapped. Once per device.
void retain_pool(int device);

// Runs `f` and maps exceptions to status codes (the reference's exception
// hierarchy, include/qv/error.hpp:10-32, is mirrored by the codes).
template <typename F>
int guarded(F&& f) {
  try {
    f();
    set_last_error("");
    return QVB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return QVB_ERR_GENERIC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return QVB_ERR_GENERIC;
  }
}

// Selects `device` for the scope and restores the caller's device after.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
      cudaGetLastError();
      fail(QVB_ERR_CUDA, "no CUDA device available (the qvb library has no CPU fallback)");
    }
    if (device < 0 || device >= count) fail(QVB_ERR_VALIDATION, "device index out of range");
    QVB_CUDA(cudaGetDevice(&prev));
    if (prev != device) QVB_CUDA(cudaSetDevice(device));
    retain_pool(device);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Stream-ordered device buffer (cudaMallocAsync pool).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) QVB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* release_ownership() {
    T* q = p;
    p = nullptr;
    n = 0;
    return q;
  }
  ~DevBuf() { release(); }
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      s = o.s;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  size_t bytes() const { return n * sizeof(T); }
};

// Persistent grid: as many blocks as fit on all SMs at once (one wave),
// capped by the work available.
template <typename Kernel>
inline unsigned resident_grid(Kernel k, int block, size_t smem, uint64_t work_blocks) {
  int dev = 0, sms = 0, per_sm = 0;
  QVB_CUDA(cudaGetDevice(&dev));
  QVB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  QVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, smem));
  uint64_t g = static_cast<uint64_t>(sms) * (per_sm > 0 ? per_sm : 1);
  if (work_blocks < g) g = work_blocks;
  return static_cast<unsigned>(g ? g : 1);
}

// resident_grid(k, block, smem, ~0) of the CURRENT device, cached per
// (kernel, device, block, smem): launch paths call it every launch, several
// stores may live on different devices, and first calls may race.
template <typename Kernel>
inline unsigned resident_grid_cached(Kernel k, int block, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, unsigned> cache;
  int dev = 0;
  QVB_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(reinterpret_cast<const void*>(k), dev, block, smem);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const unsigned g = resident_grid(k, block, smem, ~0ull);
  cache.emplace(key, g);
  return g;
}

inline unsigned grid_for(uint64_t items, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (items + block - 1) / block;
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// ---- L2 cache-policy loads/stores ------------------------------------------
// Streams that are touched once per pass (CSR columns, per-node vectors) are
// marked evict_first so they do not push the gathered vector out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
               : "=l"(v)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint16_t ld_stream(const uint16_t* a, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
               : "=h"(v)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream_u8(const uint8_t* a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
               : "=r"(v)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream(uint32_t* a, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint32_t ld_hint(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_hint(const uint64_t* a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
// Gather of one operand: mode 0 = ld.global.nc (read-only path, L1 allocate),
// 1 = ld.global.nc.L1::no_allocate, 2 = ld.global.cg (L2 only), 3 = .L2::evict_last.
__device__ __forceinline__ double ld_gather(const double* a, int mode) {
  double v;
  if (mode == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(a));
  } else if (mode == 2) {
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(a));
  } else if (mode == 3) {
    asm volatile(
        "{\n .reg .b64 p;\n createpolicy.fractional.L2::evict_last.b64 p, 1.0;\n"
        " ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], p;\n}"
        : "=d"(v)
        : "l"(a));
  } else {
    v = __ldg(a);
  }
  return v;
}
__device__ __forceinline__ void st_stream(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

// ---- SplitMix64 (rng.hpp:10-57) ------------------------------------------
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// qv::splitmix64 (rng.hpp:12-18)
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) { return mix64(x + kGamma); }
// Draw k (0-based) of RngStream{state}: next() adds gamma, then mixes.
__host__ __device__ __forceinline__ uint64_t stream_draw(uint64_t state, uint64_t k) {
  return mix64(state + (k + 1) * kGamma);
}
// RngStream::uniform (rng.hpp:35): 53-bit, exact.
__host__ __device__ __forceinline__ double to_uniform(uint64_t r) {
  return static_cast<double>(r >> 11) * 0x1.0p-53;
}
// RngStream::below (rng.hpp:42-45): high 64 bits of r * n.
__device__ __forceinline__ uint64_t to_below(uint64_t r, uint64_t n) { return __umul64hi(r, n); }

// derive_stream (rng.hpp:50-57), split after the (master, a) words so a
// prefix shared by many streams is chained once.
__host__ __device__ __forceinline__ uint64_t derive_prefix(uint64_t master, uint64_t a) {
  const uint64_t s = splitmix64(master ^ 0x6a09e667f3bcc909ULL);
  return splitmix64(s ^ splitmix64(a ^ 0xbb67ae8584caa73bULL));
}
__host__ __device__ __forceinline__ uint64_t derive_finish(uint64_t prefix, uint64_t b, uint64_t c) {
  const uint64_t mb = splitmix64(b ^ 0x3c6ef372fe94f82bULL);
  const uint64_t mc = splitmix64(c ^ 0xa54ff53a5f1d36f1ULL);
  return splitmix64(splitmix64(prefix ^ mb) ^ mc);
}
__host__ __device__ __forceinline__ uint64_t derive_state(uint64_t master, uint64_t a, uint64_t b = 0,
                                                          uint64_t c = 0) {
  return derive_finish(derive_prefix(master, a), b, c);
}

// Synthetic feature value X[f][k].
__host__ __device__ __forceinline__ float feature_value(uint64_t f, uint32_t dim, uint32_t k) {
  return static_cast<float>(splitmix64(f * dim + k) >> 40) * 0x1.0p-24f;
}

// ---- hand-written primitives (primitives.cu) --------------------------------
// Stable LSD radix sort of (key, value) pairs on bits [begin_bit, end_bit).
void sort_pairs_u32_u32(const uint32_t* kin, uint32_t* kout, const uint32_t* vin, uint32_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s);
void sort_pairs_u64_u64(const uint64_t* kin, uint64_t* kout, const uint64_t* vin, uint64_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s);
void sort_pairs_u64_u32(const uint64_t* kin, uint64_t* kout, const uint32_t* vin, uint32_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s);
// out[i] = sum_{j<i} in[j]; returns nothing (total = out[n-1] + in[n-1]).
void exclusive_sum_u32_u64(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t s);
void exclusive_sum_u8_u32(const uint8_t* in, uint32_t* out, uint64_t n, cudaStream_t s);
void inclusive_sum_u32_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s);
// Sum reduction into a device scalar.
void sum_u8_u64(const uint8_t* in, uint64_t* out, uint64_t n, cudaStream_t s);

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b == 0 ? 1 : b;
}

template <typename T>
inline T read_scalar(const T* dptr, cudaStream_t s) {
  T v{};
  QVB_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
  QVB_CUDA(cudaStreamSynchronize(s));
  return v;
}

}  // namespace qvb
