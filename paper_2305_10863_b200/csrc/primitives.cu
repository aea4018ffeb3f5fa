// primitives.cu — sort / scan / reduce building blocks used by the one-time
// preprocessing (in-CSR build) and by the ranking/read-planning kernels.
// Round 1 backs them with CUB (CUDA toolkit headers, compiled into this
// library for sm_100a); every call site goes through these wrappers so they
// can be swapped for hand-written onesweep kernels without touching callers.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace qvb {

namespace {
template <typename K, typename V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int begin_bit,
                int end_bit, cudaStream_t s) {
  if (n == 0) return;
  size_t temp = 0;
  QVB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, kin, kout, vin, vout, n, begin_bit,
                                           end_bit, s));
  DevBuf<uint8_t> t(temp, s);
  QVB_CUDA(cub::DeviceRadixSort::SortPairs(t.p, temp, kin, kout, vin, vout, n, begin_bit,
                                           end_bit, s));
}
}  // namespace

void sort_pairs_u32_u32(const uint32_t* kin, uint32_t* kout, const uint32_t* vin, uint32_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s) {
  sort_pairs(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void sort_pairs_u64_u64(const uint64_t* kin, uint64_t* kout, const uint64_t* vin, uint64_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s) {
  sort_pairs(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void sort_pairs_u64_u32(const uint64_t* kin, uint64_t* kout, const uint32_t* vin, uint32_t* vout,
                        uint64_t n, int begin_bit, int end_bit, cudaStream_t s) {
  sort_pairs(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}

void exclusive_sum_u32_u64(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  size_t temp = 0;
  QVB_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, temp, in, out, cub::Sum(), uint64_t(0), n, s));
  DevBuf<uint8_t> t(temp, s);
  QVB_CUDA(cub::DeviceScan::ExclusiveScan(t.p, temp, in, out, cub::Sum(), uint64_t(0), n, s));
}

void exclusive_sum_u8_u32(const uint8_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  size_t temp = 0;
  QVB_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, temp, in, out, cub::Sum(), uint32_t(0), n, s));
  DevBuf<uint8_t> t(temp, s);
  QVB_CUDA(cub::DeviceScan::ExclusiveScan(t.p, temp, in, out, cub::Sum(), uint32_t(0), n, s));
}

void inclusive_sum_u32_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  size_t temp = 0;
  QVB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, in, out, n, s));
  DevBuf<uint8_t> t(temp, s);
  QVB_CUDA(cub::DeviceScan::InclusiveSum(t.p, temp, in, out, n, s));
}

void sum_u8_u64(const uint8_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  if (n == 0) {
    QVB_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), s));
    return;
  }
  size_t temp = 0;
  QVB_CUDA(cub::DeviceReduce::Reduce(nullptr, temp, in, out, n, cub::Sum(), uint64_t(0), s));
  DevBuf<uint8_t> t(temp, s);
  QVB_CUDA(cub::DeviceReduce::Reduce(t.p, temp, in, out, n, cub::Sum(), uint64_t(0), s));
}

}  // namespace qvb
