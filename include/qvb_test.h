/*
 * qvb_test.h — test-only entry points of libqvb.so: direct access to the
 * hand-written sort/scan primitives so tests/test_primitives_gpu.py can check
 * them against numpy's stable sort and cumsum. Not part of the drop-in API.
 */
#ifndef QVB_TEST_H
#define QVB_TEST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Stable LSD radix sort of (key, value) on key bits [begin_bit, end_bit). */
int qvb_test_sort_pairs_u64(int device, const uint64_t* keys, const uint64_t* vals, uint64_t n,
                            int begin_bit, int end_bit, uint64_t* keys_out, uint64_t* vals_out);
/* Device time (ms per sort) of sorting n random (u64 key, u64 value) pairs on
 * key bits [0, bits). */
int qvb_test_sort_bench(int device, uint64_t n, int bits, int reps, double* ms);
/* Exclusive (inclusive=0) or inclusive scan of u32 values, widened to u64. */
int qvb_test_scan_u32(int device, const uint32_t* in, uint64_t n, int inclusive, uint64_t* out);

/* out[i] = log1p(x[i]) by the device restatement of glibc's x86-64 FMA
 * log1p that the sampler's exponential keys use (sampler.cu). */
int qvb_test_log1p(int device, const double* x, uint64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif
