// sampler.cu — K0, the k-hop neighbour sampler: the request-ID producer
// upstream of the collect call (reference src/sampler.cpp:21-149, called per
// batch from simulator.cpp:250-254). Bit-identical to qv::batch_sample.
//
// HBM layout of a qvb_sampler (n nodes, C candidates):
//   cro  u64[n+1]  candidate row offsets
//   ccol u32[C]    candidate node, in the reference's candidate order
//   cw   f64[C]    candidate weight (summed over parallel edges in CSR order);
//                  absent when every weight is 1.0
//   cpos u32[n]    positive-weight candidates per row
// Without parallel edges the candidates are the out-CSR itself.
//
// A batch runs hop by hop over the frontier of ALL seeds at once. Frontier k
// is stored seed-major, parent-major, candidate-order — the concatenation of
// the reference's per-seed frontiers[k] — as (node u32, seed slot u32):
//   k_hop_count    m_i = min(cpos[p], fanout)                 (:24-28)
//   scan           child offsets O: children of parent i at O[i]..O[i+1)
//   k_hop_sample   one warp per parent: every positive candidate when
//                  m == positive (:30-36), else the m smallest (Exp(1)/w, idx)
//                  keys (:38-51), written in candidate order; the stream is
//                  derive_stream(splitmix64(rng ^ seed*gamma), k, idx, p)
//                  (:94, :136), counter-based, so draw t is computed directly
//   k_seed_starts  seed segment starts of frontier k: ss_k[s] = O[ss_{k-1}[s]]
// then the flatten to seed-major/hop-major order and the sorted union
// (BatchSampleStats::unique_nodes, :140-146) through a node bitmap.
//
// Selection. Rows of <= 32 candidates rank the keys across the warp (one key
// per lane); rows of <= 256 keep 8 keys per lane in registers; longer rows
// take one CTA each and stage their keys in its scratch slab (on a side
// stream, concurrently with the warp kernel). The latter two find the m-th
// smallest key by an 8-bit radix select over the key bits (non-negative
// doubles order like their bit patterns) and then take keys < T plus the
// first keys == T in candidate order — exactly the reference's
// nth_element over (key, idx) pairs followed by the sort by idx.
#include <mutex>
#include <algorithm>
#include <memory>
#include <vector>

#include "common.cuh"
#include "graph.cuh"

struct qvb_sampler {
  int device = 0;
  uint64_t n = 0, e = 0, ncand = 0, max_len = 0, bytes = 0;
  bool parallel = false;
  uint64_t* cro = nullptr;
  uint32_t* ccol = nullptr;
  double* cw = nullptr;  // nullptr: unit weights
  uint32_t* cpos = nullptr;
  uint64_t* scratch = nullptr;  // long-row key slabs, large_ctas * max_len
  uint32_t large_ctas = 0;
  cudaStream_t side = nullptr;  // long-row kernel runs beside the warp kernel
  double build_ms = 0.0;
  // qvb_batch_sample shares scratch and the side stream, and returns only
  // after its batch completed: calls on one sampler are serialised here
  std::mutex mu;
  ~qvb_sampler() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    cudaFree(cro);
    cudaFree(ccol);
    cudaFree(cw);
    cudaFree(cpos);
    cudaFree(scratch);
    if (side) cudaStreamDestroy(side);
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct qvb_sample {
  int device = 0;
  uint64_t nseeds = 0, total = 0, unique_count = 0;
  uint32_t hops = 0;
  uint64_t* nodes = nullptr;
  uint64_t* counts = nullptr;
  uint64_t* unique = nullptr;
  double ms = 0.0;
  ~qvb_sample() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    cudaFree(nodes);
    cudaFree(counts);
    cudaFree(unique);
    if (prev >= 0) cudaSetDevice(prev);
  }
};

namespace qvb {
namespace {

constexpr unsigned kBlock = 256;
constexpr unsigned kWarpsPerBlock = kBlock / 32;
constexpr int kRegRounds = 8;                    // register path: L <= 256
constexpr uint32_t kRegMax = 32u * kRegRounds;
constexpr uint64_t kScratchBudget = 256ull << 20;  // long-row key slabs
constexpr uint64_t kNoKey = ~0ull;  // above every key (keys are >= +0.0, <= +inf)

// ---- glibc log1p ----------------------------------------------------------
__device__ __forceinline__ double with_hi(double x, int32_t h) {
  return __hiloint2double(h, __double2loint(x));
}

// std::log1p in RngStream::exponential (rng.hpp:38) as the reference runs it:
// glibc 2.39's x86-64 ifunc picks __log1p_fma on FMA hardware — fdlibm
// s_log1p.c with glibc's Estrin-form polynomial, compiled with FMA
// contraction. Every __fma_rn below is an FMA that build emitted; every other
// operation is a separately rounded IEEE op (this file builds with
// -fmad=false), so the result is bit-identical for every input.
__device__ double glibc_log1p(double x) {
  const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33, two54 = 0x1p54;
  const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2,
               Lp3 = 0x1.2492494229359p-2, Lp4 = 0x1.c71c51d8e78afp-3,
               Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3,
               Lp7 = 0x1.2f112df3e5244p-3;
  const int32_t hx = __double2hiint(x), ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0, u;
  if (hx < 0x3fda827a) {  // 1+x < sqrt(2)+
    if (ax >= 0x3ff00000) {  // x <= -1.0
      if (x == -1.0) return -two54 / 0.0;
      return (x - x) / (x - x);
    }
    if (ax < 0x3e200000) {  // |x| < 2**-29
      if (ax < 0x3c900000) return x;
      return __fma_rn(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= static_cast<int32_t>(0xbfd2bec3u)) {  // sqrt(2)/2- <= 1+x < sqrt(2)+
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c = c / u;
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = with_hi(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = (0.5 * f) * f;
  const double dk = static_cast<double>(k);
  if (hu == 0) {  // |f| < 2**-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
    }
    const double R = __fma_rn(-f, 0x1.5555555555555p-1, 1.0) * hfsq;
    if (k == 0) return f - R;
    return __fma_rn(dk, ln2_hi, -((R - __fma_rn(dk, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f), z = s * s;
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double z2 = z * z, z4 = z2 * z2, z6 = z2 * z4;
  double R = __fma_rn(z, Lp1, R2 * z2);
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double t = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - t);
  return __fma_rn(dk, ln2_hi, -((hfsq - (__fma_rn(dk, ln2_lo, c) + t)) - f));
}

// Exp(1)/w of draw t of the parent's stream (sampler.cpp:43-44), as the bit
// pattern of the non-negative double (order-preserving); kNoKey for w <= 0.
__device__ __forceinline__ uint64_t sample_key(uint64_t state, uint64_t t, double w) {
  const double e = -glibc_log1p(-to_uniform(stream_draw(state, t)));
  if (!(w > 0.0)) return kNoKey;
  return static_cast<uint64_t>(__double_as_longlong(w == 1.0 ? e : e / w));  // e/1.0 == e
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- sampler build --------------------------------------------------------
// key = row << 32 | column for every edge (one warp per row).
__global__ void k_edge_keys(const uint64_t* __restrict__ ro, const uint32_t* __restrict__ col,
                            uint64_t n, uint64_t* __restrict__ keys, uint32_t* __restrict__ iota) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t i = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); i < n;
       i += warps) {
    const uint64_t a = ro[i], b = ro[i + 1];
    for (uint64_t q = a + lane; q < b; q += 32) {
      keys[q] = (i << 32) | col[q];
      iota[q] = static_cast<uint32_t>(q);
    }
  }
}

// Heads of equal (row, column) runs in the stably sorted edge list: the
// head is the neighbour's first occurrence; its weight is the run summed in
// CSR order (sampler.cpp:80-89: w[first], then += w[later]).
__global__ void k_mark_heads(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx,
                             const double* __restrict__ w, uint64_t e, uint8_t* __restrict__ first,
                             double* __restrict__ wsum, unsigned long long* __restrict__ dups) {
  uint32_t local = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = skeys[i];
    if (i > 0 && skeys[i - 1] == key) {
      ++local;
      continue;
    }
    const uint32_t q0 = sidx[i];
    double sum = w ? w[q0] : 1.0;
    for (uint64_t j = i + 1; j < e && skeys[j] == key; ++j) sum = __dadd_rn(sum, w ? w[sidx[j]] : 1.0);
    first[q0] = 1;
    wsum[q0] = sum;
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(dups, (unsigned long long)local);
}

__global__ void k_compact_candidates(const uint8_t* __restrict__ first,
                                     const uint32_t* __restrict__ pos,
                                     const uint32_t* __restrict__ col,
                                     const double* __restrict__ wsum, uint64_t e,
                                     uint32_t* __restrict__ ccol, double* __restrict__ cw) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < e;
       q += (uint64_t)gridDim.x * blockDim.x) {
    if (!first[q]) continue;
    ccol[pos[q]] = col[q];
    cw[pos[q]] = wsum[q];
  }
}

__global__ void k_candidate_rows(const uint64_t* __restrict__ ro, const uint32_t* __restrict__ pos,
                                 uint64_t n, uint64_t* __restrict__ cro) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
       i += (uint64_t)gridDim.x * blockDim.x)
    cro[i] = pos[ro[i]];
}

// cpos = positive candidates per row; the all-zero-weights row check of
// Graph::validate (graph.cpp:76,86-91); the longest row.
__global__ void k_row_stats(const uint64_t* __restrict__ cro, const double* __restrict__ cw,
                            uint64_t n, uint32_t* __restrict__ cpos,
                            unsigned long long* __restrict__ bad_zero,
                            unsigned long long* __restrict__ max_len) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t i = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); i < n;
       i += warps) {
    const uint64_t a = cro[i], b = cro[i + 1];
    uint32_t cnt = 0;
    if (cw) {
      for (uint64_t q = a + lane; q < b; q += 32) cnt += cw[q] > 0.0;
      cnt = __reduce_add_sync(0xffffffffu, cnt);
    } else {
      cnt = static_cast<uint32_t>(b - a);
    }
    if (lane == 0) {
      cpos[i] = cnt;
      if (b > a && cnt == 0) atomicMin(bad_zero, (unsigned long long)i);
      if (b > a) atomicMax(max_len, (unsigned long long)(b - a));
    }
  }
}

// ---- one hop --------------------------------------------------------------
__global__ void k_hop_count(const uint32_t* __restrict__ pn, const uint64_t* __restrict__ Pp, uint64_t ub,
                            uint32_t fanout, const uint64_t* __restrict__ cro,
                            const uint32_t* __restrict__ cpos, uint32_t* __restrict__ m_out,
                            uint32_t* __restrict__ large, unsigned long long* __restrict__ nlarge) {
  // entries [P, ub] are 0, so the scan over ub + 1 entries ends in the total
  const uint64_t P = *Pp;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= ub;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i >= P) {
      m_out[i] = 0;
      continue;
    }
    const uint32_t p = pn[i];
    const uint32_t pos = cpos[p];
    const uint32_t m = pos < fanout ? pos : fanout;
    m_out[i] = m;
    if (m > 0 && m < pos && cro[p + 1] - cro[p] > kRegMax)
      large[atomicAdd(nlarge, 1ull)] = static_cast<uint32_t>(i);
  }
}

struct HopArgs {
  const uint32_t* pn;  // parents: node, seed slot
  const uint32_t* ps;
  const uint64_t* P;  // parent count (device: the previous frontier's size)
  const uint64_t* ss_prev;  // seed starts of the parents' frontier
  const uint64_t* O;        // child offsets
  // derive_prefix(splitmix64(rng ^ seed*gamma), hop) per seed: the part of
  // sample_khop's derive_stream(rs, k, idx, p) (sampler.cpp:94, :136) shared
  // by every parent of the seed at this hop
  const uint64_t* hop_state;
  uint32_t hop, fanout;
  const uint64_t* cro;
  const uint32_t* ccol;
  const double* cw;
  const uint32_t* cpos;
  uint32_t* cn;  // children: node, seed slot
  uint32_t* cs;
};

// Finds the m-th smallest key (1-based) among the keys `each` visits: 8-bit
// digits from the top, one shared 256-bin histogram per warp. Returns the
// threshold T and how many keys == T (in candidate order) belong to the m.
// Stops early once the digit's whole bin is selected: then T = prefix with
// all lower bits set and every key <= T is taken (take_eq = all).
template <typename Each>
__device__ __forceinline__ void radix_select(Each&& each, uint32_t m, uint32_t* hist, uint64_t& T,
                                             uint32_t& take_eq) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t prefix = 0, mask = 0;
  uint32_t need = m;
#pragma unroll 1
  for (int shift = 56; shift >= 0; shift -= 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) hist[lane * 8 + j] = 0;
    __syncwarp();
    each([&](uint64_t key, bool in) {
      if (in && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
    });
    __syncwarp();
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = hist[lane * 8 + j];
      sum += c[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t excl = incl - sum;
    const uint32_t owner = __ffs(__ballot_sync(0xffffffffu, excl < need && need <= incl)) - 1;
    uint32_t digit = 0, below = excl, bin = 0;
    if (lane == owner) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (below + c[j] >= need) {
          digit = lane * 8 + j;
          bin = c[j];
          break;
        }
        below += c[j];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, owner);
    below = __shfl_sync(0xffffffffu, below, owner);
    bin = __shfl_sync(0xffffffffu, bin, owner);
    need -= below;
    prefix |= static_cast<uint64_t>(digit) << shift;
    mask |= 0xFFull << shift;
    __syncwarp();
    if (bin == need) {  // the whole bin is in: keys <= prefix|~mask
      T = prefix | ~mask;
      take_eq = 0xFFFFFFFFu;
      return;
    }
  }
  T = prefix;
  take_eq = need;
}

// Writes the selected candidates (key < T, or == T among the first take_eq)
// in candidate order; `each` visits warp-uniform rounds of 32 candidates.
template <typename Each>
__device__ __forceinline__ void emit_selected(Each&& each, uint64_t T, uint32_t take_eq,
                                              const uint32_t* __restrict__ col, uint32_t s,
                                              uint32_t* __restrict__ cn, uint32_t* __restrict__ cs,
                                              uint64_t out) {
  const uint32_t lt_mask = lanemask_lt();
  uint32_t eq_seen = 0;
  each([&](uint64_t key, bool in, uint32_t t) {
    const bool eq = in && key == T;
    const uint32_t eqm = __ballot_sync(0xffffffffu, eq);
    const bool sel = (in && key < T) || (eq && eq_seen + __popc(eqm & lt_mask) < take_eq);
    const uint32_t selm = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const uint64_t at = out + __popc(selm & lt_mask);
      cn[at] = col[t];
      cs[at] = s;
    }
    out += __popc(selm);
    eq_seen += __popc(eqm);
  });
}

// One warp per parent (rows <= 256 candidates; longer selecting rows are
// left to k_hop_sample_large).
__global__ void __launch_bounds__(kBlock) k_hop_sample(HopArgs a) {
  __shared__ uint32_t hist_all[kWarpsPerBlock][256];
  uint32_t* hist = hist_all[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt_mask = lanemask_lt();
  const uint64_t warps = (uint64_t)gridDim.x * kWarpsPerBlock;
  const uint64_t P = *a.P;
  for (uint64_t i = blockIdx.x * (uint64_t)kWarpsPerBlock + (threadIdx.x >> 5); i < P;
       i += warps) {
    const uint32_t p = a.pn[i], s = a.ps[i];
    const uint64_t c0 = a.cro[p];
    const uint32_t L = static_cast<uint32_t>(a.cro[p + 1] - c0);
    const uint32_t pos = a.cpos[p];
    const uint32_t m = pos < a.fanout ? pos : a.fanout;
    uint64_t out = a.O[i];
    const uint32_t* col = a.ccol + c0;
    const double* w = a.cw ? a.cw + c0 : nullptr;
    if (m == 0) continue;
    if (m == pos) {  // every positive candidate, in order (sampler.cpp:30-36)
      for (uint32_t base = 0; base < L; base += 32) {
        const uint32_t t = base + lane;
        const bool take = t < L && (!w || w[t] > 0.0);
        const uint32_t tm = __ballot_sync(0xffffffffu, take);
        if (take) {
          const uint64_t at = out + __popc(tm & lt_mask);
          a.cn[at] = col[t];
          a.cs[at] = s;
        }
        out += __popc(tm);
      }
      continue;
    }
    if (L > kRegMax) continue;  // k_hop_sample_large
    const uint64_t state =
        derive_finish(a.hop_state[s], i - a.ss_prev[s], p);
    if (L <= 32) {
      // rank of (key, idx) among the row's keys; the m smallest are chosen
      const bool in = lane < L;
      const uint64_t key = in ? sample_key(state, lane, w ? w[lane] : 1.0) : kNoKey;
      // Rank by the high words; only when two valid keys share a high word
      // (rare: exponent and 20 mantissa bits equal) compare all 64 bits.
      const uint32_t hi = static_cast<uint32_t>(key >> 32);
      const uint32_t same_hi = __match_any_sync(0xffffffffu, hi);  // all lanes take part
      const bool tie = key != kNoKey && __popc(same_hi) > 1;
      uint32_t rank = 0;
      if (!__any_sync(0xffffffffu, tie)) {
        for (uint32_t u = 0; u < L; ++u) rank += __shfl_sync(0xffffffffu, hi, u) < hi;
      } else {
        for (uint32_t u = 0; u < L; ++u) {
          const uint64_t ku = __shfl_sync(0xffffffffu, key, u);
          rank += (ku < key) || (ku == key && u < lane);
        }
      }
      const bool sel = in && key != kNoKey && rank < m;
      const uint32_t selm = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const uint64_t at = out + __popc(selm & lt_mask);
        a.cn[at] = col[lane];
        a.cs[at] = s;
      }
      continue;
    }
    uint64_t k[kRegRounds];
#pragma unroll
    for (int r = 0; r < kRegRounds; ++r) {
      const uint32_t t = r * 32 + lane;
      k[r] = t < L ? sample_key(state, t, w ? w[t] : 1.0) : kNoKey;
    }
    const uint32_t rounds = (L + 31) / 32;
    uint64_t T;
    uint32_t take_eq;
    radix_select(
        [&](auto&& f) {
#pragma unroll
          for (int r = 0; r < kRegRounds; ++r)
            if (r < rounds) f(k[r], r * 32 + lane < L);
        },
        m, hist, T, take_eq);
    emit_selected(
        [&](auto&& f) {
#pragma unroll
          for (int r = 0; r < kRegRounds; ++r)
            if (r < rounds) f(k[r], r * 32 + lane < L, r * 32 + lane);
        },
        T, take_eq, col, s, a.cn, a.cs, out);
  }
}

// Selecting parents with more than 256 candidates: one CTA per parent, keys
// staged in the CTA's scratch slab (max_len keys), then the radix select of
// radix_select with a block-wide histogram, and the emit in candidate order
// with block-wide ballot prefixes.
__global__ void __launch_bounds__(kBlock)
    k_hop_sample_large(HopArgs a, const uint32_t* __restrict__ large,
                       const unsigned long long* __restrict__ nlarge,
                       uint64_t* __restrict__ scratch, uint64_t slab) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t wsum[kWarpsPerBlock];
  __shared__ uint32_t wsel[kWarpsPerBlock], weq[kWarpsPerBlock];
  __shared__ uint32_t s_digit, s_below, s_bin;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = lanemask_lt();
  uint64_t* K = scratch + blockIdx.x * slab;
  const uint64_t count = *nlarge;
  for (uint64_t j = blockIdx.x; j < count; j += gridDim.x) {
    const uint64_t i = large[j];
    const uint32_t p = a.pn[i], s = a.ps[i];
    const uint64_t c0 = a.cro[p];
    const uint32_t L = static_cast<uint32_t>(a.cro[p + 1] - c0);
    const uint32_t pos = a.cpos[p];
    const uint32_t m = pos < a.fanout ? pos : a.fanout;
    const uint32_t* col = a.ccol + c0;
    const double* w = a.cw ? a.cw + c0 : nullptr;
    const uint64_t state = derive_finish(a.hop_state[s], i - a.ss_prev[s], p);
    for (uint32_t t = tid; t < L; t += kBlock) K[t] = sample_key(state, t, w ? w[t] : 1.0);
    // radix select (see radix_select), block-wide
    uint64_t prefix = 0, mask = 0, T = 0;
    uint32_t need = m, take_eq = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
      hist[tid] = 0;  // kBlock == 256 bins
      __syncthreads();
      for (uint32_t t = tid; t < L; t += kBlock) {
        const uint64_t key = K[t];
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
      }
      __syncthreads();
      const uint32_t c = hist[tid];
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      uint32_t before = 0;
      for (uint32_t x = 0; x < warp; ++x) before += wsum[x];
      incl += before;
      if (incl - c < need && need <= incl) {
        s_digit = tid;
        s_below = incl - c;
        s_bin = c;
      }
      __syncthreads();
      need -= s_below;
      prefix |= static_cast<uint64_t>(s_digit) << shift;
      mask |= 0xFFull << shift;
      const uint32_t bin = s_bin;
      __syncthreads();  // s_* and wsum reused next pass
      if (bin == need) {
        T = prefix | ~mask;
        take_eq = 0xFFFFFFFFu;
        break;
      }
      T = prefix;
      take_eq = need;
    }
    // emit in candidate order: rounds of kBlock candidates
    uint64_t out = a.O[i];
    uint32_t eq_seen = 0;
    for (uint32_t base = 0; base < L; base += kBlock) {
      const uint32_t t = base + tid;
      const uint64_t key = t < L ? K[t] : kNoKey;
      const bool in = t < L;
      const bool eq = in && key == T;
      const uint32_t eqm = __ballot_sync(0xffffffffu, eq);
      if (lane == 0) weq[warp] = __popc(eqm);
      __syncthreads();
      uint32_t eq_before = eq_seen, eq_round = 0;
      for (uint32_t x = 0; x < kWarpsPerBlock; ++x) {
        if (x < warp) eq_before += weq[x];
        eq_round += weq[x];
      }
      const bool sel = (in && key < T) || (eq && eq_before + __popc(eqm & lt_mask) < take_eq);
      const uint32_t selm = __ballot_sync(0xffffffffu, sel);
      if (lane == 0) wsel[warp] = __popc(selm);
      __syncthreads();
      uint64_t sel_before = out, sel_round = 0;
      for (uint32_t x = 0; x < kWarpsPerBlock; ++x) {
        if (x < warp) sel_before += wsel[x];
        sel_round += wsel[x];
      }
      if (sel) {
        const uint64_t at = sel_before + __popc(selm & lt_mask);
        a.cn[at] = col[t];
        a.cs[at] = s;
      }
      out += sel_round;
      eq_seen += eq_round;
      __syncthreads();  // weq/wsel reused next round
    }
  }
}

__global__ void k_seed_starts(const uint64_t* __restrict__ ss_prev, const uint64_t* __restrict__ O,
                              uint64_t nseeds, uint64_t* __restrict__ ss,
                              const uint64_t* __restrict__ seeds, uint64_t rng_seed, uint32_t hop,
                              uint64_t* __restrict__ hop_state) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s <= nseeds;
       s += (uint64_t)gridDim.x * blockDim.x) {
    ss[s] = O[ss_prev[s]];
    if (s < nseeds) hop_state[s] = derive_prefix(splitmix64(rng_seed ^ (seeds[s] * kGamma)), hop);
  }
}

__global__ void k_hop0(const uint64_t* __restrict__ seeds, uint64_t nseeds, uint32_t* __restrict__ pn,
                       uint32_t* __restrict__ ps, uint64_t* __restrict__ ss) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s <= nseeds;
       s += (uint64_t)gridDim.x * blockDim.x) {
    ss[s] = s;
    if (s < nseeds) {
      pn[s] = static_cast<uint32_t>(seeds[s]);
      ps[s] = static_cast<uint32_t>(s);
    }
  }
}

__global__ void k_check_seeds(const uint64_t* __restrict__ seeds, uint64_t nseeds, uint64_t n,
                              unsigned long long* __restrict__ bad) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nseeds;
       s += (uint64_t)gridDim.x * blockDim.x)
    if (seeds[s] >= n) atomicMin(bad, (unsigned long long)s);
}

// instance_counts per (seed, hop), seed-major; entry nseeds*(H+1) = 0.
__global__ void k_instance_counts(const uint64_t* __restrict__ ss, uint64_t nseeds, uint32_t H,
                                  uint32_t* __restrict__ cnt) {
  const uint64_t total = nseeds * (H + 1);
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x <= total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    if (x == total) {
      cnt[x] = 0;
      continue;
    }
    const uint64_t s = x / (H + 1), k = x % (H + 1);
    const uint64_t* sk = ss + k * (nseeds + 1);
    cnt[x] = static_cast<uint32_t>(sk[s + 1] - sk[s]);
  }
}

// Frontier k -> flattened seed-major/hop-major position; marks the bitmap.
__global__ void k_flatten(const uint32_t* __restrict__ fn, const uint32_t* __restrict__ fs,
                          const uint64_t* __restrict__ countp, const uint64_t* __restrict__ ssk,
                          const uint64_t* __restrict__ flat_off, uint32_t H, uint32_t k,
                          uint64_t* __restrict__ nodes, uint32_t* __restrict__ bitmap) {
  const uint64_t count = *countp;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = fn[j], s = fs[j];
    nodes[flat_off[(uint64_t)s * (H + 1) + k] + (j - ssk[s])] = v;
    atomicOr(&bitmap[v >> 5], 1u << (v & 31));
  }
}

__global__ void k_widen(const uint32_t* __restrict__ in, uint64_t count, uint64_t* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = in[j];
}

__global__ void k_popc_words(const uint32_t* __restrict__ bitmap, uint64_t words,
                             uint32_t* __restrict__ pc) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= words;
       j += (uint64_t)gridDim.x * blockDim.x)
    pc[j] = j < words ? __popc(bitmap[j]) : 0u;
}

__global__ void k_emit_unique(const uint32_t* __restrict__ bitmap, uint64_t words,
                              const uint64_t* __restrict__ off, uint64_t* __restrict__ unique) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < words;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = bitmap[j];
    uint64_t at = off[j];
    while (b) {
      const int bit = __ffs(b) - 1;
      unique[at++] = j * 32 + bit;
      b &= b - 1;
    }
  }
}

__global__ void k_log1p(const double* __restrict__ x, uint64_t n, double* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = glibc_log1p(x[j]);
}

template <typename T>
T* persist(DevBuf<T>& b) {
  return b.release_ownership();
}

unsigned warp_grid(uint64_t items) { return grid_for(items * 32, kBlock); }

// Candidate rows from a device out-CSR (takes ownership of ro/col/w).
void build_candidates(qvb_sampler& sp, DevBuf<uint64_t>& ro, DevBuf<uint32_t>& col,
                      DevBuf<double>& w, cudaStream_t s) {
  const uint64_t n = sp.n, e = sp.e;
  DevBuf<unsigned long long> flags(3, s);  // dups, bad_zero, max_len
  QVB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(unsigned long long), s));
  QVB_CUDA(cudaMemsetAsync(flags.p + 1, 0xFF, sizeof(unsigned long long), s));
  QVB_CUDA(cudaMemsetAsync(flags.p + 2, 0, sizeof(unsigned long long), s));
  uint64_t dups = 0;
  DevBuf<uint8_t> first;
  DevBuf<double> wsum;
  if (e) {
    DevBuf<uint64_t> keys(e, s), skeys(e, s);
    DevBuf<uint32_t> iota(e, s), sidx(e, s);
    k_edge_keys<<<warp_grid(n), kBlock, 0, s>>>(ro.p, col.p, n, keys.p, iota.p);
    QVB_LAUNCH_CHECK();
    sort_pairs_u64_u32(keys.p, skeys.p, iota.p, sidx.p, e, 0, 32 + bits_for(n - 1), s);
    keys.release();
    iota.release();
    first.alloc(e + 1, s);
    wsum.alloc(e, s);
    QVB_CUDA(cudaMemsetAsync(first.p, 0, e + 1, s));
    k_mark_heads<<<grid_for(e, kBlock), kBlock, 0, s>>>(skeys.p, sidx.p, w.p, e, first.p, wsum.p,
                                                        flags.p);
    QVB_LAUNCH_CHECK();
    dups = read_scalar(flags.p, s);
  }
  sp.parallel = dups > 0;
  if (sp.parallel) {
    DevBuf<uint32_t> pos(e + 1, s);
    exclusive_sum_u8_u32(first.p, pos.p, e + 1, s);
    sp.ncand = e - dups;
    DevBuf<uint32_t> ccol(sp.ncand, s);
    DevBuf<double> cw(sp.ncand, s);
    DevBuf<uint64_t> cro(n + 1, s);
    k_compact_candidates<<<grid_for(e, kBlock), kBlock, 0, s>>>(first.p, pos.p, col.p, wsum.p, e,
                                                                ccol.p, cw.p);
    QVB_LAUNCH_CHECK();
    k_candidate_rows<<<grid_for(n + 1, kBlock), kBlock, 0, s>>>(ro.p, pos.p, n, cro.p);
    QVB_LAUNCH_CHECK();
    sp.cro = persist(cro);
    sp.ccol = persist(ccol);
    sp.cw = persist(cw);
  } else {
    sp.ncand = e;
    sp.cro = persist(ro);
    sp.ccol = persist(col);
    sp.cw = w.p ? persist(w) : nullptr;
  }
  first.release();
  wsum.release();
  DevBuf<uint32_t> cpos(n, s);
  k_row_stats<<<warp_grid(n), kBlock, 0, s>>>(sp.cro, sp.cw, n, cpos.p, flags.p + 1, flags.p + 2);
  QVB_LAUNCH_CHECK();
  unsigned long long st[3];
  QVB_CUDA(cudaMemcpyAsync(st, flags.p, sizeof st, cudaMemcpyDeviceToHost, s));
  QVB_CUDA(cudaStreamSynchronize(s));
  if (st[1] != ~0ull)
    fail(QVB_ERR_VALIDATION, "node " + std::to_string(st[1]) +
                                 " has out-edges but all weights are zero");
  sp.cpos = persist(cpos);
  sp.max_len = st[2];
  if (sp.max_len > kRegMax) {
    const uint64_t slab_bytes = sp.max_len * sizeof(uint64_t);
    uint64_t ctas = std::max<uint64_t>(1, kScratchBudget / slab_bytes);
    ctas = std::min<uint64_t>(ctas, 148ull * 4);
    sp.large_ctas = static_cast<uint32_t>(ctas);
    QVB_CUDA(cudaMalloc(&sp.scratch, ctas * slab_bytes));
    QVB_CUDA(cudaStreamCreateWithFlags(&sp.side, cudaStreamNonBlocking));
  }
  sp.bytes = (n + 1) * 8 + sp.ncand * (4 + (sp.cw ? 8 : 0)) + n * 4 +
             sp.large_ctas * sp.max_len * 8;
}

uint64_t* to_device_owned(DevBuf<uint64_t>& b) { return b.release_ownership(); }

}  // namespace
}  // namespace qvb

using namespace qvb;

namespace {

template <typename Build>
int make_sampler(int device, uint64_t n, uint64_t e, void* stream, qvb_sampler** out, Build&& build) {
  return guarded([&] {
    if (!out) fail(QVB_ERR_VALIDATION, "out is null");
    *out = nullptr;
    if (n == 0) fail(QVB_ERR_VALIDATION, "empty graph: node count is zero");
    if (n > kMaxNodes || e > kMaxEdges)
      fail(QVB_ERR_UNSUPPORTED, "graph exceeds the device path limits (n < 2^30, e < 2^32)");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto sp = std::make_unique<qvb_sampler>();
    sp->device = device;
    sp->n = n;
    sp->e = e;
    cudaEvent_t ea, eb;
    QVB_CUDA(cudaEventCreate(&ea));
    QVB_CUDA(cudaEventCreate(&eb));
    QVB_CUDA(cudaEventRecord(ea, s));
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> col;
    DevBuf<double> w;
    build(s, ro, col, w);
    build_candidates(*sp, ro, col, w, s);
    QVB_CUDA(cudaEventRecord(eb, s));
    QVB_CUDA(cudaEventSynchronize(eb));
    float ms = 0;
    QVB_CUDA(cudaEventElapsedTime(&ms, ea, eb));
    sp->build_ms = ms;
    cudaEventDestroy(ea);
    cudaEventDestroy(eb);
    *out = sp.release();
  });
}

}  // namespace

extern "C" int qvb_sampler_create(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                                  const uint64_t* col, const double* weights, void* stream,
                                  qvb_sampler** out) {
  return make_sampler(device, n, e, stream, out,
                      [&](cudaStream_t s, DevBuf<uint64_t>& ro, DevBuf<uint32_t>& dcol,
                          DevBuf<double>& dw) {
                        upload_out_csr(n, e, row_offsets, col, weights, s, ro, dcol, dw);
                      });
}

extern "C" int qvb_sampler_synthetic(int device, uint64_t n, uint64_t e, uint64_t seed,
                                     int weighted, int transposed, void* stream,
                                     qvb_sampler** out) {
  return make_sampler(device, n, e, stream, out,
                      [&](cudaStream_t s, DevBuf<uint64_t>& ro, DevBuf<uint32_t>& col,
                          DevBuf<double>& w) {
                        DevBuf<uint32_t> ssrc;
                        generate_out_csr(n, e, seed, weighted, transposed, s, ro, col, w, ssrc);
                      });
}

extern "C" int qvb_sampler_info_get(const qvb_sampler* sp, qvb_sampler_info* info) {
  return guarded([&] {
    if (!sp || !info) fail(QVB_ERR_VALIDATION, "null argument");
    info->node_count = sp->n;
    info->edge_count = sp->e;
    info->candidates = sp->ncand;
    info->parallel_edges = sp->parallel ? 1 : 0;
    info->unit_weights = sp->cw ? 0 : 1;
    info->max_candidates = sp->max_len;
    info->device_bytes = sp->bytes;
    info->build_ms = sp->build_ms;
  });
}

extern "C" int qvb_sampler_destroy(qvb_sampler* sp) {
  delete sp;
  return QVB_OK;
}

extern "C" int qvb_batch_sample(qvb_sampler* sp, const uint64_t* seeds, uint64_t nseeds,
                                int seeds_on_device, const uint32_t* fanouts, uint32_t hops,
                                uint64_t rng_seed, void* stream, qvb_sample** out) {
  return guarded([&] {
    if (!sp || !out) fail(QVB_ERR_VALIDATION, "null argument");
    *out = nullptr;
    // SamplingConfig::validate (metrics.cpp:13-18)
    if (hops == 0 || !fanouts) fail(QVB_ERR_VALIDATION, "sampling config needs >= 1 hop");
    for (uint32_t k = 0; k < hops; ++k)
      if (fanouts[k] < 1) fail(QVB_ERR_VALIDATION, "fanouts must be >= 1");
    if (nseeds && !seeds) fail(QVB_ERR_VALIDATION, "seeds is null");
    if (nseeds >= 0xFFFFFFFFull) fail(QVB_ERR_UNSUPPORTED, "too many seeds for one batch");
    // batch_sample's range check (sampler.cpp:119-125), host seeds
    if (!seeds_on_device)
      for (uint64_t i = 0; i < nseeds; ++i)
        if (seeds[i] >= sp->n)
          fail(QVB_ERR_VALIDATION, "batch seed at position " + std::to_string(i) + " (node " +
                                       std::to_string(seeds[i]) + ") out of range");
    DeviceGuard dg(sp->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(sp->mu);
    auto r = std::make_unique<qvb_sample>();
    r->device = sp->device;
    r->nseeds = nseeds;
    r->hops = hops;
    const uint32_t H = hops;
    DevBuf<uint64_t> dseeds(nseeds ? nseeds : 1, s);
    if (nseeds) {
      if (seeds_on_device) {
        QVB_CUDA(cudaMemcpyAsync(dseeds.p, seeds, nseeds * 8, cudaMemcpyDeviceToDevice, s));
        DevBuf<unsigned long long> bad(1, s);
        QVB_CUDA(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
        k_check_seeds<<<grid_for(nseeds, kBlock), kBlock, 0, s>>>(dseeds.p, nseeds, sp->n, bad.p);
        QVB_LAUNCH_CHECK();
        const unsigned long long b = read_scalar(bad.p, s);
        if (b != ~0ull) {
          const uint64_t node = read_scalar(dseeds.p + b, s);
          fail(QVB_ERR_VALIDATION, "batch seed at position " + std::to_string(b) + " (node " +
                                       std::to_string(node) + ") out of range");
        }
      } else {
        QVB_CUDA(cudaMemcpyAsync(dseeds.p, seeds, nseeds * 8, cudaMemcpyHostToDevice, s));
      }
    }
    cudaEvent_t ea, eb, fork, join;
    QVB_CUDA(cudaEventCreate(&ea));
    QVB_CUDA(cudaEventCreate(&eb));
    QVB_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    QVB_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    struct Events {
      cudaEvent_t* e[4];
      ~Events() {
        for (auto* x : e) cudaEventDestroy(*x);
      }
    } events{{&ea, &eb, &fork, &join}};
    QVB_CUDA(cudaEventRecord(ea, s));

    // Frontier sizes live on the device (frontier k's size = its sentinel
    // seed start ss[k][nseeds]); every kernel reads them there, so the hops
    // run without host round trips when the buffers can be sized by the
    // upper bound |frontier k| <= |frontier k-1| * fanout. Past kSyncFreeMax
    // instances the exact sizes are read back per hop instead.
    constexpr uint64_t kSyncFreeMax = 1ull << 28;
    std::vector<uint64_t> ub(H + 1);
    ub[0] = nseeds;
    bool sync_free = true;
    uint64_t ub_total = nseeds;
    for (uint32_t k = 1; k <= H; ++k) {
      const uint64_t f = fanouts[k - 1];
      ub[k] = ub[k - 1] > kSyncFreeMax / f ? kSyncFreeMax + 1 : ub[k - 1] * f;
      ub_total += ub[k];
      if (ub[k] > kSyncFreeMax || ub_total > kSyncFreeMax) sync_free = false;
    }
    // seed starts of every frontier, [H+1][nseeds+1]
    DevBuf<uint64_t> ss((H + 1) * (nseeds + 1), s);
    std::vector<DevBuf<uint32_t>> fn(H + 1), fs(H + 1);
    std::vector<uint64_t> fcap(H + 1, 0);  // allocated capacity of each frontier
    fn[0].alloc(nseeds ? nseeds : 1, s);
    fs[0].alloc(nseeds ? nseeds : 1, s);
    fcap[0] = nseeds;
    k_hop0<<<grid_for(nseeds + 1, kBlock), kBlock, 0, s>>>(dseeds.p, nseeds, fn[0].p, fs[0].p, ss.p);
    QVB_LAUNCH_CHECK();
    DevBuf<unsigned long long> nlarge(1, s);
    DevBuf<uint64_t> hop_state(nseeds ? nseeds : 1, s);
    for (uint32_t k = 1; k <= H; ++k) {
      const uint64_t Pub = fcap[k - 1];  // parents: at most the previous capacity
      const uint64_t* Pd = ss.p + (uint64_t)(k - 1) * (nseeds + 1) + nseeds;
      DevBuf<uint32_t> m(Pub + 1, s), large(Pub ? Pub : 1, s);
      DevBuf<uint64_t> O(Pub + 1, s);
      QVB_CUDA(cudaMemsetAsync(nlarge.p, 0, sizeof(unsigned long long), s));
      k_hop_count<<<grid_for(Pub + 1, kBlock), kBlock, 0, s>>>(fn[k - 1].p, Pd, Pub, fanouts[k - 1], sp->cro,
                                                               sp->cpos, m.p, large.p, nlarge.p);
      QVB_LAUNCH_CHECK();
      exclusive_sum_u32_u64(m.p, O.p, Pub + 1, s);
      uint64_t* ssk = ss.p + (uint64_t)k * (nseeds + 1);
      k_seed_starts<<<grid_for(nseeds + 1, kBlock), kBlock, 0, s>>>(
          ss.p + (uint64_t)(k - 1) * (nseeds + 1), O.p, nseeds, ssk, dseeds.p, rng_seed, k,
          hop_state.p);
      QVB_LAUNCH_CHECK();
      uint64_t C = ub[k];
      if (!sync_free) {
        C = read_scalar(ssk + nseeds, s);
        if (C >= 0xFFFFFFFFull) fail(QVB_ERR_UNSUPPORTED, "frontier exceeds 2^32 instances");
      }
      fcap[k] = C;
      fn[k].alloc(C ? C : 1, s);
      fs[k].alloc(C ? C : 1, s);
      if (Pub == 0) continue;
      HopArgs a{fn[k - 1].p, fs[k - 1].p, Pd,        ss.p + (uint64_t)(k - 1) * (nseeds + 1),
                O.p,         hop_state.p, k,
                fanouts[k - 1], sp->cro,  sp->ccol,  sp->cw,
                sp->cpos,    fn[k].p,     fs[k].p};
      if (sp->scratch) {  // fork: long rows on the side stream, concurrently
        QVB_CUDA(cudaEventRecord(fork, s));
        QVB_CUDA(cudaStreamWaitEvent(sp->side, fork, 0));
        k_hop_sample_large<<<sp->large_ctas, kBlock, 0, sp->side>>>(
            a, large.p, nlarge.p, sp->scratch, sp->max_len);
        QVB_LAUNCH_CHECK();
        QVB_CUDA(cudaEventRecord(join, sp->side));
      }
      k_hop_sample<<<warp_grid(Pub), kBlock, 0, s>>>(a);
      QVB_LAUNCH_CHECK();
      if (sp->scratch) QVB_CUDA(cudaStreamWaitEvent(s, join, 0));
      // m, large and O are freed stream-ordered after this hop's kernels
    }
    // flatten: instance_counts (seed-major) -> offsets -> scatter
    const uint64_t ncounts = nseeds * (H + 1);
    DevBuf<uint32_t> cnt(ncounts + 1, s);
    DevBuf<uint64_t> flat_off(ncounts + 1, s);
    k_instance_counts<<<grid_for(ncounts + 1, kBlock), kBlock, 0, s>>>(ss.p, nseeds, H, cnt.p);
    QVB_LAUNCH_CHECK();
    exclusive_sum_u32_u64(cnt.p, flat_off.p, ncounts + 1, s);
    uint64_t cap_total = 0;
    for (uint32_t k = 0; k <= H; ++k) cap_total += fcap[k];
    DevBuf<uint64_t> nodes(cap_total ? cap_total : 1, s), counts(ncounts ? ncounts : 1, s);
    const uint64_t words = (sp->n + 31) / 32;
    DevBuf<uint32_t> bitmap(words, s), pc(words + 1, s);
    DevBuf<uint64_t> woff(words + 1, s);
    QVB_CUDA(cudaMemsetAsync(bitmap.p, 0, words * 4, s));
    for (uint32_t k = 0; k <= H; ++k) {
      if (!fcap[k]) continue;
      k_flatten<<<grid_for(fcap[k], kBlock), kBlock, 0, s>>>(
          fn[k].p, fs[k].p, ss.p + (uint64_t)k * (nseeds + 1) + nseeds, ss.p + (uint64_t)k * (nseeds + 1),
          flat_off.p, H, k, nodes.p, bitmap.p);
      QVB_LAUNCH_CHECK();
    }
    if (ncounts) {
      k_widen<<<grid_for(ncounts, kBlock), kBlock, 0, s>>>(cnt.p, ncounts, counts.p);
      QVB_LAUNCH_CHECK();
    }
    k_popc_words<<<grid_for(words + 1, kBlock), kBlock, 0, s>>>(bitmap.p, words, pc.p);
    QVB_LAUNCH_CHECK();
    exclusive_sum_u32_u64(pc.p, woff.p, words + 1, s);
    const uint64_t ucap = std::min<uint64_t>(sp->n, cap_total);
    DevBuf<uint64_t> unique(ucap ? ucap : 1, s);
    k_emit_unique<<<grid_for(words, kBlock), kBlock, 0, s>>>(bitmap.p, words, woff.p, unique.p);
    QVB_LAUNCH_CHECK();
    // the batch's two sizes (unique nodes, instances), read back once
    DevBuf<uint64_t> sizes(2, s);
    QVB_CUDA(cudaMemcpyAsync(sizes.p, woff.p + words, 8, cudaMemcpyDeviceToDevice, s));
    QVB_CUDA(cudaMemcpyAsync(sizes.p + 1, flat_off.p + ncounts, 8, cudaMemcpyDeviceToDevice, s));
    uint64_t hsz[2] = {0, 0};
    QVB_CUDA(cudaMemcpyAsync(hsz, sizes.p, sizeof hsz, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaEventRecord(eb, s));
    QVB_CUDA(cudaEventSynchronize(eb));
    float ms = 0;
    QVB_CUDA(cudaEventElapsedTime(&ms, ea, eb));
    r->ms = ms;
    r->total = hsz[1];
    r->unique_count = hsz[0];
    r->nodes = to_device_owned(nodes);
    r->counts = to_device_owned(counts);
    r->unique = to_device_owned(unique);
    *out = r.release();
  });
}

extern "C" int qvb_sample_info_get(const qvb_sample* r, qvb_sample_info* info) {
  return guarded([&] {
    if (!r || !info) fail(QVB_ERR_VALIDATION, "null argument");
    info->seeds = r->nseeds;
    info->hops = r->hops;
    info->reserved = 0;
    info->total_instances = r->total;
    info->unique_count = r->unique_count;
    info->device_ms = r->ms;
  });
}

extern "C" int qvb_sample_copy(const qvb_sample* r, uint64_t* nodes, uint64_t* counts,
                               uint64_t* unique) {
  return guarded([&] {
    if (!r) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(r->device);
    if (nodes && r->total)
      QVB_CUDA(cudaMemcpy(nodes, r->nodes, r->total * 8, cudaMemcpyDeviceToHost));
    if (counts && r->nseeds)
      QVB_CUDA(cudaMemcpy(counts, r->counts, r->nseeds * (r->hops + 1) * 8, cudaMemcpyDeviceToHost));
    if (unique && r->unique_count)
      QVB_CUDA(cudaMemcpy(unique, r->unique, r->unique_count * 8, cudaMemcpyDeviceToHost));
  });
}

extern "C" int qvb_sample_device(const qvb_sample* r, const uint64_t** nodes,
                                 const uint64_t** counts, const uint64_t** unique) {
  return guarded([&] {
    if (!r) fail(QVB_ERR_VALIDATION, "null argument");
    if (nodes) *nodes = r->nodes;
    if (counts) *counts = r->counts;
    if (unique) *unique = r->unique;
  });
}

extern "C" int qvb_sample_destroy(qvb_sample* r) {
  delete r;
  return QVB_OK;
}

extern "C" int qvb_test_log1p(int device, const double* x, uint64_t n, double* out) {
  return guarded([&] {
    DeviceGuard dg(device);
    if (!n) return;
    DevBuf<double> dx(n, nullptr), dy(n, nullptr);
    QVB_CUDA(cudaMemcpy(dx.p, x, n * 8, cudaMemcpyHostToDevice));
    k_log1p<<<grid_for(n, kBlock), kBlock>>>(dx.p, n, dy.p);
    QVB_LAUNCH_CHECK();
    QVB_CUDA(cudaMemcpy(out, dy.p, n * 8, cudaMemcpyDeviceToHost));
  });
}
