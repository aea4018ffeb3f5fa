// access_prob.cu — K1: the analytical access-probability estimator P(n,j)
// (reference metrics.cpp:134-173, compute_access_prob_ie), as a per-layer
// pull over the sliced device in-CSR of graph.cuh.
//
// Exactness. The reference multiplies a node's factors (1 - P(s,j-1)*R(s,n))
// strictly left to right in ascending source order, and its cancellation-
// prone 1 - prod makes any re-association visible at 1e-9. So a
// node's product is ONE sequential chain of __dmul_rn in the reference order;
// every op is an explicit round-to-nearest intrinsic (no FMA contraction).
//
// Regular rows: one warp per slice of 32 destination nodes, lane l owns node
// perm[32s+l]; step k reads the 32 lanes' k-th sources as one coalesced
// 128-byte line (evict-first: streamed once per sweep), gathers the 32
// operands (8 steps in flight per lane) and each lane multiplies its own
// factor into its own chain — no shared memory, no cross-lane traffic.
// Padding slots point at operand N == 0, i.e. factor 1.0, an exact identity.
//
// Compact layout: the gathered operand is y[s] = P(s,j-1) * (1/row_sum(s)),
// produced by the previous sweep's epilogue, which equals the reference's
// P(s,j-1) * (w/row_sum(s)) bit for bit whenever w/row_sum == 1/row_sum (the
// exception table covers every other edge). One 8-byte gather per edge.
// Weighted layout: factor = 1 - P(s,j-1) * R_e with R_e streamed per edge.
//
// Long rows (in-degree above the slicing threshold): one warp per row
// gathers 32 factors per step in parallel and lane 0 multiplies them in
// order (shuffled to it), so the sequential chain is the only serial part.
// Their blocks come first in the grid so these chains start immediately.
#include <chrono>
#include <cstdlib>
#include <string>
#include <vector>
#include <algorithm>

#include "graph.cuh"

namespace qvb {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kU = 8;  // sliced steps in flight per lane
constexpr int kLongU = 4;
constexpr unsigned kFull = 0xffffffffu;

// kcode of y (graph.cuh): rint(y * 2^53) while y < 2^-22, else kBigCode.
__device__ __forceinline__ uint32_t y_code(double y) {
  return y < 0x1p-22 ? static_cast<uint32_t>(__double2ull_rn(__dmul_rn(y, 0x1p53))) : kBigCode;
}

// The factor of a code J (< 2^52): 1 - J 2^-53 is a multiple of 2^-53 in
// (1/2, 1], so it is exact, and its bit pattern is 1.0's minus J — one
// integer subtraction instead of a conversion and an FMA.
__device__ __forceinline__ double code_to_factor(uint32_t J) {
  double f;  // {lo, hi} = {-J, 0x3FF00000 - borrow}
  asm("{\n .reg .u32 lo, hi;\n sub.cc.u32 lo, 0, %1;\n subc.u32 hi, 1072693248, 0;\n"
      " mov.b64 %0, {lo, hi};\n}"
      : "=d"(f)
      : "r"(J));
  return f;
}

// The same factor from its low word L = -J mod 2^32 (the form k_codes
// stores): J in [1, 2^32) has high word 0x3FEFFFFF, J = 0 is 1.0 exactly.
__device__ __forceinline__ double low_to_factor(uint32_t L) {
  return __hiloint2double(L ? 0x3FEFFFFF : 0x3FF00000, static_cast<int>(L));
}

// Inclusive warp scan of x: shfl.up's validity predicate guards the add
// (two instructions a step instead of shuffle + lane test + select + add).
template <int O>
__device__ __forceinline__ void scan_step(uint32_t& x) {
  asm("{\n .reg .pred p;\n .reg .u32 t;\n shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n"
      " @p add.u32 %0, %0, t;\n}"
      : "+r"(x)
      : "n"(O));
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  scan_step<1>(x);
  scan_step<2>(x);
  scan_step<4>(x);
  scan_step<8>(x);
  scan_step<16>(x);
  return x;
}

__global__ void k_init(uint64_t n, const double* __restrict__ inv, double* __restrict__ p,
                       double* __restrict__ y, uint32_t* __restrict__ kc) {
  const double base = __ddiv_rn(1.0, static_cast<double>(n));  // metrics.cpp:143
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const bool real = i < n;
    p[i] = real ? base : 0.0;  // slot N: the padding operand
    const double yi = real ? __dmul_rn(base, inv[i]) : 0.0;
    if (y) y[i] = yi;
    if (kc) kc[i] = y_code(yi);
  }
}

template <bool kWeighted>
__device__ __forceinline__ double factor(uint32_t c, double v, double r,
                                         const uint32_t* __restrict__ exc_src,
                                         const double* __restrict__ exc_R,
                                         const double* __restrict__ prev) {
  if constexpr (kWeighted) {
    return __dsub_rn(1.0, __dmul_rn(v, r));  // metrics.cpp:166
  } else {
    if (c & kExcFlag) {
      const uint32_t x = c & ~kExcFlag;
      return __dsub_rn(1.0, __dmul_rn(prev[exc_src[x]], exc_R[x]));
    }
    return __dsub_rn(1.0, v);
  }
}

template <bool kWeighted>
__device__ __forceinline__ void finish(uint32_t v, double miss, const double* __restrict__ prev,
                                       const double* __restrict__ inv, double* __restrict__ out,
                                       double* __restrict__ yout, uint32_t* __restrict__ kout,
                                       uint64_t pol) {
  const double p = prev[v];
  // metrics.cpp:169: prev + (1 - prev) * (1 - miss_all)
  const double P = __dadd_rn(p, __dmul_rn(__dsub_rn(1.0, p), __dsub_rn(1.0, miss)));
  st_stream(out + v, P, pol);
  if (yout) {
    const double y = __dmul_rn(P, inv[v]);
    st_stream(yout + v, y, pol);
    if (kout) kout[v] = y_code(y);
  }
}

// Long rows: one warp per row gathers 32 factors per step in parallel and
// every lane runs the same sequential chain over them (shuffled), in order.
template <bool kWeighted>
__device__ __forceinline__ void long_row(uint64_t i, uint64_t nlong,
                                         const uint32_t* __restrict__ lnode,
                                         const uint64_t* __restrict__ lptr,
                                         const uint32_t* __restrict__ lcol,
                                         const double* __restrict__ lR,
                                         const uint32_t* __restrict__ exc_src,
                                         const double* __restrict__ exc_R,
                                         const double* __restrict__ prev,
                                         const double* __restrict__ opnd,
                                         const double* __restrict__ inv, double* __restrict__ out,
                                         double* __restrict__ yout, uint32_t* __restrict__ kout,
                                         int gmode, uint64_t pol, double fbase) {
  const int lane = threadIdx.x & 31;
  if (i >= nlong) return;
  const uint64_t a = lptr[i], b = lptr[i + 1];
  double miss = 1.0;
  for (uint64_t cs = a; cs < b; cs += 32 * kLongU) {
    double f[kLongU];
#pragma unroll
    for (int u = 0; u < kLongU; ++u) {
      const uint64_t e = cs + u * 32 + lane;
      f[u] = 1.0;
      if (e < b) {
        const uint32_t c = ld_stream(lcol + e, pol);
        const double r = kWeighted ? ld_stream(lR + e, pol) : 0.0;
        // weighted first sweep: P(s,1) = fbase for every source, no gather
        const double v = (!kWeighted && (c & kExcFlag)) ? 0.0
                         : (kWeighted && fbase != 0.0) ? fbase : ld_gather(opnd + c, gmode);
        f[u] = factor<kWeighted>(c, v, r, exc_src, exc_R, prev);
      }
    }
#pragma unroll
    for (int u = 0; u < kLongU; ++u) {
      const uint64_t base = cs + u * 32;
      const int cnt = b > base ? static_cast<int>(b - base < 32 ? b - base : 32) : 0;
      for (int j = 0; j < cnt; ++j) {
        const double x = __shfl_sync(kFull, f[u], j);
        miss = __dmul_rn(miss, x);  // every lane runs the same chain; lane 0 writes
      }
    }
  }
  if (lane == 0) finish<kWeighted>(lnode[i], miss, prev, inv, out, yout, kout, pol);
}

// One bulk L2 prefetch of [p, p + bytes) (16-byte granules).
__device__ __forceinline__ void prefetch_l2(const void* p, uint64_t bytes) {
  uint64_t a = reinterpret_cast<uint64_t>(p) & ~15ull;
  uint64_t end = (reinterpret_cast<uint64_t>(p) + bytes + 15) & ~15ull;
  while (a < end) {
    const uint32_t chunk = static_cast<uint32_t>(end - a < (1u << 16) ? end - a : (1u << 16));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(chunk) : "memory");
    a += chunk;
  }
}

// Stream lookahead for the sliced passes: blocks run roughly in launch order,
// so the block `pf` launches ahead gets its perm words and slice pointers
// pulled into L2 now, and the block pf/2 ahead its column (and R) stream —
// whose pointers were prefetched pf/2 blocks ago. The dependent
// perm/sptr -> columns -> operand chain of a new warp then starts from L2
// instead of DRAM.
template <bool kWeighted>
__device__ __forceinline__ void prefetch_ahead(uint64_t s_block, uint64_t pf, uint64_t s_end,
                                               const uint32_t* __restrict__ perm,
                                               const uint64_t* __restrict__ sptr,
                                               const uint32_t* __restrict__ scol,
                                               const double* __restrict__ sR) {
  const uint64_t sp = s_block + pf * kWarpsPerBlock;
  if (sp < s_end) {
    const uint64_t cnt = s_end - sp < kWarpsPerBlock ? s_end - sp : kWarpsPerBlock;
    prefetch_l2(perm + sp * 32, cnt * 32 * sizeof(uint32_t));
    prefetch_l2(sptr + sp, (cnt + 1) * sizeof(uint64_t));
  }
  const uint64_t sc = s_block + (pf / 2) * kWarpsPerBlock;
  if (sc < s_end) {
    const uint64_t ce = sc + kWarpsPerBlock < s_end ? sc + kWarpsPerBlock : s_end;
    const uint64_t a = sptr[sc], b = sptr[ce];
    if (b > a) {
      prefetch_l2(scol + a, (b - a) * sizeof(uint32_t));
      if constexpr (kWeighted) prefetch_l2(sR + a, (b - a) * sizeof(double));
    }
  }
}

template <bool kWeighted>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_sweep(uint64_t s0, uint64_t s1, uint64_t long_blocks, uint64_t nlong, uint64_t pf,
            uint64_t s_end, double* __restrict__ state,
            const uint32_t* __restrict__ perm, const uint64_t* __restrict__ sptr,
            const uint32_t* __restrict__ scol, const double* __restrict__ sR,
            const uint32_t* __restrict__ lnode, const uint64_t* __restrict__ lptr,
            const uint32_t* __restrict__ lcol, const double* __restrict__ lR,
            const uint32_t* __restrict__ exc_src, const double* __restrict__ exc_R,
            const double* __restrict__ prev, const double* __restrict__ yprev,
            const double* __restrict__ inv, double* __restrict__ out, double* __restrict__ yout,
            int gmode, double fbase) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  // kWeighted gathers P(s, j-1) (the first sweep: fbase = P(s,1) for every s);
  // compact gathers y(s, j-1)
  const double* __restrict__ opnd = kWeighted ? prev : yprev;

  if (blockIdx.x < long_blocks) {  // ---- long rows: one warp per row
    long_row<kWeighted>((uint64_t)blockIdx.x * kWarpsPerBlock + wib, nlong, lnode, lptr, lcol, lR,
                        exc_src, exc_R, prev, opnd, inv, out, yout, nullptr, gmode, pol, fbase);
    return;
  }

  // ---- sliced rows: one warp per slice of 32 (node, pass) slots
  const uint64_t s_block = s0 + ((uint64_t)blockIdx.x - long_blocks) * kWarpsPerBlock;
  const uint64_t s = s_block + wib;
  if (pf && wib == kWarpsPerBlock - 1 && lane == 0)
    prefetch_ahead<kWeighted>(s_block, pf, s_end, perm, sptr, scol, sR);
  if (s >= s1) return;
  const uint32_t pv = perm[s * 32 + lane];
  const uint32_t v = pv & kNodeMask;
  const uint64_t base = sptr[s];
  const uint32_t len = static_cast<uint32_t>((sptr[s + 1] - base) >> 5);
  const uint32_t* __restrict__ cp = scol + base + lane;
  const double* __restrict__ rp = kWeighted ? sR + base + lane : nullptr;
  // metrics.cpp:152 starts every product at 1.0; a later pass resumes it
  double miss = (v == kNoNode || (pv & kFirst)) ? 1.0 : ld_stream(state + v, pol);
  for (uint32_t k = 0; k < len; k += kU) {
    uint32_t c[kU];
    double r[kU], x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool in = k + u < len;
      c[u] = in ? ld_stream(cp + (uint64_t)(k + u) * 32, pol) : 0u;
      if constexpr (kWeighted) r[u] = in ? ld_stream(rp + (uint64_t)(k + u) * 32, pol) : 0.0;
      else r[u] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool in = k + u < len;
      x[u] = (in && (kWeighted || !(c[u] & kExcFlag)))
                 ? ((kWeighted && fbase != 0.0) ? fbase : ld_gather(opnd + c[u], gmode))
                 : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (k + u < len) miss = __dmul_rn(miss, factor<kWeighted>(c[u], x[u], r[u], exc_src, exc_R, prev));
  }
  if (v == kNoNode) return;
  if (pv & kLast) finish<kWeighted>(v, miss, prev, inv, out, yout, nullptr, pol);
  else st_stream(state + v, miss, pol);
}

// Node-major segmented pass k of a weighted graph (graph.cuh "nm"): one warp
// per slice of 32 consecutive node ids, lane = node in every pass, so the
// running product (carried between passes in `state`) and P are read and
// written coalesced; the lane's pass-k sources (and R) start at
// sbase(k, slice) + the prefix of the slice's lens. The first sweep gathers
// nothing (fbase = P(s,1)). Compact node-major graphs use k_codes/k_products.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_sweep_nm(int k, uint64_t S, uint64_t long_blocks, uint64_t nlong, uint64_t pf,
               const uint8_t* __restrict__ lenf, const uint64_t* __restrict__ sbase,
               const uint32_t* __restrict__ ncol, const double* __restrict__ nR,
               double* __restrict__ state, const uint32_t* __restrict__ lnode,
               const uint64_t* __restrict__ lptr, const uint32_t* __restrict__ lcol,
               const double* __restrict__ lR, const double* __restrict__ prev,
               const double* __restrict__ inv, double* __restrict__ out, int gmode, double fbase) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  if (blockIdx.x < long_blocks) {
    long_row<true>((uint64_t)blockIdx.x * kWarpsPerBlock + wib, nlong, lnode, lptr, lcol, lR, nullptr,
                   nullptr, prev, prev, inv, out, nullptr, nullptr, gmode, pol, fbase);
    return;
  }
  const uint64_t s_block = ((uint64_t)blockIdx.x - long_blocks) * kWarpsPerBlock;
  const uint64_t sl = s_block + wib;
  if (pf && wib == kWarpsPerBlock - 1 && lane == 0) {
    // L2 lookahead (see prefetch_ahead): lens, slice pointers and running
    // products of the block pf ahead, columns and R of the block pf/2 ahead
    const uint64_t sp = s_block + pf * kWarpsPerBlock;
    if (sp < S) {
      const uint64_t cnt = S - sp < kWarpsPerBlock ? S - sp : kWarpsPerBlock;
      prefetch_l2(lenf + ((uint64_t)k * S + sp) * 32, cnt * 32);
      prefetch_l2(sbase + (uint64_t)k * S + sp, (cnt + 1) * sizeof(uint64_t));
      if (k > 0) prefetch_l2(state + sp * 32, cnt * 32 * sizeof(double));
    }
    const uint64_t sc = s_block + (pf / 2) * kWarpsPerBlock;
    if (sc < S) {
      const uint64_t ce = sc + kWarpsPerBlock < S ? sc + kWarpsPerBlock : S;
      const uint64_t a = sbase[(uint64_t)k * S + sc], b = sbase[(uint64_t)k * S + ce];
      if (b > a) {
        prefetch_l2(ncol + a, (b - a) * sizeof(uint32_t));
        prefetch_l2(nR + a, (b - a) * sizeof(double));
      }
    }
  }
  if (sl >= S) return;
  const uint64_t v = sl * 32 + lane;
  const uint32_t lf = lenf[(uint64_t)k * S * 32 + v];
  if (__ballot_sync(kFull, lf != 0) == 0) return;  // slice untouched by this pass
  const uint32_t len = lf & kNmLen;
  uint32_t incl = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t maxlen = __reduce_max_sync(kFull, len);
  const uint64_t off = sbase[(uint64_t)k * S + sl] + (incl - len);
  // metrics.cpp:152 starts every product at 1.0; a later pass resumes it
  double miss = 1.0;
  if (lf != 0 && !(lf & kNmFirst)) miss = ld_stream(state + v, pol);
  for (uint32_t t = 0; t < maxlen; t += kU) {
    uint32_t c[kU];
    double r[kU], x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool in = t + u < len;
      c[u] = in ? ld_stream(ncol + off + t + u, pol) : 0u;
      r[u] = in ? ld_stream(nR + off + t + u, pol) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      x[u] = t + u < len ? (fbase != 0.0 ? fbase : ld_gather(prev + c[u], gmode)) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (t + u < len) miss = __dmul_rn(miss, factor<true>(c[u], x[u], r[u], nullptr, nullptr, prev));
  }
  if (lf & kNmLast) finish<true>(static_cast<uint32_t>(v), miss, prev, inv, out, nullptr, nullptr, pol);
  else if (len) st_stream(state + v, miss, pol);
}

// ---- first sweep over the class stream (graph.cuh "f1") ---------------------
// P(s,1) = 1/N for every source (metrics.cpp:143), so a regular edge's
// factor 1 - P(s,1) * (1/row_sum(s)) depends on the source only through its
// class; the ncls+1 factors (the last 1.0, for padding slots) sit in shared
// memory and every slot streams a 2-byte class instead of gathering.
// Exception edges (R != 1/row_sum, e.g. coalesced parallel edges) look their
// R up by slot: 1 - P(s,1) * R, as metrics.cpp:166.
__device__ __noinline__ double exc_first(uint64_t at, const uint64_t* __restrict__ xslot,
                                            const double* __restrict__ xR, uint64_t nx,
                                            double base) {
  uint64_t lo = 0, hi = nx;  // the first listed slot >= at (== at)
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (xslot[mid] < at) lo = mid + 1;
    else hi = mid;
  }
  return __dsub_rn(1.0, __dmul_rn(base, xR[lo]));
}

__device__ __forceinline__ void finish_first(uint32_t v, double miss, double base,
                                             const double* __restrict__ inv, double* __restrict__ out,
                                             double* __restrict__ yout, uint32_t* __restrict__ kout,
                                             uint64_t pol) {
  // metrics.cpp:169 with prev[v] = P(v,1) = base
  const double P = __dadd_rn(base, __dmul_rn(__dsub_rn(1.0, base), __dsub_rn(1.0, miss)));
  if (!pol) {  // L2-resident outputs: plain stores
    out[v] = P;
    if (yout || kout) {
      const double y = __dmul_rn(P, inv[v]);
      if (yout) yout[v] = y;
      if (kout) kout[v] = y_code(y);
    }
    return;
  }
  st_stream(out + v, P, pol);
  if (yout || kout) {
    const double y = __dmul_rn(P, inv[v]);
    if (yout) st_stream(yout + v, y, pol);
    if (kout) st_stream(kout + v, y_code(y), pol);
  }
}

__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void load_factors(double* fac, uint32_t ncls, double base,
                                             const double* __restrict__ cls_inv) {
  // class ncls: padding, exactly 1.0; class ncls+1: exception edges, a NaN
  // sentinel (no factor is NaN, so a NaN product flags the slice)
  for (uint32_t c = threadIdx.x; c <= ncls + 1; c += blockDim.x)
    fac[c] = c < ncls ? __dsub_rn(1.0, __dmul_rn(base, cls_inv[c])) : c == ncls ? 1.0 : __longlong_as_double(0x7ff8000000000000ll);
  __syncthreads();
}

// Long rows: one warp per row, 32 factors per step in parallel, one ordered
// chain (every lane runs it on shuffled factors; lane 0 writes).
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_first_long(uint64_t nlong, double base, uint32_t ncls, const double* __restrict__ cls_inv,
                 const uint32_t* __restrict__ lnode, const uint64_t* __restrict__ lptr,
                 const uint32_t* __restrict__ lcol, const uint16_t* __restrict__ lcls,
                 const double* __restrict__ exc_R, const double* __restrict__ inv,
                 double* __restrict__ out, double* __restrict__ yout, uint32_t* __restrict__ kout) {
  extern __shared__ double fac[];
  load_factors(fac, ncls, base, cls_inv);
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  const uint64_t warps = (uint64_t)gridDim.x * kWarpsPerBlock;
  for (uint64_t it = (uint64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); it < nlong; it += warps) {
    const uint64_t a = lptr[it], b = lptr[it + 1];
    double miss = 1.0;
    for (uint64_t cs = a; cs < b; cs += 32 * kLongU) {
      double f[kLongU];
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        const uint64_t e = cs + u * 32 + lane;
        f[u] = 1.0;
        if (e < b) {
          const uint16_t c = ld_stream(lcls + e, pol);
          f[u] = c == ncls + 1 ? __dsub_rn(1.0, __dmul_rn(base, exc_R[lcol[e] & ~kExcFlag])) : fac[c];
        }
      }
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        const uint64_t b0 = cs + u * 32;
        const int cnt = b > b0 ? static_cast<int>(b - b0 < 32 ? b - b0 : 32) : 0;
        for (int j = 0; j < cnt; ++j) miss = __dmul_rn(miss, __shfl_sync(kFull, f[u], j));
      }
    }
    if (lane == 0) finish_first(lnode[it], miss, base, inv, out, yout, kout, pol);
  }
}

// One slice's ordered product over its lane-major class stream, exception
// classes contributing the NaN sentinel.
// One slice's ordered product over its class stream (lane-major quads: the
// lane's 4 steps in one 8-byte load), exception classes contributing the NaN
// sentinel. len is a multiple of 4 (padding: class ncls, factor 1.0).
__device__ __forceinline__ double slice_product(uint32_t len, const uint16_t* __restrict__ cp,
                                                uint32_t tab, uint32_t ncls, uint64_t pol) {
  double miss = 1.0;  // metrics.cpp:152
  for (uint32_t k = 0; k < len; k += kU) {
    uint32_t c[kU];
#pragma unroll
    for (int q = 0; q < kU / 4; ++q) {
      uint64_t w = 0;
      if (k + 4 * q < len) w = ld_stream(reinterpret_cast<const uint64_t*>(cp + (uint64_t)((k >> 2) + q) * 128), pol);
      else w = 0x0001000100010001ull * ncls;
#pragma unroll
      for (int r = 0; r < 4; ++r) c[4 * q + r] = static_cast<uint32_t>(w >> (16 * r)) & 0xFFFFu;
    }
    double f[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) f[u] = lds_f64(tab + c[u] * 8);
#pragma unroll
    for (int u = 0; u < kU; ++u) miss = __dmul_rn(miss, f[u]);
  }
  return miss;
}

// The slice again, element by element, exceptions with their R (rare).
__device__ __noinline__ double slice_product_exc(uint32_t len, const uint16_t* __restrict__ cp,
                                                 uint64_t b0, uint32_t lane, uint32_t tab, uint32_t ncls,
                                                 const uint64_t* __restrict__ xslot,
                                                 const double* __restrict__ xR, uint64_t nx,
                                                 double base) {
  double miss = 1.0;
  for (uint32_t k = 0; k < len; ++k) {
    const uint64_t at = f1_slot(b0, k, lane);
    const uint32_t c = cp[at];
    const double f = c == ncls + 1 ? exc_first(at, xslot, xR, nx, base) : lds_f64(tab + c * 8);
    miss = __dmul_rn(miss, f);
  }
  return miss;
}

// Regular rows: persistent warps, one slice of 32 nodes at a time, lane =
// node, lane-major quads of classes (one coalesced 256-byte load per 4 steps). For graphs
// whose per-node outputs exceed half the L2, the slices are built without
// in-degree sorting across slices (graph.cu build_first, window 32), so a
// warp's stores of P / y / code cover its own 32 consecutive nodes and stay
// whole sectors; small graphs sort windows of 256 (less padding) and their
// scattered stores merge in L2.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_first(uint64_t s0, uint64_t S, uint64_t n, double base, uint32_t ncls, const double* __restrict__ cls_inv,
                  const uint32_t* __restrict__ perm, const uint64_t* __restrict__ sptr,
                  const uint16_t* __restrict__ cls, const uint64_t* __restrict__ xslot,
                  const double* __restrict__ xR, uint64_t nx, const double* __restrict__ inv,
                  double* __restrict__ out, double* __restrict__ yout, uint32_t* __restrict__ kout) {
  extern __shared__ double fac[];
  load_factors(fac, ncls, base, cls_inv);
  const uint32_t tab = static_cast<uint32_t>(__cvta_generic_to_shared(fac));
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  const uint64_t warps = (uint64_t)gridDim.x * kWarpsPerBlock;
  for (uint64_t sl = s0 + (uint64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); sl < S; sl += warps) {
    // node order (f1_ident): the slot names the node, no perm word to read
    const uint32_t v = perm ? (perm[sl * 32 + lane] & kNodeMask)
                            : (sl * 32 + lane < n ? static_cast<uint32_t>(sl * 32 + lane) : kNoNode);
    const uint64_t b0 = sptr[sl];
    const uint32_t len = static_cast<uint32_t>((sptr[sl + 1] - b0) >> 5);
    double miss = slice_product(len, cls + b0 + lane * 4, tab, ncls, pol);
    if (miss != miss)  // an exception edge in the slice
      miss = slice_product_exc(len, cls, b0, lane, tab, ncls, xslot, xR, nx, base);
    if (v != kNoNode) finish_first(v, miss, base, inv, out, yout, kout, 0);
  }
}

// ---- node-major graphs, compact layout: shared factor helpers --------------
// Codes of kBigCode (y >= 2^-21) fall back to y = P(s) * (1/row_sum(s)),
// recomputed exactly as the producing sweep formed it; exception edges use
// their own R.
__device__ __forceinline__ double code_factor(uint32_t c, uint32_t code, const uint32_t* __restrict__ exc_src,
                                              const double* __restrict__ exc_R,
                                              const double* __restrict__ prev,
                                              const double* __restrict__ inv) {
  if (c & kExcFlag) {
    const uint32_t x = c & ~kExcFlag;
    return __dsub_rn(1.0, __dmul_rn(prev[exc_src[x]], exc_R[x]));  // metrics.cpp:166
  }
  if (code == kBigCode) return __dsub_rn(1.0, __dmul_rn(prev[c], inv[c]));
  return code_to_factor(code);  // == 1 - y (the reference's one rounding, see graph.cuh)
}

// Long rows of a node-major graph (in-degree above kNmLen): one warp per row
// over the whole row (gathers span every segment; few rows).
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_pass_long(uint64_t nlong, const uint32_t* __restrict__ lnode, const uint64_t* __restrict__ lptr,
                const uint32_t* __restrict__ lcol, const uint32_t* __restrict__ exc_src,
                const double* __restrict__ exc_R, const double* __restrict__ prev,
                const uint32_t* __restrict__ kprev, const double* __restrict__ inv,
                double* __restrict__ out, uint32_t* __restrict__ kout) {
  const int lane = threadIdx.x & 31;
  const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= nlong) return;
  const uint64_t a = lptr[i], b = lptr[i + 1];
  double miss = 1.0;
  for (uint64_t cs = a; cs < b; cs += 32) {
    const uint64_t e = cs + lane;
    double f = 1.0;
    if (e < b) {
      const uint32_t c = lcol[e];
      f = code_factor(c, (c & kExcFlag) ? 0u : kprev[c], exc_src, exc_R, prev, inv);
    }
    const int cnt = static_cast<int>(b - cs < 32 ? b - cs : 32);
    for (int j = 0; j < cnt; ++j) miss = __dmul_rn(miss, __shfl_sync(kFull, f, j));
  }
  if (lane == 0) {
    const uint32_t v = lnode[i];
    const double pv = prev[v];
    const double P = __dadd_rn(pv, __dmul_rn(__dsub_rn(1.0, pv), __dsub_rn(1.0, miss)));
    out[v] = P;
    if (kout) kout[v] = y_code(__dmul_rn(P, inv[v]));
  }
}

// ---- later sweeps, decoupled: gather codes, then ordered products ---------
// A node-major graph's later sweep runs in two kernels instead of
// state-carrying passes.
//
// k_codes (G): every nm_col entry's 4-byte code, gathered into nm_code at the
// same position. nm_col is laid out pass by pass (source segment by source
// segment), and the persistent grid walks it in order, so the CTAs in flight
// gather from one L2-sized code segment at a time (evict_last), while the
// column and code streams go by evict_first. No per-node work at all: the
// kernel is bound by the random-gather rate of the L1 (one wavefront per
// 4-byte gather) and the stream bandwidth.
//
// k_products (P): one warp per slice of 32 consecutive nodes, lane = node;
// for pass 0..K-1 the lane reads its run of codes (its sources ascending
// inside the pass, passes in source order) and multiplies the factors
// 1 - J 2^-53 in order — the reference's left-to-right product
// (metrics.cpp:152-168) with the running product in a register across
// passes. Exception and big-code entries carry marker codes and are resolved
// from nm_col (rare).
constexpr uint32_t kExcCode = 0xFFFFFFFEu;  // code marker: exception edge
// nm_code holds each factor's low word L = -J (low_to_factor): one compare and
// select rebuild the factor. The marker's low word is 2 (-kExcCode); no code
// below kExcCode maps there.
constexpr uint32_t kExcLow = 0u - kExcCode;

constexpr int kCodesPerThread = 16;

// A factor f in (1/2, 1] is 1 - J 2^-53 for the integer J = bits(1.0) -
// bits(f): the code whose code_to_factor is f bit for bit. Factors outside
// that range, or whose J does not fit below the markers, keep a marker.
__device__ __forceinline__ uint32_t factor_to_code(double f) {
  const long long j = 0x3FF0000000000000ll - __double_as_longlong(f);
  return (f > 0.5 && j >= 0 && j < kExcCode) ? static_cast<uint32_t>(j) : kExcCode;
}

__device__ __forceinline__ uint32_t code_of(uint32_t c, uint32_t code, const uint32_t* __restrict__ exc_src,
                                           const double* __restrict__ exc_R,
                                           const double* __restrict__ prev,
                                           const double* __restrict__ inv, uint32_t& any) {
  if (code < kExcCode) return code;
  // rare: exception edge or y >= 2^-21: the exact factor's code
  double f;
  if (c & kExcFlag) {
    const uint32_t x = c & ~kExcFlag;
    f = __dsub_rn(1.0, __dmul_rn(prev[exc_src[x]], exc_R[x]));  // metrics.cpp:166
  } else {
    f = __dsub_rn(1.0, __dmul_rn(prev[c], inv[c]));  // y = P(s) * (1/row_sum(s))
  }
  const uint32_t j = factor_to_code(f);
  any |= j == kExcCode;
  return j;
}

// Each thread owns groups of 4 consecutive entries: 16-byte column loads and
// code stores (a quarter of the memory instructions of 4-byte ones); the
// region's unaligned head and tail go element by element.
__global__ void __launch_bounds__(256)
    k_codes(uint64_t e0, uint64_t e1, const uint32_t* __restrict__ ncol, const uint32_t* __restrict__ kprev,
            const uint32_t* __restrict__ exc_src, const double* __restrict__ exc_R,
            const double* __restrict__ prev, const double* __restrict__ inv,
            uint32_t* __restrict__ ncode, uint32_t* __restrict__ marked) {
  const uint64_t pol = policy_evict_first();
  uint32_t any = 0;
  const uint64_t a0 = (e0 + 3) & ~3ull, a1 = e1 & ~3ull;  // 16-byte aligned body [a0, a1)
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (a0 >= a1) {  // tiny region: element by element
    for (uint64_t i = e0 + tid; i < e1; i += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t c = ncol[i];
      ncode[i] = 0u - code_of(c, (c & kExcFlag) ? kExcCode : __ldg(kprev + c), exc_src, exc_R, prev, inv, any);
    }
  } else {
    if (tid < a0 - e0) {
      const uint64_t i = e0 + tid;
      const uint32_t c = ncol[i];
      ncode[i] = 0u - code_of(c, (c & kExcFlag) ? kExcCode : __ldg(kprev + c), exc_src, exc_R, prev, inv, any);
    }
    if (tid < e1 - a1) {
      const uint64_t i = a1 + tid;
      const uint32_t c = ncol[i];
      ncode[i] = 0u - code_of(c, (c & kExcFlag) ? kExcCode : __ldg(kprev + c), exc_src, exc_R, prev, inv, any);
    }
    const uint4* __restrict__ col4 = reinterpret_cast<const uint4*>(ncol + a0);
    uint4* __restrict__ out4 = reinterpret_cast<uint4*>(ncode + a0);
    const uint64_t g4 = (a1 - a0) / 4;
    constexpr int kG = kCodesPerThread / 4;  // 4-entry groups per thread per step
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g0 = tid; g0 < g4; g0 += stride * kG) {
      uint4 c[kG];
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const uint64_t g = g0 + u * stride;
        if (g < g4) {
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                       : "=r"(c[u].x), "=r"(c[u].y), "=r"(c[u].z), "=r"(c[u].w)
                       : "l"(col4 + g), "l"(pol));
        } else {
          c[u] = make_uint4(kExcFlag, kExcFlag, kExcFlag, kExcFlag);
        }
      }
      uint4 k[kG];
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        k[u].x = (c[u].x & kExcFlag) ? kExcCode : __ldg(kprev + c[u].x);
        k[u].y = (c[u].y & kExcFlag) ? kExcCode : __ldg(kprev + c[u].y);
        k[u].z = (c[u].z & kExcFlag) ? kExcCode : __ldg(kprev + c[u].z);
        k[u].w = (c[u].w & kExcFlag) ? kExcCode : __ldg(kprev + c[u].w);
      }
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const uint64_t g = g0 + u * stride;
        if (g >= g4) continue;
        uint4 o;
        o.x = 0u - code_of(c[u].x, k[u].x, exc_src, exc_R, prev, inv, any);
        o.y = 0u - code_of(c[u].y, k[u].y, exc_src, exc_R, prev, inv, any);
        o.z = 0u - code_of(c[u].z, k[u].z, exc_src, exc_R, prev, inv, any);
        o.w = 0u - code_of(c[u].w, k[u].w, exc_src, exc_R, prev, inv, any);
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(out4 + g), "r"(o.x),
                     "r"(o.y), "r"(o.z), "r"(o.w), "l"(pol)
                     : "memory");
      }
    }
  }
  if (__any_sync(kFull, any) && (threadIdx.x & 31) == 0) atomicOr(marked, 1u);
}

__device__ __noinline__ double marker_factor(uint32_t c, const uint32_t* __restrict__ exc_src,
                                             const double* __restrict__ exc_R,
                                             const double* __restrict__ prev,
                                             const double* __restrict__ inv) {
  if (c & kExcFlag) {
    const uint32_t x = c & ~kExcFlag;
    return __dsub_rn(1.0, __dmul_rn(prev[exc_src[x]], exc_R[x]));  // metrics.cpp:166
  }
  return __dsub_rn(1.0, __dmul_rn(prev[c], inv[c]));  // y = P(s) * (1/row_sum(s))
}

// The lane's product over every pass with marker codes resolved (rare: only
// when some factor of the sweep had no code, see k_codes).
__device__ __noinline__ double products_markers(int K, uint64_t S, uint64_t sl, int lane,
                                                const uint8_t* __restrict__ lenf,
                                                const uint64_t* __restrict__ sbase,
                                                const uint32_t* __restrict__ ncode,
                                                const uint32_t* __restrict__ ncol,
                                                const uint32_t* __restrict__ exc_src,
                                                const double* __restrict__ exc_R,
                                                const double* __restrict__ prev,
                                                const double* __restrict__ inv) {
  const uint64_t v = sl * 32 + lane;
  double miss = 1.0;
  for (int k = 0; k < K; ++k) {
    const uint32_t len = lenf[(uint64_t)k * S * 32 + v] & kNmLen;
    uint32_t incl = len;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const uint64_t q = sbase[(uint64_t)k * S + sl] + (incl - len);
    for (uint32_t t = 0; t < len; ++t) {
      const uint32_t low = ncode[q + t];
      miss = __dmul_rn(miss, low != kExcLow ? low_to_factor(low)
                                            : marker_factor(ncol[q + t], exc_src, exc_R, prev, inv));
    }
  }
  return miss;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32, 8)
    k_products(int K, uint64_t S, uint64_t n, const uint8_t* __restrict__ lenf,
               const uint64_t* __restrict__ sbase, const uint32_t* __restrict__ ncode,
               const uint32_t* __restrict__ ncol, const uint32_t* __restrict__ exc_src,
               const double* __restrict__ exc_R, const double* __restrict__ prev,
               const double* __restrict__ inv, double* __restrict__ out, uint32_t* __restrict__ kout,
               const uint32_t* __restrict__ marked) {
  const int lane = threadIdx.x & 31;
  const uint64_t sl = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sl >= S) return;
  const uint64_t pol = policy_evict_first();
  const uint64_t v = sl * 32 + lane;
  const bool real = v < n;
  double pv = 0.0, iv = 0.0;
  if (real) {  // finish operands in flight early
    pv = ld_stream(prev + v, pol);
    if (kout) iv = ld_stream(inv + v, pol);
  }
  double miss = 1.0;  // metrics.cpp:152
  uint32_t any = 0;   // a first-pass flag: regular row (long rows have their own kernel)
  const uint8_t* __restrict__ lp = lenf + v;
  const uint64_t* __restrict__ sp = sbase + sl;
  const uint64_t lstep = S * 32;
  uint32_t lf_next = K > 0 ? *lp : 0u;  // software-pipelined: pass k+1's len and base
  uint64_t sb_next = K > 0 ? *sp : 0ull;  // are in flight during pass k
  for (int k = 0; k < K; ++k) {
    const uint32_t lf = lf_next;
    const uint64_t sb = sb_next;
    lp += lstep;
    sp += S;
    if (k + 1 < K) {
      lf_next = *lp;
      sb_next = *sp;
    }
    any |= lf;
    const uint32_t len = lf & kNmLen;
    const uint32_t maxlen = __reduce_max_sync(kFull, len);
    if (maxlen == 0) continue;  // slice untouched by this pass
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t* __restrict__ cp = ncode + sb + (incl - len);
    for (uint32_t t = 0; t < maxlen; t += 4) {
      const int rem = static_cast<int>(len - t);  // this lane's entries left in the run
      uint32_t code[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) code[u] = __ldg(cp + t + u);  // ncode is padded past its end
#pragma unroll
      for (int u = 0; u < 4; ++u)
        miss = __dmul_rn(miss, low_to_factor(u < rem ? code[u] : 0u));  // past the run: 1.0
    }
  }
  if (*marked)  // uniform and rare: redo with the marker codes resolved
    miss = products_markers(K, S, sl, lane, lenf, sbase, ncode, ncol, exc_src, exc_R, prev, inv);
  if (real && (any & kNmFirst)) {
    // metrics.cpp:169: prev + (1 - prev) * (1 - miss_all)
    const double P = __dadd_rn(pv, __dmul_rn(__dsub_rn(1.0, pv), __dsub_rn(1.0, miss)));
    st_stream(out + v, P, pol);
    if (kout) st_stream(kout + v, y_code(__dmul_rn(P, iv)), pol);
  }
}

// ---- k_products_tma: the products with every pass's run staged by TMA ------
// k_products above walks the passes of a slice in lock-step: every pass
// starts with a dependent code load and a warp scan of the 32 run lengths,
// and lasts as long as its longest run (Σ_k max_lane len_k ≈ 37 steps per
// slice at C4 for 14.4 in-edges per node).
//
// Here a warp owns a slice at a time. The slice's K code ranges (one
// contiguous range of nm_code per pass, the lanes' runs back to back) are
// copied into the warp's shared-memory buffer by cp.async.bulk — one bulk
// copy per pass, issued by lane k, completing on the buffer's mbarrier — ONE
// slice ahead of the compute, so every pass's loads are in flight together
// and overlap the previous slice's multiplies. Each lane then walks its
// node's whole chain across the passes without lock-step (the warp runs
// max_lane Σ_k len_k ≈ 23 steps), jumping from run to run through a small
// per-lane table of (first, end) shared-memory addresses.
//
// Everything that places a lane's runs inside the staging buffer is static
// for the graph and precomputed once (k_build_runs):
//   desc[s*K + k]  (u64) pass k of slice s: words | staging offset << 11 |
//                  aligned source word << 22 | the slice's longest chain
//                  << 54; bit 63: the slice exceeds the buffer (global path)
//   runs[v]        (2 x u64) node v: its non-empty runs in pass order as
//                  u16 fields (staged word | len << 10), then sentinels:
//                  an empty run at the buffer's zero words (whose word says
//                  whether this kernel finishes the node: kPtSentReg)
// A lane past its chain keeps reading zero codes, i.e. factor 1.0 — an exact
// identity. Same factors, same left-to-right order: bit-identical.
constexpr int kPtWarps = 4;
constexpr int kPtKMax = 7;            // <= 7 runs + 1 sentinel in the 8 u16 fields
constexpr uint32_t kPtMaxBufw = 1024;  // words per buffer at most (10-bit run starts)
constexpr uint64_t kPtBig = 1ull << 63;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// shared memory of one warp: two staging buffers, the run table, 2 mbarriers
__host__ __device__ __forceinline__ size_t pt_warp_bytes(uint32_t bufw) {
  return (size_t)2 * bufw * 4 + 8 * 32 * 8 + 16;
}

// Largest staged size (words, 16-byte aligned ranges) of one slice.
__global__ void k_stage_words(int K, uint64_t S, const uint64_t* __restrict__ sbase,
                              unsigned* __restrict__ mx) {
  unsigned best = 0;
  for (uint64_t sl = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; sl < S;
       sl += (uint64_t)gridDim.x * blockDim.x) {
    unsigned w = 0;
    for (int k = 0; k < K; ++k) {
      const uint64_t st = sbase[(uint64_t)k * S + sl], en = sbase[(uint64_t)k * S + sl + 1];
      if (en > st) w += static_cast<unsigned>(((en + 3) & ~3ull) - (st & ~3ull));
    }
    best = max(best, w);
  }
  best = __reduce_max_sync(kFull, best);
  if ((threadIdx.x & 31) == 0) atomicMax(mx, best);
}

// One warp per slice, lane = node: the static staging layout (see above).
// zw: zero words at the end of each buffer (>= the longest chain).
__global__ void k_build_runs(int K, uint64_t S, const uint8_t* __restrict__ lenf,
                             const uint64_t* __restrict__ sbase, uint32_t bufw, uint32_t zw,
                             uint64_t* __restrict__ desc, ulonglong2* __restrict__ runs,
                             unsigned* __restrict__ big) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t zs = bufw - zw;  // sentinel start: the zero words
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t sl = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < S; sl += warps) {
    uint64_t st = 0, en = 0;
    if (lane < static_cast<uint32_t>(K)) {
      st = sbase[(uint64_t)lane * S + sl];
      en = sbase[(uint64_t)lane * S + sl + 1];
    }
    const uint64_t a = st & ~3ull;
    const uint32_t words = en > st ? static_cast<uint32_t>(((en + 3) & ~3ull) - a) : 0u;
    const uint32_t incl = warp_incl_scan(words);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const bool too_big = total > zs;
    const uint32_t off = incl - words;                          // staging offset of pass `lane`
    const uint32_t base = off + static_cast<uint32_t>(st - a);  // staged word of its first code
    uint64_t f[2] = {0, 0};
    uint32_t nj = 0, chain = 0, anyf = 0;
    for (int k = 0; k < K; ++k) {
      const uint32_t lf = lenf[(uint64_t)k * S * 32 + sl * 32 + lane];
      anyf |= lf;
      const uint32_t len = lf & kNmLen;
      const uint32_t pre = warp_incl_scan(len) - len;
      const uint32_t start = __shfl_sync(kFull, base, k) + pre;
      if (len) {
        f[nj >> 2] |= (uint64_t)((start & 0x3FFu) | (len << 10)) << (16 * (nj & 3));
        ++nj;
      }
      chain += len;
    }
    const uint64_t sent = (anyf & kNmFirst) ? zs : zs + 1;  // which sentinel: finish or not
    for (uint32_t j = nj; j < 8; ++j) f[j >> 2] |= sent << (16 * (j & 3));
    const uint32_t maxchain = __reduce_max_sync(kFull, chain);
    if (lane < static_cast<uint32_t>(K))
      desc[sl * K + lane] = (too_big ? kPtBig : 0ull) | ((uint64_t)maxchain << 54) | (a << 22) |
                            ((uint64_t)off << 11) | words;
    runs[sl * 32 + lane] = make_ulonglong2(f[0], f[1]);
    if (lane == 0 && too_big) atomicAdd(big, 1u);
  }
}

__global__ void __launch_bounds__(kPtWarps * 32)
    k_products_tma(int K, uint64_t S, uint64_t s0, uint64_t s1, uint64_t n, const uint8_t* __restrict__ lenf,
                   const uint64_t* __restrict__ desc, const ulonglong2* __restrict__ runs,
                   const uint64_t* __restrict__ sbase, const uint32_t* __restrict__ ncode,
                   const uint32_t* __restrict__ ncol, const uint32_t* __restrict__ exc_src,
                   const double* __restrict__ exc_R, const double* __restrict__ prev,
                   const double* __restrict__ inv, double* __restrict__ out,
                   uint32_t* __restrict__ kout, const uint32_t* __restrict__ marked, uint32_t bufw,
                   uint32_t zw) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* mine = smem + wid * pt_warp_bytes(bufw);
  uint32_t* const buf = reinterpret_cast<uint32_t*>(mine);  // [2][bufw]
  uint2* const tab = reinterpret_cast<uint2*>(mine + (size_t)2 * bufw * 4);  // [8][32]
  uint64_t* const bars = reinterpret_cast<uint64_t*>(mine + (size_t)2 * bufw * 4 + 8 * 32 * 8);
  for (uint32_t z = lane; z < zw; z += 32) {  // the sentinel runs' zero codes
    buf[bufw - zw + z] = 0u;
    buf[2 * bufw - zw + z] = 0u;
  }
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const bool mk = *marked != 0;  // uniform: some factor kept a marker code
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = policy_evict_first();
  const uint32_t buf0 = smem_u32(buf);
  const uint32_t sent_reg = bufw - zw;

  auto load_desc = [&](uint64_t sl) -> uint64_t {
    return (sl < s1 && lane < static_cast<uint32_t>(K)) ? ld_stream(desc + sl * K + lane, pol) : 0ull;
  };
  // Copies of a slice into buffer b: 0 nothing to copy, 1 in flight on
  // bars[b], 2 global path (too big for the buffer, or markers).
  auto issue = [&](uint64_t sl, uint64_t d, int b, uint32_t& maxt) -> uint32_t {
    const uint32_t hi0 = __shfl_sync(kFull, static_cast<uint32_t>(d >> 32), 0);
    maxt = (hi0 >> 22) & 0x1FF;
    if (sl >= s1) return 0;
    if ((hi0 & 0x80000000u) || mk) return 2;
    const uint32_t words = static_cast<uint32_t>(d & 0x7FF);
    const uint32_t total = __reduce_add_sync(kFull, words);
    if (total == 0) return 0;
    const uint32_t bar = smem_u32(&bars[b]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(total * 4)
                   : "memory");
    __syncwarp();
    if (words)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              buf0 + 4 * (b * bufw + static_cast<uint32_t>((d >> 11) & 0x7FF))),
          "l"(ncode + ((d >> 22) & 0xFFFFFFFFull)), "r"(words * 4), "r"(bar)
          : "memory");
    return 1;
  };

  uint64_t sl = s0 + gw;  // this call's slices: [s0, s1) (a rank's node range when sharded)
  uint64_t d1 = load_desc(sl);
  ulonglong2 rc = sl < s1 ? runs[sl * 32 + lane] : make_ulonglong2(0, 0);
  uint32_t maxt_cur, maxt_nxt;
  uint32_t stat_cur = issue(sl, d1, 0, maxt_cur), stat_nxt;
  d1 = load_desc(sl + nw);
  uint32_t par = 0;  // expected parity per buffer
  for (int i = 0; sl < s1; ++i, sl += nw) {
    const int b = i & 1;
    const uint64_t v = sl * 32 + lane;
    const bool real = v < n;
    double pv = 0.0, iv = 0.0;
    if (real) {  // finish operands in flight early
      pv = ld_stream(prev + v, pol);
      if (kout) iv = ld_stream(inv + v, pol);
    }
    // the next slice's copies go into the other buffer: its reads by the
    // previous iteration have completed (their values were consumed)
    stat_nxt = issue(sl + nw, d1, b ^ 1, maxt_nxt);
    const ulonglong2 rn = sl + nw < s1 ? runs[(sl + nw) * 32 + lane] : make_ulonglong2(0, 0);
    d1 = load_desc(sl + 2 * nw);

    double miss = 1.0;  // metrics.cpp:152
    if (stat_cur == 2) {  // rare: the slice's runs exceed the buffer, or markers
      miss = products_markers(K, S, sl, static_cast<int>(lane), lenf, sbase, ncode, ncol, exc_src,
                              exc_R, prev, inv);
    } else {
      // the lane's (first, end) byte addresses of runs 1..7 (run 0 stays in registers)
      const uint32_t bb = buf0 + 4 * b * bufw;
      uint32_t a0 = 0, e0 = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t f = static_cast<uint32_t>(((j < 4 ? rc.x : rc.y) >> (16 * (j & 3))) & 0xFFFF);
        const uint32_t aa = bb + 4 * (f & 0x3FFu), ee = aa + 4 * (f >> 10);
        if (j == 0) {
          a0 = aa;
          e0 = ee;
        } else {
          tab[(j - 1) * 32 + lane] = make_uint2(aa, ee);
        }
      }
      if (stat_cur == 1) {
        asm volatile(
            "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra W_%=;\n}" ::"r"(smem_u32(&bars[b])),
            "r"((par >> b) & 1u)
            : "memory");
        par ^= 1u << b;
      }
      uint32_t a = a0, e = e0, ta = smem_u32(tab + lane);
#pragma unroll 4
      for (uint32_t t = 0; t < maxt_cur; ++t) {
        uint32_t c;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(c) : "r"(a));
        miss = __dmul_rn(miss, low_to_factor(c));
        a += 4;
        if (a == e) {  // the lane's next run (or its sentinel)
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(e) : "r"(ta));
          ta += 256;
        }
      }
    }
    const uint32_t s7 = static_cast<uint32_t>(rc.y >> 48) & 0x3FFu;  // field 7: always a sentinel
    if (real && s7 == sent_reg) {
      // metrics.cpp:169: prev + (1 - prev) * (1 - miss_all)
      const double P = __dadd_rn(pv, __dmul_rn(__dsub_rn(1.0, pv), __dsub_rn(1.0, miss)));
      st_stream(out + v, P, pol);
      if (kout) st_stream(kout + v, y_code(__dmul_rn(P, iv)), pol);
    }
    __syncwarp();  // buffer b and the table are read; refilled next iteration
    rc = rn;
    stat_cur = stat_nxt;
    maxt_cur = maxt_nxt;
  }
}

// ---- k_pass_fused: gathers and ordered products of one source segment -------
// The decoupled sweep above writes every entry's code (nm_code) and reads it
// back in k_products_tma: 8 bytes of HBM per edge on top of the L1-bound
// gathers, and a second kernel whose issue-bound products do not overlap
// them. Here one launch per pass k does both. Every warp is an independent
// pipeline (no CTA barriers): it owns chunks of kFpSlices consecutive slices,
// whose pass-k entries are contiguous in nm_col ([sbase(k,c0), sbase(k,c1))).
// The warp gathers the chunk's codes (kFpU in flight per lane) into its own
// shared-memory buffer at each entry's position, then, lane = node, multiplies
// each lane's run in order into the running product carried between passes
// in `state` (coalesced, 16 bytes per node and pass instead of 8 per edge); a
// node's last pass finishes P. Passes run in source order and each run is
// ascending: the reference's left-to-right product (metrics.cpp:152-168),
// bit-identical. Lanes past their run read word 0 of the buffer's tail, a
// zero code (factor 1.0, an exact identity). Chunks with an unrepresentable
// factor (marker) or more entries than `cap` run the exact loop on nm_col
// (both rare).
constexpr int kFpWarps = 4;
constexpr int kFpSlices = 4;            // slices per warp chunk
constexpr uint32_t kFpBufw = 1024;      // words per warp buffer, the last one kept zero
constexpr int kFpU = 8;                 // gathers in flight per lane
constexpr size_t kFpSmem = (size_t)kFpWarps * kFpBufw * sizeof(uint32_t);

__global__ void __launch_bounds__(kFpWarps * 32)
    k_pass_fused(int k, uint64_t S, uint64_t s0, uint64_t s1, uint64_t n, const uint8_t* __restrict__ lenf,
                 const uint64_t* __restrict__ sbase, const uint32_t* __restrict__ ncol,
                 const uint32_t* __restrict__ kprev, const uint32_t* __restrict__ exc_src,
                 const double* __restrict__ exc_R, const double* __restrict__ prev,
                 const double* __restrict__ inv, double* __restrict__ state, double* __restrict__ out,
                 uint32_t* __restrict__ kout, uint32_t cap) {
  extern __shared__ __align__(16) uint32_t fbuf[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* const buf = fbuf + wid * kFpBufw;
  const uint32_t zero = kFpBufw - 1;
  if (lane == 0) buf[zero] = 0u;
  __syncwarp();
  const uint64_t pol = policy_evict_first();
  const uint64_t nch = (s1 - s0 + kFpSlices - 1) / kFpSlices;
  const uint64_t* const sb = sbase + (uint64_t)k * S;
  const uint8_t* const lk = lenf + (uint64_t)k * S * 32;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t ch = gw; ch < nch; ch += nw) {
    const uint64_t c0 = s0 + ch * kFpSlices, c1 = c0 + kFpSlices < s1 ? c0 + kFpSlices : s1;
    // the lane's lens of every slice (one byte each), the chunk's bounds
    uint32_t lfs = 0;
#pragma unroll
    for (int q = 0; q < kFpSlices; ++q)
      if (c0 + q < c1) lfs |= ld_stream_u8(lk + (c0 + q) * 32 + lane, pol) << (8 * q);
    const uint64_t e0 = ld_stream(sb + c0, pol), e1 = ld_stream(sb + c1, pol);
    // every slice's running product and P(j-1) in flight under the gathers
    double m[kFpSlices], pv[kFpSlices];
#pragma unroll
    for (int q = 0; q < kFpSlices; ++q) {
      const uint32_t lf = (lfs >> (8 * q)) & 0xFF;
      const uint64_t v = (c0 + q) * 32 + lane;
      m[q] = (lf != 0 && !(lf & kNmFirst)) ? ld_stream(state + v, pol) : 1.0;
      pv[q] = ((lf & kNmLast) && v < n) ? ld_stream(prev + v, pol) : 0.0;
    }
    const uint32_t cnt = static_cast<uint32_t>(e1 - e0);
    bool exact = e1 - e0 > cap;
    if (!exact) {
      uint32_t any = 0;
      for (uint32_t i0 = lane; i0 < cnt; i0 += kFpU * 32) {
        uint32_t c[kFpU], kc[kFpU];
        // all kFpU column loads, then all gathers (volatile: kept in this order)
#pragma unroll
        for (int u = 0; u < kFpU; ++u) {
          const uint32_t i = i0 + u * 32;
          c[u] = i < cnt ? ld_stream(ncol + e0 + i, pol) : kExcFlag;
        }
#pragma unroll
        for (int u = 0; u < kFpU; ++u) {
          kc[u] = kExcCode;
          if (!(c[u] & kExcFlag))
            asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(kc[u]) : "l"(kprev + c[u]));
        }
#pragma unroll
        for (int u = 0; u < kFpU; ++u) {
          const uint32_t i = i0 + u * 32;
          if (i < cnt) {
            const uint32_t j = kc[u] < kExcCode ? kc[u] : code_of(c[u], kc[u], exc_src, exc_R, prev, inv, any);
            buf[i] = 0u - j;
          }
        }
      }
      exact = __any_sync(kFull, any);
      __syncwarp();
    }
    uint32_t pre = 0;  // entries of the chunk's earlier slices
#pragma unroll
    for (int q = 0; q < kFpSlices; ++q) {
      const uint64_t sl = c0 + q;
      if (sl >= c1) break;  // warp-uniform
      const uint64_t v = sl * 32 + lane;
      const uint32_t lf = (lfs >> (8 * q)) & 0xFF;
      const uint32_t len = lf & kNmLen;
      const uint32_t incl = warp_incl_scan(len);
      const uint32_t total = __shfl_sync(kFull, incl, 31);
      const uint32_t b0 = pre + incl - len;  // the lane's run, relative to e0
      pre += total;
      double mq = m[q];
      if (!exact) {
        const uint32_t maxlen = __reduce_max_sync(kFull, len);
        for (uint32_t t = 0; t < maxlen; ++t) {
          const uint32_t L = buf[t < len ? b0 + t : zero];
          mq = __dmul_rn(mq, low_to_factor(L));
        }
      } else {
        for (uint32_t t = 0; t < len; ++t) {
          const uint32_t c = ncol[e0 + b0 + t];
          uint32_t any = 0;
          const uint32_t j = code_of(c, (c & kExcFlag) ? kExcCode : __ldg(kprev + c), exc_src, exc_R, prev, inv, any);
          mq = __dmul_rn(mq, j == kExcCode ? marker_factor(c, exc_src, exc_R, prev, inv) : low_to_factor(0u - j));
        }
      }
      if (lf & kNmLast) {
        if (v < n) {  // metrics.cpp:169: prev + (1 - prev) * (1 - miss_all)
          const double P = __dadd_rn(pv[q], __dmul_rn(__dsub_rn(1.0, pv[q]), __dsub_rn(1.0, mq)));
          st_stream(out + v, P, pol);
          if (kout) st_stream(kout + v, y_code(__dmul_rn(P, ld_stream(inv + v, pol))), pol);
        }
      } else if (len) {
        st_stream(state + v, mq, pol);
      }
    }
    __syncwarp();  // the buffer is refilled by the next chunk
  }
}

}  // namespace

namespace {

// Phase brackets of one run (graph.cuh PhaseEv), events pooled in the graph.
struct PhaseTimer {
  qvb_graph& g;
  cudaStream_t s;
  int open = -1;
  PhaseTimer(qvb_graph& gr, cudaStream_t st) : g(gr), s(st) {
    g.phase_used = 0;
    g.launches = 0;
  }
  void begin(int phase) {
    if (g.phase_used == g.phase_ev.size()) {
      qvb_graph::PhaseEv pe{phase, nullptr, nullptr};
      QVB_CUDA(cudaEventCreate(&pe.a));
      QVB_CUDA(cudaEventCreate(&pe.b));
      g.phase_ev.push_back(pe);
    }
    auto& pe = g.phase_ev[g.phase_used];
    pe.phase = phase;
    QVB_CUDA(cudaEventRecord(pe.a, s));
    open = static_cast<int>(g.phase_used);
  }
  void end(uint32_t launched) {
    QVB_CUDA(cudaEventRecord(g.phase_ev[open].b, s));
    ++g.phase_used;
    g.launches += launched;
  }
};

}  // namespace

const double* run_access_prob(qvb_graph& g, uint32_t layers, cudaStream_t s, double* final_out,
                              const Shard& sh) {
  constexpr int kPtKMaxSh = kPtKMax;
  if (layers < 1) fail(QVB_ERR_VALIDATION, "access probability needs layers >= 1");
  const uint64_t n = g.n;
  const bool compact = g.layout == 0;
  const bool codes = g.nm && compact;                    // nm compact sweeps gather 4-byte codes
  const bool f1 = compact && g.ncls > 0 && layers >= 2;  // class-stream first sweep
  // entry N of every gathered vector is the padding operand: 0 (factor 1.0);
  // set once when the buffer is made (sweeps write entries < N only). P and
  // code buffers carry kShardPad more zero entries: a sharded call's ranks
  // own chunks of ceil(n / world / 32) * 32 nodes, world * chunk <= n + 32 world
  for (int i = 0; i < 2; ++i) {
    if (!g.p[i]) {
      QVB_CUDA(cudaMalloc(&g.p[i], (n + 1 + kShardPad) * sizeof(double)));
      QVB_CUDA(cudaMemsetAsync(g.p[i] + n, 0, (1 + kShardPad) * sizeof(double), s));
    }
    if (compact && !g.nm && !g.y[i]) {
      QVB_CUDA(cudaMalloc(&g.y[i], (n + 1) * sizeof(double)));
      QVB_CUDA(cudaMemsetAsync(g.y[i] + n, 0, sizeof(double), s));
    }
    if (codes && !g.kcode[i]) {
      QVB_CUDA(cudaMalloc(&g.kcode[i], (n + 1 + kShardPad) * sizeof(uint32_t)));
      QVB_CUDA(cudaMemsetAsync(g.kcode[i] + n, 0, (1 + kShardPad) * sizeof(uint32_t), s));
    }
  }
  // Row-sharded sweeps: this rank computes the nodes of its
  // chunk, then the exchange callback all-gathers P (and the codes the next
  // sweep gathers) in place. Per-node arithmetic is unchanged, so the result
  // is bit-identical to the single-GPU call. Layouts other than the
  // node-major compact one with TMA products compute every node on every
  // rank (no exchange needed).
  bool sharded = false;
  uint64_t chunk = n, s0 = 0, s1 = g.nm ? g.nm_S : 0;
  if (sh.world > 1) {
    if (sh.rank >= sh.world || !sh.fn) fail(QVB_ERR_VALIDATION, "bad shard (rank, world, exchange)");
    chunk = ((n + sh.world - 1) / sh.world + 31) / 32 * 32;
    if ((uint64_t)sh.world * chunk > n + 1 + kShardPad) fail(QVB_ERR_UNSUPPORTED, "too many ranks for the graph");
    const int nseg_ = static_cast<int>(g.seg_slice.size()) - 1;
    sharded = layers >= 2 && codes && (!f1 || g.f1_ident) && nseg_ <= kPtKMaxSh && g.long_threshold <= 256 &&
              (!std::getenv("QVB_PRODUCTS") || std::string(std::getenv("QVB_PRODUCTS")) == "fused");
    const uint64_t lo = std::min<uint64_t>(n, (uint64_t)sh.rank * chunk);
    const uint64_t hi = std::min<uint64_t>(n, lo + chunk);
    s0 = lo / 32;
    s1 = (hi + 31) / 32;
  }
  g.last_sharded = sharded;
  if (codes && !g.nm_code) {  // +128: k_products reads whole 4-code groups past a run's end
    QVB_CUDA(cudaMalloc(&g.nm_code, (g.nm_cols + 128) * sizeof(uint32_t)));
    QVB_CUDA(cudaMalloc(&g.marked, sizeof(uint32_t)));
  }
  for (auto& e : g.ev)
    if (!e) QVB_CUDA(cudaEventCreate(&e));
  PhaseTimer pt(g, s);
  const double base = 1.0 / static_cast<double>(n);  // metrics.cpp:143
  if (!f1) {  // P(n,1) (and, for a gathering first sweep, its operands)
    k_init<<<grid_for(n + 1, 256), 256, 0, s>>>(n, g.inv, g.p[0],
                                               (compact && !g.nm && layers >= 2) ? g.y[0] : nullptr,
                                               (codes && layers >= 2) ? g.kcode[0] : nullptr);
    QVB_LAUNCH_CHECK();
    ++g.launches;
  }
  const uint64_t long_blocks = (g.nlong + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int nseg = static_cast<int>(g.seg_slice.size()) - 1;
  int gmode = 0;
  if (const char* m = std::getenv("QVB_GATHER_MODE")) gmode = std::atoi(m);
  // L2 lookahead in blocks for the segmented passes (QVB_PF_BLOCKS; 0 = off);
  // worthwhile only when the streams do not already sit in L2
  uint64_t pf = nseg > 1 ? 512 : 0;
  if (const char* m = std::getenv("QVB_PF_BLOCKS")) pf = std::strtoull(m, nullptr, 10);
  QVB_CUDA(cudaEventRecord(g.ev[0], s));
  for (uint32_t j = 2; j <= layers; ++j) {
    const int cur = (j - 2) & 1, nxt = cur ^ 1;
    const bool first = j == 2;
    double* yout = (compact && !g.nm && j < layers) ? g.y[nxt] : nullptr;
    // the last sweep writes straight into the caller's device buffer (not
    // when sharded: the exchange needs the padded buffer)
    double* const pout = (j == layers && final_out && !sharded) ? final_out : g.p[nxt];
    uint32_t* kout = (codes && j < layers) ? g.kcode[nxt] : nullptr;
    // after a sharded sweep: every rank's chunk of P_j (and of its codes,
    // which the next sweep gathers) into every rank's buffers
    auto exchange = [&]() {
      if (!sharded) return;
      const int rc = sh.fn(sh.ctx, j, pout, kout, chunk, s);
      if (rc != 0) fail(QVB_ERR_GENERIC, "exchange callback failed at layer " + std::to_string(j));
    };

    if (first && f1) {  // ---- first sweep over the class stream
      pt.begin(0);
      uint32_t launched = 0;
      const size_t smem = (g.ncls + 2) * sizeof(double);
      if (g.nlong) {
        QVB_CUDA(cudaFuncSetAttribute(k_first_long, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kMaxCls + 2) * 8));
        const unsigned lg = resident_grid(k_first_long, kWarpsPerBlock * 32, smem,
                                          (g.nlong + kWarpsPerBlock - 1) / kWarpsPerBlock);
        k_first_long<<<lg, kWarpsPerBlock * 32, smem, s>>>(g.nlong, base, g.ncls, g.cls_inv, g.lnode,
                                                           g.lptr, g.lcol, g.lcls, g.exc_R, g.inv,
                                                           pout, yout, kout);
        QVB_LAUNCH_CHECK();
        ++launched;
      }
      if (g.f1_S) {
        if (!g.f1_grid) {  // once per graph: host API calls between launches idle the GPU
          QVB_CUDA(cudaFuncSetAttribute(k_first, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kMaxCls + 2) * 8));
          g.f1_grid = resident_grid(k_first, kWarpsPerBlock * 32, smem,
                                    (g.f1_S + kWarpsPerBlock - 1) / kWarpsPerBlock);
        }
        const unsigned grid = g.f1_grid;
        k_first<<<grid, kWarpsPerBlock * 32, smem, s>>>(sharded ? s0 : 0, sharded ? s1 : g.f1_S, n, base,
                                                        g.ncls, g.cls_inv,
                                                        g.f1_ident ? nullptr : g.f1_perm,
                                                        g.f1_sptr, g.f1_cls, g.f1_xslot, g.f1_xR,
                                                        g.f1_nx, g.inv, pout, yout, kout);
        QVB_LAUNCH_CHECK();
        ++launched;
      }
      pt.end(launched);
      exchange();
      continue;
    }

    if (codes) {  // ---- node-major compact graph: code gathers, then products
      uint32_t launched = 0;
      pt.begin(1);
      QVB_CUDA(cudaMemsetAsync(g.marked, 0, sizeof(uint32_t), s));
      if (g.nlong) {  // long rows: whole rows, one warp each
        k_pass_long<<<static_cast<unsigned>((g.nlong * 32 + 255) / 256), 256, 0, s>>>(
            g.nlong, g.lnode, g.lptr, g.lcol, g.exc_src, g.exc_R, g.p[cur], g.kcode[cur], g.inv,
            pout, kout);
        QVB_LAUNCH_CHECK();
        ++launched;
      }
      const char* pm = std::getenv("QVB_PRODUCTS");  // "fused": fused passes (A/B)
      const int products_mode = pm && std::string(pm) == "fused" ? 1 : 0;
      if (products_mode == 1) {
        // one fused pass per source segment (k_pass_fused): gathers and
        // ordered products together, the running product in g.state
        uint32_t fp_cap = kFpBufw - 1;  // tests: QVB_FP_CAP forces the exact path for larger chunks
        if (const char* c = std::getenv("QVB_FP_CAP")) fp_cap = std::min<uint32_t>(kFpBufw - 1, std::atoi(c));
        if (!g.fused_grid) {
          QVB_CUDA(cudaFuncSetAttribute(k_pass_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kFpSmem)));
          g.fused_grid = resident_grid(k_pass_fused, kFpWarps * 32, kFpSmem, ~0ull);
        }
        const uint64_t nch = (s1 - s0 + kFpSlices - 1) / kFpSlices;
        const unsigned fg = static_cast<unsigned>(std::min<uint64_t>(g.fused_grid, nch ? nch : 1));
        for (int k = 0; k < nseg; ++k) {
          k_pass_fused<<<fg, kFpWarps * 32, kFpSmem, s>>>(k, g.nm_S, s0, s1, n, g.nm_lenf, g.nm_sbase, g.nm_col,
                                                   g.kcode[cur], g.exc_src, g.exc_R, g.p[cur], g.inv,
                                                   g.state, pout, kout, fp_cap);
          QVB_LAUNCH_CHECK();
          ++launched;
        }
        pt.end(launched);
        exchange();
        continue;
      }
      // one launch per source segment: the CTAs in flight gather from one
      // L2-resident code segment
      if (sharded && g.shard_key != (uint64_t)sh.world << 32 | sh.rank) {  // this rank's entries per pass
        g.shard_e.assign(2 * nseg, 0);
        for (int k = 0; k < nseg; ++k) {
          QVB_CUDA(cudaMemcpy(&g.shard_e[2 * k], g.nm_sbase + (uint64_t)k * g.nm_S + s0, 8, cudaMemcpyDeviceToHost));
          QVB_CUDA(cudaMemcpy(&g.shard_e[2 * k + 1], g.nm_sbase + (uint64_t)k * g.nm_S + s1, 8,
                              cudaMemcpyDeviceToHost));
        }
        g.shard_key = (uint64_t)sh.world << 32 | sh.rank;
      }
      for (int k = 0; k < nseg; ++k) {
        const uint64_t e0 = sharded ? g.shard_e[2 * k] : g.nm_region[k];
        const uint64_t e1 = sharded ? g.shard_e[2 * k + 1] : g.nm_region[k + 1];
        if (e1 <= e0) continue;
        if (!g.codes_grid) g.codes_grid = resident_grid(k_codes, 256, 0, ~0ull);
        const unsigned cg = static_cast<unsigned>(std::min<uint64_t>(g.codes_grid, (e1 - e0 + 2047) / 2048));
        k_codes<<<cg, 256, 0, s>>>(e0, e1, g.nm_col, g.kcode[cur], g.exc_src, g.exc_R, g.p[cur], g.inv,
                                  g.nm_code, g.marked);
        QVB_LAUNCH_CHECK();
        ++launched;
      }
      pt.end(launched);
      static const bool old_products = [] {
        const char* m = std::getenv("QVB_PRODUCTS");
        return m && std::string(m) == "lockstep";
      }();
      if (!g.prod_bufw && nseg <= kPtKMax && g.long_threshold <= 256 && !old_products) {
        // once per graph: the static staging layout of every slice; buffers
        // sized to the largest slice plus the zero words (chains <=
        // long_threshold), capped by the 10-bit run starts
        g.prod_zw = (std::max<uint32_t>(g.long_threshold, 4) + 3) & ~3u;
        DevBuf<unsigned> mx(1, s);
        QVB_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned), s));
        k_stage_words<<<grid_for(g.nm_S, 256), 256, 0, s>>>(nseg, g.nm_S, g.nm_sbase, mx.p);
        QVB_LAUNCH_CHECK();
        const unsigned most = read_scalar(mx.p, s);
        g.prod_bufw = std::min<uint32_t>(kPtMaxBufw, (most + g.prod_zw + 31) & ~31u);
        if (const char* bw = std::getenv("QVB_PT_BUFW")) {  // tests: force a buffer size (slices beyond it take the global path)
          const uint32_t w = static_cast<uint32_t>(std::atoi(bw)) & ~31u;
          if (w >= g.prod_zw + 32 && w <= kPtMaxBufw) g.prod_bufw = w;
        }
        QVB_CUDA(cudaMalloc(&g.nm_desc, g.nm_S * nseg * sizeof(uint64_t)));
        QVB_CUDA(cudaMalloc(&g.nm_runs, g.nm_S * 32 * 2 * sizeof(uint64_t)));
        g.bytes += g.nm_S * nseg * sizeof(uint64_t) + g.nm_S * 32 * 2 * sizeof(uint64_t);
        DevBuf<unsigned> big(1, s);
        QVB_CUDA(cudaMemsetAsync(big.p, 0, sizeof(unsigned), s));
        k_build_runs<<<grid_for(g.nm_S * 32, 256), 256, 0, s>>>(
            nseg, g.nm_S, g.nm_lenf, g.nm_sbase, g.prod_bufw, g.prod_zw, g.nm_desc,
            reinterpret_cast<ulonglong2*>(g.nm_runs), big.p);
        QVB_LAUNCH_CHECK();
        g.prod_big = read_scalar(big.p, s);
        const size_t smem = (size_t)kPtWarps * pt_warp_bytes(g.prod_bufw);
        // always the largest buffer any graph can ask for: graphs built on
        // other threads (or devices) set the same value, so none of them can
        // leave the attribute below another graph's launch size
        QVB_CUDA(cudaFuncSetAttribute(k_products_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>((size_t)kPtWarps * pt_warp_bytes(kPtMaxBufw))));
        g.prod_grid = resident_grid(k_products_tma, kPtWarps * 32, smem,
                                    (g.nm_S + kPtWarps - 1) / kPtWarps);
      }
      pt.begin(2);
      if (g.prod_bufw && !old_products) {
        const size_t smem = (size_t)kPtWarps * pt_warp_bytes(g.prod_bufw);
        k_products_tma<<<g.prod_grid, kPtWarps * 32, smem, s>>>(
            nseg, g.nm_S, sharded ? s0 : 0, sharded ? s1 : g.nm_S, n, g.nm_lenf, g.nm_desc, reinterpret_cast<const ulonglong2*>(g.nm_runs),
            g.nm_sbase, g.nm_code, g.nm_col, g.exc_src, g.exc_R, g.p[cur], g.inv, pout, kout,
            g.marked, g.prod_bufw, g.prod_zw);
      } else {
        k_products<<<static_cast<unsigned>((g.nm_S + kWarpsPerBlock - 1) / kWarpsPerBlock),
                     kWarpsPerBlock * 32, 0, s>>>(nseg, g.nm_S, n, g.nm_lenf, g.nm_sbase, g.nm_code,
                                                  g.nm_col, g.exc_src, g.exc_R, g.p[cur], g.inv,
                                                  pout, kout, g.marked);
      }
      QVB_LAUNCH_CHECK();
      pt.end(1);
      exchange();
      continue;
    }

    const double fbase = (first && !compact) ? base : 0.0;  // weighted first sweep: no gathers
    pt.begin(3);
    uint32_t launched = 0;
    if (g.nm) {  // node-major weighted passes, carrying the running products
      for (int k = 0; k < nseg; ++k) {
        const uint64_t lb = k == 0 ? long_blocks : 0;
        const uint64_t blocks = lb + (g.nm_S + kWarpsPerBlock - 1) / kWarpsPerBlock;
        k_sweep_nm<<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
            k, g.nm_S, lb, g.nlong, pf, g.nm_lenf, g.nm_sbase, g.nm_col, g.nm_R, g.state, g.lnode,
            g.lptr, g.lcol, g.lR, g.p[cur], g.inv, pout, gmode, fbase);
        QVB_LAUNCH_CHECK();
        ++launched;
      }
    } else {
      // sliced passes: pass k multiplies the factors of source segment k; the
      // long rows ride along in the first pass's grid (their blocks first)
      for (int k = 0; k < nseg; ++k) {
        const uint64_t s0 = g.seg_slice[k], s1 = g.seg_slice[k + 1];
        const uint64_t lb = k == 0 ? long_blocks : 0;
        const uint64_t blocks = lb + (s1 - s0 + kWarpsPerBlock - 1) / kWarpsPerBlock;
        if (blocks == 0) continue;
        if (compact) {
          k_sweep<false><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
              s0, s1, lb, g.nlong, pf, g.nslices, g.state, g.perm, g.sptr, g.scol, nullptr, g.lnode,
              g.lptr, g.lcol, nullptr, g.exc_src, g.exc_R, g.p[cur], g.y[cur], g.inv, pout, yout,
              gmode, 0.0);
        } else {
          k_sweep<true><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
              s0, s1, lb, g.nlong, pf, g.nslices, g.state, g.perm, g.sptr, g.scol, g.sR, g.lnode,
              g.lptr, g.lcol, g.lR, nullptr, nullptr, g.p[cur], nullptr, g.inv, pout, nullptr,
              gmode, fbase);
        }
        QVB_LAUNCH_CHECK();
        ++launched;
      }
    }
    pt.end(launched);
  }
  QVB_CUDA(cudaEventRecord(g.ev[1], s));
  if (final_out && (layers == 1 || sharded)) {
    QVB_CUDA(cudaMemcpyAsync(final_out, g.p[(layers - 1) & 1], n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return final_out;
  }
  return final_out ? final_out : g.p[(layers - 1) & 1];
}

}  // namespace qvb

using namespace qvb;

extern "C" int qvb_access_prob(qvb_graph* g, uint32_t layers, double* out, int out_on_device,
                               void* stream) {
  return guarded([&] {
    if (!g || !out) fail(QVB_ERR_VALIDATION, "null argument");
    if (layers < 1) fail(QVB_ERR_VALIDATION, "access probability needs layers >= 1");
    DeviceGuard dg(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g->run_mu);
    if (!g->done) QVB_CUDA(cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming));
    QVB_CUDA(cudaStreamWaitEvent(s, g->done, 0));  // the previous call's buffers are free
    if (out_on_device) {  // the last sweep writes the caller's buffer itself
      run_access_prob(*g, layers, s, out);
      QVB_CUDA(cudaEventRecord(g->done, s));
    } else {
      const double* p = run_access_prob(*g, layers, s);
      QVB_CUDA(cudaEventRecord(g->done, s));
      copy_to_host(out, p, g->n * sizeof(double), s);
    }
  });
}

extern "C" int qvb_access_prob_sharded(qvb_graph* g, uint32_t layers, uint32_t rank, uint32_t world,
                                       qvb_exchange_fn exchange, void* ctx, double* out,
                                       int out_on_device, void* stream, int* sharded) {
  return guarded([&] {
    if (!g || !out) fail(QVB_ERR_VALIDATION, "null argument");
    if (layers < 1) fail(QVB_ERR_VALIDATION, "access probability needs layers >= 1");
    if (world < 1 || rank >= world) fail(QVB_ERR_VALIDATION, "rank out of range");
    if (world > 1 && !exchange) fail(QVB_ERR_VALIDATION, "a sharded call needs an exchange callback");
    DeviceGuard dg(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g->run_mu);
    if (!g->done) QVB_CUDA(cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming));
    QVB_CUDA(cudaStreamWaitEvent(s, g->done, 0));
    Shard sh;
    sh.rank = rank;
    sh.world = world;
    sh.fn = exchange;
    sh.ctx = ctx;
    const double* p = run_access_prob(*g, layers, s, out_on_device ? out : nullptr, sh);
    QVB_CUDA(cudaEventRecord(g->done, s));
    if (!out_on_device) copy_to_host(out, p, g->n * sizeof(double), s);
    if (sharded) *sharded = g->last_sharded ? 1 : 0;
  });
}

extern "C" int qvb_compute_access_prob_ie(int device, uint64_t n, uint64_t e,
                                          const uint64_t* row_offsets, const uint64_t* col,
                                          const double* weights, uint32_t layers, double* out,
                                          double* ms_out) {
  qvb_graph* g = nullptr;
  int rc = guarded([&] {
    if (layers < 1) fail(QVB_ERR_VALIDATION, "access probability needs layers >= 1");
    if (!out) fail(QVB_ERR_VALIDATION, "null argument");
  });
  if (rc) return rc;
  cudaStream_t s = nullptr;
  cudaEvent_t ev[4] = {};
  rc = guarded([&] {
    DeviceGuard dg(device);
    QVB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (auto& x : ev) QVB_CUDA(cudaEventCreate(&x));
    QVB_CUDA(cudaEventRecord(ev[0], s));
  });
  if (rc) return rc;
  rc = qvb_graph_upload(device, n, e, row_offsets, col, weights, s, &g);
  if (rc == 0) {
    rc = guarded([&] {
      DeviceGuard dg(device);
      QVB_CUDA(cudaEventRecord(ev[1], s));
      const double* p = run_access_prob(*g, layers, s);
      QVB_CUDA(cudaEventRecord(ev[2], s));
      QVB_CUDA(cudaEventSynchronize(ev[2]));
      const auto t0 = std::chrono::steady_clock::now();
      copy_to_host(out, p, n * sizeof(double), s);  // returns when out is filled
      const double dl_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms_out) {
        for (int i = 0; i < 2; ++i) {
          float ms = 0;
          QVB_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
          ms_out[i] = ms;
        }
        ms_out[2] = dl_ms;  // host clock: the copy runs on the staging threads' streams
      }
    });
  }
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  if (g) delete g;
  for (auto& x : ev)
    if (x) cudaEventDestroy(x);
  if (s) cudaStreamDestroy(s);
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}
