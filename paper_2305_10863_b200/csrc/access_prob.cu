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
#include <cstdlib>
#include <string>

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
                                         int gmode, uint64_t pol) {
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
        const double v = (!kWeighted && (c & kExcFlag)) ? 0.0 : ld_gather(opnd + c, gmode);
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
            int gmode) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  // kWeighted gathers P(s, j-1); compact gathers y(s, j-1)
  const double* __restrict__ opnd = kWeighted ? prev : yprev;

  if (blockIdx.x < long_blocks) {  // ---- long rows: one warp per row
    long_row<kWeighted>((uint64_t)blockIdx.x * kWarpsPerBlock + wib, nlong, lnode, lptr, lcol, lR,
                        exc_src, exc_R, prev, opnd, inv, out, yout, nullptr, gmode, pol);
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
      x[u] = (in && (kWeighted || !(c[u] & kExcFlag))) ? ld_gather(opnd + c[u], gmode) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (k + u < len) miss = __dmul_rn(miss, factor<kWeighted>(c[u], x[u], r[u], exc_src, exc_R, prev));
  }
  if (v == kNoNode) return;
  if (pv & kLast) finish<kWeighted>(v, miss, prev, inv, out, yout, nullptr, pol);
  else st_stream(state + v, miss, pol);
}

// Node-major segmented pass k (graph.cuh "nm"): one warp per slice of 32
// consecutive node ids, lane = node in every pass, so the running product,
// P, y and the code are read and written coalesced and without a perm word;
// the lane's pass-k sources start at sbase(k, slice) + the prefix of the
// slice's lens. Compact sweeps gather the 4-byte code of y (exact, see
// graph.cuh) and fall back to y for kBigCode sources.
template <bool kWeighted>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_sweep_nm(int k, uint64_t S, uint64_t long_blocks, uint64_t nlong, uint64_t pf,
               const uint8_t* __restrict__ lenf, const uint64_t* __restrict__ sbase,
               const uint32_t* __restrict__ ncol, const double* __restrict__ nR,
               double* __restrict__ state, const uint32_t* __restrict__ lnode,
               const uint64_t* __restrict__ lptr, const uint32_t* __restrict__ lcol,
               const double* __restrict__ lR, const uint32_t* __restrict__ exc_src,
               const double* __restrict__ exc_R, const double* __restrict__ prev,
               const double* __restrict__ yprev, const uint32_t* __restrict__ kprev,
               const double* __restrict__ inv, double* __restrict__ out,
               double* __restrict__ yout, uint32_t* __restrict__ kout, int gmode) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t pol = policy_evict_first();
  const uint64_t keep = policy_evict_last();
  if (blockIdx.x < long_blocks) {
    long_row<kWeighted>((uint64_t)blockIdx.x * kWarpsPerBlock + wib, nlong, lnode, lptr, lcol, lR,
                        exc_src, exc_R, prev, kWeighted ? prev : yprev, inv, out, yout, kout,
                        gmode, pol);
    return;
  }
  const uint64_t s_block = ((uint64_t)blockIdx.x - long_blocks) * kWarpsPerBlock;
  const uint64_t sl = s_block + wib;
  if (pf && wib == kWarpsPerBlock - 1 && lane == 0) {
    // L2 lookahead (see prefetch_ahead): lens, slice pointers and running
    // products of the block pf ahead, columns (and R) of the block pf/2 ahead
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
        if constexpr (kWeighted) prefetch_l2(nR + a, (b - a) * sizeof(double));
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
      if constexpr (kWeighted) r[u] = in ? ld_stream(nR + off + t + u, pol) : 0.0;
      else r[u] = 0.0;
    }
    if constexpr (kWeighted) {
#pragma unroll
      for (int u = 0; u < kU; ++u) x[u] = t + u < len ? ld_gather(prev + c[u], gmode) : 0.0;
    } else {
      // all codes in flight first; the rare y fallbacks after (no load waits
      // on a branch over an earlier load)
      uint32_t code[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        code[u] = (t + u < len && !(c[u] & kExcFlag))
                      ? (gmode == 3 ? ld_hint(kprev + c[u], keep) : __ldg(kprev + c[u]))
                      : 0u;
#pragma unroll
      for (int u = 0; u < kU; ++u)  // J * 2^-53 is exact; 1 - it rounds like 1 - y
        x[u] = __dmul_rn(static_cast<double>(code[u]), 0x1p-53);
      bool big = false;
#pragma unroll
      for (int u = 0; u < kU; ++u) big |= code[u] == kBigCode;
      if (big) {
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (code[u] == kBigCode) x[u] = ld_gather(yprev + c[u], gmode);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (t + u < len) miss = __dmul_rn(miss, factor<kWeighted>(c[u], x[u], r[u], exc_src, exc_R, prev));
  }
  if (lf & kNmLast) finish<kWeighted>(static_cast<uint32_t>(v), miss, prev, inv, out, yout, kout, pol);
  else if (len) st_stream(state + v, miss, pol);
}

// ---- node-major passes with TMA-staged streams ----------------------------
// The same pass as k_sweep_nm, restructured so that a slice's only global
// reads on the critical path are its operand gathers: a producer warp
// streams each chunk of kNmChunk slices — their lenf bytes, slice pointers,
// running products and columns, all contiguous — into a shared-memory stage
// with cp.async.bulk (mbarrier full/empty pipeline, kNmStages deep), and 8
// consumer warps work from shared memory.
constexpr int kNmChunk = 16;       // slices per chunk (512 nodes)
constexpr int kNmStages = 2;
constexpr uint32_t kNmColCap = 7680;  // columns per stage; larger chunks read global
constexpr int kNmConsumers = 8;
constexpr int kNmThreads = (kNmConsumers + 1) * 32;

struct alignas(128) NmStage {
  double st[kNmChunk * 32];
  uint32_t col[kNmColCap + 8];
  uint64_t sb[kNmChunk + 4];
  uint8_t lenf[kNmChunk * 32];
  uint64_t col_lo;  // global column index of col[0]; ~0: this chunk reads global
  uint32_t ns;      // slices in the chunk
  uint32_t sb_off;  // (k*S + first slice) - index of sb[0]
};

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(kNmThreads)
    k_sweep_nm_tma(int k, uint64_t S, uint64_t nchunks, const uint8_t* __restrict__ lenf,
                   const uint64_t* __restrict__ sbase, const uint32_t* __restrict__ ncol,
                   double* __restrict__ state, const uint32_t* __restrict__ exc_src,
                   const double* __restrict__ exc_R, const double* __restrict__ prev,
                   const double* __restrict__ yprev, const uint32_t* __restrict__ kprev,
                   const double* __restrict__ inv, double* __restrict__ out,
                   double* __restrict__ yout, uint32_t* __restrict__ kout, int gmode) {
  extern __shared__ __align__(128) unsigned char smem[];
  NmStage* stg = reinterpret_cast<NmStage*>(smem);
  __shared__ __align__(8) uint64_t full[kNmStages], empty[kNmStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNmStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&full[i]))));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&empty[i]))),
                   "r"(kNmConsumers));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine =
      blockIdx.x < nchunks ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp == kNmConsumers) {  // ---- producer
    if (lane != 0) return;
    uint64_t c0n = 0, c1n = 0;
    auto bounds = [&](uint64_t it, uint64_t& i0, uint32_t& ns) {
      const uint64_t a = (blockIdx.x + it * gridDim.x) * kNmChunk;
      ns = static_cast<uint32_t>(S - a < kNmChunk ? S - a : kNmChunk);
      i0 = (uint64_t)k * S + a;
    };
    if (mine) {
      uint64_t i0;
      uint32_t ns;
      bounds(0, i0, ns);
      c0n = sbase[i0];
      c1n = sbase[i0 + ns];
    }
    for (uint64_t it = 0; it < mine; ++it) {
      const int si = static_cast<int>(it % kNmStages);
      uint64_t i0;
      uint32_t ns;
      bounds(it, i0, ns);
      const uint64_t c0 = c0n, c1 = c1n;
      if (it + 1 < mine) {  // next chunk's column range: in flight during the wait
        uint64_t j0;
        uint32_t nn;
        bounds(it + 1, j0, nn);
        c0n = sbase[j0];
        c1n = sbase[j0 + nn];
      }
      if (it >= kNmStages)
        mbar_wait(static_cast<uint32_t>(__cvta_generic_to_shared(&empty[si])),
                  static_cast<uint32_t>((it / kNmStages - 1) & 1));
      NmStage& st = stg[si];
      const uint64_t a = i0 - (uint64_t)k * S;
      const uint64_t sb_lo = i0 & ~1ull, sb_hi = (i0 + ns + 2) & ~1ull;
      const uint64_t col_lo = c0 & ~3ull, col_hi = (c1 + 3) & ~3ull;
      const bool cols_in = col_hi - col_lo <= kNmColCap;
      st.ns = ns;
      st.sb_off = static_cast<uint32_t>(i0 - sb_lo);
      st.col_lo = cols_in ? col_lo : ~0ull;
      const uint32_t b_len = ns * 32, b_sb = static_cast<uint32_t>((sb_hi - sb_lo) * 8);
      const uint32_t b_st = k > 0 ? ns * 32 * 8 : 0;
      const uint32_t b_col = cols_in ? static_cast<uint32_t>((col_hi - col_lo) * 4) : 0;
      const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&full[si]));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(b_len + b_sb + b_st + b_col)
                   : "memory");
      bulk_g2s(st.lenf, lenf + i0 * 32, b_len, bar);
      bulk_g2s(st.sb, sbase + sb_lo, b_sb, bar);
      if (b_st) bulk_g2s(st.st, state + a * 32, b_st, bar);
      if (b_col) bulk_g2s(st.col, ncol + col_lo, b_col, bar);
    }
    return;
  }

  // ---- consumers
  const uint64_t pol = policy_evict_first();
  for (uint64_t it = 0; it < mine; ++it) {
    const int si = static_cast<int>(it % kNmStages);
    mbar_wait(static_cast<uint32_t>(__cvta_generic_to_shared(&full[si])),
              static_cast<uint32_t>((it / kNmStages) & 1));
    const NmStage& st = stg[si];
    const uint32_t ns = st.ns;
    const uint64_t col_lo = st.col_lo;
    const uint64_t a = (blockIdx.x + it * gridDim.x) * kNmChunk;
    for (uint32_t q = warp; q < ns; q += kNmConsumers) {
      const uint64_t v = (a + q) * 32 + lane;
      const uint32_t lf = st.lenf[q * 32 + lane];
      if (__ballot_sync(kFull, lf != 0) == 0) continue;
      const uint32_t len = lf & kNmLen;
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t maxlen = __reduce_max_sync(kFull, len);
      const uint64_t cs = st.sb[st.sb_off + q] + (incl - len);  // global column index
      const bool last = lf & kNmLast;
      double pv = 0.0, iv = 0.0;
      if (last) {  // finish operands early, off the critical path
        pv = prev[v];
        if (yout) iv = inv[v];
      }
      double miss = (lf != 0 && !(lf & kNmFirst)) ? st.st[q * 32 + lane] : 1.0;
      for (uint32_t t = 0; t < maxlen; t += kU) {
        uint32_t c[kU], code[kU];
        double x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const bool in = t + u < len;
          c[u] = !in ? 0u
                     : (col_lo != ~0ull ? st.col[cs + t + u - col_lo]
                                        : ld_stream(ncol + cs + t + u, pol));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
          code[u] = (t + u < len && !(c[u] & kExcFlag)) ? __ldg(kprev + c[u]) : 0u;
#pragma unroll
        for (int u = 0; u < kU; ++u) x[u] = __dmul_rn(static_cast<double>(code[u]), 0x1p-53);
        bool big = false;
#pragma unroll
        for (int u = 0; u < kU; ++u) big |= code[u] == kBigCode;
        if (big) {
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if (code[u] == kBigCode) x[u] = ld_gather(yprev + c[u], gmode);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (t + u < len) miss = __dmul_rn(miss, factor<false>(c[u], x[u], 0.0, exc_src, exc_R, prev));
      }
      if (last) {
        // metrics.cpp:169, as finish()
        const double P = __dadd_rn(pv, __dmul_rn(__dsub_rn(1.0, pv), __dsub_rn(1.0, miss)));
        st_stream(out + v, P, pol);
        if (yout) {
          const double y = __dmul_rn(P, iv);
          st_stream(yout + v, y, pol);
          if (kout) kout[v] = y_code(y);
        }
      } else if (len) {
        st_stream(state + v, miss, pol);
      }
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&empty[si])))
                   : "memory");
  }
}

}  // namespace

const double* run_access_prob(qvb_graph& g, uint32_t layers, cudaStream_t s) {
  if (layers < 1) fail(QVB_ERR_VALIDATION, "access probability needs layers >= 1");
  const uint64_t n = g.n;
  const bool compact = g.layout == 0;
  for (int i = 0; i < 2; ++i) {
    if (!g.p[i]) QVB_CUDA(cudaMalloc(&g.p[i], (n + 1) * sizeof(double)));
    if (compact && !g.y[i]) QVB_CUDA(cudaMalloc(&g.y[i], (n + 1) * sizeof(double)));
  }
  // both ping-pong buffers carry the zero padding operand at index N
  const bool codes = g.nm && compact;
  if (codes)
    for (int i = 0; i < 2; ++i)
      if (!g.kcode[i]) QVB_CUDA(cudaMalloc(&g.kcode[i], (n + 1) * sizeof(uint32_t)));
  k_init<<<grid_for(n + 1, 256), 256, 0, s>>>(n, g.inv, g.p[0], (compact && layers >= 2) ? g.y[0] : nullptr,
                                             (codes && layers >= 2) ? g.kcode[0] : nullptr);
  QVB_LAUNCH_CHECK();
  if (layers >= 3) {
    QVB_CUDA(cudaMemsetAsync(g.p[1] + n, 0, sizeof(double), s));
    if (compact) QVB_CUDA(cudaMemsetAsync(g.y[1] + n, 0, sizeof(double), s));
  }
  const uint64_t long_blocks = (g.nlong + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int nseg = static_cast<int>(g.seg_slice.size()) - 1;
  for (auto& e : g.ev)
    if (!e) QVB_CUDA(cudaEventCreate(&e));
  int gmode = 0;
  if (const char* m = std::getenv("QVB_GATHER_MODE")) gmode = std::atoi(m);
  // L2 lookahead in blocks for the sliced passes (QVB_PF_BLOCKS; 0 = off);
  // worthwhile only when the streams do not already sit in L2
  uint64_t pf = nseg > 1 ? 512 : 0;
  if (const char* m = std::getenv("QVB_PF_BLOCKS")) pf = std::strtoull(m, nullptr, 10);
  int persist_mb = 0;
  if (const char* m = std::getenv("QVB_L2_PERSIST_MB")) persist_mb = std::atoi(m);
  if (persist_mb > 0) {
    QVB_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_mb << 20));
  }
  unsigned tma_grid = 0;  // persistent grid of the TMA-staged node-major kernel
  const char* nm_kernel = std::getenv("QVB_NM_KERNEL");
  if (g.nm && compact && nm_kernel && std::string(nm_kernel) == "tma") {
    const int smem = static_cast<int>(sizeof(NmStage) * kNmStages);
    QVB_CUDA(cudaFuncSetAttribute(k_sweep_nm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const uint64_t nchunks = (g.nm_S + kNmChunk - 1) / kNmChunk;
    tma_grid = resident_grid(k_sweep_nm_tma, kNmThreads, smem, nchunks);
  }
  QVB_CUDA(cudaEventRecord(g.ev[0], s));
  for (uint32_t j = 2; j <= layers; ++j) {
    const int cur = (j - 2) & 1, nxt = cur ^ 1;
    double* yout = (compact && j < layers) ? g.y[nxt] : nullptr;
    if (g.nm && compact && tma_grid) {  // node-major passes, TMA-staged
      uint32_t* kout = (codes && j < layers) ? g.kcode[nxt] : nullptr;
      const uint64_t nchunks = (g.nm_S + kNmChunk - 1) / kNmChunk;
      for (int k = 0; k < nseg; ++k) {
        if (k == 0 && long_blocks) {  // long rows: the warp-per-row path, full rows
          k_sweep_nm<false><<<static_cast<unsigned>(long_blocks), kWarpsPerBlock * 32, 0, s>>>(
              0, 0, long_blocks, g.nlong, 0, g.nm_lenf, g.nm_sbase, g.nm_col, nullptr, g.state,
              g.lnode, g.lptr, g.lcol, nullptr, g.exc_src, g.exc_R, g.p[cur], g.y[cur],
              g.kcode[cur], g.inv, g.p[nxt], yout, kout, gmode);
          QVB_LAUNCH_CHECK();
        }
        k_sweep_nm_tma<<<tma_grid, kNmThreads, sizeof(NmStage) * kNmStages, s>>>(
            k, g.nm_S, nchunks, g.nm_lenf, g.nm_sbase, g.nm_col, g.state, g.exc_src, g.exc_R,
            g.p[cur], g.y[cur], g.kcode[cur], g.inv, g.p[nxt], yout, kout, gmode);
        QVB_LAUNCH_CHECK();
      }
      continue;
    }
    if (g.nm) {  // node-major passes
      uint32_t* kout = (codes && j < layers) ? g.kcode[nxt] : nullptr;
      for (int k = 0; k < nseg; ++k) {
        const uint64_t lb = k == 0 ? long_blocks : 0;
        const uint64_t blocks = lb + (g.nm_S + kWarpsPerBlock - 1) / kWarpsPerBlock;
        if (compact)
          k_sweep_nm<false><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
              k, g.nm_S, lb, g.nlong, pf, g.nm_lenf, g.nm_sbase, g.nm_col, nullptr, g.state, g.lnode,
              g.lptr, g.lcol, nullptr, g.exc_src, g.exc_R, g.p[cur], g.y[cur], g.kcode[cur],
              g.inv, g.p[nxt], yout, kout, gmode);
        else
          k_sweep_nm<true><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
              k, g.nm_S, lb, g.nlong, pf, g.nm_lenf, g.nm_sbase, g.nm_col, g.nm_R, g.state, g.lnode,
              g.lptr, g.lcol, g.lR, nullptr, nullptr, g.p[cur], nullptr, nullptr, g.inv,
              g.p[nxt], nullptr, nullptr, gmode);
        QVB_LAUNCH_CHECK();
      }
      continue;
    }
    // pass k multiplies the factors of source segment k; the long rows ride
    // along in the first pass's grid (their blocks first)
    for (int k = 0; k < nseg; ++k) {
      const uint64_t s0 = g.seg_slice[k], s1 = g.seg_slice[k + 1];
      const uint64_t lb = k == 0 ? long_blocks : 0;
      const uint64_t blocks = lb + (s1 - s0 + kWarpsPerBlock - 1) / kWarpsPerBlock;
      if (blocks == 0) continue;
      if (persist_mb > 0 && nseg > 1) {
        // experiment: pin this pass's operand slice in the persisting L2 carve-out
        const double* opnd = compact ? g.y[cur] : g.p[cur];
        const uint64_t first = (uint64_t)k * g.seg_size;
        const uint64_t count = std::min<uint64_t>(g.seg_size, n - first);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(blocks));
        cfg.blockDim = dim3(kWarpsPerBlock * 32);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = const_cast<double*>(opnd + first);
        attr[0].val.accessPolicyWindow.num_bytes = count * sizeof(double);
        attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (compact)
          QVB_CUDA(cudaLaunchKernelEx(&cfg, k_sweep<false>, s0, s1, lb, g.nlong, pf, g.nslices, g.state,
                                      (const uint32_t*)g.perm, (const uint64_t*)g.sptr,
                                      (const uint32_t*)g.scol, (const double*)nullptr,
                                      (const uint32_t*)g.lnode, (const uint64_t*)g.lptr,
                                      (const uint32_t*)g.lcol, (const double*)nullptr,
                                      (const uint32_t*)g.exc_src, (const double*)g.exc_R,
                                      (const double*)g.p[cur], (const double*)g.y[cur],
                                      (const double*)g.inv, g.p[nxt], yout, gmode));
        else
          QVB_CUDA(cudaLaunchKernelEx(&cfg, k_sweep<true>, s0, s1, lb, g.nlong, pf, g.nslices, g.state,
                                      (const uint32_t*)g.perm, (const uint64_t*)g.sptr,
                                      (const uint32_t*)g.scol, (const double*)g.sR,
                                      (const uint32_t*)g.lnode, (const uint64_t*)g.lptr,
                                      (const uint32_t*)g.lcol, (const double*)g.lR,
                                      (const uint32_t*)nullptr, (const double*)nullptr,
                                      (const double*)g.p[cur], (const double*)nullptr,
                                      (const double*)g.inv, g.p[nxt], (double*)nullptr, gmode));
        continue;
      }
      if (compact) {
        k_sweep<false><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
            s0, s1, lb, g.nlong, pf, g.nslices, g.state, g.perm, g.sptr, g.scol, nullptr, g.lnode, g.lptr,
            g.lcol, nullptr, g.exc_src, g.exc_R, g.p[cur], g.y[cur], g.inv, g.p[nxt], yout, gmode);
      } else {
        k_sweep<true><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
            s0, s1, lb, g.nlong, pf, g.nslices, g.state, g.perm, g.sptr, g.scol, g.sR, g.lnode, g.lptr, g.lcol,
            g.lR, nullptr, nullptr, g.p[cur], nullptr, g.inv, g.p[nxt], nullptr, gmode);
      }
      QVB_LAUNCH_CHECK();
    }
  }
  QVB_CUDA(cudaEventRecord(g.ev[1], s));
  return g.p[(layers - 1) & 1];
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
    const double* p = run_access_prob(*g, layers, s);
    QVB_CUDA(cudaMemcpyAsync(out, p, g->n * sizeof(double),
                             out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    if (!out_on_device) QVB_CUDA(cudaStreamSynchronize(s));
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
      QVB_CUDA(cudaMemcpyAsync(out, p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
      QVB_CUDA(cudaEventRecord(ev[3], s));
      QVB_CUDA(cudaStreamSynchronize(s));
      if (ms_out) {
        for (int i = 0; i < 3; ++i) {
          float ms = 0;
          QVB_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
          ms_out[i] = ms;
        }
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
