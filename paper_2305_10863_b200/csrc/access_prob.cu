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

#include "graph.cuh"

namespace qvb {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kU = 8;  // sliced steps in flight per lane
constexpr int kLongU = 4;
constexpr unsigned kFull = 0xffffffffu;

__global__ void k_init(uint64_t n, const double* __restrict__ inv, double* __restrict__ p,
                       double* __restrict__ y) {
  const double base = __ddiv_rn(1.0, static_cast<double>(n));  // metrics.cpp:143
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const bool real = i < n;
    p[i] = real ? base : 0.0;  // slot N: the padding operand
    if (y) y[i] = real ? __dmul_rn(base, inv[i]) : 0.0;
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
                                       double* __restrict__ yout, uint64_t pol) {
  const double p = prev[v];
  // metrics.cpp:169: prev + (1 - prev) * (1 - miss_all)
  const double P = __dadd_rn(p, __dmul_rn(__dsub_rn(1.0, p), __dsub_rn(1.0, miss)));
  st_stream(out + v, P, pol);
  if (yout) st_stream(yout + v, __dmul_rn(P, inv[v]), pol);
}

template <bool kWeighted>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_sweep(uint64_t s0, uint64_t s1, uint64_t long_blocks, uint64_t nlong, double* __restrict__ state,
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
    const uint64_t i = (uint64_t)blockIdx.x * kWarpsPerBlock + wib;
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
    if (lane == 0) finish<kWeighted>(lnode[i], miss, prev, inv, out, yout, pol);
    return;
  }

  // ---- sliced rows: one warp per slice of 32 (node, pass) slots
  const uint64_t s = s0 + ((uint64_t)blockIdx.x - long_blocks) * kWarpsPerBlock + wib;
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
  if (pv & kLast) finish<kWeighted>(v, miss, prev, inv, out, yout, pol);
  else st_stream(state + v, miss, pol);
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
  k_init<<<grid_for(n + 1, 256), 256, 0, s>>>(n, g.inv, g.p[0], (compact && layers >= 2) ? g.y[0] : nullptr);
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
  int persist_mb = 0;
  if (const char* m = std::getenv("QVB_L2_PERSIST_MB")) persist_mb = std::atoi(m);
  if (persist_mb > 0) {
    QVB_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_mb << 20));
  }
  QVB_CUDA(cudaEventRecord(g.ev[0], s));
  for (uint32_t j = 2; j <= layers; ++j) {
    const int cur = (j - 2) & 1, nxt = cur ^ 1;
    double* yout = (compact && j < layers) ? g.y[nxt] : nullptr;
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
          QVB_CUDA(cudaLaunchKernelEx(&cfg, k_sweep<false>, s0, s1, lb, g.nlong, g.state,
                                      (const uint32_t*)g.perm, (const uint64_t*)g.sptr,
                                      (const uint32_t*)g.scol, (const double*)nullptr,
                                      (const uint32_t*)g.lnode, (const uint64_t*)g.lptr,
                                      (const uint32_t*)g.lcol, (const double*)nullptr,
                                      (const uint32_t*)g.exc_src, (const double*)g.exc_R,
                                      (const double*)g.p[cur], (const double*)g.y[cur],
                                      (const double*)g.inv, g.p[nxt], yout, gmode));
        else
          QVB_CUDA(cudaLaunchKernelEx(&cfg, k_sweep<true>, s0, s1, lb, g.nlong, g.state,
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
            s0, s1, lb, g.nlong, g.state, g.perm, g.sptr, g.scol, nullptr, g.lnode, g.lptr,
            g.lcol, nullptr, g.exc_src, g.exc_R, g.p[cur], g.y[cur], g.inv, g.p[nxt], yout, gmode);
      } else {
        k_sweep<true><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, s>>>(
            s0, s1, lb, g.nlong, g.state, g.perm, g.sptr, g.scol, g.sR, g.lnode, g.lptr, g.lcol,
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
