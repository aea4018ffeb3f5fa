// access_prob.cu — K1: the analytical access-probability estimator P(n,j)
// (reference metrics.cpp:134-173, compute_access_prob_ie), as a per-layer
// CSR pull over the device in-CSR of graph.cu.
//
// Exactness. The reference multiplies a node's factors (1 - P(s,j-1)*R(s,n))
// strictly left to right in ascending source order, and its cancellation-
// prone 1 - prod makes any re-association visible at 1e-9. So a
// node's product is ONE sequential chain of __dmul_rn in the reference order;
// every op is an explicit round-to-nearest intrinsic (no FMA contraction).
// Parallelism is across nodes and across the gathers of a chunk:
//
//   warp  = 32 consecutive destination nodes (lane l owns node 32w+l)
//   chunk = up to 256 consecutive in-edges of those nodes
//   phase A: the 32 lanes load the chunk's col (coalesced) and gather the
//            source operands (8 independent 8-byte gathers per lane in
//            flight), form the factors and stage them in shared memory
//   phase B: every lane multiplies the factors of its own node's slice of
//            the chunk into its running product, in order; the product
//            carries across chunks, so hub rows of any length work.
//
// Compact layout: the gathered operand is y[s] = P(s,j-1) * (1/row_sum(s)),
// produced by the previous sweep's epilogue, which equals the reference's
// P(s,j-1) * (w/row_sum(s)) bit for bit whenever w/row_sum == 1/row_sum (the
// exception table covers every other edge). One 8-byte gather per edge.
// Weighted layout: factor = 1 - P(s,j-1) * R_e with R_e streamed per edge.
#include "graph.cuh"

namespace qvb {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kChunk = 256;
constexpr int kPerLane = kChunk / 32;
constexpr unsigned kFull = 0xffffffffu;

__global__ void k_init(uint64_t n, const double* __restrict__ inv, double* __restrict__ p,
                       double* __restrict__ y) {
  const double base = __ddiv_rn(1.0, static_cast<double>(n));  // metrics.cpp:143
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    p[i] = base;
    if (y) y[i] = __dmul_rn(base, inv[i]);
  }
}

template <bool kWeighted>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_sweep(uint32_t n, const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ col,
            const double* __restrict__ R, const uint32_t* __restrict__ exc_src,
            const double* __restrict__ exc_R, const double* __restrict__ prev,
            const double* __restrict__ yprev, const double* __restrict__ inv,
            double* __restrict__ out, double* __restrict__ yout) {
  __shared__ double fbuf[kWarpsPerBlock][kChunk];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t node0 = ((uint64_t)blockIdx.x * kWarpsPerBlock + wib) * 32;
  if (node0 >= n) return;
  const uint64_t node = node0 + lane;
  const bool valid = node < n;
  const uint64_t last = node0 + 32 < n ? node0 + 32 : n;  // one past the warp's last node
  const uint64_t rs = uptr[valid ? node : last];
  const uint64_t end_all = uptr[last];
  uint64_t re = __shfl_down_sync(kFull, rs, 1);
  if (lane == 31) re = end_all;
  const uint64_t ebeg = __shfl_sync(kFull, rs, 0);
  double* fb = fbuf[wib];

  double miss = 1.0;  // metrics.cpp:152
  for (uint64_t cs = ebeg; cs < end_all; cs += kChunk) {
    const uint32_t cnt = static_cast<uint32_t>(end_all - cs < kChunk ? end_all - cs : kChunk);
    uint32_t c[kPerLane];
    double a[kPerLane];
    double v[kPerLane];
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
      const uint32_t idx = j * 32 + lane;
      c[j] = idx < cnt ? col[cs + idx] : 0u;
      if constexpr (kWeighted) a[j] = idx < cnt ? R[cs + idx] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
      const uint32_t idx = j * 32 + lane;
      if constexpr (kWeighted) {
        v[j] = idx < cnt ? prev[c[j]] : 0.0;
      } else {
        v[j] = (idx < cnt && !(c[j] & kExcFlag)) ? yprev[c[j]] : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
      const uint32_t idx = j * 32 + lane;
      if (idx < cnt) {
        double f;
        if constexpr (kWeighted) {
          f = __dsub_rn(1.0, __dmul_rn(v[j], a[j]));  // metrics.cpp:166
        } else if (c[j] & kExcFlag) {
          const uint32_t x = c[j] & ~kExcFlag;
          f = __dsub_rn(1.0, __dmul_rn(prev[exc_src[x]], exc_R[x]));
        } else {
          f = __dsub_rn(1.0, v[j]);
        }
        fb[idx] = f;
      }
    }
    __syncwarp();
    const uint64_t lo = rs > cs ? rs : cs;
    const uint64_t hi = re < cs + cnt ? re : cs + cnt;
    for (uint64_t e = lo; e < hi; ++e) miss = __dmul_rn(miss, fb[e - cs]);
    __syncwarp();
  }
  if (valid) {
    const double p = prev[node];
    // metrics.cpp:169: prev + (1 - prev) * (1 - miss_all)
    const double P = __dadd_rn(p, __dmul_rn(__dsub_rn(1.0, p), __dsub_rn(1.0, miss)));
    out[node] = P;
    if (yout) yout[node] = __dmul_rn(P, inv[node]);
  }
}

}  // namespace

const double* run_access_prob(qvb_graph& g, uint32_t layers, cudaStream_t s) {
  if (layers < 1) fail(QVB_ERR_VALIDATION, "access probability needs layers >= 1");
  const uint64_t n = g.n;
  for (int i = 0; i < 2; ++i) {
    if (!g.p[i]) QVB_CUDA(cudaMalloc(&g.p[i], n * sizeof(double)));
    if (g.layout == 0 && !g.y[i]) QVB_CUDA(cudaMalloc(&g.y[i], n * sizeof(double)));
  }
  const bool compact = g.layout == 0;
  k_init<<<grid_for(n, 256), 256, 0, s>>>(n, g.inv, g.p[0], (compact && layers >= 2) ? g.y[0] : nullptr);
  QVB_LAUNCH_CHECK();
  const uint64_t warps = (n + 31) / 32;
  const unsigned grid = static_cast<unsigned>((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
  for (auto& e : g.ev)
    if (!e) QVB_CUDA(cudaEventCreate(&e));
  QVB_CUDA(cudaEventRecord(g.ev[0], s));
  for (uint32_t j = 2; j <= layers; ++j) {
    const int cur = (j - 2) & 1, nxt = cur ^ 1;
    double* yout = (compact && j < layers) ? g.y[nxt] : nullptr;
    if (compact) {
      k_sweep<false><<<grid, kWarpsPerBlock * 32, 0, s>>>(
          static_cast<uint32_t>(n), g.uptr, g.col, nullptr, g.exc_src, g.exc_R, g.p[cur],
          g.y[cur], g.inv, g.p[nxt], yout);
    } else {
      k_sweep<true><<<grid, kWarpsPerBlock * 32, 0, s>>>(
          static_cast<uint32_t>(n), g.uptr, g.col, g.R, nullptr, nullptr, g.p[cur], nullptr,
          g.inv, g.p[nxt], nullptr);
    }
    QVB_LAUNCH_CHECK();
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
