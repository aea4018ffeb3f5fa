// fap.cu — the FAP visit-mass estimator (reference metrics.cpp:95-132,
// compute_fap; distribution_step metrics.cpp:42-58) on the device. This is
// the estimator the reference's own `qvserve plan` feeds to the placement
// manager (tools/qvserve.cpp:146-153); SURVEY §8(f) next-row #1.
//
//   p_0 = seed (uniform 1/|V| by default), values = p_0
//   p_k[i] = sum over in-edges (j -> i), transpose order, of
//            p_{k-1}[j] * w_e / row_sum(j)        (Neumaier-compensated)
//   values += p_k                                  for k = 1..hops
//
// Exactness: each node's compensated sum runs in the reference's order
// (ascending source, parallel edges separately, in CSR order), so the same
// sliced lane-owned-chain layout as K1 applies; padding slots add an exact
// 0.0. Unit weights: (p*1.0)/rs == p/rs, so the gathered operand is
// z(j) = p(j)/rs(j), formed once per source per hop. Real weights: the
// 16-byte pair (p(j), rs(j)) is gathered (one sector) and w_e streamed.
#include <algorithm>
#include <cmath>
#include <vector>

#include "graph.cuh"

namespace qvb {
namespace {

constexpr int kFapWarps = 8;
constexpr int kFapU = 8;
constexpr unsigned kFull = 0xffffffffu;

// NeumaierSum::add (include/qv/numeric.hpp:14-23)
__device__ __forceinline__ void nadd(double& sum, double& comp, double v) {
  const double t = __dadd_rn(sum, v);
  if (fabs(sum) >= fabs(v)) comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(sum, t), v));
  else comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(v, t), sum));
  sum = t;
}

__global__ void k_fap_operand(uint64_t n, const double* __restrict__ p, const double* __restrict__ rs,
                              double* __restrict__ z, double2* __restrict__ pr) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i == n) {  // padding operand: contributes exactly 0
      if (z) z[i] = 0.0;
      if (pr) pr[i] = make_double2(0.0, 1.0);
      continue;
    }
    const double r = rs[i];
    if (z) z[i] = r > 0.0 ? __ddiv_rn(p[i], r) : 0.0;
    if (pr) pr[i] = make_double2(p[i], r);
  }
}

template <bool kWeighted>
__device__ __forceinline__ double term(uint32_t c, double w, const double* __restrict__ z,
                                       const double2* __restrict__ pr) {
  if constexpr (kWeighted) {
    const double2 q = pr[c];
    // metrics.cpp:53 — p_in[j] * w / row_sum[j], left to right
    return q.y > 0.0 ? __ddiv_rn(__dmul_rn(q.x, w), q.y) : 0.0;
  } else {
    return z[c];
  }
}

template <bool kWeighted>
__global__ void __launch_bounds__(kFapWarps * 32)
    k_fap_step(uint64_t nslices, uint64_t long_blocks, uint64_t nlong,
               const uint32_t* __restrict__ perm, const uint64_t* __restrict__ sptr,
               const uint32_t* __restrict__ scol, const double* __restrict__ sW,
               const uint32_t* __restrict__ lnode, const uint64_t* __restrict__ lptr,
               const uint32_t* __restrict__ lcol, const double* __restrict__ lW,
               const double* __restrict__ z, const double2* __restrict__ pr,
               const double* __restrict__ values_in, double* __restrict__ values_out,
               double* __restrict__ p_out) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  if (blockIdx.x < long_blocks) {  // long rows: gathers in parallel, one sequential sum
    const uint64_t i = (uint64_t)blockIdx.x * kFapWarps + wib;
    if (i >= nlong) return;
    const uint64_t a = lptr[i], b = lptr[i + 1];
    double sum = 0.0, comp = 0.0;
    for (uint64_t cs = a; cs < b; cs += 32) {
      const uint64_t e = cs + lane;
      const double t = e < b ? term<kWeighted>(lcol[e], kWeighted ? lW[e] : 0.0, z, pr) : 0.0;
      const int cnt = static_cast<int>(b - cs < 32 ? b - cs : 32);
      for (int j = 0; j < cnt; ++j) nadd(sum, comp, __shfl_sync(kFull, t, j));
    }
    if (lane == 0) {
      const uint32_t v = lnode[i];
      const double next = __dadd_rn(sum, comp);
      p_out[v] = next;
      values_out[v] = __dadd_rn(values_in[v], next);
    }
    return;
  }
  const uint64_t s = ((uint64_t)blockIdx.x - long_blocks) * kFapWarps + wib;
  if (s >= nslices) return;
  const uint32_t v = perm[s * 32 + lane] & kNodeMask;
  const uint64_t base = sptr[s];
  const uint32_t len = static_cast<uint32_t>((sptr[s + 1] - base) >> 5);
  const uint32_t* cp = scol + base + lane;
  const double* wp = kWeighted ? sW + base + lane : nullptr;
  double sum = 0.0, comp = 0.0;
  for (uint32_t k = 0; k < len; k += kFapU) {
    uint32_t c[kFapU];
    double w[kFapU], t[kFapU];
#pragma unroll
    for (int u = 0; u < kFapU; ++u) {
      const bool in = k + u < len;
      c[u] = in ? cp[(uint64_t)(k + u) * 32] : 0u;
      w[u] = (kWeighted && in) ? wp[(uint64_t)(k + u) * 32] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kFapU; ++u) t[u] = k + u < len ? term<kWeighted>(c[u], w[u], z, pr) : 0.0;
#pragma unroll
    for (int u = 0; u < kFapU; ++u)
      if (k + u < len) nadd(sum, comp, t[u]);
  }
  if (v == kNoNode) return;
  const double next = __dadd_rn(sum, comp);  // NeumaierSum::value
  p_out[v] = next;
  values_out[v] = __dadd_rn(values_in[v], next);  // metrics.cpp:128
}

}  // namespace
}  // namespace qvb

using namespace qvb;

extern "C" int qvb_compute_fap(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                               const uint64_t* col, const double* weights, uint32_t hops,
                               const double* seed, double* values) {
  return guarded([&] {
    if (!values) fail(QVB_ERR_VALIDATION, "null argument");
    if (n == 0) fail(QVB_ERR_VALIDATION, "empty graph: node count is zero");
    // seed validation (metrics.cpp:100-112): non-negative, Neumaier total 1 +- 1e-12
    std::vector<double> p0(n);
    if (seed) {
      double sum = 0.0, comp = 0.0;
      for (uint64_t i = 0; i < n; ++i) {
        const double v = seed[i];
        if (!(v >= 0.0)) fail(QVB_ERR_VALIDATION, "seed distribution has negative mass");
        const double t = sum + v;
        if (std::fabs(sum) >= std::fabs(v)) comp += (sum - t) + v;
        else comp += (v - t) + sum;
        sum = t;
      }
      if (std::fabs((sum + comp) - 1.0) > 1e-12)
        fail(QVB_ERR_VALIDATION, "seed distribution does not sum to 1");
      std::copy(seed, seed + n, p0.begin());
    } else {
      std::fill(p0.begin(), p0.end(), 1.0 / static_cast<double>(n));
    }
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> tptr;
    DevBuf<uint32_t> tsrc;
    DevBuf<double> tw, rs;
    bool unit = true;
    device_transpose(n, e, row_offsets, col, weights, s, tptr, tsrc, tw, rs, &unit);
    const bool weighted = !unit;
    qvb_graph fg;  // slice structure over the raw (uncoalesced) transpose
    fg.device = device;
    fg.n = n;
    fg.e = e;
    fg.eu = e;
    fg.layout = weighted ? 1 : 0;
    fg.seg_size = n;  // one pass: Neumaier state stays in registers
    build_slices(fg, tptr.p, tsrc.p, tsrc.p, weighted ? tw.p : nullptr, s);
    tptr.release();
    tsrc.release();
    tw.release();

    DevBuf<double> vals[2] = {DevBuf<double>(n, s), DevBuf<double>(n, s)};
    DevBuf<double> p(n, s), z, zsl;
    DevBuf<double2> pr;
    QVB_CUDA(cudaMemcpyAsync(vals[0].p, p0.data(), n * 8, cudaMemcpyHostToDevice, s));
    QVB_CUDA(cudaMemcpyAsync(p.p, p0.data(), n * 8, cudaMemcpyHostToDevice, s));
    if (weighted) pr.alloc(n + 1, s);
    else z.alloc(n + 1, s);
    const uint64_t long_blocks = (fg.nlong + kFapWarps - 1) / kFapWarps;
    const uint64_t blocks = long_blocks + (fg.nslices + kFapWarps - 1) / kFapWarps;
    int cur = 0;
    for (uint32_t k = 1; k <= hops; ++k) {
      k_fap_operand<<<grid_for(n + 1, 256), 256, 0, s>>>(n, p.p, rs.p, z.p, pr.p);
      QVB_LAUNCH_CHECK();
      if (blocks) {
        if (weighted)
          k_fap_step<true><<<static_cast<unsigned>(blocks), kFapWarps * 32, 0, s>>>(
              fg.nslices, long_blocks, fg.nlong, fg.perm, fg.sptr, fg.scol, fg.sR, fg.lnode,
              fg.lptr, fg.lcol, fg.lR, nullptr, pr.p, vals[cur].p, vals[cur ^ 1].p, p.p);
        else
          k_fap_step<false><<<static_cast<unsigned>(blocks), kFapWarps * 32, 0, s>>>(
              fg.nslices, long_blocks, fg.nlong, fg.perm, fg.sptr, fg.scol, nullptr, fg.lnode,
              fg.lptr, fg.lcol, nullptr, z.p, nullptr, vals[cur].p, vals[cur ^ 1].p, p.p);
        QVB_LAUNCH_CHECK();
      }
      cur ^= 1;
    }
    QVB_CUDA(cudaMemcpyAsync(values, vals[cur].p, n * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}
