// graph.cu — device in-CSR build (replaces in_adjacency, graph.cpp:260-281,
// and transition_view's row sums, graph.cpp:292-318) and the device-side
// synthetic generator (tools/bench.cpp:22-34).
//
// Pipeline (all on device, one-time per graph):
//   validate + row sums      thread per out-row; sequential sum in CSR order
//                            (bit-exact with graph.cpp:305); unit weights are
//                            exact integer counts, no loop
//   source of every edge     marks at row starts + inclusive scan
//   transpose                stable radix sort by destination with the edge
//                            index as payload => inside a destination the
//                            edges keep out-CSR order = ascending source, and
//                            parallel edges keep their CSR order (exactly the
//                            counting-sort order of graph.cpp:271-279)
//   coalesce                 runs of equal (dst, src) -> one factor edge; the
//                            run's weights summed left to right
//                            (metrics.cpp:157-164); R = w_sum / row_sum(s)
//   layout                   compact (u32 col + per-source y) when almost
//                            every R equals 1/row_sum(s) bitwise, else
//                            weighted (u32 col + f64 R per edge)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "graph.cuh"

qvb_graph::~qvb_graph() {
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  if (done) cudaEventDestroy(done);
  cudaFree(perm);
  cudaFree(sptr);
  cudaFree(scol);
  cudaFree(sR);
  cudaFree(lnode);
  cudaFree(lptr);
  cudaFree(lcol);
  cudaFree(lR);
  cudaFree(exc_src);
  cudaFree(exc_R);
  cudaFree(inv);
  cudaFree(state);
  cudaFree(nm_lenf);
  cudaFree(nm_desc);
  cudaFree(nm_runs);
  cudaFree(nm_sbase);
  cudaFree(nm_col);
  cudaFree(nm_code);
  cudaFree(marked);
  cudaFree(nm_R);
  cudaFree(cls_inv);
  cudaFree(f1_perm);
  cudaFree(f1_sptr);
  cudaFree(f1_cls);
  cudaFree(f1_xslot);
  cudaFree(f1_xR);
  cudaFree(lcls);
  for (auto& pe : phase_ev) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  for (int i = 0; i < 2; ++i) {
    cudaFree(p[i]);
    cudaFree(y[i]);
    cudaFree(kcode[i]);
    if (ev[i]) cudaEventDestroy(ev[i]);
  }
  if (prev >= 0) cudaSetDevice(prev);
}

namespace qvb {
namespace {

constexpr unsigned kBlock = 256;
constexpr unsigned long long kNone = ~0ull;

__global__ void k_check_ro(const uint64_t* __restrict__ ro, uint64_t n,
                           unsigned long long* bad_mono) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (ro[i + 1] < ro[i]) atomicMin(bad_mono, (unsigned long long)i);
}

// graph.cpp:82-85 (edge-level code 2).
__global__ void k_check_weights(const double* __restrict__ w, uint64_t e,
                                unsigned long long* bad_edge) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double x = w[i];
    if (!(x >= 0.0)) atomicMin(bad_edge, (unsigned long long)((i << 2) | 2));
  }
}

// transition_view row sums (graph.cpp:301-316) + the all-zero-weights row
// check (graph.cpp:76,86-91).
__global__ void k_row_sums(const uint64_t* __restrict__ ro, const double* __restrict__ w,
                           uint64_t n, double* __restrict__ rs, double* __restrict__ inv,
                           unsigned long long* bad_zero) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = ro[i], b = ro[i + 1];
    double sum;
    if (w) {
      sum = 0.0;
      bool any_positive = a == b;
      for (uint64_t k = a; k < b; ++k) {
        double x = w[k];
        sum = __dadd_rn(sum, x);
        any_positive |= x > 0.0;
      }
      if (!any_positive) atomicMin(bad_zero, (unsigned long long)i);
    } else {
      sum = static_cast<double>(b - a);  // sum of (b-a) ones, exact
    }
    rs[i] = sum;
    inv[i] = sum > 0.0 ? __ddiv_rn(1.0, sum) : 0.0;
  }
}

__global__ void k_row_marks(const uint64_t* __restrict__ ro, uint64_t n, uint64_t e,
                            uint32_t* __restrict__ marks) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t a = ro[i];
    if (a < e && ro[i + 1] > a) atomicAdd(&marks[a], 1u);
  }
}

// marks[p] = 1 where a non-empty row starts; the inclusive scan then gives
// 1 + the rank of each edge's row among non-empty rows (row_of_rank maps it
// back to the row id).
__global__ void k_src_from_rank(const uint32_t* __restrict__ incl, const uint32_t* __restrict__ row_of_rank,
                                uint64_t e, uint32_t* __restrict__ src) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x)
    src[k] = row_of_rank[incl[k] - 1];
}

__global__ void k_rank_rows(const uint64_t* __restrict__ ro, uint64_t n, const uint32_t* __restrict__ incl,
                            uint64_t e, uint32_t* __restrict__ row_of_rank) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t a = ro[i];
    if (a < e && ro[i + 1] > a) row_of_rank[incl[a] - 1] = static_cast<uint32_t>(i);
  }
}

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = static_cast<uint32_t>(i);
}

// For every transposed position k: its source and whether it starts a run
// of equal (destination, source).
__global__ void k_runs(const uint32_t* __restrict__ sdst, const uint32_t* __restrict__ seid,
                       const uint32_t* __restrict__ src, uint64_t e, uint32_t* __restrict__ ssrc,
                       uint8_t* __restrict__ head) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = src[seid[k]];
    bool h = k == 0;
    if (!h) h = sdst[k] != sdst[k - 1] || s != src[seid[k - 1]];
    ssrc[k] = s;
    head[k] = h ? 1 : 0;
  }
}

// Run heads over sorted (destination, source) pairs (unit-weight graphs).
__global__ void k_heads(const uint32_t* __restrict__ sdst, const uint32_t* __restrict__ ssrc, uint64_t e,
                        uint8_t* __restrict__ head) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x)
    head[k] = (k == 0 || sdst[k] != sdst[k - 1] || ssrc[k] != ssrc[k - 1]) ? 1 : 0;
}

// One thread per run head: coalesce the run (metrics.cpp:157-164), form
// R = w_sum / row_sum(s) and flag it when it differs bitwise from
// 1/row_sum(s); also writes the in-row pointers of every destination whose
// first edge this is (and of the empty rows before it).
__global__ void k_coalesce(const uint32_t* __restrict__ sdst, const uint32_t* __restrict__ seid,
                           const uint32_t* __restrict__ ssrc, const uint8_t* __restrict__ head,
                           const uint32_t* __restrict__ uidx, const double* __restrict__ w,
                           const double* __restrict__ rs, const double* __restrict__ inv,
                           uint64_t e, uint64_t n, uint64_t eu, uint32_t* __restrict__ ucol,
                           double* __restrict__ uR, uint8_t* __restrict__ uexc,
                           uint64_t* __restrict__ uptr) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x) {
    if (k == e - 1) {  // tail rows after the last destination
      for (uint64_t d = (uint64_t)sdst[k] + 1; d <= n; ++d) uptr[d] = eu;
    }
    if (!head[k]) continue;
    const uint32_t s = ssrc[k];
    const uint32_t u = uidx[k];
    double W;
    uint64_t k2 = k + 1;
    if (w) {
      W = w[seid[k]];
      while (k2 < e && !head[k2]) {
        W = __dadd_rn(W, w[seid[k2]]);
        ++k2;
      }
    } else {
      while (k2 < e && !head[k2]) ++k2;
      W = static_cast<double>(k2 - k);  // sum of ones, exact
    }
    ucol[u] = s;
    if (!w && k2 == k + 1) {
      // unit weight, single edge: R = 1/row_sum(s) is inv[s] bit for bit, no
      // exception; uR is filled by k_fill_unit_R only if the weighted layout
      // is chosen (the compact layout reads uR of exceptions alone)
      uexc[u] = 0;
    } else {
      const double R = __ddiv_rn(W, rs[s]);
      uR[u] = R;
      uexc[u] = __double_as_longlong(R) != __double_as_longlong(inv[s]) ? 1 : 0;
    }
    const uint32_t d = sdst[k];
    if (k == 0 || sdst[k - 1] != d) {
      const uint64_t d0 = k == 0 ? 0 : (uint64_t)sdst[k - 1] + 1;
      for (uint64_t dd = d0; dd <= d; ++dd) uptr[dd] = u;
    }
  }
}

__global__ void k_count_sources(const uint32_t* __restrict__ ucol, uint64_t eu,
                                uint32_t* __restrict__ distinct) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < eu;
       u += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&distinct[ucol[u]], 1u);
}

// uR of the single unit-weight edges k_coalesce skipped: inv[s].
__global__ void k_fill_unit_R(const uint32_t* __restrict__ ucol, const uint8_t* __restrict__ uexc,
                              const double* __restrict__ inv, uint64_t eu, double* __restrict__ uR) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < eu;
       u += (uint64_t)gridDim.x * blockDim.x)
    if (!uexc[u]) uR[u] = inv[ucol[u]];
}

__global__ void k_compact(const uint32_t* __restrict__ ucol, const double* __restrict__ uR,
                          const uint8_t* __restrict__ uexc, const uint32_t* __restrict__ xidx,
                          uint64_t eu, uint32_t* __restrict__ col, uint32_t* __restrict__ exc_src,
                          double* __restrict__ exc_R) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < eu;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = ucol[u];
    if (uexc[u]) {
      const uint32_t x = xidx[u];
      col[u] = kExcFlag | x;
      exc_src[x] = s;
      exc_R[x] = uR[u];
    } else {
      col[u] = s;
    }
  }
}

// ---- segmented slicing (see graph.cuh) ---------------------------------------
// (node, segment) pairs: for every regular row, one pair per source segment
// its (source-sorted) in-row touches; zero-degree rows get one empty pair in
// pass 0 so their P(n,j) = P(n,j-1) is written too. Long rows get none.
__global__ void k_pair_count(const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ src,
                             uint64_t n, uint32_t thr, uint64_t seg, uint32_t* __restrict__ cnt) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = uptr[v], b = uptr[v + 1];
    uint32_t c = 0;
    if (b == a) {
      c = 1;
    } else if (b - a <= thr) {
      uint64_t prev = ~0ull;
      for (uint64_t u = a; u < b; ++u) {
        const uint64_t k = src[u] / seg;
        c += k != prev;
        prev = k;
      }
    }
    cnt[v] = c;
  }
}

__global__ void k_pair_emit(const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ src,
                            uint64_t n, uint32_t thr, uint64_t seg, const uint64_t* __restrict__ po,
                            uint32_t* __restrict__ pk, uint32_t* __restrict__ pv,
                            uint64_t* __restrict__ pstart, uint32_t* __restrict__ pdeg) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = uptr[v], b = uptr[v + 1];
    uint64_t at = po[v];
    if (b == a) {
      pk[at] = 0;
      pv[at] = static_cast<uint32_t>(v) | kFirst | kLast;
      pstart[at] = 0;
      pdeg[at] = 0;
      continue;
    }
    if (b - a > thr) continue;
    uint64_t run = a;
    for (uint64_t u = a; u < b; ++u) {
      const uint64_t k = src[u] / seg;
      const bool end = u + 1 == b || src[u + 1] / seg != k;
      if (end) {
        uint32_t flags = (run == a ? kFirst : 0u) | (u + 1 == b ? kLast : 0u);
        pk[at] = static_cast<uint32_t>(k);
        pv[at] = static_cast<uint32_t>(v) | flags;
        pstart[at] = run;
        pdeg[at] = static_cast<uint32_t>(u + 1 - run);
        ++at;
        run = u + 1;
      }
    }
  }
}

// One CTA per group of up to 256 pairs of one pass: order them by degree
// (descending, node id ascending) into the group's 256 slots, so each slice
// of 32 holds similar row lengths and pads little.
template <uint32_t W = kWindow>
__global__ void __launch_bounds__(W)
    k_group_sort(const uint32_t* __restrict__ sorted_idx, const uint64_t* __restrict__ seg_pair_begin,
                 const uint64_t* __restrict__ seg_group_begin, int nseg,
                 const uint32_t* __restrict__ pv, const uint32_t* __restrict__ pdeg,
                 uint32_t* __restrict__ slot_pair) {
  __shared__ uint32_t sdeg[W];
  __shared__ uint32_t snode[W];
  const uint64_t grp = blockIdx.x;
  int k = 0;
  while (k + 1 < nseg && seg_group_begin[k + 1] <= grp) ++k;
  const uint64_t q0 = seg_pair_begin[k] + (grp - seg_group_begin[k]) * W;
  const uint64_t q1 = seg_pair_begin[k + 1];
  const uint32_t t = threadIdx.x;
  const bool real = q0 + t < q1;
  uint32_t idx = 0, d = 0, node = 0;
  if (real) {
    idx = sorted_idx[q0 + t];
    d = pdeg[idx];
    node = pv[idx] & kNodeMask;
  }
  sdeg[t] = real ? d : 0u;
  snode[t] = real ? node : 0xFFFFFFFFu;
  __syncthreads();
  const uint32_t cnt = static_cast<uint32_t>(q1 - q0 < W ? q1 - q0 : W);
  if (real) {
    uint32_t rank = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint32_t dj = sdeg[j], nj = snode[j];
      rank += (dj > d) || (dj == d && nj < node);
    }
    slot_pair[grp * W + rank] = idx;
  } else {
    slot_pair[grp * W + t] = 0xFFFFFFFFu;
  }
}

__global__ void k_slot_lens(const uint32_t* __restrict__ slot_pair, const uint32_t* __restrict__ pdeg,
                            uint64_t nslices, uint32_t* __restrict__ len32, uint32_t quantum = 1,
                            bool sorted = true) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= nslices;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t len = 0;
    if (j < nslices) {
      const uint32_t i = slot_pair[j * 32];  // first slot holds the slice maximum
        len = i == 0xFFFFFFFFu ? 0u : pdeg[i];
      if (!sorted) {  // unsorted slices: the longest of the 32 rows
        for (int l = 1; l < 32; ++l) {
          const uint32_t il = slot_pair[j * 32 + l];
          if (il != 0xFFFFFFFFu && pdeg[il] > len) len = pdeg[il];
        }
      }
      len = (len + quantum - 1) / quantum * quantum;
    }
    len32[j] = 32u * len;
  }
}

template <bool kWithR>
__global__ void k_fill_slots(const uint32_t* __restrict__ slot_pair, const uint32_t* __restrict__ pv,
                             const uint64_t* __restrict__ pstart, const uint32_t* __restrict__ pdeg,
                             const uint64_t* __restrict__ sptr, const uint32_t* __restrict__ col,
                             const double* __restrict__ R, uint64_t nslices, uint32_t pad,
                             uint32_t* __restrict__ perm, uint32_t* __restrict__ scol,
                             double* __restrict__ sR) {
  const uint64_t slots = nslices * 32;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < slots;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = p >> 5, lane = p & 31;
    const uint64_t base = sptr[s];
    const uint64_t len = (sptr[s + 1] - base) >> 5;
    const uint32_t i = slot_pair[p];
    uint64_t r0 = 0, deg = 0;
    if (i != 0xFFFFFFFFu) {
      perm[p] = pv[i];
      r0 = pstart[i];
      deg = pdeg[i];
    } else {
      perm[p] = kNoNode;
    }
    for (uint64_t k = 0; k < len; ++k) {
      const uint64_t at = base + k * 32 + lane;
      if (k < deg) {
        scol[at] = col[r0 + k];
        if (kWithR) sR[at] = R[r0 + k];
      } else {
        scol[at] = pad;
        if (kWithR) sR[at] = 0.0;
      }
    }
  }
}

__global__ void k_long_marks(const uint64_t* __restrict__ uptr, uint64_t n, uint32_t thr,
                             uint8_t* __restrict__ mark) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    mark[v] = (uptr[v + 1] - uptr[v]) > thr ? 1 : 0;
}

__global__ void k_long_list(const uint8_t* __restrict__ mark, const uint32_t* __restrict__ lidx,
                            const uint64_t* __restrict__ uptr, uint64_t n,
                            uint32_t* __restrict__ lnode, uint32_t* __restrict__ ldeg) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    if (mark[v]) {
      lnode[lidx[v]] = static_cast<uint32_t>(v);
      ldeg[lidx[v]] = static_cast<uint32_t>(uptr[v + 1] - uptr[v]);
    }
}

// One warp per long row: copy its CSR segment.
__global__ void k_long_copy(const uint32_t* __restrict__ lnode, const uint64_t* __restrict__ lptr,
                            const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ col,
                            const double* __restrict__ R, uint64_t nlong,
                            uint32_t* __restrict__ lcol, double* __restrict__ lR) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp >= nlong) return;
  const uint64_t src = uptr[lnode[warp]];
  const uint64_t dst = lptr[warp], len = lptr[warp + 1] - dst;
  for (uint64_t k = lane; k < len; k += 32) {
    lcol[dst + k] = col[src + k];
    if (R) lR[dst + k] = R[src + k];
  }
}

// tools/bench.cpp:22-34 on the device: edge i consumes draws 3i, 3i+1, 3i+2
// of derive_stream(seed, 0xBE9C4).
__global__ void k_gen_edges(uint64_t n, uint64_t e, uint64_t state, int weighted, int transposed,
                            uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                            double* __restrict__ w) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double u = to_uniform(stream_draw(state, 3 * i));
    uint64_t s = __double2ull_rz(__dmul_rn(__dmul_rn(u, u), static_cast<double>(n)));
    uint64_t d = to_below(stream_draw(state, 3 * i + 1), n);
    if (s > n - 1) s = n - 1;
    if (transposed) {
      uint64_t t = s;
      s = d;
      d = t;
    }
    src[i] = static_cast<uint32_t>(s);
    dst[i] = static_cast<uint32_t>(d);
    if (w) w[i] = weighted ? __dadd_rn(1.0, to_uniform(stream_draw(state, 3 * i + 2))) : 1.0;
  }
}

// Row offsets from sorted row keys: ro[r] = first position with key >= r.
__global__ void k_offsets_from_sorted(const uint32_t* __restrict__ keys, uint64_t e, uint64_t n,
                                      uint64_t* __restrict__ ro) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = keys[k];
    const uint64_t d0 = k == 0 ? 0 : (uint64_t)keys[k - 1] + 1;
    if (k == 0 || keys[k - 1] != keys[k])
      for (uint64_t dd = d0; dd <= d; ++dd) ro[dd] = k;
    if (k == e - 1)
      for (uint64_t dd = d + 1; dd <= n; ++dd) ro[dd] = e;
  }
}

template <typename T>
__global__ void k_gather_by(const T* __restrict__ in, const uint32_t* __restrict__ idx, uint64_t e,
                            T* __restrict__ out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x)
    out[k] = in[idx[k]];
}

template <typename T>
T* persist(DevBuf<T>& b) {
  return b.release_ownership();
}

// ---- node-major segmented layout (graph.cuh "nm") --------------------------
// Per node: its sources per segment (rows are source-sorted, so one walk),
// flagged with the first and last pass that touch it. Long rows (> thr) stay
// 0 everywhere (long path); in-degree-0 nodes finish in pass 0.
__global__ void k_nm_lens(const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ src,
                          uint64_t n, uint64_t npad, uint32_t thr, uint64_t seg0, uint64_t seg,
                          uint8_t* __restrict__ lenf) {
  // source segment: [0, seg0), then every seg sources
  auto segment = [&](uint64_t x) -> uint64_t { return x < seg0 ? 0 : 1 + (x - seg0) / seg; };
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = uptr[v], b = uptr[v + 1];
    if (b - a > thr) continue;
    if (b == a) {
      lenf[v] = kNmFirst | kNmLast;
      continue;
    }
    bool first = true;
    uint64_t u = a;
    while (u < b) {
      const uint64_t k = segment(src[u]);
      uint32_t cnt = 0;
      while (u < b && segment(src[u]) == k) {
        ++u;
        ++cnt;
      }
      uint8_t f = static_cast<uint8_t>(cnt);
      if (first) f |= kNmFirst;
      if (u == b) f |= kNmLast;
      first = false;
      lenf[k * npad + v] = f;
    }
  }
}

// Columns of slice (k, s): sum of its 32 lens; entry nseg*S is 0.
__global__ void k_nm_slice_sums(const uint8_t* __restrict__ lenf, uint64_t S, int nseg,
                                uint32_t* __restrict__ cnt) {
  const uint64_t total = S * nseg;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x <= total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    if (x == total) {
      cnt[x] = 0;
      continue;
    }
    const uint8_t* l = lenf + x * 32;  // (k, s) -> k*S*32 + s*32 == x*32
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) c += l[i] & kNmLen;
    cnt[x] = c;
  }
}

// One warp per slice: lane = node; pass by pass, the lane's next len sources
// go to sbase(k, s) + (prefix of the slice's lens).
__global__ void k_nm_fill(const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ col,
                          const double* __restrict__ R, const uint8_t* __restrict__ lenf,
                          const uint64_t* __restrict__ sbase, uint64_t n, uint64_t S, int nseg,
                          uint32_t* __restrict__ ncol, double* __restrict__ nR) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t sl = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); sl < S;
       sl += warps) {
    const uint64_t v = sl * 32 + lane;
    uint64_t u = v < n ? uptr[v] : 0;
    for (int k = 0; k < nseg; ++k) {
      const uint32_t len = lenf[(uint64_t)k * S * 32 + v] & kNmLen;
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint64_t dst = sbase[(uint64_t)k * S + sl] + (incl - len);
      for (uint32_t t = 0; t < len; ++t) {
        ncol[dst + t] = col[u + t];
        if (R) nR[dst + t] = R[u + t];
      }
      u += len;
    }
  }
}


// ---- first-sweep classes (graph.cuh "f1") ------------------------------------
__global__ void k_cls_keys(const double* __restrict__ inv, uint64_t n, uint64_t* __restrict__ keys,
                           uint32_t* __restrict__ vals) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    keys[i] = static_cast<uint64_t>(__double_as_longlong(inv[i]));
    vals[i] = static_cast<uint32_t>(i);
  }
}

__global__ void k_cls_heads(const uint64_t* __restrict__ skeys, uint64_t n, uint8_t* __restrict__ head) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x)
    head[k] = (k == 0 || skeys[k] != skeys[k - 1]) ? 1 : 0;
}

__global__ void k_cls_assign(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
                             const uint8_t* __restrict__ head, const uint32_t* __restrict__ cidx,
                             uint64_t n, uint32_t* __restrict__ cls_of, double* __restrict__ cls_inv) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cidx[k] + head[k] - 1;
    cls_of[svals[k]] = c;
    if (head[k]) cls_inv[c] = __longlong_as_double(static_cast<long long>(skeys[k]));
  }
}

// k_fill_slots for the class stream (lane-major quads, f1_slot): exceptions
// get class ncls+1 and are appended
// (slot, exception index) for a later sort by slot.
__global__ void k_fill_cls(const uint32_t* __restrict__ slot_pair, const uint32_t* __restrict__ pv,
                           const uint64_t* __restrict__ pstart, const uint32_t* __restrict__ pdeg,
                           const uint64_t* __restrict__ sptr, const uint32_t* __restrict__ col,
                           const uint32_t* __restrict__ cls_of, uint64_t nslices, uint16_t pad,
                           uint16_t exc_cls,
                           uint32_t* __restrict__ perm, uint16_t* __restrict__ scls,
                           unsigned long long* __restrict__ xcount, uint64_t* __restrict__ xslot,
                           uint32_t* __restrict__ xidx) {
  const uint64_t slots = nslices * 32;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < slots;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = p >> 5, lane = p & 31;
    const uint64_t base = sptr[s];
    const uint64_t len = (sptr[s + 1] - base) >> 5;
    const uint32_t i = slot_pair[p];
    uint64_t r0 = 0, deg = 0;
    if (i != 0xFFFFFFFFu) {
      perm[p] = pv[i];
      r0 = pstart[i];
      deg = pdeg[i];
    } else {
      perm[p] = kNoNode;
    }
    for (uint64_t k = 0; k < len; ++k) {
      const uint64_t at = f1_slot(base, k, lane);
      uint16_t c = pad;
      if (k < deg) {
        const uint32_t x = col[r0 + k];
        if (x & kExcFlag) {
          c = exc_cls;
          const unsigned long long j = atomicAdd(xcount, 1ull);
          xslot[j] = at;
          xidx[j] = x & ~kExcFlag;
        } else {
          c = static_cast<uint16_t>(cls_of[x]);
        }
      }
      scls[at] = c;
    }
  }
}

__global__ void k_x_values(const uint32_t* __restrict__ sidx, const double* __restrict__ exc_R,
                           uint64_t nx, double* __restrict__ xR) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nx;
       i += (uint64_t)gridDim.x * blockDim.x)
    xR[i] = exc_R[sidx[i]];
}

__global__ void k_long_cls(const uint32_t* __restrict__ lcol, const uint32_t* __restrict__ cls_of,
                           uint64_t m, uint16_t exc_cls, uint16_t* __restrict__ lcls) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = lcol[i];
    lcls[i] = (x & kExcFlag) ? exc_cls : static_cast<uint16_t>(cls_of[x]);
  }
}

}  // namespace

void build_in_csr(qvb_graph& g, const uint64_t* d_ro, const uint32_t* d_col, const double* d_w,
                  const uint32_t* d_src, cudaStream_t s, ViewOut view) {
  const uint64_t n = g.n, e = g.e;
  DevBuf<double> rs(n, s), inv(n + 2, s);  // +2: 16-byte bulk-copy spans (f1)
  QVB_CUDA(cudaMemsetAsync(inv.p + n, 0, 2 * sizeof(double), s));
  DevBuf<unsigned long long> flags(1, s);
  QVB_CUDA(cudaMemsetAsync(flags.p, 0xFF, sizeof(unsigned long long), s));
  k_row_sums<<<grid_for(n, kBlock), kBlock, 0, s>>>(d_ro, d_w, n, rs.p, inv.p, flags.p);
  QVB_LAUNCH_CHECK();
  unsigned long long bad_zero = read_scalar(flags.p, s);
  if (bad_zero != kNone)
    fail(QVB_ERR_VALIDATION, "node " + std::to_string(bad_zero) +
                                 " has out-edges but all weights are zero");
  if (view.row_sums)
    QVB_CUDA(cudaMemcpyAsync(view.row_sums, rs.p, n * 8, cudaMemcpyDeviceToDevice, s));
  if (view.distinct) QVB_CUDA(cudaMemsetAsync(view.distinct, 0, n * 4, s));

  DevBuf<uint64_t> uptr(n + 1, s);
  if (e == 0) {
    QVB_CUDA(cudaMemsetAsync(uptr.p, 0, (n + 1) * sizeof(uint64_t), s));
    g.eu = 0;
    g.nexc = 0;
    g.layout = 0;
    DevBuf<uint32_t> none(1, s);
    build_slices(g, uptr.p, none.p, none.p, nullptr, s);
    g.inv = persist(inv);
    g.bytes += n * 8;
    QVB_CUDA(cudaStreamSynchronize(s));
    return;
  }

  // Source of every out-CSR edge.
  DevBuf<uint32_t> src_buf;
  if (!d_src) {
    src_buf.alloc(e, s);
    DevBuf<uint32_t> marks(e, s), incl(e, s);
    QVB_CUDA(cudaMemsetAsync(marks.p, 0, e * sizeof(uint32_t), s));
    k_row_marks<<<grid_for(n, kBlock), kBlock, 0, s>>>(d_ro, n, e, marks.p);
    QVB_LAUNCH_CHECK();
    inclusive_sum_u32_u32(marks.p, incl.p, e, s);
    DevBuf<uint32_t> row_of_rank(n, s);
    k_rank_rows<<<grid_for(n, kBlock), kBlock, 0, s>>>(d_ro, n, incl.p, e, row_of_rank.p);
    QVB_LAUNCH_CHECK();
    k_src_from_rank<<<grid_for(e, kBlock), kBlock, 0, s>>>(incl.p, row_of_rank.p, e, src_buf.p);
    QVB_LAUNCH_CHECK();
    d_src = src_buf.p;
  }

  // Transpose: stable sort by destination. Weighted graphs carry the
  // out-CSR edge index (the weights are gathered through it); unit-weight
  // graphs carry the source itself, so the sorted sources come out of the
  // sort instead of a random gather per edge (stable over source-major input:
  // ascending sources within every destination either way).
  DevBuf<uint32_t> sdst(e, s), seid, ssrc(e, s);
  DevBuf<uint8_t> head(e, s);
  if (d_w) {
    seid.alloc(e, s);
    {
      DevBuf<uint32_t> iota(e, s);
      k_iota<<<grid_for(e, kBlock), kBlock, 0, s>>>(iota.p, e);
      QVB_LAUNCH_CHECK();
      sort_pairs_u32_u32(d_col, sdst.p, iota.p, seid.p, e, 0, bits_for(n - 1), s);
    }
    k_runs<<<grid_for(e, kBlock), kBlock, 0, s>>>(sdst.p, seid.p, d_src, e, ssrc.p, head.p);
  } else {
    sort_pairs_u32_u32(d_col, sdst.p, d_src, ssrc.p, e, 0, bits_for(n - 1), s);
    k_heads<<<grid_for(e, kBlock), kBlock, 0, s>>>(sdst.p, ssrc.p, e, head.p);
  }
  QVB_LAUNCH_CHECK();
  src_buf.release();
  DevBuf<uint32_t> uidx(e, s);
  exclusive_sum_u8_u32(head.p, uidx.p, e, s);
  uint32_t last_idx = read_scalar(uidx.p + (e - 1), s);
  uint8_t last_head = read_scalar(head.p + (e - 1), s);
  const uint64_t eu = (uint64_t)last_idx + last_head;

  DevBuf<uint32_t> ucol(eu, s);
  DevBuf<double> uR(eu, s);
  DevBuf<uint8_t> uexc(eu, s);
  k_coalesce<<<grid_for(e, kBlock), kBlock, 0, s>>>(sdst.p, seid.p, ssrc.p, head.p, uidx.p, d_w,
                                                    rs.p, inv.p, e, n, eu, ucol.p, uR.p, uexc.p,
                                                    uptr.p);
  QVB_LAUNCH_CHECK();
  sdst.release();
  seid.release();
  ssrc.release();
  head.release();
  uidx.release();
  if (view.distinct) {  // each coalesced in-edge is one distinct out-neighbour of its source
    k_count_sources<<<grid_for(eu, kBlock), kBlock, 0, s>>>(ucol.p, eu, view.distinct);
    QVB_LAUNCH_CHECK();
  }

  DevBuf<uint64_t> cnt(1, s);
  sum_u8_u64(uexc.p, cnt.p, eu, s);
  const uint64_t nexc = read_scalar(cnt.p, s);
  g.eu = eu;
  g.nexc = nexc;
  if (nexc * 16 <= eu) {  // compact layout
    g.layout = 0;
    DevBuf<uint32_t> xidx(eu, s), col(eu, s), xsrc(nexc ? nexc : 1, s);
    DevBuf<double> xR(nexc ? nexc : 1, s);
    exclusive_sum_u8_u32(uexc.p, xidx.p, eu, s);
    k_compact<<<grid_for(eu, kBlock), kBlock, 0, s>>>(ucol.p, uR.p, uexc.p, xidx.p, eu, col.p,
                                                      xsrc.p, xR.p);
    QVB_LAUNCH_CHECK();
    uR.release();
    uexc.release();
    g.exc_src = persist(xsrc);
    g.exc_R = persist(xR);
    g.bytes = (nexc ? nexc : 1) * 12;
    build_slices(g, uptr.p, col.p, ucol.p, nullptr, s);
    build_first(g, uptr.p, col.p, inv.p, s);
  } else {
    g.layout = 1;
    if (!d_w) {
      k_fill_unit_R<<<grid_for(eu, kBlock), kBlock, 0, s>>>(ucol.p, uexc.p, inv.p, eu, uR.p);
      QVB_LAUNCH_CHECK();
    }
    uexc.release();
    build_slices(g, uptr.p, ucol.p, ucol.p, uR.p, s);
  }
  g.inv = persist(inv);
  g.bytes += n * 8;
  QVB_CUDA(cudaStreamSynchronize(s));
}

uint64_t segment_size(uint64_t n) {
  uint64_t mb = 64;
  if (const char* e = std::getenv("QVB_SEG_MB")) mb = std::strtoull(e, nullptr, 10);
  uint64_t seg = std::max<uint64_t>(1, (mb << 20) / 8);
  if (const char* e = std::getenv("QVB_SEG_SOURCES")) seg = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  return std::min<uint64_t>(seg, std::max<uint64_t>(n, 1));
}

// Rows with in-degree above thr: a plain CSR, one warp per row.
void build_long_rows(qvb_graph& g, const uint64_t* uptr, const uint32_t* col, const double* R,
                     uint32_t thr, cudaStream_t s) {
  const uint64_t n = g.n;
  DevBuf<uint8_t> mark(n, s);
  DevBuf<uint32_t> lidx(n, s);
  k_long_marks<<<grid_for(n, kBlock), kBlock, 0, s>>>(uptr, n, thr, mark.p);
  QVB_LAUNCH_CHECK();
  exclusive_sum_u8_u32(mark.p, lidx.p, n, s);
  g.nlong = (uint64_t)read_scalar(lidx.p + (n - 1), s) + read_scalar(mark.p + (n - 1), s);
  if (g.nlong) {
    const uint64_t L = g.nlong;
    DevBuf<uint32_t> lnode(L, s), ldeg(L + 1, s);
    DevBuf<uint64_t> lptr(L + 1, s);
    k_long_list<<<grid_for(n, kBlock), kBlock, 0, s>>>(mark.p, lidx.p, uptr, n, lnode.p, ldeg.p);
    QVB_LAUNCH_CHECK();
    QVB_CUDA(cudaMemsetAsync(ldeg.p + L, 0, sizeof(uint32_t), s));
    exclusive_sum_u32_u64(ldeg.p, lptr.p, L + 1, s);
    const uint64_t lsum = read_scalar(lptr.p + L, s);
    DevBuf<uint32_t> lcol(lsum, s);
    DevBuf<double> lR;
    if (R) lR.alloc(lsum, s);
    k_long_copy<<<static_cast<unsigned>((L * 32 + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        lnode.p, lptr.p, uptr, col, R, L, lcol.p, lR.p);
    QVB_LAUNCH_CHECK();
    g.lnode = persist(lnode);
    g.lptr = persist(lptr);
    g.lcol = persist(lcol);
    g.lR = lR.p ? persist(lR) : nullptr;
    g.bytes += L * 12 + lsum * (R ? 12 : 4);
  }
}

// The nm layout (graph.cuh) for more than one source segment.
void build_nm(qvb_graph& g, const uint64_t* uptr, const uint32_t* col, const uint32_t* src,
              const double* R, cudaStream_t s) {
  const uint64_t n = g.n;
  const uint32_t thr = std::min<uint32_t>(g.long_threshold, kNmLen);
  g.long_threshold = thr;
  // compact sweeps gather 4-byte codes: twice the sources per segment, and
  // by default a 64 MiB code slice — the per-segment code gathers (k_codes)
  // stay L2-resident up to about that size next to their column and code
  // streams (C4: 48 MiB 7.2 ms, 64 MiB 7.5 ms, 96 MiB 11.6 ms), and fewer
  // segments mean fewer runs per node for k_products (48: 5.0, 64: 4.1 ms)
  uint64_t seg = R ? g.seg_size : g.seg_size * 2;
  if (!R && !std::getenv("QVB_SEG_MB") && !std::getenv("QVB_SEG_SOURCES")) seg = (64ull << 20) / 4;
  seg = std::min<uint64_t>(n, seg);
  g.seg_size = seg;
  // the first segment may be wider (QVB_SEG0_MB of codes): its sources are
  // the hottest, so its gathers keep hitting L2 over a larger range
  uint64_t seg0 = seg;
  if (const char* m = std::getenv("QVB_SEG0_MB")) seg0 = std::max<uint64_t>(1, (std::strtoull(m, nullptr, 10) << 20) / 4);
  seg0 = std::min<uint64_t>(n, std::max<uint64_t>(seg0, 1));
  g.seg0_size = seg0;
  const int nseg = n <= seg0 ? 1 : 1 + static_cast<int>((n - seg0 + seg - 1) / seg);
  if (nseg > 255) fail(QVB_ERR_UNSUPPORTED, "too many source segments (raise QVB_SEG_MB)");
  g.seg_slice.assign(nseg + 1, 0);
  const uint64_t S = (n + 31) / 32, npad = S * 32;
  DevBuf<uint8_t> lenf(npad * nseg, s);
  QVB_CUDA(cudaMemsetAsync(lenf.p, 0, npad * nseg, s));
  k_nm_lens<<<grid_for(n, kBlock), kBlock, 0, s>>>(uptr, src, n, npad, thr, seg0, seg, lenf.p);
  QVB_LAUNCH_CHECK();
  DevBuf<uint32_t> cnt(S * nseg + 1, s);
  DevBuf<uint64_t> sbase(S * nseg + 3, s);  // +2: 16-byte bulk-copy windows
  k_nm_slice_sums<<<grid_for(S * nseg + 1, kBlock), kBlock, 0, s>>>(lenf.p, S, nseg, cnt.p);
  QVB_LAUNCH_CHECK();
  exclusive_sum_u32_u64(cnt.p, sbase.p, S * nseg + 1, s);
  cnt.release();
  const uint64_t total = read_scalar(sbase.p + S * nseg, s);
  g.nm_region.resize(nseg + 1);
  g.nm_region_count = nseg;
  for (int k = 0; k <= nseg; ++k) g.nm_region[k] = read_scalar(sbase.p + S * k, s);
  DevBuf<uint32_t> ncol(total + 4, s);  // +4: 16-byte bulk-copy windows
  DevBuf<double> nR;
  if (R) nR.alloc(total ? total : 1, s);
  k_nm_fill<<<grid_for(S * 32, kBlock), kBlock, 0, s>>>(uptr, col, R, lenf.p, sbase.p, n, S, nseg,
                                                        ncol.p, nR.p);
  QVB_LAUNCH_CHECK();
  QVB_CUDA(cudaMalloc(&g.state, npad * sizeof(double)));  // whole slices: bulk-copied
  QVB_CUDA(cudaMemsetAsync(sbase.p + S * nseg + 1, 0, 2 * sizeof(uint64_t), s));
  QVB_CUDA(cudaMemsetAsync(ncol.p + total, 0, 4 * sizeof(uint32_t), s));
  build_long_rows(g, uptr, col, R, thr, s);
  g.nm = true;
  g.nm_S = S;
  g.nm_cols = total;
  g.slots = total;
  g.nslices = 0;
  g.nm_lenf = persist(lenf);
  g.nm_sbase = persist(sbase);
  g.nm_col = persist(ncol);
  g.nm_R = nR.p ? persist(nR) : nullptr;
  g.bytes += npad * nseg + (S * nseg + 1) * 8 + total * (R ? 12 : 4) + n * 8;
}

void build_first(qvb_graph& g, const uint64_t* uptr, const uint32_t* col, const double* inv,
                 cudaStream_t s) {
  const char* mode = std::getenv("QVB_FIRST");
  if (mode && std::string(mode) == "gather") return;
  const uint64_t n = g.n;
  if (n == 0 || g.eu == 0 || g.layout != 0) return;
  // classes: distinct bit patterns of 1/row_sum, by a sort of (inv, node)
  DevBuf<uint32_t> cls_of(n, s);
  uint32_t ncls = 0;
  {
    DevBuf<uint64_t> keys(n, s), skeys(n, s);
    DevBuf<uint32_t> vals(n, s), svals(n, s);
    k_cls_keys<<<grid_for(n, kBlock), kBlock, 0, s>>>(inv, n, keys.p, vals.p);
    QVB_LAUNCH_CHECK();
    sort_pairs_u64_u32(keys.p, skeys.p, vals.p, svals.p, n, 0, 64, s);
    keys.release();
    vals.release();
    DevBuf<uint8_t> head(n, s);
    DevBuf<uint32_t> cidx(n, s);
    k_cls_heads<<<grid_for(n, kBlock), kBlock, 0, s>>>(skeys.p, n, head.p);
    QVB_LAUNCH_CHECK();
    exclusive_sum_u8_u32(head.p, cidx.p, n, s);
    ncls = read_scalar(cidx.p + (n - 1), s) + read_scalar(head.p + (n - 1), s);
    if (ncls > kMaxCls) return;  // (ncls+1 must also fit the u16 class stream)
    DevBuf<double> cinv(ncls, s);
    k_cls_assign<<<grid_for(n, kBlock), kBlock, 0, s>>>(skeys.p, svals.p, head.p, cidx.p, n, cls_of.p,
                                                       cinv.p);
    QVB_LAUNCH_CHECK();
    g.cls_inv = persist(cinv);
  }
  g.ncls = ncls;
  // one pass over every regular row (in-degree <= long_threshold): pairs are
  // the rows themselves, in node order
  const uint32_t thr = g.long_threshold;
  const uint64_t one = ~0ull;  // a single source segment
  DevBuf<uint32_t> cnt(n + 1, s);
  DevBuf<uint64_t> po(n + 1, s);
  QVB_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(uint32_t), s));
  k_pair_count<<<grid_for(n, kBlock), kBlock, 0, s>>>(uptr, col, n, thr, one, cnt.p);
  QVB_LAUNCH_CHECK();
  exclusive_sum_u32_u64(cnt.p, po.p, n + 1, s);
  cnt.release();
  const uint64_t H = read_scalar(po.p + n, s);
  DevBuf<uint32_t> pk(H ? H : 1, s), pv(H ? H : 1, s), pdeg(H ? H : 1, s), iota(H ? H : 1, s);
  DevBuf<uint64_t> pstart(H ? H : 1, s);
  k_pair_emit<<<grid_for(n, kBlock), kBlock, 0, s>>>(uptr, col, n, thr, one, po.p, pk.p, pv.p,
                                                     pstart.p, pdeg.p);
  QVB_LAUNCH_CHECK();
  po.release();
  pk.release();
  k_iota<<<grid_for(H, kBlock), kBlock, 0, s>>>(iota.p, H);
  QVB_LAUNCH_CHECK();
  // Nodes are sorted by in-degree into slices inside windows of W nodes:
  // wider windows pad less, but scatter a warp's per-node stores across the
  // window. Those merge in L2 while the outputs (24 B per node) fit half of
  // it; beyond that W = 32 keeps every warp's stores whole sectors (C4: the
  // first sweep 2.7 ms at W = 256 with 2x the DRAM reads, 1.8 ms at W = 32).
  uint32_t W = n * 24 <= (64ull << 20) ? 256 : 32;
  if (const char* m = std::getenv("QVB_F1_WINDOW")) W = static_cast<uint32_t>(std::atoi(m));
  if (W != 32 && W != 64 && W != 128) W = 256;
  const uint64_t groups = (H + W - 1) / W;
  const uint64_t S = groups * (W / 32);
  DevBuf<uint64_t> spb(2, s), sgb(2, s);
  {
    const uint64_t hb[2] = {0, H}, gb[2] = {0, groups};
    QVB_CUDA(cudaMemcpyAsync(spb.p, hb, sizeof(hb), cudaMemcpyHostToDevice, s));
    QVB_CUDA(cudaMemcpyAsync(sgb.p, gb, sizeof(gb), cudaMemcpyHostToDevice, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  }
  DevBuf<uint32_t> slot_pair(S * 32 ? S * 32 : 1, s);
  // windows of 32 are single slices: sorting them cannot pad less, so their
  // nodes keep node order (k_first then derives the node from the slot)
  const bool ident = W == 32;
  if (groups && ident) {
    QVB_CUDA(cudaMemsetAsync(slot_pair.p, 0xFF, S * 32 * sizeof(uint32_t), s));
    QVB_CUDA(cudaMemcpyAsync(slot_pair.p, iota.p, H * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  } else if (groups)
    switch (W) {
      case 32:
        k_group_sort<32><<<static_cast<unsigned>(groups), 32, 0, s>>>(iota.p, spb.p, sgb.p, 1, pv.p, pdeg.p, slot_pair.p);
        break;
      case 64:
        k_group_sort<64><<<static_cast<unsigned>(groups), 64, 0, s>>>(iota.p, spb.p, sgb.p, 1, pv.p, pdeg.p, slot_pair.p);
        break;
      case 128:
        k_group_sort<128><<<static_cast<unsigned>(groups), 128, 0, s>>>(iota.p, spb.p, sgb.p, 1, pv.p, pdeg.p, slot_pair.p);
        break;
      default:
        k_group_sort<256><<<static_cast<unsigned>(groups), 256, 0, s>>>(iota.p, spb.p, sgb.p, 1, pv.p, pdeg.p, slot_pair.p);
    }
  QVB_LAUNCH_CHECK();
  iota.release();
  DevBuf<uint32_t> len32(S + 1, s);
  DevBuf<uint64_t> sptr(S + 1, s);
  // slices padded to a multiple of 4 steps: lane-major quads (graph.cuh)
  k_slot_lens<<<grid_for(S + 1, kBlock), kBlock, 0, s>>>(slot_pair.p, pdeg.p, S, len32.p, 4, !ident);
  QVB_LAUNCH_CHECK();
  exclusive_sum_u32_u64(len32.p, sptr.p, S + 1, s);
  len32.release();
  const uint64_t slots = read_scalar(sptr.p + S, s);
  DevBuf<uint32_t> perm(S * 32 ? S * 32 : 1, s);
  DevBuf<uint16_t> scls(slots ? slots : 1, s);
  const uint64_t xcap = g.nexc ? g.nexc : 1;
  DevBuf<unsigned long long> xcount(1, s);
  DevBuf<uint64_t> xslot(xcap, s);
  DevBuf<uint32_t> xidx(xcap, s);
  QVB_CUDA(cudaMemsetAsync(xcount.p, 0, sizeof(unsigned long long), s));
  k_fill_cls<<<grid_for(S * 32, kBlock), kBlock, 0, s>>>(slot_pair.p, pv.p, pstart.p, pdeg.p, sptr.p,
                                                         col, cls_of.p, S,
                                                         static_cast<uint16_t>(ncls),
                                                         static_cast<uint16_t>(ncls + 1), perm.p, scls.p,
                                                         xcount.p, xslot.p, xidx.p);
  QVB_LAUNCH_CHECK();
  const uint64_t nx = read_scalar(xcount.p, s);
  if (nx) {  // exception slots ascending, with their R
    DevBuf<uint64_t> sslot(nx, s);
    DevBuf<uint32_t> sidx(nx, s);
    sort_pairs_u64_u32(xslot.p, sslot.p, xidx.p, sidx.p, nx, 0, bits_for(slots), s);
    DevBuf<double> xR(nx, s);
    k_x_values<<<grid_for(nx, kBlock), kBlock, 0, s>>>(sidx.p, g.exc_R, nx, xR.p);
    QVB_LAUNCH_CHECK();
    g.f1_xslot = persist(sslot);
    g.f1_xR = persist(xR);
  }
  g.f1_nx = nx;
  if (g.nlong) {
    const uint64_t m = read_scalar(g.lptr + g.nlong, s);
    DevBuf<uint16_t> lc(m ? m : 1, s);
    k_long_cls<<<grid_for(m, kBlock), kBlock, 0, s>>>(g.lcol, cls_of.p, m,
                                                      static_cast<uint16_t>(ncls + 1), lc.p);
    QVB_LAUNCH_CHECK();
    g.lcls = persist(lc);
    g.bytes += m * 2;
  }
  g.f1_S = S;
  g.f1_slots = slots;
  g.f1_ident = ident && g.nlong == 0;  // slot (s, l) is node 32 s + l
  g.f1_perm = persist(perm);
  g.f1_sptr = persist(sptr);
  g.f1_cls = persist(scls);
  g.bytes += S * 32 * 4 + (S + 1) * 8 + slots * 2 + nx * 16 + (uint64_t)ncls * 8;
  QVB_CUDA(cudaStreamSynchronize(s));
}

void build_slices(qvb_graph& g, const uint64_t* uptr, const uint32_t* col, const uint32_t* src,
                  const double* R, cudaStream_t s) {
  const uint64_t n = g.n;
  const uint64_t avg = g.eu ? (g.eu + n - 1) / n : 1;
  g.long_threshold = static_cast<uint32_t>(std::max<uint64_t>(64, 4 * avg));
  const uint32_t thr = g.long_threshold;
  g.seg_size = g.seg_size ? g.seg_size : segment_size(n);
  const char* layout_env = std::getenv("QVB_SEG_LAYOUT");
  if (n > g.seg_size && !(layout_env && std::string(layout_env) == "slices")) {
    build_nm(g, uptr, col, src, R, s);
    return;
  }
  const uint64_t seg = g.seg_size;
  const int nseg = static_cast<int>((n + seg - 1) / seg);
  if (nseg > 255) fail(QVB_ERR_UNSUPPORTED, "too many source segments (raise QVB_SEG_MB)");

  // (node, segment) pairs
  DevBuf<uint32_t> cnt(n + 1, s);
  DevBuf<uint64_t> po(n + 1, s);
  QVB_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(uint32_t), s));
  k_pair_count<<<grid_for(n, kBlock), kBlock, 0, s>>>(uptr, src, n, thr, seg, cnt.p);
  QVB_LAUNCH_CHECK();
  exclusive_sum_u32_u64(cnt.p, po.p, n + 1, s);
  cnt.release();
  const uint64_t H = read_scalar(po.p + n, s);
  g.pairs = H;
  DevBuf<uint32_t> pk(H, s), pv(H, s), pdeg(H, s);
  DevBuf<uint64_t> pstart(H, s);
  k_pair_emit<<<grid_for(n, kBlock), kBlock, 0, s>>>(uptr, src, n, thr, seg, po.p, pk.p, pv.p,
                                                     pstart.p, pdeg.p);
  QVB_LAUNCH_CHECK();
  po.release();

  // group the pairs by pass (stable: node order inside a pass)
  DevBuf<uint32_t> sorted_idx(H, s);
  DevBuf<uint64_t> seg_pair_begin(nseg + 1, s);
  {
    DevBuf<uint32_t> iota(H, s), sk(H, s);
    k_iota<<<grid_for(H, kBlock), kBlock, 0, s>>>(iota.p, H);
    QVB_LAUNCH_CHECK();
    sort_pairs_u32_u32(pk.p, sk.p, iota.p, sorted_idx.p, H, 0, bits_for(nseg - 1), s);
    k_offsets_from_sorted<<<grid_for(H, kBlock), kBlock, 0, s>>>(sk.p, H, nseg, seg_pair_begin.p);
    QVB_LAUNCH_CHECK();
  }
  pk.release();
  std::vector<uint64_t> spb(nseg + 1), sgb(nseg + 1);
  QVB_CUDA(cudaMemcpyAsync(spb.data(), seg_pair_begin.p, (nseg + 1) * 8, cudaMemcpyDeviceToHost, s));
  QVB_CUDA(cudaStreamSynchronize(s));
  sgb[0] = 0;
  for (int k = 0; k < nseg; ++k) sgb[k + 1] = sgb[k] + (spb[k + 1] - spb[k] + kWindow - 1) / kWindow;
  const uint64_t groups = sgb[nseg];
  DevBuf<uint64_t> seg_group_begin(nseg + 1, s);
  QVB_CUDA(cudaMemcpyAsync(seg_group_begin.p, sgb.data(), (nseg + 1) * 8, cudaMemcpyHostToDevice, s));
  g.nslices = groups * (kWindow / 32);
  g.seg_slice.resize(nseg + 1);
  for (int k = 0; k <= nseg; ++k) g.seg_slice[k] = sgb[k] * (kWindow / 32);
  const uint64_t S = g.nslices;

  DevBuf<uint32_t> slot_pair(S * 32 ? S * 32 : 1, s);
  if (groups)
    k_group_sort<<<static_cast<unsigned>(groups), kWindow, 0, s>>>(
        sorted_idx.p, seg_pair_begin.p, seg_group_begin.p, nseg, pv.p, pdeg.p, slot_pair.p);
  QVB_LAUNCH_CHECK();
  sorted_idx.release();
  DevBuf<uint32_t> len32(S + 1, s);
  DevBuf<uint64_t> sptr(S + 1, s);
  k_slot_lens<<<grid_for(S + 1, kBlock), kBlock, 0, s>>>(slot_pair.p, pdeg.p, S, len32.p);
  QVB_LAUNCH_CHECK();
  exclusive_sum_u32_u64(len32.p, sptr.p, S + 1, s);
  len32.release();
  g.slots = read_scalar(sptr.p + S, s);
  DevBuf<uint32_t> perm(S * 32 ? S * 32 : 1, s), scol(g.slots ? g.slots : 1, s);
  DevBuf<double> sR;
  const uint32_t pad = static_cast<uint32_t>(n);  // operand slot N holds 0
  if (R) {
    sR.alloc(g.slots ? g.slots : 1, s);
    k_fill_slots<true><<<grid_for(S * 32, kBlock), kBlock, 0, s>>>(
        slot_pair.p, pv.p, pstart.p, pdeg.p, sptr.p, col, R, S, pad, perm.p, scol.p, sR.p);
  } else {
    k_fill_slots<false><<<grid_for(S * 32, kBlock), kBlock, 0, s>>>(
        slot_pair.p, pv.p, pstart.p, pdeg.p, sptr.p, col, nullptr, S, pad, perm.p, scol.p, nullptr);
  }
  QVB_LAUNCH_CHECK();
  if (nseg > 1) QVB_CUDA(cudaMalloc(&g.state, n * sizeof(double)));

  build_long_rows(g, uptr, col, R, thr, s);
  g.perm = persist(perm);
  g.sptr = persist(sptr);
  g.scol = persist(scol);
  g.sR = sR.p ? persist(sR) : nullptr;
  g.bytes += S * 32 * 4 + (S + 1) * 8 + g.slots * (R ? 12 : 4) + (nseg > 1 ? n * 8 : 0);
}

}  // namespace qvb

using namespace qvb;

namespace qvb {

// tools/bench.cpp:22-34 + Graph::from_edges/build_csr (graph.cpp:16-47) on
// the device: out-CSR with rows in input order (stable sort by source).
// ssrc receives the source of every CSR edge.
void generate_out_csr(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                      cudaStream_t s, DevBuf<uint64_t>& ro, DevBuf<uint32_t>& col,
                      DevBuf<double>& w, DevBuf<uint32_t>& ssrc) {
  ro.alloc(n + 1, s);
  col.alloc(e, s);
  ssrc.alloc(e, s);
  if (e == 0) {
    QVB_CUDA(cudaMemsetAsync(ro.p, 0, (n + 1) * 8, s));
    return;
  }
  DevBuf<uint32_t> src(e, s), dst(e, s), iota(e, s), perm(e, s);
  DevBuf<double> w_in;
  if (weighted) w_in.alloc(e, s);
  const uint64_t state = derive_state(seed, 0xBE9C4ULL);
  k_gen_edges<<<grid_for(e, kBlock), kBlock, 0, s>>>(n, e, state, weighted, transposed, src.p,
                                                    dst.p, w_in.p);
  QVB_LAUNCH_CHECK();
  k_iota<<<grid_for(e, kBlock), kBlock, 0, s>>>(iota.p, e);
  QVB_LAUNCH_CHECK();
  sort_pairs_u32_u32(src.p, ssrc.p, iota.p, perm.p, e, 0, bits_for(n - 1), s);
  k_gather_by<uint32_t><<<grid_for(e, kBlock), kBlock, 0, s>>>(dst.p, perm.p, e, col.p);
  QVB_LAUNCH_CHECK();
  if (weighted) {
    w.alloc(e, s);
    k_gather_by<double><<<grid_for(e, kBlock), kBlock, 0, s>>>(w_in.p, perm.p, e, w.p);
    QVB_LAUNCH_CHECK();
  }
  k_offsets_from_sorted<<<grid_for(e, kBlock), kBlock, 0, s>>>(ssrc.p, e, n, ro.p);
  QVB_LAUNCH_CHECK();
}

namespace {

__global__ void k_u32_to_u64(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                             uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

}  // namespace
}  // namespace qvb

namespace {

void finish_build(qvb_graph* g, cudaEvent_t a, cudaEvent_t b, cudaStream_t s) {
  QVB_CUDA(cudaEventRecord(b, s));
  QVB_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  QVB_CUDA(cudaEventElapsedTime(&ms, a, b));
  g->build_ms = ms;
}

}  // namespace

namespace qvb {

// Columns host -> device as u32, with the range check of graph.cpp:78-81
// (edge-level code 1): host threads narrow (and range-check) the
// caller's u64 columns chunk by chunk into pinned staging slots, each chunk
// DMA'd on the thread's stream as soon as it is written — half the PCIe bytes
// of shipping u64, at pinned rather than pageable speed, with the narrowing
// overlapped with the copies. The slots are kept for the process (the first
// call pays for pinning them). Returns the first out-of-range column index
// as (i << 2) | 1, or kNone.
struct ColStage {
  uint32_t* pinned = nullptr;  // threads * 2 slots of kChunk entries
  unsigned threads = 0;
  static constexpr uint64_t kChunk = 1ull << 21;
};

void ensure_pinned(ColStage& cs) {  // by the lease holder only
  if (cs.pinned) return;
  const char* te = std::getenv("QVB_UPLOAD_THREADS");
  unsigned t = te ? static_cast<unsigned>(std::atoi(te)) : std::thread::hardware_concurrency();
  cs.threads = std::max(1u, std::min(16u, t));
  QVB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&cs.pinned),
                         cs.threads * 2 * ColStage::kChunk * sizeof(uint32_t), cudaHostAllocPortable));
}

// A small pool of staging sets (each threads x 2 pinned 8 MB slots): large
// host<->device copies of different graphs, stores or threads proceed
// concurrently, one set each; a caller waits only when QVB_STAGE_SETS (4)
// copies are already in flight. Sets are pinned on first use and kept.
class StagePool {
 public:
  static StagePool& get() {
    static StagePool p;
    return p;
  }
  ColStage* acquire() {
    std::unique_lock<std::mutex> lock(mu_);
    cv_.wait(lock, [&] { return !free_.empty() || all_.size() < max_; });
    ColStage* cs;
    if (!free_.empty()) {
      cs = free_.back();
      free_.pop_back();
    } else {
      all_.push_back(std::make_unique<ColStage>());
      cs = all_.back().get();
    }
    return cs;
  }
  void release(ColStage* cs) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      free_.push_back(cs);
    }
    cv_.notify_one();
  }

 private:
  StagePool() {
    const char* e = std::getenv("QVB_STAGE_SETS");
    max_ = e ? std::max<size_t>(1, std::strtoull(e, nullptr, 10)) : 4;
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<std::unique_ptr<ColStage>> all_;
  std::vector<ColStage*> free_;
  size_t max_ = 4;
};

struct StageLease {
  ColStage* cs;
  StageLease() : cs(StagePool::get().acquire()) {
    try {
      ensure_pinned(*cs);
    } catch (...) {
      StagePool::get().release(cs);
      throw;
    }
  }
  ~StageLease() { StagePool::get().release(cs); }
  StageLease(const StageLease&) = delete;
  StageLease& operator=(const StageLease&) = delete;
};

// Device -> pageable host copy through the same pinned slots: each thread
// DMAs its chunks into its two slots (one in flight while it copies the
// other out), instead of the driver's single-threaded pageable staging.
// Stream-ordered after the work queued on s; returns when the data is in dst.
void copy_to_host(void* dst, const void* src, uint64_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  constexpr uint64_t kBytes = ColStage::kChunk * sizeof(uint32_t);
  if (bytes < 4 * kBytes) {  // small: one pageable copy
    QVB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
    return;
  }
  StageLease lease;  // one staging set for this copy; others may run concurrently
  ColStage& cs = *lease.cs;
  const uint64_t nchunks = (bytes + kBytes - 1) / kBytes;
  const unsigned T = static_cast<unsigned>(std::min<uint64_t>(cs.threads, nchunks));
  cudaEvent_t start;
  QVB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  QVB_CUDA(cudaEventRecord(start, s));
  std::vector<cudaStream_t> st(T, nullptr);
  std::vector<cudaEvent_t> ev(2 * T, nullptr);
  for (unsigned t = 0; t < T; ++t) {
    QVB_CUDA(cudaStreamCreateWithFlags(&st[t], cudaStreamNonBlocking));
    QVB_CUDA(cudaStreamWaitEvent(st[t], start, 0));
    for (int k = 0; k < 2; ++k) QVB_CUDA(cudaEventCreateWithFlags(&ev[2 * t + k], cudaEventDisableTiming));
  }
  std::vector<int> err(T, 0);
  int dev = 0;
  QVB_CUDA(cudaGetDevice(&dev));
  auto work = [&](unsigned t) {
    cudaSetDevice(dev);
    auto issue = [&](uint64_t c, uint64_t k) {
      char* slot = reinterpret_cast<char*>(cs.pinned) + (2 * t + (k & 1)) * kBytes;
      const uint64_t a = c * kBytes, len = std::min(kBytes, bytes - a);
      return cudaMemcpyAsync(slot, static_cast<const char*>(src) + a, len, cudaMemcpyDeviceToHost, st[t]) ==
                 cudaSuccess &&
             cudaEventRecord(ev[2 * t + (k & 1)], st[t]) == cudaSuccess;
    };
    uint64_t k = 0;
    if (t < nchunks && !issue(t, 0)) { err[t] = 1; return; }
    for (uint64_t c = t; c < nchunks; c += T, ++k) {
      if (c + T < nchunks && !issue(c + T, k + 1)) { err[t] = 1; return; }  // next chunk in flight
      if (cudaEventSynchronize(ev[2 * t + (k & 1)]) != cudaSuccess) { err[t] = 1; return; }
      const uint64_t a = c * kBytes, len = std::min(kBytes, bytes - a);
      std::memcpy(static_cast<char*>(dst) + a, reinterpret_cast<char*>(cs.pinned) + (2 * t + (k & 1)) * kBytes, len);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  int failed = 0;
  for (unsigned t = 0; t < T; ++t) {
    failed |= err[t];
    cudaStreamSynchronize(st[t]);
    cudaStreamDestroy(st[t]);
    cudaEventDestroy(ev[2 * t]);
    cudaEventDestroy(ev[2 * t + 1]);
  }
  cudaEventDestroy(start);
  if (failed) fail(QVB_ERR_CUDA, "device to host copy failed");
}

unsigned long long upload_columns(const uint64_t* col, uint64_t e, uint64_t n, uint32_t* dcol,
                                  cudaStream_t s) {
  constexpr unsigned long long kNoBad = ~0ull;
  StageLease lease;  // one staging set for this copy; others may run concurrently
  ColStage& cs = *lease.cs;
  const uint64_t nchunks = (e + ColStage::kChunk - 1) / ColStage::kChunk;
  const unsigned T = static_cast<unsigned>(std::min<uint64_t>(cs.threads, nchunks));
  cudaEvent_t start;
  QVB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  QVB_CUDA(cudaEventRecord(start, s));  // dcol is allocated in stream order on s
  std::vector<cudaStream_t> st(T, nullptr);
  std::vector<cudaEvent_t> ev(2 * T, nullptr), fin(T, nullptr);
  for (unsigned t = 0; t < T; ++t) {
    QVB_CUDA(cudaStreamCreateWithFlags(&st[t], cudaStreamNonBlocking));
    QVB_CUDA(cudaStreamWaitEvent(st[t], start, 0));
    for (int k = 0; k < 2; ++k) QVB_CUDA(cudaEventCreateWithFlags(&ev[2 * t + k], cudaEventDisableTiming));
    QVB_CUDA(cudaEventCreateWithFlags(&fin[t], cudaEventDisableTiming));
  }
  std::vector<unsigned long long> bad(T, kNoBad);
  std::vector<int> err(T, 0);
  int dev = 0;
  QVB_CUDA(cudaGetDevice(&dev));
  auto work = [&](unsigned t) {
    cudaSetDevice(dev);
    uint64_t k = 0;
    for (uint64_t c = t; c < nchunks; c += T, ++k) {
      uint32_t* slot = cs.pinned + (2 * t + (k & 1)) * ColStage::kChunk;
      if (k >= 2 && cudaEventSynchronize(ev[2 * t + (k & 1)]) != cudaSuccess) { err[t] = 1; return; }
      const uint64_t a = c * ColStage::kChunk, len = std::min(ColStage::kChunk, e - a);
      const uint64_t* in = col + a;
      for (uint64_t i = 0; i < len; ++i) {
        const uint64_t v = in[i];
        if (v >= n && bad[t] == kNoBad) bad[t] = ((a + i) << 2) | 1;
        slot[i] = static_cast<uint32_t>(v < n ? v : 0);
      }
      if (cudaMemcpyAsync(dcol + a, slot, len * sizeof(uint32_t), cudaMemcpyHostToDevice, st[t]) !=
              cudaSuccess ||
          cudaEventRecord(ev[2 * t + (k & 1)], st[t]) != cudaSuccess) {
        err[t] = 1;
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  int failed = 0;
  for (unsigned t = 0; t < T; ++t) {
    failed |= err[t];
    QVB_CUDA(cudaEventRecord(fin[t], st[t]));
    QVB_CUDA(cudaStreamWaitEvent(s, fin[t], 0));
  }
  // the slots are reused by the next call: this one's copies must be done
  for (unsigned t = 0; t < T; ++t) QVB_CUDA(cudaStreamSynchronize(st[t]));
  for (unsigned t = 0; t < T; ++t) {
    cudaStreamDestroy(st[t]);
    cudaEventDestroy(ev[2 * t]);
    cudaEventDestroy(ev[2 * t + 1]);
    cudaEventDestroy(fin[t]);
  }
  cudaEventDestroy(start);
  if (failed) fail(QVB_ERR_CUDA, "column upload failed");
  unsigned long long first = kNoBad;
  for (auto b : bad) first = std::min(first, b);
  return first;
}

// Host out-CSR -> device (row offsets u64, columns u32, weights f64 or none)
// with Graph::validate's checks and messages (graph.cpp:58-93); the
// all-zero-weights row check runs with the row sums (k_row_sums).
void upload_out_csr(uint64_t n, uint64_t e, const uint64_t* row_offsets, const uint64_t* col,
                    const double* weights, cudaStream_t s, DevBuf<uint64_t>& ro,
                    DevBuf<uint32_t>& dcol, DevBuf<double>& dw) {
  if (n == 0) fail(QVB_ERR_VALIDATION, "empty graph: node count is zero");
  if (!row_offsets || (e && !col)) fail(QVB_ERR_VALIDATION, "null graph arrays");
  if (n > kMaxNodes || e > kMaxEdges)
    fail(QVB_ERR_UNSUPPORTED, "graph exceeds the device path limits (n < 2^31, e < 2^32)");
  if (row_offsets[0] != 0 || row_offsets[n] != e)
    fail(QVB_ERR_VALIDATION, "row_offsets endpoints invalid");
  ro.alloc(n + 1, s);
  QVB_CUDA(cudaMemcpyAsync(ro.p, row_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
  DevBuf<unsigned long long> flags(2, s);
  QVB_CUDA(cudaMemsetAsync(flags.p, 0xFF, 2 * sizeof(unsigned long long), s));
  k_check_ro<<<grid_for(n, kBlock), kBlock, 0, s>>>(ro.p, n, flags.p);
  QVB_LAUNCH_CHECK();
  unsigned long long bad_mono = read_scalar(flags.p, s);
  if (bad_mono != kNone)
    fail(QVB_ERR_VALIDATION, "row_offsets not non-decreasing at node " + std::to_string(bad_mono));

  dcol.alloc(e, s);
  unsigned long long bad_col = kNone;
  if (e) {
    bad_col = upload_columns(col, e, n, dcol.p, s);
    if (weights) {
      dw.alloc(e, s);
      QVB_CUDA(cudaMemcpyAsync(dw.p, weights, e * 8, cudaMemcpyHostToDevice, s));
      k_check_weights<<<grid_for(e, kBlock), kBlock, 0, s>>>(dw.p, e, flags.p + 1);
      QVB_LAUNCH_CHECK();
    }
  }
  unsigned long long bad_edge = std::min(read_scalar(flags.p + 1, s), bad_col);
  if (bad_edge != kNone) {
    // The first failing edge names its row (graph.cpp:75-91 walks rows in
    // order; a zero-weight row before it would be reported first).
    const uint64_t ei = bad_edge >> 2;
    const uint64_t row =
        static_cast<uint64_t>(std::upper_bound(row_offsets, row_offsets + n + 1, ei) - row_offsets) - 1;
    // Rows before `row` may still fail the all-zero check: run it on them.
    bool zero_before = false;
    uint64_t zrow = 0;
    if (weights) {
      for (uint64_t i = 0; i < row && !zero_before; ++i) {
        bool anyp = row_offsets[i] == row_offsets[i + 1];
        for (uint64_t k = row_offsets[i]; k < row_offsets[i + 1]; ++k) anyp |= weights[k] > 0.0;
        if (!anyp) {
          zero_before = true;
          zrow = i;
        }
      }
    }
    if (zero_before)
      fail(QVB_ERR_VALIDATION,
           "node " + std::to_string(zrow) + " has out-edges but all weights are zero");
    if ((bad_edge & 3) == 1)
      fail(QVB_ERR_VALIDATION, "column index out of range at node " + std::to_string(row));
    fail(QVB_ERR_VALIDATION, "negative or NaN edge weight at node " + std::to_string(row));
  }
}

}  // namespace qvb

extern "C" int qvb_graph_upload(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                                const uint64_t* col, const double* weights, void* stream,
                                qvb_graph** out) {
  return guarded([&] {
    if (!out) fail(QVB_ERR_VALIDATION, "out is null");
    *out = nullptr;
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto g = std::make_unique<qvb_graph>();
    g->device = device;
    g->n = n;
    g->e = e;
    cudaEvent_t ea, eb;
    QVB_CUDA(cudaEventCreate(&ea));
    QVB_CUDA(cudaEventCreate(&eb));
    QVB_CUDA(cudaEventRecord(ea, s));
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> dcol;
    DevBuf<double> dw;
    const bool trace = std::getenv("QVB_TRACE_UPLOAD") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    upload_out_csr(n, e, row_offsets, col, weights, s, ro, dcol, dw);
    if (trace) QVB_CUDA(cudaStreamSynchronize(s));
    auto t1 = std::chrono::steady_clock::now();
    build_in_csr(*g, ro.p, dcol.p, dw.p, nullptr, s);
    if (trace) QVB_CUDA(cudaStreamSynchronize(s));
    auto t2 = std::chrono::steady_clock::now();
    finish_build(g.get(), ea, eb, s);
    if (trace)
      std::fprintf(stderr, "qvb_graph_upload: upload %.2f ms, in-CSR build %.2f ms (host clock)\n",
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(t2 - t1).count());
    cudaEventDestroy(ea);
    cudaEventDestroy(eb);
    *out = g.release();
  });
}

extern "C" int qvb_graph_synthetic(int device, uint64_t n, uint64_t e, uint64_t seed, int weighted,
                                   int transposed, void* stream, qvb_graph** out) {
  return guarded([&] {
    if (!out) fail(QVB_ERR_VALIDATION, "out is null");
    *out = nullptr;
    if (n == 0) fail(QVB_ERR_VALIDATION, "empty graph: node count is zero");
    if (n > kMaxNodes || e > kMaxEdges)
      fail(QVB_ERR_UNSUPPORTED, "graph exceeds the device path limits (n < 2^31, e < 2^32)");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto g = std::make_unique<qvb_graph>();
    g->device = device;
    g->n = n;
    g->e = e;
    cudaEvent_t ea, eb;
    QVB_CUDA(cudaEventCreate(&ea));
    QVB_CUDA(cudaEventCreate(&eb));
    QVB_CUDA(cudaEventRecord(ea, s));
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> col, ssrc;
    DevBuf<double> w;
    generate_out_csr(n, e, seed, weighted, transposed, s, ro, col, w, ssrc);
    build_in_csr(*g, ro.p, col.p, w.p, ssrc.p, s);
    finish_build(g.get(), ea, eb, s);
    cudaEventDestroy(ea);
    cudaEventDestroy(eb);
    *out = g.release();
  });
}

extern "C" int qvb_synthetic_csr(int device, uint64_t n, uint64_t e, uint64_t seed, int weighted,
                                 int transposed, uint64_t* row_offsets, uint64_t* col,
                                 double* weights) {
  return guarded([&] {
    if (n == 0) fail(QVB_ERR_VALIDATION, "empty graph: node count is zero");
    if (n > kMaxNodes || e > kMaxEdges)
      fail(QVB_ERR_UNSUPPORTED, "graph exceeds the device path limits (n < 2^31, e < 2^32)");
    if (!row_offsets || (e && (!col || !weights))) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> c, ssrc;
    DevBuf<double> w;
    generate_out_csr(n, e, seed, weighted, transposed, s, ro, c, w, ssrc);
    ssrc.release();
    QVB_CUDA(cudaMemcpyAsync(row_offsets, ro.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (e) {
      const uint64_t chunk = 1ull << 26;
      DevBuf<uint64_t> wide(std::min(chunk, e), s);
      for (uint64_t b = 0; b < e; b += chunk) {
        const uint64_t m = std::min(chunk, e - b);
        k_u32_to_u64<<<grid_for(m, kBlock), kBlock, 0, s>>>(c.p + b, wide.p, m);
        QVB_LAUNCH_CHECK();
        QVB_CUDA(cudaMemcpyAsync(col + b, wide.p, m * 8, cudaMemcpyDeviceToHost, s));
      }
      if (weighted) {
        QVB_CUDA(cudaMemcpyAsync(weights, w.p, e * 8, cudaMemcpyDeviceToHost, s));
      } else {
        QVB_CUDA(cudaStreamSynchronize(s));
        std::fill(weights, weights + e, 1.0);
      }
    }
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}

namespace qvb {
namespace {

// qvb_graph_in_rows: one thread per listed node walks its runs of the
// node-major layout (pass by pass = ascending source) or its long row; with
// src == nullptr it only counts.
struct InRowsView {  // the device arrays k_in_rows reads
  uint32_t layout;
  uint64_t nlong, nm_S, nm_region_count;
  const uint32_t *lnode, *lcol, *exc_src, *nm_col;
  const uint64_t *lptr, *nm_sbase;
  const double *lR, *exc_R, *inv, *nm_R;
  const uint8_t* nm_lenf;
};

__global__ void k_in_rows(const InRowsView g, const uint64_t* __restrict__ nodes, uint64_t count,
                          const uint64_t* __restrict__ row_ptr, uint32_t* __restrict__ src,
                          double* __restrict__ R, uint64_t* __restrict__ lens) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t v = nodes[i];
  uint64_t at = src ? row_ptr[i] : 0, m = 0;
  auto emit = [&](uint32_t c, double r_weighted, bool weighted) {
    if (src) {
      uint32_t s = c;
      double r;
      if (weighted) {
        r = r_weighted;
      } else if (c & kExcFlag) {
        s = g.exc_src[c & ~kExcFlag];
        r = g.exc_R[c & ~kExcFlag];
      } else {
        r = g.inv[c];
      }
      src[at] = s;
      R[at] = r;
      ++at;
    }
    ++m;
  };
  const bool weighted = g.layout == 1;
  // long row?
  uint64_t lo = 0, hi = g.nlong;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (g.lnode[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  if (lo < g.nlong && g.lnode[lo] == v) {
    for (uint64_t e = g.lptr[lo]; e < g.lptr[lo + 1]; ++e) emit(g.lcol[e], weighted ? g.lR[e] : 0.0, weighted);
  } else {
    const uint64_t S = g.nm_S, sl = v / 32, lane = v % 32;
    const int nseg = static_cast<int>(g.nm_region_count);
    for (int k = 0; k < nseg; ++k) {
      const uint8_t* lf = g.nm_lenf + (uint64_t)k * S * 32 + sl * 32;
      uint64_t off = 0;
      for (uint64_t l = 0; l < lane; ++l) off += lf[l] & kNmLen;
      const uint64_t len = lf[lane] & kNmLen;
      const uint64_t b = g.nm_sbase[(uint64_t)k * S + sl] + off;
      for (uint64_t t = 0; t < len; ++t) emit(g.nm_col[b + t], weighted ? g.nm_R[b + t] : 0.0, weighted);
    }
  }
  if (!src) lens[i] = m;
}

}  // namespace
}  // namespace qvb

extern "C" int qvb_graph_in_rows(const qvb_graph* g, const uint64_t* nodes, uint64_t count,
                                 uint64_t* row_ptr, uint32_t* src, double* R) {
  return guarded([&] {
    if (!g || (count && (!nodes || !row_ptr))) fail(QVB_ERR_VALIDATION, "null argument");
    if (!g->nm) fail(QVB_ERR_UNSUPPORTED, "in_rows needs the node-major (segmented) layout");
    DeviceGuard dg(g->device);
    cudaStream_t s = nullptr;
    for (uint64_t i = 0; i < count; ++i)
      if (nodes[i] >= g->n) fail(QVB_ERR_VALIDATION, "node " + std::to_string(nodes[i]) + " out of range");
    DevBuf<uint64_t> dn(count ? count : 1, s), dl(count ? count : 1, s), dp(count + 1, s);
    QVB_CUDA(cudaMemcpyAsync(dn.p, nodes, count * 8, cudaMemcpyHostToDevice, s));
    const InRowsView gv{g->layout, g->nlong, g->nm_S, g->nm_region_count, g->lnode, g->lcol,
                        g->exc_src, g->nm_col, g->lptr, g->nm_sbase, g->lR, g->exc_R, g->inv,
                        g->nm_R, g->nm_lenf};
    const unsigned blocks = static_cast<unsigned>((count + 127) / 128);
    std::vector<uint64_t> lens(count);
    if (count) {
      k_in_rows<<<blocks, 128, 0, s>>>(gv, dn.p, count, nullptr, nullptr, nullptr, dl.p);
      QVB_LAUNCH_CHECK();
      QVB_CUDA(cudaMemcpyAsync(lens.data(), dl.p, count * 8, cudaMemcpyDeviceToHost, s));
      QVB_CUDA(cudaStreamSynchronize(s));
    }
    row_ptr[0] = 0;
    for (uint64_t i = 0; i < count; ++i) row_ptr[i + 1] = row_ptr[i] + lens[i];
    if (src && R && count) {
      const uint64_t tot = row_ptr[count];
      DevBuf<uint32_t> ds(tot ? tot : 1, s);
      DevBuf<double> dr(tot ? tot : 1, s);
      QVB_CUDA(cudaMemcpyAsync(dp.p, row_ptr, (count + 1) * 8, cudaMemcpyHostToDevice, s));
      k_in_rows<<<blocks, 128, 0, s>>>(gv, dn.p, count, dp.p, ds.p, dr.p, nullptr);
      QVB_LAUNCH_CHECK();
      QVB_CUDA(cudaMemcpyAsync(src, ds.p, tot * 4, cudaMemcpyDeviceToHost, s));
      QVB_CUDA(cudaMemcpyAsync(R, dr.p, tot * 8, cudaMemcpyDeviceToHost, s));
      QVB_CUDA(cudaStreamSynchronize(s));
    }
  });
}


extern "C" int qvb_graph_last_sweep_ms(const qvb_graph* g, double* ms) {
  return guarded([&] {
    if (!g || !ms) fail(QVB_ERR_VALIDATION, "null argument");
    if (!g->ev[0]) fail(QVB_ERR_VALIDATION, "no sweep has run on this graph");
    DeviceGuard dg(g->device);
    QVB_CUDA(cudaEventSynchronize(g->ev[1]));
    float f = 0;
    QVB_CUDA(cudaEventElapsedTime(&f, g->ev[0], g->ev[1]));
    *ms = f;
  });
}

extern "C" int qvb_graph_phase_ms(const qvb_graph* g, double* ms, uint32_t* launches) {
  return guarded([&] {
    if (!g || !ms) fail(QVB_ERR_VALIDATION, "null argument");
    for (int i = 0; i < 4; ++i) ms[i] = 0.0;
    DeviceGuard dg(g->device);
    for (size_t i = 0; i < g->phase_used; ++i) {
      const auto& pe = g->phase_ev[i];
      QVB_CUDA(cudaEventSynchronize(pe.b));
      float f = 0;
      QVB_CUDA(cudaEventElapsedTime(&f, pe.a, pe.b));
      ms[pe.phase] += f;
    }
    if (launches) *launches = g->launches;
  });
}

extern "C" int qvb_graph_info_get(const qvb_graph* g, qvb_graph_info* info) {
  return guarded([&] {
    if (!g || !info) fail(QVB_ERR_VALIDATION, "null argument");
    std::memset(info, 0, sizeof *info);
    info->node_count = g->n;
    info->edge_count = g->e;
    info->unique_edge_count = g->eu;
    info->exception_count = g->nexc;
    info->layout = g->layout;
    info->device = static_cast<uint32_t>(g->device);
    info->device_bytes = g->bytes;
    info->build_ms = g->build_ms;
    info->classes = g->ncls;
    info->segments = g->seg_slice.empty() ? 1u : static_cast<uint32_t>(g->seg_slice.size() - 1);
    info->first_slots = g->f1_slots;
    info->segment_columns = g->nm ? g->nm_cols : 0;
  });
}

extern "C" int qvb_graph_destroy(qvb_graph* g) {
  return guarded([&] { delete g; });
}

namespace qvb {
namespace {

__global__ void k_transpose_out(const uint32_t* __restrict__ seid, const uint32_t* __restrict__ src,
                                const double* __restrict__ w, uint64_t e, uint64_t* __restrict__ tcol,
                                double* __restrict__ tw) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = seid[k];
    tcol[k] = src[i];
    tw[k] = w ? w[i] : 1.0;
  }
}

}  // namespace
}  // namespace qvb

// in_adjacency (graph.cpp:260-281) on the device: the transposed graph with
// parallel edges kept, rows in ascending source order (stable sort by
// destination over the source-major edge order).
namespace qvb {
namespace {
__global__ void k_unit_check(const double* __restrict__ w, uint64_t e, int* __restrict__ non_unit) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (w[i] != 1.0) *non_unit = 1;
}
__global__ void k_gather_weights(const uint32_t* __restrict__ seid, const double* __restrict__ w,
                                 uint64_t e, double* __restrict__ tw) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x)
    tw[k] = w[seid[k]];
}
__global__ void k_gather_src(const uint32_t* __restrict__ seid, const uint32_t* __restrict__ src,
                             uint64_t e, uint32_t* __restrict__ tsrc) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x)
    tsrc[k] = src[seid[k]];
}
}  // namespace

void device_transpose(uint64_t n, uint64_t e, const uint64_t* ro_h, const uint64_t* col_h,
                      const double* w_h, cudaStream_t s, DevBuf<uint64_t>& tptr,
                      DevBuf<uint32_t>& tsrc, DevBuf<double>& tw, DevBuf<double>& rs,
                      bool* unit_weights) {
  DevBuf<uint64_t> ro;
  DevBuf<uint32_t> dcol;
  DevBuf<double> dw;
  upload_out_csr(n, e, ro_h, col_h, w_h, s, ro, dcol, dw);
  rs.alloc(n, s);
  {
    DevBuf<double> inv(n, s);
    DevBuf<unsigned long long> flag(1, s);
    QVB_CUDA(cudaMemsetAsync(flag.p, 0xFF, sizeof(unsigned long long), s));
    k_row_sums<<<grid_for(n, kBlock), kBlock, 0, s>>>(ro.p, dw.p, n, rs.p, inv.p, flag.p);
    QVB_LAUNCH_CHECK();
    const unsigned long long z = read_scalar(flag.p, s);
    if (z != kNone)
      fail(QVB_ERR_VALIDATION, "node " + std::to_string(z) + " has out-edges but all weights are zero");
  }
  *unit_weights = true;
  if (dw.p && e) {
    DevBuf<int> nu(1, s);
    QVB_CUDA(cudaMemsetAsync(nu.p, 0, sizeof(int), s));
    k_unit_check<<<grid_for(e, kBlock), kBlock, 0, s>>>(dw.p, e, nu.p);
    QVB_LAUNCH_CHECK();
    *unit_weights = read_scalar(nu.p, s) == 0;
  }
  tptr.alloc(n + 1, s);
  tsrc.alloc(e ? e : 1, s);
  if (e == 0) {
    QVB_CUDA(cudaMemsetAsync(tptr.p, 0, (n + 1) * 8, s));
    return;
  }
  DevBuf<uint32_t> src(e, s);
  {
    DevBuf<uint32_t> marks(e, s), incl(e, s), row_of_rank(n, s);
    QVB_CUDA(cudaMemsetAsync(marks.p, 0, e * sizeof(uint32_t), s));
    k_row_marks<<<grid_for(n, kBlock), kBlock, 0, s>>>(ro.p, n, e, marks.p);
    QVB_LAUNCH_CHECK();
    inclusive_sum_u32_u32(marks.p, incl.p, e, s);
    k_rank_rows<<<grid_for(n, kBlock), kBlock, 0, s>>>(ro.p, n, incl.p, e, row_of_rank.p);
    QVB_LAUNCH_CHECK();
    k_src_from_rank<<<grid_for(e, kBlock), kBlock, 0, s>>>(incl.p, row_of_rank.p, e, src.p);
    QVB_LAUNCH_CHECK();
  }
  DevBuf<uint32_t> sdst(e, s), seid(e, s);
  {
    DevBuf<uint32_t> iota(e, s);
    k_iota<<<grid_for(e, kBlock), kBlock, 0, s>>>(iota.p, e);
    QVB_LAUNCH_CHECK();
    sort_pairs_u32_u32(dcol.p, sdst.p, iota.p, seid.p, e, 0, bits_for(n - 1), s);
  }
  k_offsets_from_sorted<<<grid_for(e, kBlock), kBlock, 0, s>>>(sdst.p, e, n, tptr.p);
  QVB_LAUNCH_CHECK();
  k_gather_src<<<grid_for(e, kBlock), kBlock, 0, s>>>(seid.p, src.p, e, tsrc.p);
  QVB_LAUNCH_CHECK();
  if (dw.p) {
    tw.alloc(e, s);
    k_gather_weights<<<grid_for(e, kBlock), kBlock, 0, s>>>(seid.p, dw.p, e, tw.p);
    QVB_LAUNCH_CHECK();
  }
}

}  // namespace qvb

extern "C" int qvb_in_adjacency(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                                const uint64_t* col, const double* weights, uint64_t* t_row_offsets,
                                uint64_t* t_col, double* t_weights) {
  return guarded([&] {
    if (!t_row_offsets || (e && (!t_col || !t_weights))) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> dcol;
    DevBuf<double> dw;
    upload_out_csr(n, e, row_offsets, col, weights, s, ro, dcol, dw);
    {
      DevBuf<double> rs(n, s), inv(n, s);
      DevBuf<unsigned long long> flag(1, s);
      QVB_CUDA(cudaMemsetAsync(flag.p, 0xFF, sizeof(unsigned long long), s));
      k_row_sums<<<grid_for(n, kBlock), kBlock, 0, s>>>(ro.p, dw.p, n, rs.p, inv.p, flag.p);
      QVB_LAUNCH_CHECK();
      const unsigned long long z = read_scalar(flag.p, s);
      if (z != kNone)
        fail(QVB_ERR_VALIDATION, "node " + std::to_string(z) + " has out-edges but all weights are zero");
    }
    DevBuf<uint64_t> tro(n + 1, s);
    if (e == 0) {
      QVB_CUDA(cudaMemsetAsync(tro.p, 0, (n + 1) * 8, s));
    } else {
      DevBuf<uint32_t> src(e, s), marks(e, s), incl(e, s), row_of_rank(n, s);
      QVB_CUDA(cudaMemsetAsync(marks.p, 0, e * sizeof(uint32_t), s));
      k_row_marks<<<grid_for(n, kBlock), kBlock, 0, s>>>(ro.p, n, e, marks.p);
      QVB_LAUNCH_CHECK();
      inclusive_sum_u32_u32(marks.p, incl.p, e, s);
      k_rank_rows<<<grid_for(n, kBlock), kBlock, 0, s>>>(ro.p, n, incl.p, e, row_of_rank.p);
      QVB_LAUNCH_CHECK();
      k_src_from_rank<<<grid_for(e, kBlock), kBlock, 0, s>>>(incl.p, row_of_rank.p, e, src.p);
      QVB_LAUNCH_CHECK();
      DevBuf<uint32_t> iota(e, s), sdst(e, s), seid(e, s);
      k_iota<<<grid_for(e, kBlock), kBlock, 0, s>>>(iota.p, e);
      QVB_LAUNCH_CHECK();
      sort_pairs_u32_u32(dcol.p, sdst.p, iota.p, seid.p, e, 0, bits_for(n - 1), s);
      k_offsets_from_sorted<<<grid_for(e, kBlock), kBlock, 0, s>>>(sdst.p, e, n, tro.p);
      QVB_LAUNCH_CHECK();
      DevBuf<uint64_t> tcol(e, s);
      DevBuf<double> tw(e, s);
      k_transpose_out<<<grid_for(e, kBlock), kBlock, 0, s>>>(seid.p, src.p, dw.p, e, tcol.p, tw.p);
      QVB_LAUNCH_CHECK();
      QVB_CUDA(cudaMemcpyAsync(t_col, tcol.p, e * 8, cudaMemcpyDeviceToHost, s));
      QVB_CUDA(cudaMemcpyAsync(t_weights, tw.p, e * 8, cudaMemcpyDeviceToHost, s));
    }
    QVB_CUDA(cudaMemcpyAsync(t_row_offsets, tro.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}

// ---- drop-in construction/validation on the device -----------------------------
namespace qvb {
namespace {

// from_edges input checks in input order (graph.cpp:21-33): the first edge
// with an endpoint out of range (code 0) or a bad weight (code 1) wins;
// splits the AoS edges into u32 source / destination and the weights.
__global__ void k_split_edges(const qvb_edge* __restrict__ edges, uint64_t e, uint64_t n,
                              uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                              double* __restrict__ w, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const qvb_edge ed = edges[i];
    if (ed.src >= n || ed.dst >= n) atomicMin(bad, (unsigned long long)(i << 1));
    else if (!(ed.weight >= 0.0)) atomicMin(bad, (unsigned long long)((i << 1) | 1));
    src[i] = static_cast<uint32_t>(ed.src < n ? ed.src : 0);
    dst[i] = static_cast<uint32_t>(ed.dst < n ? ed.dst : 0);
    w[i] = ed.weight;
  }
}

__global__ void k_u32_to_u64_out(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                 uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

void check_zero_rows(const uint64_t* d_ro, const double* d_w, uint64_t n, cudaStream_t s) {
  DevBuf<double> rs(n, s), inv(n, s);
  DevBuf<unsigned long long> flag(1, s);
  QVB_CUDA(cudaMemsetAsync(flag.p, 0xFF, sizeof(unsigned long long), s));
  k_row_sums<<<grid_for(n, kBlock), kBlock, 0, s>>>(d_ro, d_w, n, rs.p, inv.p, flag.p);
  QVB_LAUNCH_CHECK();
  const unsigned long long z = read_scalar(flag.p, s);
  if (z != kNone)
    fail(QVB_ERR_VALIDATION, "node " + std::to_string(z) + " has out-edges but all weights are zero");
}

}  // namespace
}  // namespace qvb

extern "C" int qvb_graph_validate(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                                  const uint64_t* col, const double* weights) {
  return guarded([&] {
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> dcol;
    DevBuf<double> dw;
    upload_out_csr(n, e, row_offsets, col, weights, s, ro, dcol, dw);
    check_zero_rows(ro.p, dw.p, n, s);
  });
}

extern "C" int qvb_build_csr(int device, uint64_t n, const qvb_edge* edges, uint64_t e,
                             uint64_t* row_offsets, uint64_t* col, double* weights) {
  return guarded([&] {
    if (n == 0) fail(QVB_ERR_VALIDATION, "empty graph: node count is zero");
    if (!row_offsets || (e && (!edges || !col || !weights))) fail(QVB_ERR_VALIDATION, "null argument");
    if (n > kMaxNodes || e > kMaxEdges)
      fail(QVB_ERR_UNSUPPORTED, "graph exceeds the device path limits (n < 2^31, e < 2^32)");
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> ro(n + 1, s);
    if (e == 0) {
      QVB_CUDA(cudaMemsetAsync(ro.p, 0, (n + 1) * 8, s));
      QVB_CUDA(cudaMemcpyAsync(row_offsets, ro.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
      QVB_CUDA(cudaStreamSynchronize(s));
      return;
    }
    DevBuf<uint32_t> src(e, s), dst(e, s), iota(e, s), perm(e, s), ssrc(e, s);
    DevBuf<double> w(e, s), sw(e, s);
    {
      DevBuf<qvb_edge> dedges(e, s);
      QVB_CUDA(cudaMemcpyAsync(dedges.p, edges, e * sizeof(qvb_edge), cudaMemcpyHostToDevice, s));
      DevBuf<unsigned long long> bad(1, s);
      QVB_CUDA(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
      k_split_edges<<<grid_for(e, kBlock), kBlock, 0, s>>>(dedges.p, e, n, src.p, dst.p, w.p, bad.p);
      QVB_LAUNCH_CHECK();
      const unsigned long long b = read_scalar(bad.p, s);
      if (b != kNone) {
        const qvb_edge& ed = edges[b >> 1];
        if ((b & 1) == 0)
          fail(QVB_ERR_VALIDATION, "edge endpoint " + std::to_string(std::max(ed.src, ed.dst)) +
                                       " out of range for node count " + std::to_string(n));
        fail(QVB_ERR_VALIDATION, "negative or NaN edge weight on edge " + std::to_string(ed.src) +
                                     " -> " + std::to_string(ed.dst));
      }
    }
    // stable by source: build_csr's cursor walk keeps input order in a row
    k_iota<<<grid_for(e, kBlock), kBlock, 0, s>>>(iota.p, e);
    QVB_LAUNCH_CHECK();
    sort_pairs_u32_u32(src.p, ssrc.p, iota.p, perm.p, e, 0, bits_for(n - 1), s);
    k_offsets_from_sorted<<<grid_for(e, kBlock), kBlock, 0, s>>>(ssrc.p, e, n, ro.p);
    QVB_LAUNCH_CHECK();
    k_gather_by<double><<<grid_for(e, kBlock), kBlock, 0, s>>>(w.p, perm.p, e, sw.p);
    QVB_LAUNCH_CHECK();
    check_zero_rows(ro.p, sw.p, n, s);  // the validate() at the end of build_csr
    {
      DevBuf<uint32_t> scol(e, s);
      k_gather_by<uint32_t><<<grid_for(e, kBlock), kBlock, 0, s>>>(dst.p, perm.p, e, scol.p);
      QVB_LAUNCH_CHECK();
      DevBuf<uint64_t> col64(e, s);
      k_u32_to_u64_out<<<grid_for(e, kBlock), kBlock, 0, s>>>(scol.p, col64.p, e);
      QVB_LAUNCH_CHECK();
      copy_to_host(col, col64.p, e * 8, s);
    }
    copy_to_host(weights, sw.p, e * 8, s);
    QVB_CUDA(cudaMemcpyAsync(row_offsets, ro.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int qvb_transition_view(int device, uint64_t n, uint64_t e, const uint64_t* row_offsets,
                                   const uint64_t* col, const double* weights, double* row_sums,
                                   uint64_t* distinct_out, int* has_parallel_edges,
                                   qvb_graph** keep) {
  return guarded([&] {
    if (!row_sums || !distinct_out || !has_parallel_edges) fail(QVB_ERR_VALIDATION, "null argument");
    if (keep) *keep = nullptr;
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    auto g = std::make_unique<qvb_graph>();
    g->device = device;
    g->n = n;
    g->e = e;
    cudaEvent_t ea, eb;
    QVB_CUDA(cudaEventCreate(&ea));
    QVB_CUDA(cudaEventCreate(&eb));
    QVB_CUDA(cudaEventRecord(ea, s));
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> dcol;
    DevBuf<double> dw;
    upload_out_csr(n, e, row_offsets, col, weights, s, ro, dcol, dw);
    DevBuf<double> rs(n, s);
    DevBuf<uint32_t> distinct(n, s);
    ViewOut view;
    view.row_sums = rs.p;
    view.distinct = distinct.p;
    build_in_csr(*g, ro.p, dcol.p, dw.p, nullptr, s, view);
    finish_build(g.get(), ea, eb, s);
    cudaEventDestroy(ea);
    cudaEventDestroy(eb);
    ro.release();
    dcol.release();
    dw.release();
    DevBuf<uint64_t> d64(n, s);
    k_u32_to_u64_out<<<grid_for(n, kBlock), kBlock, 0, s>>>(distinct.p, d64.p, n);
    QVB_LAUNCH_CHECK();
    copy_to_host(row_sums, rs.p, n * 8, s);
    copy_to_host(distinct_out, d64.p, n * 8, s);
    QVB_CUDA(cudaStreamSynchronize(s));
    *has_parallel_edges = g->eu != e ? 1 : 0;
    if (keep) *keep = g.release();
  });
}
