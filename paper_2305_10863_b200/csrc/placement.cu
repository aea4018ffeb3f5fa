// placement.cu — the placement manager and the feature lookup table.
//
//   K2  rank: stable radix sort of order-preserving 64-bit keys of the values
//       (descending) with the feature id as payload: ties keep ascending id,
//       which is exactly std::stable_sort's order in fap_ranking
//       (placement.cpp:79-87).
//   plan: the reference's sequential planner (placement.cpp:94-226) on the
//       host over the device ranking — the greedy LPT balance is sequential
//       by definition — plus the gpu_replicated_capacity extension (hot rows
//       on every GPU, next range LPT-partitioned; 0 == reference).
//   K3  lookup table (placement.cpp:306-342): the reference walks features
//       in id order bumping cursor[loc] for every copy, so a copy's offset is
//       the number of lower-id features holding a copy at that location. On
//       the device that is a per-location exclusive prefix count: per-tile
//       counts (block-wide __syncthreads_count), one scan over all
//       (location, tile) pairs, then an in-tile ballot prefix. The chosen
//       copy is the first of the feature's locations in the reader's
//       (cost, id) order — the reference's min-cost, lowest-id rule.
#include <algorithm>
#include <memory>
#include <vector>
#include <numeric>
#include <string>
#include <thread>

#include "placement.cuh"

namespace qvb {
namespace {

constexpr unsigned kTile = 256;
constexpr unsigned kFull = 0xffffffffu;

// Order-preserving map of a double to u64, inverted for descending order.
// -0.0 is folded onto +0.0 (they compare equal in the reference).
__global__ void k_rank_keys(const double* __restrict__ v, uint64_t n, uint64_t* __restrict__ keys,
                            uint64_t* __restrict__ ids, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double x = v[i];
    if (x != x) atomicMin(bad, (unsigned long long)i);
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    if (b == 0x8000000000000000ull) b = 0;
    b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending total order
    keys[i] = ~b;                                       // descending
    ids[i] = i;
  }
}

// vr[r] = v[ranks[r]], pos[ranks[r]] = r
__global__ void k_rank_views(const double* __restrict__ v, const uint64_t* __restrict__ ranks, uint64_t n,
                             double* __restrict__ vr, uint64_t* __restrict__ pos) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = ranks[r];
    vr[r] = v[f];
    pos[f] = r;
  }
}

__global__ void k_masks(const uint64_t* __restrict__ lo, const int64_t* __restrict__ ids,
                        uint64_t n, int nloc, uint64_t* __restrict__ masks,
                        unsigned long long* bad) {
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < n;
       f += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t m = 0;
    for (uint64_t k = lo[f]; k < lo[f + 1]; ++k) {
      const int64_t id = ids[k];
      if (id < 0 || id >= nloc) {
        atomicMin(bad, (unsigned long long)(f << 1));
        continue;
      }
      const uint64_t bit = 1ull << id;
      if (m & bit) atomicMin(bad, (unsigned long long)((f << 1) | 1));
      m |= bit;
    }
    masks[f] = m;
  }
}

__global__ void __launch_bounds__(kTile)
    k_tile_counts(const uint64_t* __restrict__ masks, uint64_t n, int nloc, uint64_t ntiles,
                  uint32_t* __restrict__ counts) {
  const uint64_t t = blockIdx.x;
  const uint64_t f = t * kTile + threadIdx.x;
  const uint64_t m = f < n ? masks[f] : 0;
  for (int l = 0; l < nloc; ++l) {
    const int c = __syncthreads_count(static_cast<int>((m >> l) & 1));
    if (threadIdx.x == 0) counts[(uint64_t)l * ntiles + t] = static_cast<uint32_t>(c);
  }
}

__global__ void k_tile_off(const uint64_t* __restrict__ scanned, uint64_t ntiles, int nloc,
                           uint64_t* __restrict__ tile_off) {
  const uint64_t total = (uint64_t)nloc * ntiles;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t l = i / ntiles;
    tile_off[i] = scanned[i] - scanned[l * ntiles];
  }
}

__global__ void k_location_totals(const uint64_t* __restrict__ scanned,
                                  const uint32_t* __restrict__ counts, uint64_t ntiles, int nloc,
                                  uint64_t* __restrict__ starts) {
  const int l = threadIdx.x;
  if (l <= nloc) {
    const uint64_t i = (uint64_t)l * ntiles;
    starts[l] = l < nloc ? scanned[i] : scanned[i - 1] + counts[i - 1];
  }
}

struct Order {
  int8_t loc[kMaxLocations];
};

// Block-wide exclusive count of features (in id order) that hold location
// `want` before this thread's feature. All threads of the block call it.
__device__ __forceinline__ uint32_t block_prefix(uint64_t m, int want, int nloc,
                                                 uint32_t (*wcnt)[kMaxLocations]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t mine = 0;
  for (int l = 0; l < nloc; ++l) {
    const uint32_t b = __ballot_sync(kFull, (m >> l) & 1);
    if (l == want) mine = __popc(b & lt);
    if (lane == 0) wcnt[warp][l] = __popc(b);
  }
  __syncthreads();
  if (want >= 0)
    for (int w = 0; w < warp; ++w) mine += wcnt[w][want];
  return mine;
}

__global__ void __launch_bounds__(kTile)
    k_lut_choose(const uint64_t* __restrict__ masks, const uint64_t* __restrict__ tile_off,
                 uint64_t n, int nloc, uint64_t ntiles, Order order, int64_t* __restrict__ out_loc,
                 uint64_t* __restrict__ out_off, uint64_t* __restrict__ packed,
                 unsigned long long* used_mask) {
  __shared__ uint32_t wcnt[kTile / 32][kMaxLocations];
  const uint64_t t = blockIdx.x;
  const uint64_t f = t * kTile + threadIdx.x;
  const uint64_t m = f < n ? masks[f] : 0;
  int best = -1;
  for (int i = 0; i < nloc; ++i) {
    const int l = order.loc[i];
    if ((m >> l) & 1) {
      best = l;
      break;
    }
  }
  const uint32_t pre = block_prefix(m, best, nloc, wcnt);
  if (f < n) {
    const uint64_t off = best >= 0 ? tile_off[(uint64_t)best * ntiles + t] + pre : 0;
    if (out_loc) out_loc[f] = best;
    if (out_off) out_off[f] = off;
    if (packed) packed[f] = best >= 0 ? ((uint64_t)best << kOffsetBits) | off : ~0ull;
  }
  const uint64_t bit = best >= 0 ? (1ull << best) : 0;
  const uint32_t lo = __reduce_or_sync(kFull, static_cast<uint32_t>(bit));
  const uint32_t hi = __reduce_or_sync(kFull, static_cast<uint32_t>(bit >> 32));
  if ((threadIdx.x & 31) == 0 && (lo | hi))
    atomicOr(used_mask, ((unsigned long long)hi << 32) | lo);
  if (f < n && best < 0) atomicMin(used_mask + 1, (unsigned long long)f);  // no copy at all
}

__global__ void __launch_bounds__(kTile)
    k_rows_of_location(const uint64_t* __restrict__ masks, const uint64_t* __restrict__ tile_off,
                       uint64_t n, int nloc, uint64_t ntiles, int loc,
                       uint64_t* __restrict__ feat_of_row) {
  __shared__ uint32_t wcnt[kTile / 32][kMaxLocations];
  const uint64_t t = blockIdx.x;
  const uint64_t f = t * kTile + threadIdx.x;
  const uint64_t m = f < n ? masks[f] : 0;
  const uint32_t pre = block_prefix(m, loc, nloc, wcnt);
  if (f < n && ((m >> loc) & 1)) feat_of_row[tile_off[(uint64_t)loc * ntiles + t] + pre] = f;
}

// ---- K3 for any number of locations (multi-server topologies: S x (G+2)
// location ids can exceed one 64-bit mask). Copies are listed feature by
// feature, so a stable sort of copy indices by location id leaves each
// location's copies in ascending feature order: a copy's offset is its rank
// inside its location's run — the reference's cursor[loc]++ (placement.cpp:
// 318-330) computed for all copies at once.
__global__ void k_copy_keys(const uint64_t* __restrict__ lo, const int64_t* __restrict__ ids,
                            uint64_t n, int nloc, uint64_t* __restrict__ keys,
                            uint64_t* __restrict__ idx, unsigned long long* bad) {
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < n;
       f += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = lo[f], b = lo[f + 1];
    for (uint64_t k = a; k < b; ++k) {
      const int64_t id = ids[k];
      if (id < 0 || id >= nloc) {
        atomicMin(bad, (unsigned long long)(f << 1));
        keys[k] = 0;
      } else {
        keys[k] = static_cast<uint64_t>(id);  // a repeated location consumes a slot per copy
      }
      idx[k] = k;
    }
  }
}

// run starts: first sorted position of every location id present
__global__ void k_run_starts(const uint64_t* __restrict__ skeys, uint64_t copies,
                             uint64_t* __restrict__ start) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < copies;
       p += (uint64_t)gridDim.x * blockDim.x)
    if (p == 0 || skeys[p] != skeys[p - 1]) start[skeys[p]] = p;
}

__global__ void k_copy_offsets(const uint64_t* __restrict__ skeys, const uint64_t* __restrict__ sidx,
                               uint64_t copies, const uint64_t* __restrict__ start,
                               uint64_t* __restrict__ copy_off) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < copies;
       p += (uint64_t)gridDim.x * blockDim.x)
    copy_off[sidx[p]] = p - start[skeys[p]];
}

// per feature: the copy whose location ranks first in the reader's
// (cost, id) order (placement.cpp:323-337)
__global__ void k_choose_general(const uint64_t* __restrict__ lo, const int64_t* __restrict__ ids,
                                 const uint64_t* __restrict__ copy_off,
                                 const uint32_t* __restrict__ rank_of_loc, uint64_t n,
                                 int64_t* __restrict__ out_loc, uint64_t* __restrict__ out_off) {
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < n;
       f += (uint64_t)gridDim.x * blockDim.x) {
    int64_t best = -1;
    uint32_t best_rank = 0xFFFFFFFFu;
    uint64_t off = 0;
    for (uint64_t k = lo[f]; k < lo[f + 1]; ++k) {
      const uint32_t r = rank_of_loc[ids[k]];
      if (r < best_rank) {
        best_rank = r;
        best = ids[k];
        off = copy_off[k];
      }
    }
    out_loc[f] = best;  // -1, offset 0 for a feature without copies, as the reference
    out_off[f] = off;
  }
}

void lut_build_general(const uint64_t* d_lo, const int64_t* d_ids, uint64_t n, uint64_t copies,
                       int nloc, const std::vector<int>& order, int64_t* d_loc, uint64_t* d_off,
                       cudaStream_t s) {
  DevBuf<unsigned long long> flags(1, s);
  QVB_CUDA(cudaMemsetAsync(flags.p, 0xFF, sizeof(unsigned long long), s));
  const uint64_t c = copies ? copies : 1;
  DevBuf<uint64_t> keys(c, s), skeys(c, s), idx(c, s), sidx(c, s), off(c, s), start(nloc, s);
  k_copy_keys<<<grid_for(n, 256), 256, 0, s>>>(d_lo, d_ids, n, nloc, keys.p, idx.p, flags.p);
  QVB_LAUNCH_CHECK();
  const unsigned long long b = read_scalar(flags.p, s);
  if (b != ~0ull) {
    const uint64_t f = b >> 1;
    if (b & 1) fail(QVB_ERR_VALIDATION, "feature " + std::to_string(f) + " lists a location twice");
    fail(QVB_ERR_VALIDATION, "unknown location id for feature " + std::to_string(f));
  }
  if (copies) {
    sort_pairs_u64_u64(keys.p, skeys.p, idx.p, sidx.p, copies, 0, bits_for((uint64_t)nloc - 1), s);
    k_run_starts<<<grid_for(copies, 256), 256, 0, s>>>(skeys.p, copies, start.p);
    QVB_LAUNCH_CHECK();
    k_copy_offsets<<<grid_for(copies, 256), 256, 0, s>>>(skeys.p, sidx.p, copies, start.p, off.p);
    QVB_LAUNCH_CHECK();
  }
  std::vector<uint32_t> rank(nloc);
  for (int i = 0; i < nloc; ++i) rank[order[i]] = static_cast<uint32_t>(i);
  DevBuf<uint32_t> drank(nloc, s);
  QVB_CUDA(cudaMemcpyAsync(drank.p, rank.data(), nloc * 4, cudaMemcpyHostToDevice, s));
  k_choose_general<<<grid_for(n, 256), 256, 0, s>>>(d_lo, d_ids, off.p, drank.p, n, d_loc, d_off);
  QVB_LAUNCH_CHECK();
}

// LPT over one NUMA group's slots (placement.cpp:100-115).
// vr: the run's values in rank order (read sequentially, not through the ids).
void lpt(const double* vr, uint64_t len, uint32_t gpn, uint64_t cap, std::vector<uint8_t>& slot) {
  std::vector<double> load(gpn, 0.0);
  std::vector<uint64_t> used(gpn, 0);
  slot.resize(len);
  for (uint64_t i = 0; i < len; ++i) {
    uint32_t best = gpn;
    for (uint32_t s = 0; s < gpn; ++s) {
      if (used[s] >= cap) continue;
      if (best == gpn || load[s] < load[best]) best = s;
    }
    if (best == gpn) fail(QVB_ERR_GENERIC, "gpu range exceeds numa group capacity");
    load[best] += vr[i];
    ++used[best];
    slot[i] = static_cast<uint8_t>(best);
  }
}

// One server's share of a run (place_server_run, placement.cpp:158-169).
struct ServerRun {
  uint64_t lo = 0, hi = 0;  // rank positions of the run
  uint64_t rep = 0, g = 0, h = 0;
  std::vector<uint8_t> slot;  // LPT slot for positions [rep, g) of the run
};

}  // namespace

void rank_desc_device(const double* d_values, uint64_t n, uint64_t* d_ranks, cudaStream_t s) {
  DevBuf<uint64_t> keys(n, s), ids(n, s), skeys(n, s);
  DevBuf<unsigned long long> bad(1, s);
  QVB_CUDA(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
  k_rank_keys<<<grid_for(n, 256), 256, 0, s>>>(d_values, n, keys.p, ids.p, bad.p);
  QVB_LAUNCH_CHECK();
  sort_pairs_u64_u64(keys.p, skeys.p, ids.p, d_ranks, n, 0, 64, s);
  const unsigned long long b = read_scalar(bad.p, s);
  if (b != ~0ull) fail(QVB_ERR_VALIDATION, "NaN value for feature " + std::to_string(b));
}

// vr[r] = value of the feature at rank position r; pos[f] = rank position of
// feature f (both computed on the device, see qvb_plan_placement).
HostPlan plan_from_ranks(const double* vr, const uint64_t* pos, uint64_t n,
                         const qvb_topology& t) {
  const uint32_t G = t.gpus_per_server, S = t.servers;
  const uint32_t gpn = gpus_per_numa(t);
  const bool nvl = t.nvlink_within_numa != 0;
  const uint64_t rep_cap = nvl ? t.gpu_replicated_capacity : 0;
  // placement.cpp:147-152 (+ extension: rep_cap rows of every GPU replicate)
  const uint64_t gpu_range_size =
      G == 0 ? 0 : (nvl ? rep_cap + gpn * (t.gpu_feature_capacity - rep_cap) : t.gpu_feature_capacity);

  auto make_run = [&](uint64_t lo, uint64_t hi) {
    ServerRun r;
    r.lo = lo;
    r.hi = hi;
    const uint64_t len = hi - lo;
    r.g = std::min(len, gpu_range_size);
    r.rep = std::min(r.g, rep_cap);
    if (G > 0 && nvl) lpt(vr + lo + r.rep, r.g - r.rep, gpn, t.gpu_feature_capacity - rep_cap, r.slot);
    r.h = std::min(len - r.g, t.host_feature_capacity);
    return r;
  };

  std::vector<ServerRun> runs;  // per server (no-IB: one shared run)
  uint64_t partitioned = n, remainder = 0, rem_base = 0, rem_extra = 0;
  if (!t.infiniband) {
    const uint64_t per_server = gpu_range_size + t.host_feature_capacity + t.disk_feature_capacity;
    if (n > per_server)
      fail(QVB_ERR_PLACEMENT, "placement infeasible without infiniband: " + std::to_string(n) +
                                  " features vs per-server capacity " + std::to_string(per_server) +
                                  " (short by " + std::to_string(n - per_server) + ")");
    runs.push_back(make_run(0, n));
  } else {
    const uint64_t ns = gpu_range_size + t.host_feature_capacity;
    partitioned = std::min<uint64_t>(n, (uint64_t)S * ns);
    for (uint32_t s = 0; s < S; ++s) {
      uint64_t lo = std::min<uint64_t>(partitioned, (uint64_t)s * ns);
      uint64_t hi = std::min<uint64_t>(partitioned, (uint64_t)(s + 1) * ns);
      runs.push_back(make_run(lo, hi));
    }
    remainder = n - partitioned;
    if (remainder > 0) {
      const uint64_t disk_total = (uint64_t)S * t.disk_feature_capacity;
      if (remainder > disk_total)
        fail(QVB_ERR_PLACEMENT, "placement infeasible: remainder " + std::to_string(remainder) +
                                    " features exceed total disk capacity " +
                                    std::to_string(disk_total) + " (short by " +
                                    std::to_string(remainder - disk_total) + ")");
      rem_base = remainder / S;
      rem_extra = remainder % S;
    }
  }

  const int64_t stride = (int64_t)G + 2;

  // Copies of the feature at rank position r, canonical order (ascending id).
  auto emit = [&](uint64_t r, int64_t* out) -> uint32_t {
    uint32_t c = 0;
    auto server_copies = [&](uint32_t s, const ServerRun& run, uint64_t i) {
      const int64_t base = (int64_t)s * stride;
      if (i < run.g) {
        if (i < run.rep || !nvl) {
          for (uint32_t d = 0; d < G; ++d) out[c++] = base + d;
        } else {
          const uint32_t slot = run.slot[i - run.rep];
          for (uint32_t grp = 0; grp < t.numa_per_server; ++grp) out[c++] = base + grp * gpn + slot;
        }
      } else if (i < run.g + run.h) {
        out[c++] = base + G;
      } else {
        out[c++] = base + G + 1;
      }
    };
    if (!t.infiniband) {
      for (uint32_t s = 0; s < S; ++s) server_copies(s, runs[0], r);
    } else if (r < partitioned) {
      // find the server whose run holds r (runs are contiguous, ascending)
      for (uint32_t s = 0; s < S; ++s)
        if (r >= runs[s].lo && r < runs[s].hi) {
          server_copies(s, runs[s], r - runs[s].lo);
          break;
        }
    } else {
      uint64_t at = partitioned;
      for (uint32_t s = 0; s < S; ++s) {
        const uint64_t len = rem_base + (s < rem_extra ? 1 : 0);
        if (r < at + len) {
          out[c++] = (int64_t)s * stride + G + 1;
          break;
        }
        at += len;
      }
    }
    return c;
  };

  // Every feature's copies depend only on its rank position, so the two
  // emit passes (copy counts, then the copies) run over feature ranges on
  // host threads; per-thread location counts are summed afterwards.
  HostPlan plan;
  plan.offsets.assign(n + 1, 0);
  const int64_t nloc_all = (int64_t)S * stride;
  const unsigned T = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())),
                                                n / 65536)));
  const uint64_t per = (n + T - 1) / T;
  std::vector<uint64_t> part(T + 1, 0);
  std::vector<std::vector<uint64_t>> tcounts(T, std::vector<uint64_t>(nloc_all, 0));
  std::vector<uint64_t> missing(T, ~0ull);
  auto parallel = [&](auto&& body) {
    std::vector<std::thread> pool;
    for (unsigned k = 1; k < T; ++k) pool.emplace_back(body, k);
    body(0u);
    for (auto& th : pool) th.join();
  };
  parallel([&](unsigned k) {  // pass 1: copies per feature, range totals
    std::vector<int64_t> buf((size_t)S * (G + 1) + 2);
    const uint64_t a = std::min(n, k * per), b = std::min(n, a + per);
    uint64_t sum = 0;
    for (uint64_t f = a; f < b; ++f) {
      const uint32_t c = emit(pos[f], buf.data());
      plan.offsets[f + 1] = c;
      sum += c;
    }
    part[k + 1] = sum;
  });
  for (unsigned k = 0; k < T; ++k) part[k + 1] += part[k];
  parallel([&](unsigned k) {  // prefix within the range
    const uint64_t a = std::min(n, k * per), b = std::min(n, a + per);
    uint64_t at = part[k];
    for (uint64_t f = a; f < b; ++f) {
      at += plan.offsets[f + 1];
      plan.offsets[f + 1] = at;
    }
  });
  plan.ids.resize(plan.offsets[n]);
  parallel([&](unsigned k) {  // pass 2: the copies, and the location counts
    const uint64_t a = std::min(n, k * per), b = std::min(n, a + per);
    std::vector<uint64_t>& cnt = tcounts[k];
    for (uint64_t f = a; f < b; ++f) {
      const uint32_t c = emit(pos[f], plan.ids.data() + plan.offsets[f]);
      if (c == 0 && missing[k] == ~0ull) missing[k] = f;
      for (uint32_t q = 0; q < c; ++q) ++cnt[plan.ids[plan.offsets[f] + q]];
    }
  });
  for (unsigned k = 0; k < T; ++k)
    if (missing[k] != ~0ull) fail(QVB_ERR_GENERIC, "feature " + std::to_string(missing[k]) + " has no location");
  std::vector<uint64_t> counts(nloc_all, 0);
  for (unsigned k = 0; k < T; ++k)
    for (int64_t id = 0; id < nloc_all; ++id) counts[id] += tcounts[k][id];
  // PlacementPlan::validate (placement.cpp:53-74)
  static const char* tier_names[3] = {"gpu", "host", "disk"};
  for (int64_t id = 0; id < nloc_all; ++id) {
    uint32_t srv, tier, dev;
    decode_location(t, id, &srv, &tier, &dev);
    const uint64_t cap = tier == QVB_TIER_GPU    ? t.gpu_feature_capacity
                         : tier == QVB_TIER_HOST ? t.host_feature_capacity
                                                 : t.disk_feature_capacity;
    if (counts[id] > cap)
      fail(QVB_ERR_GENERIC, std::string("placement overfills ") + tier_names[tier] + " on server " +
                                std::to_string(srv) + ": " + std::to_string(counts[id]) + " > " +
                                std::to_string(cap));
  }
  return plan;
}

void lut_prepare(DeviceLut& L, const uint64_t* d_lo, const int64_t* d_ids, uint64_t n, int nloc,
                 cudaStream_t s) {
  if (nloc > kMaxLocations)
    fail(QVB_ERR_UNSUPPORTED, "the device lookup table supports at most 64 locations");
  L.n = n;
  L.nloc = nloc;
  L.ntiles = (n + kTile - 1) / kTile;
  L.masks.alloc(n, s);
  DevBuf<unsigned long long> bad(1, s);
  QVB_CUDA(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), s));
  k_masks<<<grid_for(n, 256), 256, 0, s>>>(d_lo, d_ids, n, nloc, L.masks.p, bad.p);
  QVB_LAUNCH_CHECK();
  const unsigned long long b = read_scalar(bad.p, s);
  if (b != ~0ull) {
    const uint64_t f = b >> 1;
    if (b & 1) fail(QVB_ERR_VALIDATION, "feature " + std::to_string(f) + " lists a location twice");
    fail(QVB_ERR_VALIDATION, "unknown location id for feature " + std::to_string(f));
  }
  const uint64_t cells = (uint64_t)nloc * L.ntiles;
  DevBuf<uint32_t> counts(cells, s);
  DevBuf<uint64_t> scanned(cells, s), starts(nloc + 1, s);
  k_tile_counts<<<static_cast<unsigned>(L.ntiles), kTile, 0, s>>>(L.masks.p, n, nloc, L.ntiles, counts.p);
  QVB_LAUNCH_CHECK();
  exclusive_sum_u32_u64(counts.p, scanned.p, cells, s);
  L.tile_off.alloc(cells, s);
  k_tile_off<<<grid_for(cells, 256), 256, 0, s>>>(scanned.p, L.ntiles, nloc, L.tile_off.p);
  QVB_LAUNCH_CHECK();
  k_location_totals<<<1, kMaxLocations + 1, 0, s>>>(scanned.p, counts.p, L.ntiles, nloc, starts.p);
  QVB_LAUNCH_CHECK();
  std::vector<uint64_t> st(nloc + 1);
  QVB_CUDA(cudaMemcpyAsync(st.data(), starts.p, (nloc + 1) * 8, cudaMemcpyDeviceToHost, s));
  QVB_CUDA(cudaStreamSynchronize(s));
  L.location_rows.resize(nloc);
  for (int l = 0; l < nloc; ++l) L.location_rows[l] = st[l + 1] - st[l];
}

uint64_t lut_choose(const DeviceLut& L, const std::vector<int>& order, int64_t* d_loc,
                    uint64_t* d_off, uint64_t* d_packed, cudaStream_t s, uint64_t* first_missing) {
  Order o;
  for (int i = 0; i < kMaxLocations; ++i) o.loc[i] = i < (int)order.size() ? (int8_t)order[i] : 0;
  DevBuf<unsigned long long> used(2, s);
  QVB_CUDA(cudaMemsetAsync(used.p, 0, sizeof(unsigned long long), s));
  QVB_CUDA(cudaMemsetAsync(used.p + 1, 0xFF, sizeof(unsigned long long), s));
  if (L.n)
    k_lut_choose<<<static_cast<unsigned>(L.ntiles), kTile, 0, s>>>(
        L.masks.p, L.tile_off.p, L.n, L.nloc, L.ntiles, o, d_loc, d_off, d_packed, used.p);
  QVB_LAUNCH_CHECK();
  unsigned long long h[2];
  QVB_CUDA(cudaMemcpyAsync(h, used.p, sizeof h, cudaMemcpyDeviceToHost, s));
  QVB_CUDA(cudaStreamSynchronize(s));
  if (first_missing) *first_missing = h[1];
  return h[0];
}

void lut_rows_of_location(const DeviceLut& L, int loc, uint64_t* d_feat_of_row, cudaStream_t s) {
  if (L.n)
    k_rows_of_location<<<static_cast<unsigned>(L.ntiles), kTile, 0, s>>>(
        L.masks.p, L.tile_off.p, L.n, L.nloc, L.ntiles, loc, d_feat_of_row);
  QVB_LAUNCH_CHECK();
}

std::vector<int> replica_order(const qvb_topology& t, uint32_t home, uint32_t reader) {
  const int nloc = static_cast<int>((uint64_t)t.servers * (t.gpus_per_server + 2));
  std::vector<int> order(nloc);
  std::iota(order.begin(), order.end(), 0);
  std::vector<double> cost(nloc);
  for (int l = 0; l < nloc; ++l) cost[l] = nominal_read_cost(t, home, reader, l);
  // strict (cost, id) order == placement.cpp:331-336 walking copies in id order
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (cost[a] < cost[b]) return true;
    if (cost[b] < cost[a]) return false;
    return a < b;
  });
  return order;
}

}  // namespace qvb

using namespace qvb;

extern "C" int qvb_rank_desc(int device, const double* values, uint64_t n, uint64_t* ranks,
                             int on_device, void* stream) {
  return guarded([&] {
    if (n == 0) return;
    if (!values || !ranks) fail(QVB_ERR_VALIDATION, "null argument");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (on_device) {
      rank_desc_device(values, n, ranks, s);
      return;
    }
    DevBuf<double> dv(n, s);
    DevBuf<uint64_t> dr(n, s);
    QVB_CUDA(cudaMemcpyAsync(dv.p, values, n * 8, cudaMemcpyHostToDevice, s));
    rank_desc_device(dv.p, n, dr.p, s);
    QVB_CUDA(cudaMemcpyAsync(ranks, dr.p, n * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}

struct qvb_plan {
  HostPlan p;
};

namespace {
HostPlan plan_on_device(int device, const double* values, uint64_t n, const qvb_topology* topo) {
  if (!topo) fail(QVB_ERR_VALIDATION, "null topology");
  topology_validate(*topo);  // placement.cpp:139
  if (n == 0) fail(QVB_ERR_VALIDATION, "placement needs at least one feature");
  if (!values) fail(QVB_ERR_VALIDATION, "null argument");
  if (topo->nvlink_within_numa && gpus_per_numa(*topo) > 255)
    fail(QVB_ERR_UNSUPPORTED, "more than 255 GPUs per NUMA group");
  // the device ranks the features and hands the sequential planner its
  // inputs in the order it walks them: values in rank order and each
  // feature's rank position (no random host reads over n values)
  std::vector<double> vr(n);
  std::vector<uint64_t> pos(n);
  {
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<double> dv(n, s), dvr(n, s);
    DevBuf<uint64_t> dr(n, s), dpos(n, s);
    QVB_CUDA(cudaMemcpyAsync(dv.p, values, n * 8, cudaMemcpyHostToDevice, s));
    rank_desc_device(dv.p, n, dr.p, s);
    k_rank_views<<<grid_for(n, 256), 256, 0, s>>>(dv.p, dr.p, n, dvr.p, dpos.p);
    QVB_LAUNCH_CHECK();
    copy_to_host(vr.data(), dvr.p, n * 8, s);
    copy_to_host(pos.data(), dpos.p, n * 8, s);
  }
  return plan_from_ranks(vr.data(), pos.data(), n, *topo);
}
}  // namespace

extern "C" int qvb_plan_placement(int device, const double* values, uint64_t n,
                                  const qvb_topology* topo, uint64_t* loc_offsets,
                                  int64_t* loc_ids, uint64_t loc_capacity, uint64_t* copies_out) {
  return guarded([&] {
    if (!loc_offsets || !copies_out) fail(QVB_ERR_VALIDATION, "null argument");
    HostPlan p = plan_on_device(device, values, n, topo);
    *copies_out = p.ids.size();
    if (p.ids.size() > loc_capacity)
      fail(QVB_ERR_VALIDATION, "loc_capacity " + std::to_string(loc_capacity) + " too small, need " +
                                   std::to_string(p.ids.size()));
    std::copy(p.offsets.begin(), p.offsets.end(), loc_offsets);
    if (!p.ids.empty()) std::copy(p.ids.begin(), p.ids.end(), loc_ids);
  });
}

extern "C" int qvb_plan_placement_create(int device, const double* values, uint64_t n,
                                         const qvb_topology* topo, qvb_plan** out) {
  return guarded([&] {
    if (!out) fail(QVB_ERR_VALIDATION, "null argument");
    *out = nullptr;
    auto h = std::make_unique<qvb_plan>();
    h->p = plan_on_device(device, values, n, topo);
    *out = h.release();
  });
}

extern "C" int qvb_plan_size(const qvb_plan* plan, uint64_t* n, uint64_t* copies) {
  return guarded([&] {
    if (!plan || !n || !copies) fail(QVB_ERR_VALIDATION, "null argument");
    *n = plan->p.offsets.size() - 1;
    *copies = plan->p.ids.size();
  });
}

extern "C" int qvb_plan_copy(const qvb_plan* plan, uint64_t* loc_offsets, int64_t* loc_ids) {
  return guarded([&] {
    if (!plan || !loc_offsets || (!loc_ids && !plan->p.ids.empty()))
      fail(QVB_ERR_VALIDATION, "null argument");
    std::copy(plan->p.offsets.begin(), plan->p.offsets.end(), loc_offsets);
    std::copy(plan->p.ids.begin(), plan->p.ids.end(), loc_ids);
  });
}

extern "C" int qvb_plan_destroy(qvb_plan* plan) {
  return guarded([&] { delete plan; });
}

extern "C" int qvb_build_lookup_table(int device, const uint64_t* loc_offsets,
                                      const int64_t* loc_ids, uint64_t n,
                                      const qvb_topology* topo, uint32_t home_server,
                                      uint32_t reader_device, int64_t* location_ids,
                                      uint64_t* offsets) {
  return guarded([&] {
    if (!topo) fail(QVB_ERR_VALIDATION, "null topology");
    if (home_server >= topo->servers) fail(QVB_ERR_VALIDATION, "home server out of range");
    if (n == 0) return;
    if (!loc_offsets || !location_ids || !offsets) fail(QVB_ERR_VALIDATION, "null argument");
    const uint64_t copies = loc_offsets[n];
    const int nloc = static_cast<int>((uint64_t)topo->servers * (topo->gpus_per_server + 2));
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> dlo(n + 1, s);
    DevBuf<int64_t> dids(copies ? copies : 1, s);
    QVB_CUDA(cudaMemcpyAsync(dlo.p, loc_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
    if (copies) QVB_CUDA(cudaMemcpyAsync(dids.p, loc_ids, copies * 8, cudaMemcpyHostToDevice, s));
    DevBuf<int64_t> dloc(n, s);
    DevBuf<uint64_t> doff(n, s);
    const char* gen = std::getenv("QVB_LUT_GENERAL");  // tests: force the any-location path
    if (nloc <= kMaxLocations && !(gen && *gen == '1')) {  // one location mask per feature
      DeviceLut L;
      lut_prepare(L, dlo.p, dids.p, n, nloc, s);
      lut_choose(L, replica_order(*topo, home_server, reader_device), dloc.p, doff.p, nullptr, s);
    } else {
      lut_build_general(dlo.p, dids.p, n, copies, nloc, replica_order(*topo, home_server, reader_device),
                        dloc.p, doff.p, s);
    }
    QVB_CUDA(cudaMemcpyAsync(location_ids, dloc.p, n * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaMemcpyAsync(offsets, doff.p, n * 8, cudaMemcpyDeviceToHost, s));
    QVB_CUDA(cudaStreamSynchronize(s));
  });
}

// ---- the reference's collect cost model (placement.cpp:269-302,382-404) ------
namespace {
bool translated(int c) {  // address-translated links pay the TLB penalty
  return c == QVB_LINK_PCIE || c == QVB_LINK_UPI || c == QVB_LINK_INFINIBAND ||
         c == QVB_LINK_ETHERNET;
}
}  // namespace

extern "C" int qvb_classify_link(const qvb_topology* t, uint32_t reader_server, uint32_t reader_tier,
                                 uint32_t reader_device, int64_t location_id, int* first,
                                 int* second) {
  return guarded([&] {
    if (!t || !first || !second) fail(QVB_ERR_VALIDATION, "null argument");
    *first = classify_link_from(*t, reader_server, reader_tier, reader_device,
                                location_id, second);
  });
}

extern "C" int qvb_fetch_cost(const qvb_topology* t, uint32_t reader_server, uint32_t reader_tier,
                              uint32_t reader_device, uint64_t groups, const int64_t* group_loc,
                              const uint64_t* group_count, const uint64_t* group_transitions,
                              uint64_t feature_bytes, double* per_location_s, double* total_s) {
  return guarded([&] {
    if (!t || !total_s || (groups && (!group_loc || !group_count || !group_transitions ||
                                      !per_location_s)))
      fail(QVB_ERR_VALIDATION, "null argument");
    const int64_t nloc = static_cast<int64_t>(t->servers) * (static_cast<int64_t>(t->gpus_per_server) + 2);
    double worst = 0.0;
    for (uint64_t g = 0; g < groups; ++g) {
      const int64_t id = group_loc[g];
      if (id < 0 || id >= nloc) fail(QVB_ERR_VALIDATION, "unknown location id " + std::to_string(id));
      int second = -1;
      const int first = classify_link_from(*t, reader_server, reader_tier, reader_device, id, &second);
      const double* lat = t->link_latency_s;
      const double* bw = t->link_bandwidth_Bps;
      const double setup = second < 0 ? lat[first] : lat[first] + lat[second];
      const double rate = second < 0 ? bw[first] : std::min(bw[first], bw[second]);
      const double bytes = static_cast<double>(feature_bytes) * static_cast<double>(group_count[g]);
      double s = setup + bytes / rate;
      if (translated(first) || (second >= 0 && translated(second)))
        s += t->tlb_miss_penalty_s * static_cast<double>(group_transitions[g]);
      per_location_s[g] = s;
      worst = std::max(worst, s);
    }
    *total_s = worst;
  });
}
