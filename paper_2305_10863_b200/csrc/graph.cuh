// graph.cuh — the device-resident in-CSR that replaces the transpose the
// reference rebuilds inside every compute_access_prob_ie call
// (metrics.cpp:145 -> in_adjacency, graph.cpp:260-281) plus the row sums of
// transition_view (graph.cpp:292-318).
//
// HBM layout (N nodes, E_u coalesced in-edges) — "sliced" in-CSR:
//   windows of 256 consecutive destination ids are sorted by in-degree
//   (descending, ties by id) and cut into slices of 32 nodes; slice s holds
//   its nodes' in-edges lane-major: edge k of the node in lane l sits at
//   sptr[s] + 32*k + l, padded to the slice's longest row with a sentinel
//   source (index N, whose operand is 0, so its factor is exactly 1.0 and
//   multiplying by it leaves the product bit-identical). A warp therefore
//   reads one coalesced 128-byte line of sources per step and every lane
//   owns its node's whole product chain in registers, in the reference's
//   ascending-source order.
//   perm   u32[S*32]   node of each slot (kNoNode: padding / long row)
//   sptr   u64[S+1]    slice starts (elements)
//   scol   u32[...]    sources, lane-major; compact layout: bit 31 set =>
//                      index into the exception table instead
//   sR     f64[...]    weighted layout only: R = w_sum / row_sum(s)
//   long rows (in-degree > long_threshold) keep a plain CSR (lnode, lptr,
//   lcol, lR) and are multiplied by one warp each (the chain is sequential
//   by definition; the gathers are warp-parallel).
//   exc_*              compact layout: (source, R) of the few edges whose R
//                      differs bitwise from 1/row_sum(s)
//   inv    f64[N]      1/row_sum(s) (0 for sinks)
//   p[2], y[2] f64[N+1] ping-pong P_{j-1}/P_j and y = P * inv; entry N = 0
//
// Source segments. At papers scale the gathered vector (8 B x N) is far
// larger than L2 and every random 8-byte gather that misses pulls a whole
// line from HBM. The sweep is therefore split into passes over source
// ranges small enough to stay L2-resident; a node's running product is
// carried between passes (state), and because each in-row is sorted by
// source, pass order == the reference's factor order: still bit-exact.
// Each pass has its own slices built only over the nodes it touches.
//
// Node-major passes (nm, default when there is more than one segment). The
// per-pass slices above re-sort every pass's nodes by degree, so the running
// product is read and written through a scattered perm word per (node, pass)
// pair and the warp's chain starts with perm -> state and sptr -> columns.
// The nm layout keeps node v in lane v%32 of slice v/32 in EVERY pass:
//   nm_lenf  u8[nseg][S*32]  len | first<<6 | last<<7  (len <= 63)
//   nm_sbase u64[nseg*S+1]   start of slice (k, s)'s columns in nm_col
//   nm_col   u32 / nm_R f64  each node's pass-k sources (ascending), nodes
//                            in id order, no padding
// so the state, P and y accesses are coalesced and need no perm, and a lane
// finds its columns by a warp prefix sum of the 32 lens. The compact layout
// then gathers a 4-byte code instead of y (see kcode), which halves the
// operand bytes and so the number of passes.
//
// First sweep ("f1"). P(s,1) = 1/N for every s (metrics.cpp:143), so the
// first sweep's operand P(s,1) * (1/row_sum(s)) depends on the source only
// through row_sum(s). Sources are grouped into classes of equal 1/row_sum
// (bitwise), and the first sweep streams a 2-byte class per in-edge instead
// of gathering: factor = table[class], the table holding
// 1 - (1/N) * inv(class) in shared memory. It is a one-pass sliced layout
// (windows of 256 nodes — 32 for large graphs — sorted by in-degree, slices
// of 32 padded to a multiple of 4 steps, lane-major quads: f1_slot), built
// over every regular row whatever the segmentation of later sweeps:
//   f1_perm u32[S*32], f1_sptr u64[S+1], f1_cls u16[...]
// Class ncls is padding (factor exactly 1.0). Exception edges
// (R != 1/row_sum) carry class ncls+1, whose table entry is a NaN sentinel:
// a slice whose product comes out NaN is recomputed with their R, looked up
// by slot in the ascending list (f1_xslot, f1_xR). Long rows use lcls next
// to lcol. Graphs with more than kMaxCls classes keep the gathering sweep.
//
// kcode: round(1 - y) in fp64 depends on y only through J = rint(y * 2^53)
// while y <= 1/2: the doubles in [1/2, 1] are the multiples of 2^-53, so
// __dsub_rn(1, y) == 1 - J * 2^-53 exactly (ties: J even <=> result even).
// kcode[s] = J when J < 2^32 - 1 (y < 2^-21), else kBigCode and the sweep
// gathers y itself. Both arrays are written by every sweep epilogue.
#pragma once

#include <mutex>
#include <vector>

#include "common.cuh"

struct qvb_graph {
  int device = 0;
  uint64_t n = 0, e = 0, eu = 0, nexc = 0;
  uint32_t layout = 0;  // 0 compact, 1 weighted
  // source segments: sweep pass k multiplies the factors whose source lies
  // in [k*seg_size, (k+1)*seg_size); its slices are seg_slice[k]..seg_slice[k+1]
  uint64_t seg_size = 0;
  uint64_t seg0_size = 0;  // node-major layout: sources of the first segment
  std::vector<uint64_t> seg_slice;  // host, nseg + 1
  double* state = nullptr;          // running products between passes (nseg > 1)
  uint64_t pairs = 0;               // (node, segment) pairs with slots
  uint64_t nslices = 0;
  uint32_t* perm = nullptr;
  uint64_t* sptr = nullptr;
  uint32_t* scol = nullptr;
  double* sR = nullptr;
  uint64_t slots = 0;  // sptr[nslices] (padded elements)
  uint64_t nlong = 0;
  uint32_t long_threshold = 0;
  uint32_t* lnode = nullptr;
  uint64_t* lptr = nullptr;
  uint32_t* lcol = nullptr;
  double* lR = nullptr;
  uint32_t* exc_src = nullptr;
  double* exc_R = nullptr;
  double* inv = nullptr;
  double* p[2] = {nullptr, nullptr};
  double* y[2] = {nullptr, nullptr};
  // node-major segmented passes
  bool nm = false;
  uint64_t nm_S = 0;   // slices of 32 node ids
  uint64_t nm_cols = 0;
  uint8_t* nm_lenf = nullptr;
  uint64_t* nm_sbase = nullptr;
  uint32_t* nm_col = nullptr;
  uint32_t* nm_code = nullptr;      // compact: the gathered code of every nm_col entry (per sweep)
  std::vector<uint64_t> nm_region;  // host: start of each pass's columns in nm_col (nseg + 1)
  uint64_t nm_region_count = 0;     // passes (nseg) of the node-major layout
  uint32_t* marked = nullptr;       // device flag: a sweep's codes kept a marker (see k_codes)
  double* nm_R = nullptr;
  uint32_t* kcode[2] = {nullptr, nullptr};
  // first sweep ("f1", see above): out-degree classes and their streams
  uint32_t ncls = 0;            // 0: no class stream (the first sweep gathers)
  double* cls_inv = nullptr;    // [ncls] 1/row_sum of each class
  uint64_t f1_S = 0;            // slices of the one-pass sliced layout
  uint64_t f1_slots = 0;        // f1_sptr[f1_S]
  bool f1_ident = false;        // unsorted slices and no long rows: slot (s, l) is node 32 s + l
  uint32_t* f1_perm = nullptr;  // node of each slot (kNoNode: padding)
  uint64_t* f1_sptr = nullptr;  // slice starts (elements)
  uint16_t* f1_cls = nullptr;   // class per slot, lane-major; ncls: pad, ncls+1: exception
  uint64_t f1_nx = 0;           // exception slots, ascending, with their R
  uint64_t* f1_xslot = nullptr;
  double* f1_xR = nullptr;
  uint16_t* lcls = nullptr;     // class per long-row edge (ncls+1: see lcol)
  uint64_t bytes = 0;
  double build_ms = 0.0;
  cudaEvent_t ev[2] = {nullptr, nullptr};  // bracket the sweeps of the last run
  bool last_sharded = false;                // the last run split its sweeps over ranks
  uint64_t shard_key = ~0ull;               // (world << 32 | rank) of shard_e
  std::vector<uint64_t> shard_e;            // per pass: this rank's nm_col entry range
  // per-phase brackets of the last run: (phase, start, end); phase 0 = first
  // sweep (class stream), 1 = code gather (k_codes), 2 = ordered products,
  // 3 = any other sweep kernel
  struct PhaseEv { int phase; cudaEvent_t a, b; };
  std::vector<PhaseEv> phase_ev;
  size_t phase_used = 0;
  uint32_t launches = 0;  // kernels launched by the last run
  unsigned f1_grid = 0, codes_grid = 0, fused_grid = 0;  // resident grids, computed on first use
  // k_products_tma's static staging layout (access_prob.cu), built on first use
  uint64_t* nm_desc = nullptr;  // [S][K] bulk-copy descriptor per (slice, pass)
  uint64_t* nm_runs = nullptr;  // [N pad][2] per node: staged run of every pass
  uint32_t prod_bufw = 0;       // words per staging buffer (0: not built)
  uint32_t prod_zw = 0;         // zero words closing each buffer (sentinel runs)
  uint32_t prod_big = 0;        // slices too large for the buffer (global path)   // k_products_tma: words per staging buffer (0: not sized yet)
  unsigned prod_grid = 0;
  // qvb_access_prob reuses the buffers above: calls are serialised on the
  // host (run_mu) and, across streams, on the device (each call's stream
  // waits for the previous call's done event)
  std::mutex run_mu;
  cudaEvent_t done = nullptr;
  ~qvb_graph();
};

namespace qvb {
// Device -> pageable host copy through pinned staging slots and host threads
// (graph.cu); stream-ordered after the work queued on s, returns when done.
void copy_to_host(void* dst, const void* src, uint64_t bytes, cudaStream_t s);
}  // namespace qvb

namespace qvb {

constexpr uint32_t kExcFlag = 0x80000000u;
// perm slot = node | kFirst (first pass touching the node: start from 1.0)
//                  | kLast  (last pass: finish P instead of storing the state)
constexpr uint32_t kFirst = 0x80000000u;
constexpr uint32_t kLast = 0x40000000u;
constexpr uint32_t kNodeMask = 0x3FFFFFFFu;
constexpr uint32_t kNoNode = kNodeMask;  // padding slot
constexpr uint32_t kWindow = 256;  // slots sorted together (one CTA of 8 warps)
constexpr uint64_t kMaxNodes = (1ull << 30) - 2;
constexpr uint32_t kBigCode = 0xFFFFFFFFu;  // kcode: gather y instead
constexpr uint8_t kNmFirst = 0x40, kNmLast = 0x80, kNmLen = 0x3F;
constexpr uint64_t kMaxEdges = 0xFFFFFFFFull;
constexpr uint32_t kMaxCls = 12288;   // shared-memory table of ncls+2 doubles
// f1 slot of step k of the lane's node in the slice starting at `base`:
// lane-major quads, so a lane reads 4 consecutive steps with one 8-byte load
// and a warp's 32 loads cover 256 contiguous bytes
__host__ __device__ __forceinline__ uint64_t f1_slot(uint64_t base, uint64_t k, uint64_t lane) {
  return base + (k >> 2) * 128 + lane * 4 + (k & 3);
}

// transition_view (graph.cpp:292-318) by-products of the in-CSR build, on
// the device (each nullable): row_sums[n] (sequential CSR-order sums) and
// distinct[n] (coalesced (source, destination) pairs per source).
struct ViewOut {
  double* row_sums = nullptr;
  uint32_t* distinct = nullptr;
};

// Builds the in-CSR from a device out-CSR. d_w == nullptr means unit weights.
// d_src (nullable): source of every out-CSR edge if already known.
void build_in_csr(qvb_graph& g, const uint64_t* d_ro, const uint32_t* d_col, const double* d_w,
                  const uint32_t* d_src, cudaStream_t s, ViewOut view = {});

// Segmented sliced layout + long-row CSR from the coalesced in-CSR (uptr,
// col as stored (flagged exceptions), true sources src, R).
void build_slices(qvb_graph& g, const uint64_t* uptr, const uint32_t* col, const uint32_t* src,
                  const double* R, cudaStream_t s);
// The first-sweep class stream (f1) of a compact graph; no-op when the
// graph has more than kMaxCls classes or QVB_FIRST=gather.
void build_first(qvb_graph& g, const uint64_t* uptr, const uint32_t* col, const double* inv,
                 cudaStream_t s);
// Segment size in sources: QVB_SEG_MB (default 64) MiB of 8-byte operands.
uint64_t segment_size(uint64_t n);

// Raw transpose of a host out-CSR on the device (in_adjacency,
// graph.cpp:260-281): row pointers tptr[n+1], sources tsrc[e] ascending in
// each row with parallel edges kept in CSR order, carried weights tw[e]
// (left empty for unit weights), and transition_view's row sums rs[n].
// Validates like Graph::validate. *unit_weights: every weight is 1.0.
void device_transpose(uint64_t n, uint64_t e, const uint64_t* ro_h, const uint64_t* col_h,
                      const double* w_h, cudaStream_t s, DevBuf<uint64_t>& tptr,
                      DevBuf<uint32_t>& tsrc, DevBuf<double>& tw, DevBuf<double>& rs,
                      bool* unit_weights);

// Host out-CSR (qv::Graph layout) -> device: row offsets u64, columns u32,
// weights f64 (left empty when weights == nullptr), with Graph::validate's
// checks and messages (graph.cpp:58-93).
void upload_out_csr(uint64_t n, uint64_t e, const uint64_t* row_offsets, const uint64_t* col,
                    const double* weights, cudaStream_t s, DevBuf<uint64_t>& ro,
                    DevBuf<uint32_t>& dcol, DevBuf<double>& dw);
// tools/bench.cpp:22-34 generator + build_csr on the device (w left empty
// when !weighted; ssrc = source of every CSR edge).
void generate_out_csr(uint64_t n, uint64_t e, uint64_t seed, int weighted, int transposed,
                      cudaStream_t s, DevBuf<uint64_t>& ro, DevBuf<uint32_t>& col,
                      DevBuf<double>& w, DevBuf<uint32_t>& ssrc);

// Row-sharded P call (qvb_access_prob_sharded): rank of world, and the
// caller's exchange (an in-place all-gather of each sweep's P and codes).
struct Shard {
  uint32_t rank = 0, world = 1;
  qvb_exchange_fn fn = nullptr;
  void* ctx = nullptr;
};
// zero entries past N in the P / code buffers: chunks of ceil(n/world/32)*32
// nodes for up to 64 ranks
constexpr uint64_t kShardPad = 32 * 64;

// Runs layers-1 sweeps; returns the device buffer holding P_layers
// (final_out, when given: the last sweep writes it directly).
const double* run_access_prob(qvb_graph& g, uint32_t layers, cudaStream_t s,
                              double* final_out = nullptr, const Shard& sh = Shard{});

}  // namespace qvb
