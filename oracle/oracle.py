"""ctypes wrappers for the test-infrastructure oracles. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline. The product path (paper_2305_10863_b200) never does.

* ``Oracle``   — liboracle.so, the C restatement (oracle.c) of the reference.
* ``RefLib``   — _ref/libqvref.so, the UNMODIFIED reference sources
  (/root/reference/proj/src/*.cpp) compiled by oracle/Makefile, behind the
  marshalling shim ref_shim.cpp. Present only where it was built.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqvref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
LINK_COUNT = 7
_BATCH_SAMPLE_ARGS = [C.c_uint64, C.c_uint64] + [C.c_void_p] * 4 + [C.c_uint64, C.c_void_p,
                                                                     C.c_uint32, C.c_uint64] \
    + [C.POINTER(C.c_uint64)] * 2 + [C.c_void_p] * 3


class Topology(C.Structure):
    """Layout of ``qvb_topology`` (include/qvb.h) == qv::ClusterTopology."""

    _fields_ = [
        ("servers", C.c_uint32),
        ("numa_per_server", C.c_uint32),
        ("gpus_per_server", C.c_uint32),
        ("nvlink_within_numa", C.c_uint32),
        ("infiniband", C.c_uint32),
        ("_pad0", C.c_uint32),
        ("gpu_feature_capacity", C.c_uint64),
        ("host_feature_capacity", C.c_uint64),
        ("disk_feature_capacity", C.c_uint64),
        ("link_latency_s", C.c_double * LINK_COUNT),
        ("link_bandwidth_Bps", C.c_double * LINK_COUNT),
        ("tlb_miss_penalty_s", C.c_double),
        ("gpu_replicated_capacity", C.c_uint64),
    ]


def topology_defaults(**kw) -> Topology:
    """ClusterTopology::with_defaults (topology.cpp:27-40) + overrides."""
    t = Topology()
    t.servers = 1
    t.numa_per_server = 1
    t.gpus_per_server = 1
    lat = [0.0, 2e-6, 1e-5, 5e-6, 2e-6, 5e-5, 1e-4]
    bw = [1e12, 300e9, 16e9, 20e9, 12.5e9, 1.25e9, 0.5e9]
    for i in range(LINK_COUNT):
        t.link_latency_s[i] = lat[i]
        t.link_bandwidth_Bps[i] = bw[i]
    t.tlb_miss_penalty_s = 1e-7
    for k, v in kw.items():
        setattr(t, k, v)
    return t


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and _ref/libqvref.so when the reference exists)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets.append("ref")
        # the reference's own test files against the qv:: drop-in (needs it built)
        if os.path.exists(os.path.join(HERE, "..", "paper_2305_10863_b200", "libqv_b200.so")):
            targets.append("reftests")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class _Lib:
    prefix = ""

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(rc, getattr(self._lib, self.prefix + "last_error")().decode())


class Oracle(_Lib):
    """The C restatement (oracle.c)."""

    prefix = "qvo_"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self._lib = L
        L.qvo_last_error.restype = C.c_char_p
        L.qvo_splitmix64.restype = C.c_uint64
        L.qvo_splitmix64.argtypes = [C.c_uint64]
        L.qvo_derive_state.restype = C.c_uint64
        L.qvo_derive_state.argtypes = [C.c_uint64] * 4
        L.qvo_synthetic_graph.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                          u64p, u64p, f64p]
        L.qvo_synthetic_graph_mt.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                             C.c_int, u64p, u64p, f64p]
        L.qvo_features_mt.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, f32p, C.c_int]
        L.qvo_feature_rows.argtypes = [u64p, C.c_uint64, C.c_uint32, f32p, C.c_int]
        L.qvo_build_csr.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, u64p, u64p, f64p]
        L.qvo_validate.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p]
        L.qvo_in_adjacency.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, u64p, u64p, f64p]
        L.qvo_row_sums.argtypes = [C.c_uint64, u64p, f64p, f64p]
        L.qvo_access_prob.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, C.c_uint32, f64p]
        L.qvo_access_prob_sweep_nodes.argtypes = [C.c_uint64, u64p, u64p, f64p, f64p, f64p, u64p,
                                                  C.c_uint64, f64p]
        L.qvo_rank_desc.argtypes = [f64p, C.c_uint64, u64p]
        L.qvo_compute_fap.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, C.c_uint32,
                                      C.c_void_p, f64p]
        L.qvo_plan_placement.argtypes = [f64p, C.c_uint64, C.POINTER(Topology), u64p, i64p,
                                         C.c_uint64, C.POINTER(C.c_uint64)]
        L.qvo_build_lookup_table.argtypes = [u64p, i64p, C.c_uint64, C.POINTER(Topology),
                                             C.c_uint32, C.c_uint32, i64p, u64p]
        L.qvo_page_transitions.argtypes = [u64p, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        L.qvo_plan_reads.argtypes = [i64p, u64p, C.c_uint64, u64p, C.c_uint64, C.c_uint64, i64p,
                                     u64p, u64p, C.POINTER(C.c_uint64), u64p]
        L.qvo_features.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, f32p]
        L.qvo_request_ids.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p, C.c_uint64]
        L.qvo_gather.argtypes = [f32p, C.c_uint64, C.c_uint32, u64p, C.c_uint64, f32p, C.c_int]
        L.qvo_batch_sample.argtypes = _BATCH_SAMPLE_ARGS

    # rng / generators -------------------------------------------------------
    def splitmix64(self, x: int) -> int:
        return self._lib.qvo_splitmix64(x)

    def derive_state(self, master: int, a: int, b: int = 0, c: int = 0) -> int:
        return self._lib.qvo_derive_state(master, a, b, c)

    def synthetic_graph(self, n: int, e: int, seed: int = 7, weighted: bool = False,
                        transposed: bool = False, threads: int = 1):
        """tools/bench.cpp:22-34 -> out-CSR (row_offsets, col, weights).
        threads > 1: the counter-based threaded build (same bytes)."""
        ro = np.zeros(n + 1, np.uint64)
        col = np.empty(max(e, 1), np.uint64)
        w = np.empty(max(e, 1), np.float64)
        if threads > 1:
            self._check(self._lib.qvo_synthetic_graph_mt(n, e, seed, int(weighted), int(transposed),
                                                         threads, ro, col, w))
        else:
            self._check(self._lib.qvo_synthetic_graph(n, e, seed, int(weighted), int(transposed),
                                                      ro, col, w))
        return ro, col[:e], w[:e]

    def build_csr(self, n: int, src, dst, w):
        e = len(src)
        ro = np.zeros(n + 1, np.uint64)
        col = np.zeros(max(e, 1), np.uint64)
        wo = np.zeros(max(e, 1), np.float64)
        s = np.ascontiguousarray(src, np.uint64)
        d = np.ascontiguousarray(dst, np.uint64)
        ww = np.ascontiguousarray(w, np.float64)
        if e == 0:
            s = np.zeros(1, np.uint64)
            d = np.zeros(1, np.uint64)
            ww = np.zeros(1, np.float64)
        self._check(self._lib.qvo_build_csr(n, e, s, d, ww, ro, col, wo))
        return ro, col[:e].copy(), wo[:e].copy()

    def in_adjacency(self, ro, col, w):
        n = len(ro) - 1
        e = len(col)
        tro = np.zeros(n + 1, np.uint64)
        tcol = np.zeros(max(e, 1), np.uint64)
        tw = np.zeros(max(e, 1), np.float64)
        self._check(self._lib.qvo_in_adjacency(n, e, ro, _pad(col, np.uint64), _pad(w, np.float64),
                                               tro, tcol, tw))
        return tro, tcol[:e].copy(), tw[:e].copy()

    def row_sums(self, ro, w):
        n = len(ro) - 1
        rs = np.zeros(n, np.float64)
        self._check(self._lib.qvo_row_sums(n, ro, _pad(w, np.float64), rs))
        return rs

    def access_prob(self, ro, col, w, layers: int):
        """compute_access_prob_ie (metrics.cpp:134-173)."""
        n = len(ro) - 1
        out = np.zeros(n, np.float64)
        self._check(self._lib.qvo_access_prob(n, len(col), ro, _pad(col, np.uint64),
                                              _pad(w, np.float64), layers, out))
        return out

    def sweep_nodes(self, tro, tcol, tw, rs, prev, nodes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        out = np.zeros(len(nodes), np.float64)
        self._check(self._lib.qvo_access_prob_sweep_nodes(len(tro) - 1, tro, _pad(tcol, np.uint64),
                                                          _pad(tw, np.float64), rs, prev, nodes,
                                                          len(nodes), out))
        return out

    def batch_sample(self, ro, col, w, seeds, fanouts, rng_seed: int):
        """batch_sample (sampler.cpp:114-149) -> (nodes, counts[seed][hop], unique)."""
        return _batch_sample(self._lib.qvo_batch_sample, self._check, ro, col, w, seeds, fanouts,
                             rng_seed)

    def compute_fap(self, ro, col, w, hops: int, seed=None):
        """compute_fap (metrics.cpp:95-132)."""
        n = len(ro) - 1
        out = np.zeros(n, np.float64)
        sd = None if seed is None else np.ascontiguousarray(seed, np.float64)
        self._check(self._lib.qvo_compute_fap(n, len(col), ro, _pad(col, np.uint64),
                                              _pad(w, np.float64), hops,
                                              None if sd is None else sd.ctypes.data, out))
        return out

    # placement ---------------------------------------------------------------
    def rank_desc(self, values):
        v = np.ascontiguousarray(values, np.float64)
        r = np.zeros(len(v), np.uint64)
        self._check(self._lib.qvo_rank_desc(v, len(v), r))
        return r

    def plan_placement(self, values, topo: Topology):
        v = np.ascontiguousarray(values, np.float64)
        n = len(v)
        cap = max(1, n * topo.servers * (topo.gpus_per_server + 1))
        lo = np.zeros(n + 1, np.uint64)
        ids = np.zeros(cap, np.int64)
        copies = C.c_uint64(0)
        self._check(self._lib.qvo_plan_placement(v, n, C.byref(topo), lo, ids, cap,
                                                 C.byref(copies)))
        return lo, ids[: copies.value].copy()

    def build_lookup_table(self, lo, ids, topo: Topology, home: int = 0, reader: int = 0):
        n = len(lo) - 1
        loc = np.zeros(n, np.int64)
        off = np.zeros(n, np.uint64)
        self._check(self._lib.qvo_build_lookup_table(lo, _pad(ids, np.int64), n, C.byref(topo),
                                                     home, reader, loc, off))
        return loc, off

    def page_transitions(self, offsets, page: int) -> int:
        o = _pad(offsets, np.uint64)
        out = C.c_uint64(0)
        self._check(self._lib.qvo_page_transitions(o, len(offsets), page, C.byref(out)))
        return out.value

    def plan_reads(self, loc, off, ids, page: int = 8):
        ids = _pad(ids, np.uint64)
        b = len(ids) if len(ids) else 0
        return _plan_reads_call(self._lib.qvo_plan_reads, self._check, loc, off, ids, b, page)

    # features / requests / gather -------------------------------------------
    def features(self, n: int, dim: int, first: int = 0, threads: int = 1):
        x = np.empty((n, dim), np.float32)
        if threads > 1:
            self._lib.qvo_features_mt(first, n, dim, x.reshape(-1), threads)
        else:
            self._lib.qvo_features(first, n, dim, x.reshape(-1))
        return x

    def feature_rows(self, ids, dim: int, threads: int = 1):
        """X[ids] from the generator, without the table."""
        ids = np.ascontiguousarray(ids, np.uint64)
        out = np.empty((max(len(ids), 1), dim), np.float32)
        self._lib.qvo_feature_rows(_pad(ids, np.uint64), len(ids), dim, out.reshape(-1), threads)
        return out[: len(ids)]

    def request_ids(self, seed: int, batch: int, n: int, b: int):
        ids = np.zeros(b, np.uint64)
        self._lib.qvo_request_ids(seed, batch, n, ids, b)
        return ids

    def gather(self, x, ids, threads: int = 1):
        x = np.ascontiguousarray(x, np.float32)
        ids = np.ascontiguousarray(ids, np.uint64)
        out = np.zeros((len(ids), x.shape[1]), np.float32)
        self._check(self._lib.qvo_gather(x.reshape(-1), x.shape[0], x.shape[1], _pad(ids, np.uint64),
                                         len(ids), out.reshape(-1) if len(ids) else
                                         np.zeros(1, np.float32), threads))
        return out


class RefLib(_Lib):
    """The unmodified reference (oracle/_ref/libqvref.so)."""

    prefix = "qvr_"

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        L = C.CDLL(path)
        self._lib = L
        dp = C.POINTER(C.c_double)
        L.qvr_last_error.restype = C.c_char_p
        L.qvr_max_threads.restype = C.c_int
        L.qvr_set_threads.argtypes = [C.c_int]
        L.qvr_topology_defaults.argtypes = [C.POINTER(Topology)]
        L.qvr_access_prob.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, C.c_uint32, C.c_int,
                                      f64p, dp]
        L.qvr_in_adjacency.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, u64p, u64p, f64p]
        L.qvr_compute_fap.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, C.c_uint32, C.c_int,
                                      C.c_void_p, f64p]
        L.qvr_row_sums.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, f64p]
        L.qvr_transition_view.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, f64p, u64p,
                                          C.POINTER(C.c_int)]
        L.qvr_from_edges.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, u64p, u64p, f64p]
        L.qvr_validate.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p]
        L.qvr_classify_link.argtypes = [C.POINTER(Topology), C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.qvr_fetch_cost.argtypes = [C.POINTER(Topology), C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint64, i64p, u64p, u64p, C.c_uint64, f64p, dp]
        L.qvr_plan_placement.argtypes = [f64p, C.c_uint64, C.POINTER(Topology), u64p, i64p,
                                         C.c_uint64, C.POINTER(C.c_uint64), dp]
        L.qvr_build_lookup_table.argtypes = [u64p, i64p, C.c_uint64, C.POINTER(Topology),
                                             C.c_uint32, i64p, u64p, dp]
        L.qvr_page_transitions.argtypes = [u64p, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        L.qvr_plan_reads.argtypes = [i64p, u64p, C.c_uint64, u64p, C.c_uint64, C.c_uint64, i64p,
                                     u64p, u64p, C.POINTER(C.c_uint64), u64p, dp]
        L.qvr_batch_sample.argtypes = _BATCH_SAMPLE_ARGS + [dp]
        self.last_ms = 0.0

    def max_threads(self) -> int:
        return self._lib.qvr_max_threads()

    def set_threads(self, t: int) -> None:
        self._lib.qvr_set_threads(t)

    def topology_defaults(self) -> Topology:
        t = Topology()
        self._lib.qvr_topology_defaults(C.byref(t))
        return t

    def access_prob(self, ro, col, w, layers: int, parallel: bool = True):
        n = len(ro) - 1
        out = np.zeros(n, np.float64)
        ms = C.c_double(0)
        self._check(self._lib.qvr_access_prob(n, len(col), ro, _pad(col, np.uint64),
                                              _pad(w, np.float64), layers, int(parallel), out,
                                              C.byref(ms)))
        self.last_ms = ms.value
        return out

    def batch_sample(self, ro, col, w, seeds, fanouts, rng_seed: int):
        ms = C.c_double(0)
        res = _batch_sample(self._lib.qvr_batch_sample, self._check, ro, col, w, seeds, fanouts,
                            rng_seed, (C.byref(ms),))
        self.last_ms = ms.value
        return res

    def compute_fap(self, ro, col, w, hops: int, seed=None, parallel: bool = True):
        n = len(ro) - 1
        out = np.zeros(n, np.float64)
        sd = None if seed is None else np.ascontiguousarray(seed, np.float64)
        self._check(self._lib.qvr_compute_fap(n, len(col), ro, _pad(col, np.uint64),
                                              _pad(w, np.float64), hops, int(parallel),
                                              None if sd is None else sd.ctypes.data, out))
        return out

    def in_adjacency(self, ro, col, w):
        n = len(ro) - 1
        e = len(col)
        tro = np.zeros(n + 1, np.uint64)
        tcol = np.zeros(max(e, 1), np.uint64)
        tw = np.zeros(max(e, 1), np.float64)
        self._check(self._lib.qvr_in_adjacency(n, e, ro, _pad(col, np.uint64), _pad(w, np.float64),
                                               tro, tcol, tw))
        return tro, tcol[:e].copy(), tw[:e].copy()

    def row_sums(self, ro, col, w):
        n = len(ro) - 1
        rs = np.zeros(n, np.float64)
        self._check(self._lib.qvr_row_sums(n, len(col), ro, _pad(col, np.uint64),
                                           _pad(w, np.float64), rs))
        return rs

    def classify_link(self, topo: Topology, loc: int, rs: int = 0, rtier: int = 0, rdev: int = 0):
        a, b = C.c_int(0), C.c_int(0)
        self._check(self._lib.qvr_classify_link(C.byref(topo), rs, rtier, rdev, loc, C.byref(a),
                                                C.byref(b)))
        return a.value, (b.value if b.value >= 0 else None)

    def fetch_cost(self, groups, topo: Topology, feature_bytes: int, rs: int = 0, rtier: int = 0,
                   rdev: int = 0):
        gl = np.ascontiguousarray(groups[0], np.int64)
        gc = np.ascontiguousarray(groups[1], np.uint64)
        gt = np.ascontiguousarray(groups[2], np.uint64)
        per = np.zeros(max(len(gl), 1), np.float64)
        tot = C.c_double(0)
        self._check(self._lib.qvr_fetch_cost(C.byref(topo), rs, rtier, rdev, len(gl), _pad(gl, np.int64),
                                             _pad(gc, np.uint64), _pad(gt, np.uint64), feature_bytes,
                                             per, C.byref(tot)))
        return tot.value, per[: len(gl)]

    def transition_view(self, ro, col, w):
        """transition_view(g): (row_sums, distinct_out, has_parallel_edges)."""
        n = len(ro) - 1
        rs = np.zeros(n, np.float64)
        dist = np.zeros(n, np.uint64)
        par = C.c_int(0)
        self._check(self._lib.qvr_transition_view(n, len(col), ro, _pad(col, np.uint64),
                                                  _pad(w, np.float64), rs, dist, C.byref(par)))
        return rs, dist, bool(par.value)

    def from_edges(self, n: int, src, dst, w):
        e = len(src)
        ro = np.zeros(n + 1, np.uint64)
        col = np.zeros(max(e, 1), np.uint64)
        wo = np.zeros(max(e, 1), np.float64)
        self._check(self._lib.qvr_from_edges(n, e, _pad(src, np.uint64), _pad(dst, np.uint64),
                                             _pad(w, np.float64), ro, col, wo))
        return ro, col[:e].copy(), wo[:e].copy()

    def validate(self, ro, col, w) -> None:
        self._check(self._lib.qvr_validate(len(ro) - 1, len(col), _pad(ro, np.uint64),
                                           _pad(col, np.uint64), _pad(w, np.float64)))

    def plan_placement(self, values, topo: Topology):
        v = np.ascontiguousarray(values, np.float64)
        n = len(v)
        cap = max(1, n * topo.servers * (topo.gpus_per_server + 1))
        lo = np.zeros(n + 1, np.uint64)
        ids = np.zeros(cap, np.int64)
        copies = C.c_uint64(0)
        ms = C.c_double(0)
        self._check(self._lib.qvr_plan_placement(v, n, C.byref(topo), lo, ids, cap,
                                                 C.byref(copies), C.byref(ms)))
        self.last_ms = ms.value
        return lo, ids[: copies.value].copy()

    def build_lookup_table(self, lo, ids, topo: Topology, home: int = 0):
        n = len(lo) - 1
        loc = np.zeros(n, np.int64)
        off = np.zeros(n, np.uint64)
        ms = C.c_double(0)
        self._check(self._lib.qvr_build_lookup_table(lo, _pad(ids, np.int64), n, C.byref(topo),
                                                     home, loc, off, C.byref(ms)))
        self.last_ms = ms.value
        return loc, off

    def page_transitions(self, offsets, page: int) -> int:
        out = C.c_uint64(0)
        self._check(self._lib.qvr_page_transitions(_pad(offsets, np.uint64), len(offsets), page,
                                                   C.byref(out)))
        return out.value

    def plan_reads(self, loc, off, ids, page: int = 8):
        ids = _pad(ids, np.uint64)
        ms = C.c_double(0)

        def call(*args):
            return self._lib.qvr_plan_reads(*args, C.byref(ms))

        res = _plan_reads_call(call, self._check, loc, off, ids, len(ids), page)
        self.last_ms = ms.value
        return res


def _batch_sample(fn, check, ro, col, w, seeds, fanouts, rng_seed, extra=()):
    """Shared two-call driver of qvo_/qvr_batch_sample -> (nodes, counts, unique)."""
    n = len(ro) - 1
    s = _pad(seeds, np.uint64)
    f = np.ascontiguousarray(fanouts, np.uint32)
    hops = len(f)
    tot, uc = C.c_uint64(0), C.c_uint64(0)
    ro = np.ascontiguousarray(ro, np.uint64)
    col_, w_ = _pad(col, np.uint64), _pad(w, np.float64)  # keep alive across both calls
    args = [n, len(col), ro.ctypes.data, col_.ctypes.data, w_.ctypes.data, s.ctypes.data,
            len(seeds), f.ctypes.data, hops, rng_seed, C.byref(tot), C.byref(uc)]
    check(fn(*args, None, None, None, *extra))
    nodes = np.zeros(max(tot.value, 1), np.uint64)
    counts = np.zeros(max(len(seeds) * (hops + 1), 1), np.uint64)
    uniq = np.zeros(max(uc.value, 1), np.uint64)
    check(fn(*args, nodes.ctypes.data, counts.ctypes.data, uniq.ctypes.data, *extra))
    return nodes[: tot.value], counts[: len(seeds) * (hops + 1)].reshape(len(seeds), hops + 1), \
        uniq[: uc.value]


def _pad(a, dtype):
    """ctypes ndpointer needs a non-empty contiguous array."""
    a = np.ascontiguousarray(a, dtype)
    return a if a.size else np.zeros(1, dtype)


def _plan_reads_call(fn, check, loc, off, ids, b, page):
    loc = _pad(loc, np.int64)
    off = _pad(off, np.uint64)
    table_n = len(loc)
    m = max(b, 1)
    gl = np.zeros(m, np.int64)
    gc = np.zeros(m, np.uint64)
    gt = np.zeros(m, np.uint64)
    ng = C.c_uint64(0)
    oo = np.zeros(m, np.uint64)
    check(fn(loc, off, table_n, ids, b, page, gl, gc, gt, C.byref(ng), oo))
    g = ng.value
    return gl[:g].copy(), gc[:g].copy(), gt[:g].copy(), oo[:b].copy()
