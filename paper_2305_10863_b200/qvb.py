"""Python mirror of the reference's hot-path interface over the qvb C-ABI.

The reference is the C++ library ``qv`` (/root/reference/proj). This module
exposes the same operations under the same names and argument meanings —
``compute_access_prob_ie``, ``plan_placement``, ``build_lookup_table``,
``plan_reads``, ``page_transitions``, ``encode_location`` — plus the real
feature gather (``FeatureStore.gather``) that the reference only models with
``fetch_cost``. Errors raise the same exception family as the reference
(include/qv/error.hpp:10-32): ``ValidationError``, ``PlacementError`` …

Everything runs through ``libqvb.so`` (include/qvb.h). There is no CPU
fallback: importing this module without the built library, or calling a
compute function without a usable CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqvb.so")

LINK_LOCAL, LINK_NVLINK, LINK_PCIE, LINK_UPI, LINK_INFINIBAND, LINK_ETHERNET, LINK_DISK = range(7)
TIER_GPU, TIER_HOST, TIER_DISK = 0, 1, 2


# ---- errors (include/qv/error.hpp:10-32) ------------------------------------
class Error(RuntimeError):
    """qv::Error"""


class ValidationError(Error):
    """qv::ValidationError (also ParseError/ConfigError at this boundary)."""


class PlacementError(Error):
    """qv::PlacementError"""


class ParseError(Error):
    """qv::ParseError (file formats; error.hpp:14-16)"""


class CudaError(Error):
    """CUDA failure or no usable device (the library has no CPU fallback)."""


class UnsupportedError(Error):
    """Valid input outside the device path's limits."""


_CODES = {1: Error, 2: ValidationError, 3: PlacementError, 10: CudaError, 11: UnsupportedError}


class Topology(C.Structure):
    """qvb_topology == qv::ClusterTopology (topology.hpp:32-54) + extension."""

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
        ("link_latency_s", C.c_double * 7),
        ("link_bandwidth_Bps", C.c_double * 7),
        ("tlb_miss_penalty_s", C.c_double),
        ("gpu_replicated_capacity", C.c_uint64),
    ]

    @staticmethod
    def with_defaults(**kw) -> "Topology":
        """ClusterTopology::with_defaults (topology.cpp:27-40) + overrides."""
        t = Topology()
        _lib().qvb_topology_defaults(C.byref(t))
        for k, v in kw.items():
            setattr(t, k, v)
        return t

    def validate(self) -> None:
        _check(_lib().qvb_topology_validate(C.byref(self)))

    def gpus_per_numa(self) -> int:
        return self.gpus_per_server // self.numa_per_server


class GraphInfo(C.Structure):
    _fields_ = [
        ("node_count", C.c_uint64),
        ("edge_count", C.c_uint64),
        ("unique_edge_count", C.c_uint64),
        ("exception_count", C.c_uint64),
        ("layout", C.c_uint32),
        ("device", C.c_uint32),
        ("device_bytes", C.c_uint64),
        ("build_ms", C.c_double),
        ("classes", C.c_uint32),
        ("segments", C.c_uint32),
        ("first_slots", C.c_uint64),
        ("segment_columns", C.c_uint64),
    ]


class StoreInfo(C.Structure):
    _fields_ = [
        ("feature_count", C.c_uint64),
        ("dim", C.c_uint32),
        ("reader_device", C.c_uint32),
        ("row_stride_bytes", C.c_uint64),
        ("local_rows", C.c_uint64),
        ("host_rows", C.c_uint64),
        ("lut_bytes", C.c_uint64),
        ("location_count", C.c_uint32),
        ("_pad", C.c_uint32),
    ]


class SamplerInfo(C.Structure):
    _fields_ = [
        ("node_count", C.c_uint64),
        ("edge_count", C.c_uint64),
        ("candidates", C.c_uint64),
        ("parallel_edges", C.c_int32),
        ("unit_weights", C.c_int32),
        ("max_candidates", C.c_uint64),
        ("device_bytes", C.c_uint64),
        ("build_ms", C.c_double),
    ]


class SampleInfo(C.Structure):
    _fields_ = [
        ("seeds", C.c_uint64),
        ("hops", C.c_uint32),
        ("reserved", C.c_uint32),
        ("total_instances", C.c_uint64),
        ("unique_count", C.c_uint64),
        ("device_ms", C.c_double),
    ]


_LIB = None
# qvb_exchange_fn: int (*)(void* ctx, uint32_t layer, void* p, void* codes, uint64_t chunk, void* stream)
ExchangeFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
vp = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int
P = C.POINTER

_SIGNATURES = {
    "qvb_last_error": (C.c_char_p, []),
    "qvb_version": (C.c_char_p, []),
    "qvb_device_count": (i32, [P(i32)]),
    "qvb_topology_defaults": (None, [P(Topology)]),
    "qvb_topology_validate": (i32, [P(Topology)]),
    "qvb_encode_location": (C.c_int64, [P(Topology), u32, u32, u32]),
    "qvb_decode_location": (i32, [P(Topology), C.c_int64, P(u32), P(u32), P(u32)]),
    "qvb_graph_upload": (i32, [i32, u64, u64, vp, vp, vp, vp, P(vp)]),
    "qvb_graph_synthetic": (i32, [i32, u64, u64, u64, i32, i32, vp, P(vp)]),
    "qvb_graph_info_get": (i32, [vp, P(GraphInfo)]),
    "qvb_synthetic_csr": (i32, [i32, u64, u64, u64, i32, i32, vp, vp, vp]),
    "qvb_in_adjacency": (i32, [i32, u64, u64, vp, vp, vp, vp, vp, vp]),
    "qvb_graph_last_sweep_ms": (i32, [vp, P(C.c_double)]),
    "qvb_graph_phase_ms": (i32, [vp, P(C.c_double), P(C.c_uint32)]),
    "qvb_graph_in_rows": (i32, [vp, vp, u64, vp, vp, vp]),
    "qvb_graph_destroy": (i32, [vp]),
    "qvb_graph_validate": (i32, [i32, u64, u64, vp, vp, vp]),
    "qvb_build_csr": (i32, [i32, u64, vp, u64, vp, vp, vp]),
    "qvb_transition_view": (i32, [i32, u64, u64, vp, vp, vp, vp, vp, P(i32), P(vp)]),
    "qvb_classify_link": (i32, [P(Topology), u32, u32, u32, C.c_int64, P(i32), P(i32)]),
    "qvb_fetch_cost": (i32, [P(Topology), u32, u32, u32, u64, vp, vp, vp, u64, vp, P(C.c_double)]),
    "qvb_access_prob": (i32, [vp, u32, vp, i32, vp]),
    "qvb_compute_access_prob_ie": (i32, [i32, u64, u64, vp, vp, vp, u32, vp, vp]),
    "qvb_access_prob_sharded": (i32, [vp, u32, u32, u32, vp, vp, vp, i32, vp, P(i32)]),
    "qvb_compute_fap": (i32, [i32, u64, u64, vp, vp, vp, u32, vp, vp]),
    "qvb_rank_desc": (i32, [i32, vp, u64, vp, i32, vp]),
    "qvb_plan_placement": (i32, [i32, vp, u64, P(Topology), vp, vp, u64, P(u64)]),
    "qvb_plan_placement_create": (i32, [i32, vp, u64, P(Topology), P(vp)]),
    "qvb_plan_size": (i32, [vp, P(u64), P(u64)]),
    "qvb_plan_copy": (i32, [vp, vp, vp]),
    "qvb_plan_destroy": (i32, [vp]),
    "qvb_build_lookup_table": (i32, [i32, vp, vp, u64, P(Topology), u32, u32, vp, vp]),
    "qvb_page_transitions": (i32, [vp, u64, u64, P(u64)]),
    "qvb_plan_reads": (i32, [i32, vp, vp, u64, vp, u64, u64, vp, vp, vp, P(u64), vp]),
    "qvb_store_create": (i32, [i32, vp, vp, u64, u32, P(Topology), u32, vp, P(vp)]),
    "qvb_store_info_get": (i32, [vp, P(StoreInfo)]),
    "qvb_store_export_handle": (i32, [vp, vp]),
    "qvb_store_attach_peer": (i32, [vp, u32, vp]),
    "qvb_store_attach_local_peer": (i32, [vp, u32, vp]),
    "qvb_store_destroy": (i32, [vp]),
    "qvb_gather": (i32, [vp, vp, u64, vp, vp]),
    "qvb_gather_planned": (i32, [vp, vp, u64, vp, vp]),
    "qvb_gather_host": (i32, [vp, vp, u64, vp, vp]),
    "qvb_store_check_error": (i32, [vp]),
    "qvb_store_plan_reads": (i32, [vp, vp, u64, i32, u64, vp, vp, vp, P(u64), vp, vp]),
    "qvb_plan_reads_device": (i32, [i32, vp, vp, u64, vp, u64, u64, vp, vp, vp, P(u64), vp, vp]),
    "qvb_request_ids_synthetic": (i32, [i32, u64, u64, u64, vp, u64, vp]),
    "qvb_sampler_create": (i32, [i32, u64, u64, vp, vp, vp, vp, P(vp)]),
    "qvb_sampler_synthetic": (i32, [i32, u64, u64, u64, i32, i32, vp, P(vp)]),
    "qvb_sampler_info_get": (i32, [vp, P(SamplerInfo)]),
    "qvb_sampler_destroy": (i32, [vp]),
    "qvb_batch_sample": (i32, [vp, vp, u64, i32, vp, u32, u64, vp, P(vp)]),
    "qvb_sample_info_get": (i32, [vp, P(SampleInfo)]),
    "qvb_sample_copy": (i32, [vp, vp, vp, vp]),
    "qvb_sample_device": (i32, [vp, P(vp), P(vp), P(vp)]),
    "qvb_sample_destroy": (i32, [vp]),
    # include/qvb_test.h
    "qvb_test_sort_pairs_u64": (i32, [i32, vp, vp, u64, i32, i32, vp, vp]),
    "qvb_test_scan_u32": (i32, [i32, vp, u64, i32, vp]),
    "qvb_test_sort_bench": (i32, [i32, u64, i32, i32, P(C.c_double)]),
    "qvb_test_log1p": (i32, [i32, vp, u64, vp]),
}


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2305_10863_b200.build` "
                "(the qvb path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            f = getattr(L, name)  # every declared entry point must be exported
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def exported_symbols():
    return list(_SIGNATURES)


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib().qvb_last_error().decode()
        raise _CODES.get(rc, Error)(msg)


def _ptr(a) -> int | None:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):  # torch tensor (device or host)
        return a.data_ptr()
    return int(a)


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def device_count() -> int:
    c = C.c_int(0)
    _check(_lib().qvb_device_count(C.byref(c)))
    return c.value


def version() -> str:
    return _lib().qvb_version().decode()


# ---- locations (placement.cpp:25-51) ------------------------------------------
def encode_location(topo: Topology, server: int, tier: int, device: int) -> int:
    return _lib().qvb_encode_location(C.byref(topo), server, tier, device)


def decode_location(topo: Topology, loc: int):
    s, t, d = u32(), u32(), u32()
    _check(_lib().qvb_decode_location(C.byref(topo), loc, C.byref(s), C.byref(t), C.byref(d)))
    return s.value, t.value, d.value


# ---- graph + K1 ----------------------------------------------------------------
class DeviceGraph:
    """Device-resident in-CSR (qvb_graph): in_adjacency + transition_view once."""

    def __init__(self, handle: int):
        self._h = handle

    @classmethod
    def upload(cls, row_offsets, col, weights=None, device: int = 0, stream=None):
        ro = np.ascontiguousarray(row_offsets, np.uint64)
        c = np.ascontiguousarray(col, np.uint64)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        h = vp()
        _check(_lib().qvb_graph_upload(device, len(ro) - 1, len(c), _ptr(ro), _ptr(c) if len(c) else None,
                                       _ptr(w) if w is not None and len(w) else None,
                                       _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    @classmethod
    def synthetic(cls, n: int, e: int, seed: int = 7, weighted: bool = False,
                  transposed: bool = False, device: int = 0, stream=None):
        """tools/bench.cpp:22-34 generator, directly on the device."""
        h = vp()
        _check(_lib().qvb_graph_synthetic(device, n, e, seed, int(weighted), int(transposed),
                                          _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    def info(self) -> GraphInfo:
        i = GraphInfo()
        _check(_lib().qvb_graph_info_get(self._h, C.byref(i)))
        return i

    def access_prob(self, layers: int, out=None, stream=None):
        """P(n, layers) for every node. ``out``: a host numpy array (default)
        or a device tensor of n float64."""
        n = self.info().node_count
        if out is None:
            out = np.zeros(n, np.float64)
        on_dev = 0 if isinstance(out, np.ndarray) else 1
        _check(_lib().qvb_access_prob(self._h, layers, _ptr(out), on_dev, _stream_ptr(stream)))
        return out

    def access_prob_sharded(self, layers: int, rank: int, world: int, exchange, out=None,
                            stream=None):
        """Row-sharded P (qvb_access_prob_sharded): this rank computes its
        node chunk of every sweep; ``exchange(layer, p_ptr, codes_ptr, chunk,
        stream_ptr)`` must all-gather the chunks in place and return. Returns
        (P for every node, whether the layout was actually split)."""
        n = self.info().node_count
        if out is None:
            out = np.zeros(n, np.float64)
        on_dev = 0 if isinstance(out, np.ndarray) else 1
        err = []

        def cb(_ctx, layer, p, codes, chunk, st):
            try:
                exchange(layer, p, codes, chunk, st)
                return 0
            except Exception as ex:  # noqa: BLE001 - reported by the library as a failure
                err.append(ex)
                return 1

        fn = ExchangeFn(cb)
        sh = C.c_int(0)
        rc = _lib().qvb_access_prob_sharded(self._h, layers, rank, world, C.cast(fn, C.c_void_p), None,
                                             _ptr(out), on_dev, _stream_ptr(stream), C.byref(sh))
        if err:
            raise err[0]
        _check(rc)
        return out, bool(sh.value)

    def last_sweep_ms(self) -> float:
        """Device time of the P sweeps of the last access_prob call."""
        ms = C.c_double(0)
        _check(_lib().qvb_graph_last_sweep_ms(self._h, C.byref(ms)))
        return ms.value

    def phase_ms(self):
        """Device ms of the last access_prob call by phase: first sweep (class
        stream), code gathers, ordered products, other sweep kernels; and the
        number of kernels it launched."""
        ms = (C.c_double * 4)()
        n = C.c_uint32()
        _check(_lib().qvb_graph_phase_ms(self._h, ms, C.byref(n)))
        return {"first": ms[0], "gather": ms[1], "products": ms[2], "other": ms[3],
                "launches": n.value}

    def in_rows(self, nodes):
        """The coalesced in-rows the sweeps multiply for ``nodes``: (row_ptr,
        sources ascending, R = w_sum / row_sum(source)). Node-major graphs."""
        nd = np.ascontiguousarray(nodes, np.uint64)
        rp = np.zeros(len(nd) + 1, np.uint64)
        _check(_lib().qvb_graph_in_rows(self._h, _ptr(nd), len(nd), _ptr(rp), None, None))
        src = np.zeros(max(int(rp[-1]), 1), np.uint32)
        R = np.zeros(max(int(rp[-1]), 1), np.float64)
        _check(_lib().qvb_graph_in_rows(self._h, _ptr(nd), len(nd), _ptr(rp), _ptr(src), _ptr(R)))
        return rp, src[: int(rp[-1])], R[: int(rp[-1])]

    def close(self):
        if self._h:
            _lib().qvb_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def synthetic_csr(n: int, e: int, seed: int = 7, weighted: bool = False,
                  transposed: bool = False, device: int = 0):
    """tools/bench.cpp:22-34 generator run on the device, returned as a host
    out-CSR (row_offsets u64[n+1], col u64[e], weights f64[e])."""
    ro = np.zeros(n + 1, np.uint64)
    col = np.zeros(max(e, 1), np.uint64)
    w = np.zeros(max(e, 1), np.float64)
    _check(_lib().qvb_synthetic_csr(device, n, e, seed, int(weighted), int(transposed), _ptr(ro),
                                    _ptr(col), _ptr(w)))
    return ro, col[:e], w[:e]


def transition_view(row_offsets, col, weights=None, device: int = 0, keep: bool = False):
    """qv::transition_view (graph.cpp:292-318) on the device:
    (row_sums, distinct_out, has_parallel_edges[, DeviceGraph]). keep=True
    also returns the device graph the same upload built (for access_prob)."""
    ro = np.ascontiguousarray(row_offsets, np.uint64)
    c = np.ascontiguousarray(col, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    n, e = len(ro) - 1, len(c)
    rs = np.empty(max(n, 1), np.float64)
    dist = np.empty(max(n, 1), np.uint64)
    par = C.c_int(0)
    h = C.c_void_p()
    _check(_lib().qvb_transition_view(device, n, e, _ptr(ro), _ptr(c) if e else None, _ptr(w),
                                      _ptr(rs), _ptr(dist), C.byref(par), C.byref(h) if keep else None))
    out = (rs[:n], dist[:n], bool(par.value))
    return out + (DeviceGraph(h.value),) if keep else out


def graph_validate(row_offsets, col, weights=None, device: int = 0) -> None:
    """qv::Graph::validate (graph.cpp:58-93) on the device."""
    ro = np.ascontiguousarray(row_offsets, np.uint64)
    c = np.ascontiguousarray(col, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    _check(_lib().qvb_graph_validate(device, len(ro) - 1, len(c), _ptr(ro), _ptr(c) if len(c) else None,
                                     _ptr(w)))


def from_edges(n: int, src, dst, weights, device: int = 0):
    """qv::Graph::from_edges (graph.cpp:16-56) on the device -> out-CSR."""
    e = len(src)
    edges = np.empty(max(e, 1), dtype=[("src", "<u8"), ("dst", "<u8"), ("w", "<f8")])
    edges["src"][:e] = np.asarray(src, np.uint64)
    edges["dst"][:e] = np.asarray(dst, np.uint64)
    edges["w"][:e] = np.asarray(weights, np.float64)
    ro = np.empty(n + 1, np.uint64)
    col = np.empty(max(e, 1), np.uint64)
    w = np.empty(max(e, 1), np.float64)
    _check(_lib().qvb_build_csr(device, n, edges.ctypes.data, e, _ptr(ro), _ptr(col), _ptr(w)))
    return ro, col[:e], w[:e]


def in_adjacency(row_offsets, col, weights=None, device: int = 0):
    """qv::in_adjacency (graph.cpp:260-281) on the device -> host transpose."""
    ro = np.ascontiguousarray(row_offsets, np.uint64)
    c = np.ascontiguousarray(col, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    n, e = len(ro) - 1, len(c)
    tro = np.zeros(n + 1, np.uint64)
    tcol = np.zeros(max(e, 1), np.uint64)
    tw = np.zeros(max(e, 1), np.float64)
    _check(_lib().qvb_in_adjacency(device, n, e, _ptr(ro), _ptr(c) if e else None,
                                   _ptr(w) if w is not None and e else None, _ptr(tro), _ptr(tcol),
                                   _ptr(tw)))
    return tro, tcol[:e], tw[:e]


@dataclass
class AccessProbTable:
    """qv::AccessProbTable (metrics.hpp:38-45)."""

    values: np.ndarray
    layers: int


def compute_access_prob_ie(row_offsets, col, weights, layers: int, device: int = 0,
                           timings: list | None = None) -> AccessProbTable:
    """qv::compute_access_prob_ie(g, transition_view(g), layers) (metrics.hpp:53-54)
    from a host out-CSR, end to end on the GPU."""
    ro = np.ascontiguousarray(row_offsets, np.uint64)
    c = np.ascontiguousarray(col, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    n = len(ro) - 1
    out = np.zeros(max(n, 1), np.float64)
    ms = (C.c_double * 3)()
    _check(_lib().qvb_compute_access_prob_ie(device, n, len(c), _ptr(ro), _ptr(c) if len(c) else None,
                                             _ptr(w) if w is not None and len(w) else None, layers,
                                             _ptr(out), ms))
    if timings is not None:
        timings[:] = list(ms)
    return AccessProbTable(out[:n], layers)


@dataclass
class FapTable:
    """qv::FapTable (metrics.hpp:32-36)."""

    values: np.ndarray
    hops: int
    seed_distribution: np.ndarray


def compute_fap(row_offsets, col, weights, hops: int, seed=None, device: int = 0) -> FapTable:
    """qv::compute_fap(transition_view(g), hops, seed) (metrics.cpp:95-132) on the GPU."""
    ro = np.ascontiguousarray(row_offsets, np.uint64)
    c = np.ascontiguousarray(col, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    n = len(ro) - 1
    sd = None if seed is None else np.ascontiguousarray(seed, np.float64)
    if sd is not None and len(sd) != n:
        raise ValidationError("seed distribution size does not match node count")
    out = np.zeros(max(n, 1), np.float64)
    _check(_lib().qvb_compute_fap(device, n, len(c), _ptr(ro), _ptr(c) if len(c) else None,
                                  _ptr(w) if w is not None and len(w) else None, hops, _ptr(sd),
                                  _ptr(out)))
    p0 = sd if sd is not None else np.full(n, 1.0 / n) if n else np.zeros(0)
    return FapTable(out[:n], hops, p0)


# ---- K2 / placement (placement.cpp:79-226) ------------------------------------
def rank_desc(values, device: int = 0) -> np.ndarray:
    """fap_ranking (placement.cpp:79-87): ids by value desc, id asc on ties."""
    v = np.ascontiguousarray(values, np.float64)
    r = np.zeros(max(len(v), 1), np.uint64)
    _check(_lib().qvb_rank_desc(device, _ptr(v), len(v), _ptr(r), 0, None))
    return r[: len(v)]


def plan_placement(values, topo: Topology, device: int = 0):
    """qv::plan_placement(FapTable{values}, topo) in canonical CSR form:
    (loc_offsets[n+1], loc_ids[copies]) — feature f's copies are
    loc_ids[loc_offsets[f]:loc_offsets[f+1]], ascending encoded location ids."""
    v = np.ascontiguousarray(values, np.float64)
    n = len(v)
    h = C.c_void_p()
    _check(_lib().qvb_plan_placement_create(device, _ptr(v) if n else None, n, C.byref(topo),
                                            C.byref(h)))
    try:
        nn, copies = u64(0), u64(0)
        _check(_lib().qvb_plan_size(h, C.byref(nn), C.byref(copies)))
        lo = np.zeros(n + 1, np.uint64)
        ids = np.zeros(max(1, copies.value), np.int64)
        _check(_lib().qvb_plan_copy(h, _ptr(lo), _ptr(ids)))
    finally:
        _lib().qvb_plan_destroy(h)
    return lo, ids[: copies.value]


def build_lookup_table(loc_offsets, loc_ids, topo: Topology, home_server: int = 0,
                       reader: int = 0, device: int = 0):
    """qv::build_lookup_table(plan, topo, home_server) -> (location_ids, offsets).
    ``reader`` > 0 is the per-reader extension (the reference reads from GPU 0)."""
    lo = np.ascontiguousarray(loc_offsets, np.uint64)
    ids = np.ascontiguousarray(loc_ids, np.int64)
    n = len(lo) - 1
    loc = np.zeros(max(n, 1), np.int64)
    off = np.zeros(max(n, 1), np.uint64)
    _check(_lib().qvb_build_lookup_table(device, _ptr(lo), _ptr(ids) if len(ids) else None, n,
                                         C.byref(topo), home_server, reader, _ptr(loc), _ptr(off)))
    return loc[:n], off[:n]


# ---- K4 read planner (placement.cpp:344-380) -----------------------------------
def page_transitions(offsets, page_size: int) -> int:
    o = np.ascontiguousarray(offsets, np.uint64)
    out = u64(0)
    _check(_lib().qvb_page_transitions(_ptr(o) if len(o) else None, len(o), page_size, C.byref(out)))
    return out.value


def plan_reads(location_ids, offsets, ids, page_size: int = 8, device: int = 0):
    """qv::plan_reads flattened: (group_loc, group_count, group_transitions,
    offsets) — groups ascending by location, offsets ascending per group."""
    loc = np.ascontiguousarray(location_ids, np.int64)
    off = np.ascontiguousarray(offsets, np.uint64)
    req = np.ascontiguousarray(ids, np.uint64)
    b = len(req)
    m = max(b, 1)
    gl = np.zeros(m, np.int64)
    gc = np.zeros(m, np.uint64)
    gt = np.zeros(m, np.uint64)
    oo = np.zeros(m, np.uint64)
    ng = u64(0)
    _check(_lib().qvb_plan_reads(device, _ptr(loc), _ptr(off), len(loc), _ptr(req) if b else None, b,
                                 page_size, _ptr(gl), _ptr(gc), _ptr(gt), C.byref(ng), _ptr(oo)))
    g = ng.value
    return gl[:g].copy(), gc[:g].copy(), gt[:g].copy(), oo[:b].copy()


def _plan_out(b: int, groups_cap: int):
    m = max(b, 1)
    g = max(1, min(m, groups_cap))
    return (np.empty(g, np.int64), np.empty(g, np.uint64), np.empty(g, np.uint64),
            np.empty(m, np.uint64), u64(0))


def classify_link(topo: Topology, location_id: int, reader_server: int = 0,
                  reader_tier: int = TIER_GPU, reader_device: int = 0):
    """classify_link (placement.cpp:228-267) -> (first, second or None)."""
    a, b = C.c_int(0), C.c_int(0)
    _check(_lib().qvb_classify_link(C.byref(topo), reader_server, reader_tier, reader_device,
                                    location_id, C.byref(a), C.byref(b)))
    return a.value, (b.value if b.value >= 0 else None)


def fetch_cost(groups, topo: Topology, feature_bytes: int, reader_server: int = 0,
               reader_tier: int = TIER_GPU, reader_device: int = 0):
    """fetch_cost (placement.cpp:382-404) over a flattened read plan
    (group_loc, group_count, group_transitions) -> (total_s, per_location_s)."""
    gl = np.ascontiguousarray(groups[0], np.int64)
    gc = np.ascontiguousarray(groups[1], np.uint64)
    gt = np.ascontiguousarray(groups[2], np.uint64)
    per = np.zeros(max(len(gl), 1), np.float64)
    tot = C.c_double(0)
    _check(_lib().qvb_fetch_cost(C.byref(topo), reader_server, reader_tier, reader_device, len(gl),
                                 _ptr(gl), _ptr(gc), _ptr(gt), feature_bytes, _ptr(per), C.byref(tot)))
    return tot.value, per[: len(gl)]


def plan_reads_device(location_ids, offsets, ids, page_size: int = 8, device: int = 0, stream=None):
    """qv::plan_reads over a lookup table already on the device (torch tensors
    location_ids int64[n], offsets uint64/int64[n], ids [b]): no table upload."""
    for t in (location_ids, offsets, ids):
        if not t.is_cuda or not t.is_contiguous() or t.element_size() != 8:
            raise ValidationError("table and ids must be contiguous 64-bit device tensors")
    b = int(ids.numel())
    gl, gc, gt, oo, ng = _plan_out(b, b)
    _check(_lib().qvb_plan_reads_device(device, _ptr(location_ids), _ptr(offsets),
                                        int(location_ids.numel()), _ptr(ids), b, page_size,
                                        _ptr(gl), _ptr(gc), _ptr(gt), C.byref(ng), _ptr(oo),
                                        _stream_ptr(stream)))
    g = ng.value
    return gl[:g], gc[:g], gt[:g], oo[:b]


# ---- K5 feature store + gather ---------------------------------------------------
class FeatureStore:
    """One reader GPU's view of the placed feature table (qvb_store).

    Built from a single-server plan (``plan_placement`` output); holds this
    GPU's shard in HBM, the host tier in pinned mapped memory and the
    reader's lookup table; peers are attached with ``attach_peer``."""

    def __init__(self, loc_offsets, loc_ids, dim: int, topo: Topology, reader: int = 0,
                 features=None, device: int | None = None):
        lo = np.ascontiguousarray(loc_offsets, np.uint64)
        ids = np.ascontiguousarray(loc_ids, np.int64)
        self.n = len(lo) - 1
        self.dim = dim
        self.device = reader if device is None else device
        x = None if features is None else np.ascontiguousarray(features, np.float32)
        if x is not None and x.shape != (self.n, dim):
            raise ValidationError(f"features must be ({self.n}, {dim})")
        h = vp()
        _check(_lib().qvb_store_create(self.device, _ptr(lo), _ptr(ids) if len(ids) else None, self.n,
                                       dim, C.byref(topo), reader, _ptr(x), C.byref(h)))
        self._h = h.value
        self._keep = x

    def info(self) -> StoreInfo:
        i = StoreInfo()
        _check(_lib().qvb_store_info_get(self._h, C.byref(i)))
        return i

    def export_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        _check(_lib().qvb_store_export_handle(self._h, buf))
        return bytes(buf)

    def attach_peer(self, peer_device: int, handle: bytes) -> None:
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        _check(_lib().qvb_store_attach_peer(self._h, peer_device, buf))

    def attach_local_peer(self, peer_device: int, peer: "FeatureStore") -> None:
        """Map another store of this process (P2P when on another device)."""
        _check(_lib().qvb_store_attach_local_peer(self._h, peer_device, peer._h))
        self._peers = getattr(self, "_peers", []) + [peer]

    def gather(self, ids, out, stream=None, planned: bool = False) -> None:
        """Device gather: ids (uint64/int64) and out (float32, b x dim) are
        contiguous device tensors; stream-ordered, no synchronisation."""
        import torch

        b = int(ids.numel())
        if ids.dtype not in (torch.int64, torch.uint64) or not ids.is_contiguous():
            raise ValidationError("ids must be a contiguous 64-bit integer tensor")
        if out.dtype != torch.float32 or not out.is_contiguous() or out.numel() < b * self.dim:
            raise ValidationError(f"out must be a contiguous float32 tensor of at least "
                                  f"{b} x {self.dim} values")
        if not ids.is_cuda or not out.is_cuda:
            raise ValidationError("ids and out must be device tensors (use gather_host for host buffers)")
        fn = _lib().qvb_gather_planned if planned else _lib().qvb_gather
        _check(fn(self._h, _ptr(ids), b, _ptr(out), _stream_ptr(stream)))

    def check_error(self) -> None:
        _check(_lib().qvb_store_check_error(self._h))

    def plan_reads(self, ids, page_size: int = 8, stream=None):
        """qv::plan_reads over this store's resident lookup table; ids are a
        host array or a device tensor. Same flattened result as plan_reads."""
        on_dev = hasattr(ids, "is_cuda") and ids.is_cuda
        if on_dev:
            if not ids.is_contiguous() or ids.element_size() != 8:
                raise ValidationError("ids must be a contiguous 64-bit tensor")
            req, b = ids, int(ids.numel())
        else:
            req = np.ascontiguousarray(ids, np.uint64)
            b = len(req)
        gl, gc, gt, oo, ng = _plan_out(b, self.info().location_count)
        _check(_lib().qvb_store_plan_reads(self._h, _ptr(req) if b else None, b, int(on_dev), page_size,
                                           _ptr(gl), _ptr(gc), _ptr(gt), C.byref(ng), _ptr(oo),
                                           _stream_ptr(stream)))
        g = ng.value
        return gl[:g], gc[:g], gt[:g], oo[:b]

    def gather_host(self, ids, out=None, stream=None) -> np.ndarray:
        """End-to-end collect from host buffers (H2D ids, gather, D2H rows)."""
        req = np.ascontiguousarray(ids, np.uint64)  # copies strided / other-typed ids
        if out is None:
            out = np.zeros((len(req), self.dim), np.float32)
        elif not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous
                  and out.shape == (len(req), self.dim)):
            raise ValidationError(f"out must be a C-contiguous float32 array of shape "
                                  f"({len(req)}, {self.dim})")
        _check(_lib().qvb_gather_host(self._h, _ptr(req), len(req), _ptr(out), _stream_ptr(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib().qvb_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def request_ids_synthetic(seed: int, batch: int, n: int, out, device: int = 0, stream=None):
    """ids[k] = derive_stream(seed, 0x5EED, batch).below(n) draw k, on device."""
    _check(_lib().qvb_request_ids_synthetic(device, seed, batch, n, _ptr(out), int(out.numel()),
                                            _stream_ptr(stream)))
    return out


# ---- K0: k-hop sampler (sampler.cpp:21-149) -----------------------------------
@dataclass
class SampleResult:
    """qv::SampleResult (sampler.hpp:14-28) for one seed."""

    seed: int
    frontiers: list
    instance_counts: list
    unique_nodes: np.ndarray

    def total_instances(self) -> int:
        return int(sum(self.instance_counts))


class BatchSample:
    """Result of one batch_sample on the device (qvb_sample). ``nodes`` is
    every per-seed frontier flattened seed-major then hop-major, ``counts``
    [seeds, hops+1] the instance counts, ``unique`` the sorted union
    (BatchSampleStats::unique_nodes)."""

    def __init__(self, handle: int):
        self._h = handle

    def info(self) -> SampleInfo:
        i = SampleInfo()
        _check(_lib().qvb_sample_info_get(self._h, C.byref(i)))
        return i

    def arrays(self):
        i = self.info()
        nodes = np.zeros(max(i.total_instances, 1), np.uint64)
        counts = np.zeros(max(i.seeds * (i.hops + 1), 1), np.uint64)
        uniq = np.zeros(max(i.unique_count, 1), np.uint64)
        _check(_lib().qvb_sample_copy(self._h, _ptr(nodes), _ptr(counts), _ptr(uniq)))
        return (nodes[: i.total_instances], counts[: i.seeds * (i.hops + 1)].reshape(i.seeds, i.hops + 1),
                uniq[: i.unique_count])

    def device_unique(self):
        """(device pointer, count) of the sorted union — qvb_gather's ids."""
        u = vp()
        _check(_lib().qvb_sample_device(self._h, None, None, C.byref(u)))
        return u.value, self.info().unique_count

    def per_seed(self, seeds) -> list:
        """The reference's BatchSampleResult::per_seed view."""
        nodes, counts, _ = self.arrays()
        out, at = [], 0
        for s, row in zip(seeds, counts):
            fr = []
            for c in row:
                fr.append(nodes[at: at + int(c)])
                at += int(c)
            out.append(SampleResult(int(s), fr, [int(c) for c in row],
                                    np.unique(np.concatenate(fr)) if fr else np.zeros(0, np.uint64)))
        return out

    def close(self):
        if self._h:
            _lib().qvb_sample_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Sampler:
    """Device-resident sampling candidates (qvb_sampler) of an out-CSR."""

    def __init__(self, handle: int):
        self._h = handle

    @classmethod
    def upload(cls, row_offsets, col, weights=None, device: int = 0, stream=None):
        ro = np.ascontiguousarray(row_offsets, np.uint64)
        c = np.ascontiguousarray(col, np.uint64)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        h = vp()
        _check(_lib().qvb_sampler_create(device, len(ro) - 1, len(c), _ptr(ro), _ptr(c) if len(c) else None,
                                         _ptr(w) if w is not None and len(w) else None,
                                         _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    @classmethod
    def synthetic(cls, n: int, e: int, seed: int = 7, weighted: bool = False,
                  transposed: bool = False, device: int = 0, stream=None):
        h = vp()
        _check(_lib().qvb_sampler_synthetic(device, n, e, seed, int(weighted), int(transposed),
                                            _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    def info(self) -> SamplerInfo:
        i = SamplerInfo()
        _check(_lib().qvb_sampler_info_get(self._h, C.byref(i)))
        return i

    def batch_sample(self, seeds, fanouts, rng_seed: int, stream=None) -> BatchSample:
        """qv::batch_sample(t, seeds, SamplingConfig{fanouts}, rng_seed). ``seeds``:
        host numpy array or device tensor of uint64/int64 node ids."""
        f = np.ascontiguousarray(fanouts, np.uint32)
        on_dev = 0
        if isinstance(seeds, np.ndarray) or isinstance(seeds, (list, tuple)):
            sd = np.ascontiguousarray(seeds, np.uint64)
            n = len(sd)
        else:
            sd, on_dev, n = seeds, 1, int(seeds.numel())
        h = vp()
        _check(_lib().qvb_batch_sample(self._h, _ptr(sd) if n else None, n, on_dev,
                                       _ptr(f) if len(f) else None, len(f), rng_seed,
                                       _stream_ptr(stream), C.byref(h)))
        return BatchSample(h.value)

    def close(self):
        if self._h:
            _lib().qvb_sampler_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def batch_sample(row_offsets, col, weights, seeds, fanouts, rng_seed: int, device: int = 0):
    """One-shot qv::batch_sample from a host out-CSR -> (nodes, counts, unique)."""
    with Sampler.upload(row_offsets, col, weights, device=device) as s:
        r = s.batch_sample(seeds, fanouts, rng_seed)
        try:
            return r.arrays()
        finally:
            r.close()


def test_log1p(x, device: int = 0) -> np.ndarray:
    """Device glibc-log1p restatement (test entry point)."""
    a = np.ascontiguousarray(x, np.float64)
    out = np.zeros(max(len(a), 1), np.float64)
    _check(_lib().qvb_test_log1p(device, _ptr(a), len(a), _ptr(out)))
    return out[: len(a)]
