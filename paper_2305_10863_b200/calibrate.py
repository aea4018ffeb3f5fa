"""Calibrate the reference's fetch-cost link model from measured B200 gathers
(model: placement.cpp:269-302,382-404, defaults
topology.cpp:27-40).

The reference costs a collect per location as
    setup_latency + bytes / bandwidth (+ tlb_penalty * page transitions)
with hand-set LinkSpec values. Here the `local` (HBM) and `pcie` (host
zero-copy) links are measured with the real gather kernel: latency from a
1-row gather, bandwidth from a large batch. NVLink cannot be measured on one
GPU; it keeps the pool's measured peer-copy figure (770 GB/s per direction,
B200_PROFILING.md) unless `nvlink_Bps` is given.
"""
from __future__ import annotations

import numpy as np

from . import qvb

NVLINK_MEASURED_BPS = 770e9


def _time_gather(store, ids_dev, out, reps: int = 20) -> float:
    import torch

    s = torch.cuda.current_stream()
    for _ in range(3):
        store.gather(ids_dev, out, stream=s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        store.gather(ids_dev, out, stream=s)
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def measure_link(tier: str, n: int = 1 << 20, dim: int = 128, batch: int = 1 << 20,
                 device: int = 0):
    """(latency_s, bandwidth_Bps) of gathering `dim`-float rows that live on
    `tier` ('local' HBM or 'pcie' = pinned host memory, zero-copy)."""
    import torch

    t = qvb.Topology.with_defaults(gpus_per_server=1,
                                   gpu_feature_capacity=n if tier == "local" else 0,
                                   host_feature_capacity=n)
    lo, ids = qvb.plan_placement(np.arange(n, 0, -1, dtype=np.float64), t, device=device)
    store = qvb.FeatureStore(lo, ids, dim, t, reader=0, device=device)
    try:
        dev = torch.device("cuda", device)
        one = torch.zeros(1, dtype=torch.int64, device=dev)
        out1 = torch.empty((1, dim), dtype=torch.float32, device=dev)
        lat = _time_gather(store, one, out1)
        big = torch.empty(batch, dtype=torch.int64, device=dev)
        qvb.request_ids_synthetic(11, 0, n, big, device=device)
        outb = torch.empty((batch, dim), dtype=torch.float32, device=dev)
        tb = _time_gather(store, big, outb, reps=5)
        bw = batch * dim * 4 / max(tb - lat, 1e-9)
        return lat, bw
    finally:
        store.close()


def calibrated_topology(base: qvb.Topology | None = None, device: int = 0,
                        nvlink_Bps: float | None = None) -> qvb.Topology:
    """A ClusterTopology whose local / nvlink / pcie LinkSpecs come from
    measurements on this GPU (others keep the reference defaults)."""
    t = base if base is not None else qvb.Topology.with_defaults()
    lat, bw = measure_link("local", device=device)
    t.link_latency_s[qvb.LINK_LOCAL] = lat
    t.link_bandwidth_Bps[qvb.LINK_LOCAL] = bw
    lat, bw = measure_link("pcie", batch=1 << 18, device=device)
    t.link_latency_s[qvb.LINK_PCIE] = lat
    t.link_bandwidth_Bps[qvb.LINK_PCIE] = bw
    t.link_bandwidth_Bps[qvb.LINK_NVLINK] = nvlink_Bps or NVLINK_MEASURED_BPS
    return t


def fetch_cost(groups, topo: qvb.Topology, feature_bytes: int, reader_device: int = 0,
               home_server: int = 0) -> float:
    """The reference's fetch_cost model (placement.cpp:382-404) over a flat
    read plan groups = (group_loc, group_count, group_transitions), through
    the library's qvb_fetch_cost."""
    return qvb.fetch_cost(groups, topo, feature_bytes, reader_server=home_server,
                          reader_device=reader_device)[0]
