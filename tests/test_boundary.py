"""CPU: the C-ABI library loads, exports exactly what include/qvb.h declares,
and its pure-host helpers agree with the reference (no compute without a GPU).
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def q():
    from paper_2305_10863_b200 import build

    build.build()
    from paper_2305_10863_b200 import qvb

    return qvb


def declared():
    import glob

    src = "".join(open(p).read() for p in glob.glob(os.path.join(ROOT, "include", "*.h")))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qvb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ["qvb_graph_upload", "qvb_access_prob", "qvb_compute_access_prob_ie",
                 "qvb_rank_desc", "qvb_plan_placement", "qvb_build_lookup_table",
                 "qvb_plan_reads", "qvb_page_transitions", "qvb_store_create", "qvb_gather",
                 "qvb_gather_host", "qvb_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(q):
    lib = ctypes.CDLL(q.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(q.exported_symbols()) == declared()


def test_library_is_sm100a(q):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", q.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_host_helpers(q, ref):
    t = q.Topology.with_defaults()
    rt = ref.topology_defaults()
    assert list(t.link_bandwidth_Bps) == list(rt.link_bandwidth_Bps)
    assert list(t.link_latency_s) == list(rt.link_latency_s)
    assert t.tlb_miss_penalty_s == rt.tlb_miss_penalty_s
    t = q.Topology.with_defaults(servers=2, gpus_per_server=4, numa_per_server=2)
    assert q.encode_location(t, 1, q.TIER_HOST, 0) == 10
    assert q.decode_location(t, 11) == (1, q.TIER_DISK, 0)
    assert q.decode_location(t, 7) == (1, q.TIER_GPU, 1)
    bad = q.Topology.with_defaults(gpus_per_server=3, numa_per_server=2)
    with pytest.raises(q.ValidationError, match="divisible"):
        bad.validate()
    assert q.page_transitions([2, 10, 3, 11], 2) == 4
    assert q.page_transitions([2, 3, 10, 11], 2) == 2
    assert q.page_transitions([], 2) == 0
    with pytest.raises(q.ValidationError):
        q.page_transitions([1], 0)


def test_no_cpu_fallback(q):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(q.CudaError):
        q.compute_access_prob_ie(np.array([0, 1, 1], np.uint64), np.array([1], np.uint64), None, 2)
    with pytest.raises(q.CudaError):
        q.device_count()


def test_fetch_cost_and_classify_match_reference(q):
    """The reference's cost model through the C-ABI (host arithmetic, runs on
    CPU) against the unmodified reference (oracle/_ref) on random topologies,
    every location, every reader tier, random flattened plans."""
    from oracle.oracle import RefLib
    from tests.util import derive_stream

    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    ref = RefLib()
    rng = derive_stream(191, 1)
    for _ in range(40):
        t = q.Topology.with_defaults(servers=1 + rng.below(3), numa_per_server=1 + rng.below(2))
        t.gpus_per_server = t.numa_per_server * rng.below(4)
        t.nvlink_within_numa = rng.below(2)
        t.infiniband = rng.below(2)
        for i in range(7):
            t.link_latency_s[i] = rng.uniform() * 1e-5
            t.link_bandwidth_Bps[i] = 1e9 + rng.uniform() * 1e12
        t.tlb_miss_penalty_s = rng.uniform() * 1e-6
        ot = ref.topology_defaults()
        for f, _ in q.Topology._fields_:
            if f.startswith("link_"):
                for i in range(7):
                    getattr(ot, f)[i] = getattr(t, f)[i]
            else:
                setattr(ot, f, getattr(t, f))
        nloc = t.servers * (t.gpus_per_server + 2)
        for rs in range(t.servers):
            for rtier in (q.TIER_GPU, q.TIER_HOST):
                rdev = rng.below(max(1, t.gpus_per_server))
                for loc in range(nloc):
                    assert q.classify_link(t, loc, rs, rtier, rdev) == ref.classify_link(ot, loc, rs, rtier, rdev)
                k = 1 + rng.below(nloc)
                groups = (list(range(nloc))[:k], [rng.below(5000) for _ in range(k)],
                          [rng.below(300) for _ in range(k)])
                a = q.fetch_cost(groups, t, 400, rs, rtier, rdev)
                b = ref.fetch_cost(groups, ot, 400, rs, rtier, rdev)
                assert a[0] == b[0] and (a[1] == b[1]).all()
    with pytest.raises(q.ValidationError, match="unknown location id"):
        q.fetch_cost(([99], [1], [1]), q.Topology.with_defaults(), 512)
