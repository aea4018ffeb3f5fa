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
