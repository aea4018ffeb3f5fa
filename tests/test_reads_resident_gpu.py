"""K4 on a resident lookup table: the per-batch read plan of the serving loop
(simulator.cpp:320-321) over the table a FeatureStore (or the caller) keeps in
HBM — no per-call table upload — equal to the reference's plan_reads
(placement.cpp:355-380) through the oracle restatement pinned to it.
"""
import numpy as np
import pytest

from tests.test_gather_gpu import plan
from tests.test_placement_gpu import otopo_from

pytestmark = pytest.mark.gpu


def same(a, b):
    return len(a) == len(b) and all((np.asarray(x) == np.asarray(y)).all() for x, y in zip(a, b))


@pytest.mark.parametrize("gpus,rep,host", [(1, 0, None), (4, 100, 3000), (8, 0, 1000)])
def test_store_plan_reads_matches_reference_plan(qvb, oracle, gpus, rep, host):
    import torch

    n = 20000
    t, lo, ids = plan(qvb, n, gpus=gpus, cap=n // gpus // 2 + rep if gpus > 1 else n, rep=rep,
                      host=n if host is None else host + n)
    ot = otopo_from(t)
    for reader in sorted({0, gpus - 1}):
        st = qvb.FeatureStore(lo, ids, 16, t, reader=reader, device=0)
        loc, off = oracle.build_lookup_table(lo, ids, ot, 0, reader)
        for k, (b, page) in enumerate([(1, 8), (777, 1), (5000, 8), (65536, 3)]):
            req = oracle.request_ids(11, 40 + k, n, b)
            exp = oracle.plan_reads(loc, off, req, page)
            assert same(st.plan_reads(req, page), exp)
            d = torch.from_numpy(req.view(np.int64)).cuda()
            assert same(st.plan_reads(d, page), exp)
            dl = torch.from_numpy(loc).cuda()
            do = torch.from_numpy(off.view(np.int64)).cuda()
            assert same(qvb.plan_reads_device(dl, do, d, page), exp)
        st.close()


def test_resident_plan_errors(qvb, oracle):
    import torch

    n = 1000
    t, lo, ids = plan(qvb, n)
    st = qvb.FeatureStore(lo, ids, 8, t, reader=0)
    with pytest.raises(qvb.ValidationError, match="page size"):
        st.plan_reads(np.array([1, 2], np.uint64), 0)
    with pytest.raises(qvb.ValidationError, match="feature id 1000 outside lookup table"):
        st.plan_reads(np.array([3, 1000, 1001], np.uint64), 8)
    d = torch.tensor([5, 7, 5000], dtype=torch.int64, device="cuda")
    with pytest.raises(qvb.ValidationError, match="feature id 5000 outside lookup table"):
        st.plan_reads(d, 8)
    assert [len(x) for x in st.plan_reads(np.zeros(0, np.uint64))] == [0, 0, 0, 0]
    st.close()


def test_resident_plan_c2_full_batch(qvb, oracle):
    """C2 table (2.4M features), a 1M-id batch: identical to the oracle."""
    from tests.util import CONFIGS

    n = CONFIGS["C2"]["n"]
    t = qvb.Topology.with_defaults(gpus_per_server=1, gpu_feature_capacity=n, host_feature_capacity=n)
    v = np.random.default_rng(2).random(n)
    lo, ids = qvb.plan_placement(v, t)
    st = qvb.FeatureStore(lo, ids, 4, t, reader=0)
    loc, off = qvb.build_lookup_table(lo, ids, t, 0)
    req = oracle.request_ids(11, 0, n, 1 << 20)
    assert same(st.plan_reads(req, 8), oracle.plan_reads(loc, off, req, 8))
    st.close()
