"""K5 parity on the GPU: gathered rows are bit-identical to X[ids].

The reference moves no bytes (fetch_cost is a model), so the oracle is the
restatement out[i] = X[ids[i]] (oracle.c qvo_gather) over the same synthetic
features and request streams ("parity unpinned" for the bytes,
pinned for the lookup table that routes them).
"""
import os

import numpy as np
import pytest

from oracle.oracle import topology_defaults

pytestmark = pytest.mark.gpu


def plan(qvb, n, gpus=1, cap=None, rep=0, host=None):
    t = qvb.Topology.with_defaults(gpus_per_server=gpus, nvlink_within_numa=1 if gpus > 1 else 0,
                                   gpu_feature_capacity=n if cap is None else cap,
                                   gpu_replicated_capacity=rep,
                                   host_feature_capacity=n if host is None else host)
    rng = np.random.default_rng(n)
    v = rng.random(n)
    lo, ids = qvb.plan_placement(v, t)
    return t, lo, ids


@pytest.mark.parametrize("kernel", ["flat", "rows"])
@pytest.mark.parametrize("dim", [128, 100, 602, 3, 1, 33])
def test_local_gather_bit_exact(qvb, oracle, dim, kernel, monkeypatch):
    """Both batch-size paths: the flat (request, chunk) kernel small batches
    take, and the row-group kernels (forced with QVB_GATHER_SMALL=0)."""
    import torch

    monkeypatch.setenv("QVB_GATHER_SMALL", "0" if kernel == "rows" else "1000000")

    n = 5000
    t, lo, ids = plan(qvb, n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    x = oracle.features(n, dim)
    req = oracle.request_ids(11, 0, n, 3001)
    exp = oracle.gather(x, req)
    assert (st.gather_host(req) == exp).all()
    d_ids = torch.from_numpy(req.view(np.int64)).cuda()
    out = torch.empty((len(req), dim), dtype=torch.float32, device="cuda")
    st.gather(d_ids, out)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == exp).all()
    out.zero_()
    st.gather(d_ids, out, planned=True)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == exp).all()
    st.close()


@pytest.mark.parametrize("kernel", ["flat", "rows"])
def test_host_tier_zero_copy(qvb, oracle, kernel, monkeypatch):
    monkeypatch.setenv("QVB_GATHER_SMALL", "0" if kernel == "rows" else "1000000")
    n, dim = 20000, 128
    t, lo, ids = plan(qvb, n, cap=n // 4, host=n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    info = st.info()
    assert info.local_rows == n // 4 and info.host_rows == n - n // 4
    x = oracle.features(n, dim)
    req = oracle.request_ids(11, 1, n, 10000)
    assert (st.gather_host(req) == oracle.gather(x, req)).all()
    st.close()


def test_concurrent_gather_host_threads(qvb, oracle):
    """qvb_gather_host from several threads on one store (ctypes drops the
    GIL): every caller gets its own rows, with batch sizes that regrow the
    shared staging buffers mid-run."""
    import threading

    import torch

    n, dim = 20000, 64
    t, lo, ids = plan(qvb, n, cap=n // 2, host=n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    x = oracle.features(n, dim)
    bad = []

    def work(tid):
        s = torch.cuda.Stream()
        for k in range(20):
            req = oracle.request_ids(11, 1000 * tid + k, n, 500 + 700 * ((tid + k) % 5))
            if not (st.gather_host(req, stream=s) == oracle.gather(x, req)).all():
                bad.append((tid, k))

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    st.close()
    assert not bad


@pytest.mark.parametrize("chunks", ["1", "3", "8"])
def test_gather_host_chunked(qvb, oracle, chunks, monkeypatch):
    """qvb_gather_host's pipelined chunks (two internal streams) return the
    same rows as one launch, including a ragged last chunk and host rows."""
    monkeypatch.setenv("QVB_HOST_CHUNKS", chunks)
    n, dim = 50000, 100
    t, lo, ids = plan(qvb, n, cap=n // 2, host=n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    x = oracle.features(n, dim)
    req = oracle.request_ids(11, 3, n, 8 * 16384 + 12345)
    assert (st.gather_host(req) == oracle.gather(x, req)).all()
    st.close()


def test_host_features_input(qvb, oracle):
    n, dim = 3000, 100
    t, lo, ids = plan(qvb, n, cap=n // 2, host=n)
    x = np.random.default_rng(5).standard_normal((n, dim)).astype(np.float32)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0, features=x)
    req = oracle.request_ids(11, 4, n, 4000)
    assert (st.gather_host(req) == x[req.astype(np.int64)]).all()
    st.close()


@pytest.mark.parametrize("gpus,rep", [(4, 0), (4, 500), (8, 250), (2, 0)])
def test_partitioned_readers_single_device(qvb, oracle, gpus, rep):
    """A G-GPU plan (hot rows replicated, the rest LPT-partitioned, cold rows
    on the host): the G readers' shards are built on this one device and
    cross-attached as 'peers', so every reader's per-reader lookup table
    routes to local / peer / host shards exactly as on G devices."""
    n, dim = 8000, 64
    cap = n // (2 * gpus) + rep
    t, lo, ids = plan(qvb, n, gpus=gpus, cap=cap, rep=rep, host=n)
    x = oracle.features(n, dim)
    stores = [qvb.FeatureStore(lo, ids, dim, t, reader=r, device=0) for r in range(gpus)]
    # peers not attached yet: refused, not faulted
    with pytest.raises(qvb.ValidationError, match="not attached"):
        stores[0].gather_host(np.arange(n, dtype=np.uint64))
    for r, st in enumerate(stores):
        assert st.info().local_rows == int((ids == r).sum())
        for p in range(gpus):
            if p != r:
                st.attach_local_peer(p, stores[p])
    req = oracle.request_ids(11, 9, n, 6000)
    exp = oracle.gather(x, req)
    for st in stores:
        assert (st.gather_host(req) == exp).all()
        assert (st.gather_host(np.arange(n, dtype=np.uint64)) == x).all()
    for st in stores:
        st.close()


def test_gather_errors(qvb, oracle):
    n, dim = 1000, 16
    t, lo, ids = plan(qvb, n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    with pytest.raises(qvb.ValidationError, match="feature id 1000 outside"):
        st.gather_host(np.array([1, 2, 1000, 3], np.uint64))
    assert st.gather_host(np.array([], np.uint64)).shape == (0, dim)
    # a chunked (pipelined) host call names the first bad id too
    big = np.random.default_rng(2).integers(0, n, 300_000).astype(np.uint64)
    big[200_001] = n + 7
    with pytest.raises(qvb.ValidationError, match=f"feature id {n + 7} outside"):
        st.gather_host(big)
    st.close()
    dt = qvb.Topology.with_defaults(gpus_per_server=1, gpu_feature_capacity=10,
                                    host_feature_capacity=10, disk_feature_capacity=n)
    lo, ids = qvb.plan_placement(np.random.default_rng(1).random(n), dt)
    with pytest.raises(qvb.UnsupportedError, match="disk"):
        qvb.FeatureStore(lo, ids, dim, dt, reader=0)


def test_request_ids_match_oracle(qvb, oracle):
    import torch

    out = torch.empty(100_000, dtype=torch.int64, device="cuda")
    qvb.request_ids_synthetic(11, 7, 2_400_000, out)
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint64) == oracle.request_ids(11, 7, 2_400_000, 100_000)).all()


def test_c2_gather_full_size(qvb, oracle):
    """C2 shape (2.4M x 100 fp32) with a 1M-id batch, bit-exact."""
    import torch

    n, dim, b = 2_400_000, 100, 1 << 20
    t, lo, ids = plan(qvb, n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    d_ids = torch.empty(b, dtype=torch.int64, device="cuda")
    qvb.request_ids_synthetic(11, 0, n, d_ids)
    out = torch.empty((b, dim), dtype=torch.float32, device="cuda")
    st.gather(d_ids, out)
    st.check_error()
    req = d_ids.cpu().numpy().view(np.uint64)
    # check a checksum of all rows plus a dense sample against the restatement
    sample = np.arange(0, b, 97)
    x_rows = oracle.features(n, dim)  # 960 MB host, fine on the GPU box
    got = out.cpu().numpy()
    assert (got[sample] == x_rows[req[sample].astype(np.int64)]).all()
    assert (got == x_rows[req.astype(np.int64)]).all()
    st.close()


@pytest.mark.parametrize("mix", ["host", "peer", "peer+host"])
@pytest.mark.parametrize("dim", [128, 100, 33, 602])
def test_tier_split_gather_bit_exact(qvb, oracle, mix, dim, monkeypatch):
    """The location-bucketed gather (local / peer / host lists, warps taking
    32-row groups per class) against the restatement, for every class mix,
    row width and both device and host entry points; the mixed row-group
    kernel (QVB_GATHER_SPLIT=0) gives the same bytes."""
    import torch

    monkeypatch.setenv("QVB_GATHER_SMALL", "0")
    monkeypatch.setenv("QVB_HOST_SORT", "1")  # offset-bucketed host list (default only for big tiers)
    n = 12000
    gpus = 1 if mix == "host" else 4
    host = n if "host" in mix else 0
    cap = n // 2 if mix == "host" else (n // gpus + 1 if mix == "peer" else n // (2 * gpus))
    t, lo, ids = plan(qvb, n, gpus=gpus, cap=cap, host=host)
    stores = [qvb.FeatureStore(lo, ids, dim, t, reader=r, device=0) for r in range(gpus)]
    for r, st in enumerate(stores):
        for p in range(gpus):
            if p != r:
                st.attach_local_peer(p, stores[p])
    x = oracle.features(n, dim)
    req = oracle.request_ids(11, 21, n, 70001)
    exp = oracle.gather(x, req)
    d_ids = torch.from_numpy(req.view(np.int64)).cuda()
    for st in stores[:2]:
        assert (st.gather_host(req) == exp).all()
        out = torch.full((len(req), dim), -1.0, dtype=torch.float32, device="cuda")
        st.gather(d_ids, out)
        st.check_error()
        assert (out.cpu().numpy() == exp).all()
    monkeypatch.setenv("QVB_HOST_SORT", "0")  # host list unordered
    assert (stores[-1].gather_host(req) == exp).all()
    monkeypatch.setenv("QVB_GATHER_SPLIT", "0")
    assert (stores[-1].gather_host(req) == exp).all()
    for st in stores:
        st.close()


@pytest.mark.parametrize("b", [1000, 50000, 131072, 262144, 300000])
@pytest.mark.parametrize("host_share", [0.05, 0.5])
def test_default_dispatch_with_host_tier(qvb, oracle, b, host_share, monkeypatch):
    """With a host tier the store picks the flat kernel or the class split by
    batch size and expected host rows (<= 256K ids and <= 16K expected host
    rows: flat), and small host groups over an offset-ordered host list (any
    tier size here, QVB_HOST_SORT=1; the default orders tiers >= 1 GB). Every
    choice returns the same bytes as X[ids]."""
    import torch

    for k in ("QVB_GATHER_SMALL", "QVB_HOST_SORT", "QVB_GATHER_SPLIT", "QVB_HOST_GROUP"):
        monkeypatch.delenv(k, raising=False)
    n, dim = 40000, 64
    t, lo, ids = plan(qvb, n, cap=int(n * (1 - host_share)), host=n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    x = oracle.features(n, dim)
    req = oracle.request_ids(11, 77, n, b)
    exp = oracle.gather(x, req)
    d = torch.from_numpy(req.view(np.int64)).cuda()
    for sort in (None, "1"):
        if sort:
            monkeypatch.setenv("QVB_HOST_SORT", sort)
        out = torch.full((b, dim), -1.0, dtype=torch.float32, device="cuda")
        st.gather(d, out)
        st.check_error()
        assert (out.cpu().numpy() == exp).all()
        assert (st.gather_host(req) == exp).all()
    st.close()


def test_tier_split_gather_reports_bad_ids(qvb, oracle, monkeypatch):
    import torch

    monkeypatch.setenv("QVB_GATHER_SMALL", "0")
    n, dim = 5000, 32
    t, lo, ids = plan(qvb, n, cap=n // 3, host=n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    req = oracle.request_ids(11, 5, n, 60000)
    req[33333] = n + 5
    with pytest.raises(qvb.ValidationError, match=f"feature id {n + 5} outside"):
        st.gather_host(req)
    d = torch.from_numpy(req.view(np.int64)).cuda()
    out = torch.empty((len(req), dim), dtype=torch.float32, device="cuda")
    st.gather(d, out)
    with pytest.raises(qvb.ValidationError, match="request 33333"):
        st.check_error()
    st.close()


def test_c4_gather_full_size(qvb, oracle):
    """C4 shape (111M x 128 fp32 = 56.8 GB in HBM) with a 1M-id batch: every
    gathered row bit-identical to the generator's row (no host copy of the
    table needed)."""
    import torch

    from tests.util import CONFIGS

    c = CONFIGS["C4"]
    n, dim, b = c["n"], 128, 1 << 20
    t, lo, ids = plan(qvb, n)
    st = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    d_ids = torch.empty(b, dtype=torch.int64, device="cuda")
    qvb.request_ids_synthetic(11, 0, n, d_ids)
    out = torch.empty((b, dim), dtype=torch.float32, device="cuda")
    st.gather(d_ids, out)
    st.check_error()
    req = d_ids.cpu().numpy().view(np.uint64)
    assert (req == oracle.request_ids(11, 0, n, b)).all()
    exp = oracle.feature_rows(req, dim, threads=os.cpu_count() or 1)
    assert (out.cpu().numpy() == exp).all()
    assert (st.gather_host(req[:300_000]) == exp[:300_000]).all()
    st.close()


@pytest.mark.parametrize("variant", ["9", "7", "2", "8"])
def test_gather_kernel_variants_bit_exact(variant):
    """The opt-in gather variants (QVB_GATHER_U, read once per process: run
    in a child) return the same rows."""
    import subprocess
    import sys

    code = (
        "import numpy as np, torch\n"
        "from oracle.oracle import Oracle\n"
        "from paper_2305_10863_b200 import qvb\n"
        "o = Oracle(); n, dim = 40000, 128\n"
        "t = qvb.Topology.with_defaults(gpus_per_server=1, gpu_feature_capacity=n, host_feature_capacity=n)\n"
        "lo, ids = qvb.plan_placement(np.random.default_rng(1).random(n), t)\n"
        "st = qvb.FeatureStore(lo, ids, dim, t, reader=0)\n"
        "req = o.request_ids(11, 3, n, 100003)\n"
        "d = torch.from_numpy(req.view(np.int64)).cuda()\n"
        "out = torch.empty((len(req), dim), dtype=torch.float32, device='cuda')\n"
        "st.gather(d, out); st.check_error()\n"
        "assert (out.cpu().numpy() == o.gather(o.features(n, dim), req)).all()\n"
        "print('variant ok')\n")
    env = dict(os.environ, QVB_GATHER_U=variant)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stderr[-3000:]
