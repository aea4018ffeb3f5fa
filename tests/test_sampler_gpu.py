"""K0 sampler on the GPU vs the reference goldens
and the oracle, instance for instance (sampler.cpp:21-149, test_sampler.cpp)."""
import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

from tests.util import CONFIGS, derive_stream, fig8_edges, random_edges

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
S = GOLD["sampler"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def check(qvb, ro, col, ww, ent, weighted=True):
    nodes, counts, uniq = qvb.batch_sample(ro, col, ww if weighted else None,
                                           np.array(ent["seeds"], np.uint64), ent["fanouts"],
                                           ent["rng_seed"])
    assert nodes.tolist() == ent["nodes"]
    assert counts.tolist() == (ent["counts"] if ent["seeds"] else [])
    assert uniq.tolist() == ent["unique"]


def test_log1p_matches_glibc(qvb):
    """The device log1p restatement equals the host glibc log1p the reference
    calls (rng.hpp:38), on the inputs the sampler feeds it and the branch edges."""
    libm = ctypes.CDLL("libm.so.6")
    libm.log1p.restype = ctypes.c_double
    libm.log1p.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(5)
    u = (rng.integers(0, 1 << 53, 200_000, dtype=np.uint64) >> np.uint64(0)).astype(np.float64) * 2.0 ** -53
    edge = np.array([0.0, 1e-300, 1e-20, 1e-17, 1e-10, 1e-9, 0.5, 0.99999999, 0.2928, 0.29289,
                     0.29290, 0.41, 1.0 - 2.0 ** -53, 2.0 ** -20, 2.0 ** -21, 2.0 ** -29, 2.0 ** -54])
    x = -np.concatenate([u, u * 1e-3, u * 1e-7, edge])
    got = qvb.test_log1p(x)
    exp = np.array([libm.log1p(float(v)) for v in x])
    bad = np.nonzero(got.view(np.uint64) != exp.view(np.uint64))[0]
    assert bad.size == 0, [(x[i], got[i], exp[i]) for i in bad[:5]]


def test_sampler_goldens(qvb, oracle):
    n, s, d, w = fig8_edges()
    ro, col, ww = oracle.build_csr(n, s, d, w)
    for name in ("fig8_full", "fig8_batch", "fig8_dup", "fig8_empty"):
        check(qvb, ro, col, ww, S[name], weighted=False)
    ro, col, ww = oracle.build_csr(3, [0, 1], [1, 2], [1.0, 1.0])
    check(qvb, ro, col, ww, S["chain3"])
    ro, col, ww = oracle.build_csr(3, [0, 0, 0, 0], [1, 1, 1, 2], [1.0] * 4)
    for ent in S["parallel"]:
        check(qvb, ro, col, ww, ent, weighted=False)
    for ent in S["random"]:
        n, s, d, w = ent["edges"]
        ro, col, ww = oracle.build_csr(n, s, d, w)
        check(qvb, ro, col, ww, ent)


@pytest.mark.parametrize("weighted", [False, True])
def test_sampler_c1_bench_golden(qvb, weighted):
    """qv_bench's batch_sample(4096 seeds, {15, 10}, 3) (tools/bench.cpp:89-94)."""
    c = CONFIGS["C1"]
    g = S["c1_bench"]["weighted" if weighted else "uniform"]
    with qvb.Sampler.synthetic(c["n"], c["e"], 7, weighted) as smp:
        st = derive_stream(11, 0x5EED)
        seeds = np.array([st.below(c["n"]) for _ in range(4096)], np.uint64)
        r = smp.batch_sample(seeds, [15, 10], 3)
        nodes, counts, uniq = r.arrays()
        assert (len(nodes), len(uniq)) == (g["total"], g["unique"])
        assert (sha(nodes), sha(counts), sha(uniq)) == (g["nodes_sha256"], g["counts_sha256"],
                                                         g["unique_sha256"])
        r.close()


@pytest.mark.parametrize("weighted", [False, True])
def test_sampler_random_vs_oracle(qvb, oracle, weighted):
    rng = derive_stream(211, int(weighted))
    for it in range(40):
        n, s, d, w = random_edges(rng, 80, 900, weighted)
        ro, col, ww = oracle.build_csr(n, s, d, w)
        if weighted and it % 3 == 1:  # zero-weight candidates inside positive rows
            ww = ww.copy()
            ww[::3] = 0.0
            for i in range(n):
                a, b = int(ro[i]), int(ro[i + 1])
                if b > a and not (ww[a:b] > 0).any():
                    ww[a] = 1.0
        seeds = np.array([rng.below(n) for _ in range(40)], np.uint64)
        fan = [1 + rng.below(6) for _ in range(1 + rng.below(3))]
        got = qvb.batch_sample(ro, col, ww if weighted else None, seeds, fan, 77 + it)
        exp = oracle.batch_sample(ro, col, ww, seeds, fan, 77 + it)
        for x, y in zip(got, exp):
            assert x.tolist() == y.tolist(), (it, fan)


def test_sampler_long_rows_vs_oracle(qvb, oracle):
    """Rows of 33..256 candidates (register radix select) and > 256 (scratch
    slabs), with ties impossible to avoid only by luck: many equal weights."""
    rng = derive_stream(223, 1)
    n = 3000
    src, dst, w = [], [], []
    for i in range(60):  # hub rows of 40..2000 out-edges, some parallel
        deg = 40 + rng.below(2000)
        for _ in range(deg):
            src.append(i)
            dst.append(rng.below(n))
            w.append(float(1 + rng.below(3)))
    for _ in range(20000):
        src.append(rng.below(n))
        dst.append(rng.below(60) if rng.below(2) else rng.below(n))
        w.append(0.5 + rng.uniform())
    ro, col, ww = oracle.build_csr(n, src, dst, w)
    seeds = np.array([rng.below(60) for _ in range(300)] + [rng.below(n) for _ in range(300)],
                     np.uint64)
    for fan in ([25, 10], [100, 3], [7, 7, 7]):
        for weighted in (True, False):
            got = qvb.batch_sample(ro, col, ww if weighted else None, seeds, fan, 5)
            exp = oracle.batch_sample(ro, col, ww if weighted else np.ones_like(ww), seeds, fan, 5)
            for x, y in zip(got, exp):
                assert x.tolist() == y.tolist(), (fan, weighted)


def test_sampler_concurrent_threads(qvb, oracle):
    """batch_sample from several threads on one sampler, each on its own
    stream, over a graph with long rows (shared scratch slabs and side
    stream): every batch equals the serial one."""
    import threading

    import torch

    rng = derive_stream(224, 1)
    n = 3000
    src, dst, w = [], [], []
    for i in range(40):
        for _ in range(300 + rng.below(1500)):
            src.append(i)
            dst.append(rng.below(n))
            w.append(0.5 + rng.uniform())
    for _ in range(20000):
        src.append(rng.below(n))
        dst.append(rng.below(n))
        w.append(0.5 + rng.uniform())
    ro, col, ww = oracle.build_csr(n, src, dst, w)
    seeds = np.array([rng.below(40) for _ in range(200)] + [rng.below(n) for _ in range(200)], np.uint64)
    with qvb.Sampler.upload(ro, col, ww) as sp:
        def one(seed, stream=None):
            r = sp.batch_sample(seeds, [20, 5], seed, stream=stream)
            try:
                return [a.tolist() for a in r.arrays()]
            finally:
                r.close()

        exp = {k: one(k) for k in range(8)}
        bad = []

        def work(tid):
            st = torch.cuda.Stream()
            for k in range(8):
                if one((k + tid) % 8, st) != exp[(k + tid) % 8]:
                    bad.append((tid, k))

        th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
        for h in th:
            h.start()
        for h in th:
            h.join()
    assert not bad


def test_sampler_c2_vs_oracle(qvb, oracle):
    """Full-size C2 graph (hubs of 40K out-edges), 8192 seeds, {15, 10}."""
    c = CONFIGS["C2"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, False)
    seeds = oracle.request_ids(11, 0, c["n"], 8192)
    seeds[:4] = np.arange(4, dtype=np.uint64)  # the longest rows
    with qvb.Sampler.synthetic(c["n"], c["e"], 7, False) as smp:
        info = smp.info()
        assert info.parallel_edges and info.candidates < len(col) and info.max_candidates > 256
        r = smp.batch_sample(seeds, [15, 10], 3)
        got = r.arrays()
        r.close()
    exp = oracle.batch_sample(ro, col, w, seeds, [15, 10], 3)
    for x, y in zip(got, exp):
        assert (x == y).all()


def test_sampler_properties_and_device_seeds(qvb, oracle):
    import torch

    n, s, d, w = fig8_edges()
    ro, col, ww = oracle.build_csr(n, s, d, w)
    with qvb.Sampler.upload(ro, col, None) as smp:
        # order independence and duplicate seeds (test_sampler.cpp:118-130)
        ra = smp.batch_sample(np.array([1, 3, 4], np.uint64), [2, 2], 11).per_seed([1, 3, 4])
        rb = smp.batch_sample(np.array([4, 1, 3], np.uint64), [2, 2], 11).per_seed([4, 1, 3])
        assert [f.tolist() for f in ra[1].frontiers] == [f.tolist() for f in rb[2].frontiers]
        dev = torch.tensor([0, 0, 3, 0], dtype=torch.int64, device="cuda")
        rd = smp.batch_sample(dev, [2, 2], 7)
        host = smp.batch_sample(np.array([0, 0, 3, 0], np.uint64), [2, 2], 7)
        for x, y in zip(rd.arrays(), host.arrays()):
            assert (x == y).all()
        ptr, cnt = rd.device_unique()
        assert ptr and cnt == len(rd.arrays()[2])


def test_sampler_marginals(qvb, oracle):
    """Fanout-1 marginals follow the transition probabilities (test_sampler.cpp:82-96)."""
    ro, col, ww = oracle.build_csr(3, [0, 0], [1, 2], [1.0, 3.0])
    with qvb.Sampler.upload(ro, col, ww) as smp:
        trials = 2000
        seeds = np.zeros(1, np.uint64)
        took1 = sum(int(smp.batch_sample(seeds, [1], 1000 + i).arrays()[0][1] == 1)
                    for i in range(trials))
        assert abs(took1 / trials - 0.25) < 3 * np.sqrt(0.25 * 0.75 / trials)


def test_sampler_errors(qvb, oracle):
    ro, col, ww = oracle.build_csr(3, [0, 1], [1, 2], [1.0, 1.0])
    with qvb.Sampler.upload(ro, col, ww) as smp:
        with pytest.raises(qvb.ValidationError, match="position 1"):
            smp.batch_sample(np.array([0, 7], np.uint64), [1], 1)
        with pytest.raises(qvb.ValidationError, match=">= 1 hop"):
            smp.batch_sample(np.array([0], np.uint64), [], 1)
        with pytest.raises(qvb.ValidationError, match="fanouts must be"):
            smp.batch_sample(np.array([0], np.uint64), [1, 0], 1)
        import torch

        with pytest.raises(qvb.ValidationError, match=r"position 2 \(node 9\)"):
            smp.batch_sample(torch.tensor([0, 1, 9], dtype=torch.int64, device="cuda"), [1], 1)
    with pytest.raises(qvb.ValidationError, match="all weights are zero"):
        qvb.Sampler.upload(ro, col, np.array([0.0, 1.0]))
