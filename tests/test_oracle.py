"""CPU: pin the oracle restatement (oracle/oracle.c) to the reference.

Every check compares the restatement with tests/golden/golden.json, which
tests/golden/make_golden.py produced by running the UNMODIFIED reference
(oracle/_ref). Where the reference library is built (this container) the
restatement is also compared with it directly on fresh random inputs.
"""
import hashlib
import itertools
import json
import os

import numpy as np
import pytest

from oracle.oracle import topology_defaults
from tests.util import bits, derive_stream, fig8_edges, random_edges

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def topo(d, mod):
    t = mod()
    for k, v in d.items():
        if k.startswith("link_"):
            arr = getattr(t, k)
            for i, x in enumerate(v):
                arr[i] = x
        else:
            setattr(t, k, v)
    return t


def otopo(d):
    return topo(d, lambda: topology_defaults())


def hexs(a):
    return [f"{int(x):016x}" for x in bits(a)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_fig8_golden(oracle):
    n, s, d, w = fig8_edges()
    ro, col, ww = oracle.build_csr(n, s, d, w)
    for L, gold in GOLD["fig8"].items():
        assert hexs(oracle.access_prob(ro, col, ww, int(L))) == gold


@pytest.mark.parametrize("name,weighted,transposed,layers", [("uniform_L2", False, False, 2),
                                                             ("uniform_L3", False, False, 3),
                                                             ("weighted_L3", True, False, 3),
                                                             ("transposed_L3", False, True, 3)])
def test_c1_golden(oracle, name, weighted, transposed, layers):
    ro, col, w = oracle.synthetic_graph(100_000, 1_000_000, 7, weighted, transposed)
    g = GOLD["c1"][name]
    assert sha(np.concatenate([ro.view(np.uint8), col.view(np.uint8), w.view(np.uint8)])) == \
        g["graph_sha256"]
    p = oracle.access_prob(ro, col, w, layers)
    assert sha(p) == g["sha256"]
    if "placement8" in g:
        t = otopo(g["placement8"]["topology"])
        lo, ids = oracle.plan_placement(p, t)
        assert sha(np.concatenate([lo.view(np.uint8), ids.view(np.uint8)])) == \
            g["placement8"]["plan_sha256"]
        loc, off = oracle.build_lookup_table(lo, ids, t)
        assert sha(np.concatenate([loc.view(np.uint8), off.view(np.uint8)])) == \
            g["placement8"]["lut_sha256"]
        gl, gc, gt, oo = oracle.plan_reads(loc, off, oracle.request_ids(11, 0, 100_000, 4096), 8)
        rd = g["placement8"]["reads"]
        assert gl.tolist() == rd["group_loc"] and gc.tolist() == rd["group_count"]
        assert gt.tolist() == rd["group_transitions"] and sha(oo) == rd["offsets_sha256"]


@pytest.mark.parametrize("name", ["a", "b", "c", "d", "closest_replica"])
def test_scenarios_golden(oracle, name):
    g = GOLD["scenarios"][name]
    t = otopo(g["topology"])
    lo, ids = oracle.plan_placement(np.array([0.5, 0.4, 0.3, 0.2, 0.1]), t)
    assert lo.tolist() == g["loc_offsets"] and ids.tolist() == g["loc_ids"]
    loc, off = oracle.build_lookup_table(lo, ids, t, 0)
    assert loc.tolist() == g["lut_loc"] and off.tolist() == g["lut_off"]
    got = [x.tolist() for x in oracle.plan_reads(loc, off, [4, 1, 0, 3, 1], 2)]
    assert got == g["reads_41031_p2"]


def test_short_by_3(oracle):
    g = GOLD["short_by_3"]
    with pytest.raises(Exception) as ei:
        oracle.plan_placement(np.array([0.5, 0.4, 0.3, 0.2, 0.1]), otopo(g["topology"]))
    assert ei.value.code == 3 and ei.value.msg == g["msg"]


def test_random_placements_golden(oracle):
    for ent in GOLD["random_placements"]:
        t = otopo(ent["topology"])
        v = np.array(ent["values"])
        if "error" in ent:
            with pytest.raises(Exception) as ei:
                oracle.plan_placement(v, t)
            assert ei.value.code == ent["error"]["code"] and ei.value.msg == ent["error"]["msg"]
            continue
        lo, ids = oracle.plan_placement(v, t)
        assert lo.tolist() == ent["loc_offsets"] and ids.tolist() == ent["loc_ids"]
        for home, (gl, go) in ent["luts"].items():
            loc, off = oracle.build_lookup_table(lo, ids, t, int(home))
            assert loc.tolist() == gl and off.tolist() == go


def test_page_transitions_golden(oracle):
    for offs, page, exp in GOLD["page_transitions"]:
        assert oracle.page_transitions(np.array(offs, np.uint64), page) == exp


def test_sorted_order_minimal(oracle):
    # acceptance.cpp:280-321 / test_placement.cpp:293-317
    rng = derive_stream(113, 4)
    for _ in range(25):
        count = 1 + rng.below(7)
        offs = [rng.below(16) for _ in range(count)]
        page = 1 + rng.below(4)
        planned = oracle.page_transitions(np.array(sorted(offs), np.uint64), page)
        best = min(oracle.page_transitions(np.array(p, np.uint64), page)
                   for p in set(itertools.permutations(offs)))
        assert planned == best == len({o // page for o in offs})


def test_restatement_matches_reference_random(oracle, ref):
    rng = derive_stream(59, 5)
    for it in range(30):
        n, s, d, w = random_edges(rng, 40, 250, it % 2 == 0)
        ro, col, ww = oracle.build_csr(n, s, d, w)
        tro, tcol, tw = oracle.in_adjacency(ro, col, ww)
        rro, rcol, rw = ref.in_adjacency(ro, col, ww)
        assert (tro == rro).all() and (tcol == rcol).all() and (bits(tw) == bits(rw)).all()
        assert (bits(oracle.row_sums(ro, ww)) == bits(ref.row_sums(ro, col, ww))).all()
        for L in range(1, 5):
            assert (bits(oracle.access_prob(ro, col, ww, L)) ==
                    bits(ref.access_prob(ro, col, ww, L))).all()


def test_restatement_matches_reference_placement_replicas(oracle, ref):
    # reader 0 of every home server, all random topologies incl. 8-GPU NVLink
    rng = derive_stream(131, 7)
    for _ in range(30):
        n = 1 + rng.below(300)
        v = np.array([float(rng.below(8)) / 8 for _ in range(n)])  # many exact ties
        t = topology_defaults(servers=1 + rng.below(2), numa_per_server=1 + rng.below(2))
        t.gpus_per_server = t.numa_per_server * (1 + rng.below(4))
        t.gpu_feature_capacity = rng.below(40)
        t.host_feature_capacity = rng.below(100)
        t.disk_feature_capacity = n
        t.nvlink_within_numa = rng.below(2)
        t.infiniband = rng.below(2)
        lo, ids = oracle.plan_placement(v, t)
        lo2, ids2 = ref.plan_placement(v, t)
        assert (lo == lo2).all() and (ids == ids2).all()
        for home in range(t.servers):
            a = oracle.build_lookup_table(lo, ids, t, home)
            b = ref.build_lookup_table(lo, ids, t, home)
            assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        req = np.array([rng.below(n) for _ in range(50)], np.uint64)
        for x, y in zip(oracle.plan_reads(a[0], a[1], req, 3), ref.plan_reads(a[0], a[1], req, 3)):
            assert (x == y).all()


def test_replication_extension_reduces_to_reference(oracle):
    # gpu_replicated_capacity = 0 is the reference; = N_g equals no-NVLink
    # full replication of the hottest N_g.
    rng = derive_stream(137, 1)
    v = np.array([rng.uniform() for _ in range(200)])
    base = dict(gpus_per_server=4, gpu_feature_capacity=10, host_feature_capacity=300,
                nvlink_within_numa=1)
    full = oracle.plan_placement(v, topology_defaults(**base, gpu_replicated_capacity=10))
    nonv = oracle.plan_placement(v, topology_defaults(**dict(base, nvlink_within_numa=0)))
    assert (full[0] == nonv[0]).all() and (full[1] == nonv[1]).all()
    part = oracle.plan_placement(v, topology_defaults(**base, gpu_replicated_capacity=4))
    ranks = oracle.rank_desc(v)
    lo, ids = part
    for r, f in enumerate(ranks):
        cp = ids[lo[f]:lo[f + 1]].tolist()
        if r < 4:
            assert cp == [0, 1, 2, 3]
        elif r < 4 + 4 * 6:
            assert len(cp) == 1 and cp[0] < 4
        else:
            assert cp == [4]


def test_gather_restatement(oracle):
    x = oracle.features(1000, 37)
    assert x[3, 5] == np.float32((oracle.splitmix64(3 * 37 + 5) >> 40) * 2.0 ** -24)
    ids = oracle.request_ids(11, 2, 1000, 500)
    s = derive_stream(11, 0x5EED, 2)
    assert ids.tolist() == [s.below(1000) for _ in range(500)]
    out = oracle.gather(x, ids, threads=4)
    assert (out == x[ids.astype(np.int64)]).all()


def test_fap_golden(oracle):
    n, s, d, w = fig8_edges()
    ro, col, ww = oracle.build_csr(n, s, d, w)
    for K, gold in GOLD["fap_fig8"].items():
        assert hexs(oracle.compute_fap(ro, col, ww, int(K))) == gold
    sd = GOLD["fap_fig8_seeded"]
    assert hexs(oracle.compute_fap(ro, col, ww, 2, np.array(sd["seed"]))) == sd["values"]
    # test_metrics.cpp worked example: node 3's visit mass is 1/2 at K=2
    assert abs(oracle.compute_fap(ro, col, ww, 2)[3] - 0.5) < 1e-12
    for name, weighted in [("uniform_K2", False), ("weighted_K3", True)]:
        ro, col, ww = oracle.synthetic_graph(100_000, 1_000_000, 7, weighted, False)
        assert sha(oracle.compute_fap(ro, col, ww, 2 if not weighted else 3)) == GOLD["fap_c1"][name]


def test_fap_matches_reference_random(oracle, ref):
    rng = derive_stream(5, 5)
    for it in range(30):
        n, s, d, w = random_edges(rng, 60, 400, it % 2 == 0)
        ro, col, ww = oracle.build_csr(n, s, d, w)
        seed = None
        if it % 3 == 0:
            x = np.array([rng.uniform() for _ in range(n)])
            seed = x / x.sum()
        for hops in range(4):
            assert (bits(oracle.compute_fap(ro, col, ww, hops, seed)) ==
                    bits(ref.compute_fap(ro, col, ww, hops, seed))).all()
    with pytest.raises(Exception, match="negative mass"):
        oracle.compute_fap(ro, col, ww, 2, -np.ones(len(ro) - 1))
    with pytest.raises(Exception, match="does not sum to 1"):
        oracle.compute_fap(ro, col, ww, 2, np.ones(len(ro) - 1))


# ---- sampler (sampler.cpp:21-149) ---------------------------------------------
def _sample_case(oracle, ro, col, ww, ent):
    nodes, counts, uniq = oracle.batch_sample(ro, col, ww, np.array(ent["seeds"], np.uint64),
                                              ent["fanouts"], ent["rng_seed"])
    assert nodes.tolist() == ent["nodes"]
    assert counts.tolist() == (ent["counts"] if ent["seeds"] else [])
    assert uniq.tolist() == ent["unique"]


def test_sampler_golden(oracle):
    S = GOLD["sampler"]
    n, s, d, w = fig8_edges()
    ro, col, ww = oracle.build_csr(n, s, d, w)
    for name in ("fig8_full", "fig8_batch", "fig8_dup", "fig8_empty"):
        _sample_case(oracle, ro, col, ww, S[name])
    # test_sampler.cpp:15-26: 4 -> 0 -> {3, 5}
    assert S["fig8_full"]["nodes"] == [4, 0, 3, 5]
    ro, col, ww = oracle.build_csr(3, [0, 1], [1, 2], [1.0, 1.0])
    _sample_case(oracle, ro, col, ww, S["chain3"])
    assert S["chain3"]["nodes"] == [0, 1, 2]
    ro, col, ww = oracle.build_csr(3, [0, 0, 0, 0], [1, 1, 1, 2], [1.0] * 4)
    for ent in S["parallel"]:
        _sample_case(oracle, ro, col, ww, ent)
        assert sorted(ent["nodes"][1:]) == [1, 2]  # coalesced: two distinct neighbours
    for ent in S["random"]:
        n, s, d, w = ent["edges"]
        ro, col, ww = oracle.build_csr(n, s, d, w)
        _sample_case(oracle, ro, col, ww, ent)
    for name, weighted in [("uniform", False), ("weighted", True)]:
        ro, col, ww = oracle.synthetic_graph(100_000, 1_000_000, 7, weighted, False)
        seeds = oracle.request_ids(11, 0, 100_000, 4096)
        nodes, counts, uniq = oracle.batch_sample(ro, col, ww, seeds, [15, 10], 3)
        g = S["c1_bench"][name]
        assert (len(nodes), len(uniq)) == (g["total"], g["unique"])
        assert (sha(nodes), sha(counts), sha(uniq)) == (g["nodes_sha256"], g["counts_sha256"],
                                                         g["unique_sha256"])


def test_sampler_matches_reference_random(oracle, ref):
    rng = derive_stream(9, 9)
    for it in range(40):
        n, s, d, w = random_edges(rng, 60, 400, it % 2 == 0)
        ro, col, ww = oracle.build_csr(n, s, d, w)
        if it % 4 == 1:  # zero-weight edges inside positive rows
            ww = ww.copy()
            ww[::3] = 0.0
            ro2 = ro.astype(np.int64)
            for i in range(n):
                a, b = ro2[i], ro2[i + 1]
                if b > a and not (ww[a:b] > 0).any():
                    ww[a] = 1.0
        seeds = np.array([rng.below(n) for _ in range(25)], np.uint64)
        fan = [1 + rng.below(5) for _ in range(1 + rng.below(3))]
        a = oracle.batch_sample(ro, col, ww, seeds, fan, 1000 + it)
        b = ref.batch_sample(ro, col, ww, seeds, fan, 1000 + it)
        for x, y in zip(a, b):
            assert (x == y).all(), it
    with pytest.raises(Exception, match="position 1"):
        oracle.batch_sample(ro, col, ww, np.array([0, 10**6], np.uint64), [1], 1)
    with pytest.raises(Exception, match=">= 1 hop"):
        oracle.batch_sample(ro, col, ww, np.array([0], np.uint64), [], 1)
    with pytest.raises(Exception, match="fanouts must be"):
        oracle.batch_sample(ro, col, ww, np.array([0], np.uint64), [2, 0], 1)


@pytest.mark.parametrize("n,e,weighted,transposed", [(100_000, 1_000_000, False, False),
                                                     (100_000, 1_000_000, True, True),
                                                     (2_000, 300_000, True, False), (3, 50, False, True)])
def test_threaded_generator_matches_sequential(oracle, n, e, weighted, transposed):
    """The threaded bench.cpp generator (used for papers-scale host graphs)
    writes the same CSR bytes as the sequential one, at several thread counts."""
    a = oracle.synthetic_graph(n, e, 7, weighted, transposed)
    for t in (2, 7, 16):
        b = oracle.synthetic_graph(n, e, 7, weighted, transposed, threads=t)
        assert all((x.view(np.uint64) == y.view(np.uint64)).all() for x, y in zip(a, b))
    x = oracle.features(1000, 37, first=5)
    assert (x == oracle.features(1000, 37, first=5, threads=5)).all()


def test_feature_rows_match_table(oracle):
    x = oracle.features(3000, 41)
    ids = oracle.request_ids(5, 1, 3000, 20000)
    assert (oracle.feature_rows(ids, 41, threads=3) == x[ids.astype(np.int64)]).all()
