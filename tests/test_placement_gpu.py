"""K2/K3/K4 parity on the GPU: ranking, placement, lookup table and read plan
against the reference goldens (tests/golden) and the oracle, exactly.

Mirrors tests/test_placement.cpp (scenarios, shortfall, random topologies,
closest replica, dense offsets, locality dominance, read plans).
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import topology_defaults
from tests.util import c4_reference_enabled, CONFIGS, bits, derive_stream

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
FIVE = np.array([0.5, 0.4, 0.3, 0.2, 0.1])


def qtopo(q, d):
    t = q.Topology.with_defaults()
    for k, v in d.items():
        if k.startswith("link_"):
            arr = getattr(t, k)
            for i, x in enumerate(v):
                arr[i] = x
        else:
            setattr(t, k, v)
    return t


def otopo_from(q_t):
    t = topology_defaults()
    for f, _ in q_t._fields_:
        if f.startswith("link_"):
            for i in range(7):
                getattr(t, f)[i] = getattr(q_t, f)[i]
        else:
            setattr(t, f, getattr(q_t, f))
    return t


def test_rank_ties_and_signs(qvb, oracle):
    rng = derive_stream(141, 1)
    for n in (1, 2, 7, 1000, 100_003):
        v = np.array([float(rng.below(50)) / 7 for _ in range(n)])  # heavy ties
        assert (qvb.rank_desc(v) == oracle.rank_desc(v)).all()
    v = np.array([0.0, -0.0, 1.5, -2.0, np.inf, -np.inf, 0.0, 1e-300, -1e-300])
    assert (qvb.rank_desc(v) == oracle.rank_desc(v)).all()
    with pytest.raises(qvb.ValidationError):
        qvb.rank_desc(np.array([1.0, np.nan]))


@pytest.mark.parametrize("name", ["a", "b", "c", "d", "closest_replica"])
def test_scenarios_golden(qvb, name):
    g = GOLD["scenarios"][name]
    t = qtopo(qvb, g["topology"])
    lo, ids = qvb.plan_placement(FIVE, t)
    assert lo.tolist() == g["loc_offsets"] and ids.tolist() == g["loc_ids"]
    loc, off = qvb.build_lookup_table(lo, ids, t, 0)
    assert loc.tolist() == g["lut_loc"] and off.tolist() == g["lut_off"]
    got = [x.tolist() for x in qvb.plan_reads(loc, off, [4, 1, 0, 3, 1], 2)]
    assert got == g["reads_41031_p2"]


def test_shortfall_error(qvb):
    g = GOLD["short_by_3"]
    with pytest.raises(qvb.PlacementError) as ei:
        qvb.plan_placement(FIVE, qtopo(qvb, g["topology"]))
    assert str(ei.value) == g["msg"]


def test_random_placements_golden(qvb):
    for ent in GOLD["random_placements"]:
        t = qtopo(qvb, ent["topology"])
        v = np.array(ent["values"])
        if "error" in ent:
            with pytest.raises(qvb.Error) as ei:
                qvb.plan_placement(v, t)
            assert str(ei.value) == ent["error"]["msg"]
            continue
        lo, ids = qvb.plan_placement(v, t)
        assert lo.tolist() == ent["loc_offsets"] and ids.tolist() == ent["loc_ids"]
        for home, (gl, go) in ent["luts"].items():
            loc, off = qvb.build_lookup_table(lo, ids, t, int(home))
            assert loc.tolist() == gl and off.tolist() == go


def test_random_vs_oracle_with_readers(qvb, oracle):
    rng = derive_stream(149, 2)
    for _ in range(25):
        n = 1 + rng.below(3000)
        v = np.array([float(rng.below(64)) / 64 for _ in range(n)])
        t = qvb.Topology.with_defaults(servers=1 + rng.below(2), numa_per_server=1 + rng.below(2))
        t.gpus_per_server = t.numa_per_server * (1 + rng.below(4))
        t.gpu_feature_capacity = rng.below(400)
        t.gpu_replicated_capacity = rng.below(t.gpu_feature_capacity + 1)
        t.host_feature_capacity = rng.below(1000)
        t.disk_feature_capacity = n
        t.nvlink_within_numa = rng.below(2)
        t.infiniband = rng.below(2)
        ot = otopo_from(t)
        lo, ids = qvb.plan_placement(v, t)
        lo2, ids2 = oracle.plan_placement(v, ot)
        assert (lo == lo2).all() and (ids == ids2).all()
        for home in range(t.servers):
            for reader in range(max(1, t.gpus_per_server)):
                a = qvb.build_lookup_table(lo, ids, t, home, reader)
                b = oracle.build_lookup_table(lo2, ids2, ot, home, reader)
                assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        req = np.array([rng.below(n) for _ in range(777)], np.uint64)
        page = 1 + rng.below(5)
        for x, y in zip(qvb.plan_reads(a[0], a[1], req, page), oracle.plan_reads(b[0], b[1], req, page)):
            assert (x == y).all()


@pytest.mark.parametrize("servers,gpus", [(8, 8), (12, 6), (3, 30)])
def test_lookup_table_beyond_64_locations(qvb, oracle, servers, gpus):
    """S x (G+2) > 64 location ids (e.g. 8 servers x 8 GPUs = 80): the
    any-location K3 path, equal to the reference restatement for every home
    server and a few readers (the mask path stopped at 64)."""
    rng = derive_stream(163, servers * 100 + gpus)
    n = 5000
    v = np.array([float(rng.below(97)) / 97 for _ in range(n)])
    for ib in (0, 1):
        t = qvb.Topology.with_defaults(servers=servers, numa_per_server=2, gpus_per_server=gpus,
                                       gpu_feature_capacity=n // (servers * gpus) + 3,
                                       host_feature_capacity=n // servers + 1,
                                       disk_feature_capacity=n, nvlink_within_numa=1, infiniband=ib)
        ot = otopo_from(t)
        lo, ids = qvb.plan_placement(v, t)
        lo2, ids2 = oracle.plan_placement(v, ot)
        assert (lo == lo2).all() and (ids == ids2).all()
        assert servers * (gpus + 2) > 64
        for home in range(servers):
            for reader in (0, gpus - 1):
                a = qvb.build_lookup_table(lo, ids, t, home, reader)
                b = oracle.build_lookup_table(lo2, ids2, ot, home, reader)
                assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        req = np.array([rng.below(n) for _ in range(4096)], np.uint64)
        for x, y in zip(qvb.plan_reads(a[0], a[1], req, 4), oracle.plan_reads(b[0], b[1], req, 4)):
            assert (x == y).all()


def test_lookup_table_general_path_matches_mask_path(qvb, oracle, monkeypatch):
    """The any-location K3 path forced on small topologies (QVB_LUT_GENERAL=1)
    gives the same tables as the mask path and the oracle."""
    rng = derive_stream(167, 3)
    for _ in range(12):
        n = 1 + rng.below(4000)
        v = np.array([float(rng.below(64)) / 64 for _ in range(n)])
        t = qvb.Topology.with_defaults(servers=1 + rng.below(3), numa_per_server=1 + rng.below(2))
        t.gpus_per_server = t.numa_per_server * (1 + rng.below(4))
        t.gpu_feature_capacity = rng.below(600)
        t.host_feature_capacity = rng.below(2000)
        t.disk_feature_capacity = n
        t.nvlink_within_numa = rng.below(2)
        t.infiniband = rng.below(2)
        lo, ids = qvb.plan_placement(v, t)
        ot = otopo_from(t)
        for home in range(t.servers):
            reader = rng.below(t.gpus_per_server)
            monkeypatch.delenv("QVB_LUT_GENERAL", raising=False)
            a = qvb.build_lookup_table(lo, ids, t, home, reader)
            monkeypatch.setenv("QVB_LUT_GENERAL", "1")
            g = qvb.build_lookup_table(lo, ids, t, home, reader)
            b = oracle.build_lookup_table(lo, ids, ot, home, reader)
            assert (a[0] == g[0]).all() and (a[1] == g[1]).all()
            assert (g[0] == b[0]).all() and (g[1] == b[1]).all()
    monkeypatch.delenv("QVB_LUT_GENERAL", raising=False)


def test_lut_properties(qvb):
    # test_placement.cpp:216-234 dense distinct offsets; :236-275 dominance
    rng = derive_stream(107, 2)
    for _ in range(15):
        n = 1 + rng.below(40)
        v = np.array([rng.uniform() for _ in range(n)])
        t = qvb.Topology.with_defaults(servers=2, numa_per_server=1, gpus_per_server=1,
                                       gpu_feature_capacity=1, host_feature_capacity=1,
                                       disk_feature_capacity=n, infiniband=1)
        lo, ids = qvb.plan_placement(v, t)
        loc, off = qvb.build_lookup_table(lo, ids, t, 1)
        assert len({(a, b) for a, b in zip(loc.tolist(), off.tolist())}) == n


def test_read_plan_errors(qvb):
    g = GOLD["scenarios"]["d"]
    t = qtopo(qvb, g["topology"])
    lo, ids = qvb.plan_placement(FIVE, t)
    loc, off = qvb.build_lookup_table(lo, ids, t, 0)
    with pytest.raises(qvb.ValidationError, match="feature id 99 outside lookup table"):
        qvb.plan_reads(loc, off, [0, 99], 4)
    with pytest.raises(qvb.ValidationError):
        qvb.plan_reads(loc, off, [0], 0)
    empty = qvb.plan_reads(loc, off, [], 4)
    assert all(len(x) == 0 for x in empty)


def test_c1_chain_golden(qvb, oracle):
    """P -> placement(8 GPUs, NVLink) -> LUT -> read plan on C1, against the
    reference's own outputs (golden hashes)."""
    import hashlib

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    g = GOLD["c1"]["uniform_L2"]
    c = CONFIGS["C1"]
    dg = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    p = dg.access_prob(2)
    dg.close()
    assert sha(p) == g["sha256"]
    pl = g["placement8"]
    t = qtopo(qvb, pl["topology"])
    lo, ids = qvb.plan_placement(p, t)
    assert sha(np.concatenate([lo.view(np.uint8), ids.view(np.uint8)])) == pl["plan_sha256"]
    loc, off = qvb.build_lookup_table(lo, ids, t)
    assert sha(np.concatenate([loc.view(np.uint8), off.view(np.uint8)])) == pl["lut_sha256"]
    gl, gc, gt, oo = qvb.plan_reads(loc, off, oracle.request_ids(11, 0, c["n"], 4096), 8)
    assert gl.tolist() == pl["reads"]["group_loc"] and gc.tolist() == pl["reads"]["group_count"]
    assert gt.tolist() == pl["reads"]["group_transitions"] and sha(oo) == pl["reads"]["offsets_sha256"]


def test_c2_rank_and_lut_vs_oracle(qvb, oracle):
    c = CONFIGS["C2"]
    dg = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    p = dg.access_prob(2)
    dg.close()
    assert (qvb.rank_desc(p) == oracle.rank_desc(p)).all()
    t = qvb.Topology.with_defaults(gpus_per_server=8, nvlink_within_numa=1,
                                   gpu_feature_capacity=c["n"] // 16,
                                   gpu_replicated_capacity=c["n"] // 64,
                                   host_feature_capacity=c["n"])
    ot = otopo_from(t)
    lo, ids = qvb.plan_placement(p, t)
    lo2, ids2 = oracle.plan_placement(p, ot)
    assert (lo == lo2).all() and (ids == ids2).all()
    for reader in (0, 5):
        a = qvb.build_lookup_table(lo, ids, t, 0, reader)
        b = oracle.build_lookup_table(lo2, ids2, ot, 0, reader)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    req = oracle.request_ids(11, 3, c["n"], 1 << 20)
    for x, y in zip(qvb.plan_reads(a[0], a[1], req, 8), oracle.plan_reads(b[0], b[1], req, 8)):
        assert (x == y).all()


@pytest.mark.skipif(not c4_reference_enabled(),
                    reason="needs >= 150 GB host RAM (QVB_C4_REFERENCE=1 forces, =0 skips)")
def test_c4_full_placement_against_reference(qvb):
    """C4 at full size (111M features, 8 GPUs, capacity N/16): plan, lookup
    table and a 1M-id read plan equal the unmodified reference's own."""
    from oracle.oracle import Oracle, RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    c = CONFIGS["C4"]
    n = c["n"]
    g = qvb.DeviceGraph.synthetic(n, c["e"], 7, False, False)
    p = g.access_prob(c["layers"])
    g.close()
    t = qvb.Topology.with_defaults(gpus_per_server=8, nvlink_within_numa=1, gpu_feature_capacity=n // 16,
                                   host_feature_capacity=n)
    ot = otopo_from(t)
    ref = RefLib()
    lo, ids = qvb.plan_placement(p, t)
    lo2, ids2 = ref.plan_placement(p, ot)
    assert (lo == lo2).all() and (ids == ids2).all()
    loc, off = qvb.build_lookup_table(lo, ids, t, 0)
    loc2, off2 = ref.build_lookup_table(lo2, ids2, ot, 0)
    assert (loc == loc2).all() and (off == off2).all()
    req = Oracle().request_ids(11, 0, n, 1 << 20)
    for x, y in zip(qvb.plan_reads(loc, off, req, 8), ref.plan_reads(loc2, off2, req, 8)):
        assert (x == y).all()
