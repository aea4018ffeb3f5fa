"""Generates tests/golden/golden.json from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It loads oracle/_ref/libqvref.so — the reference's own graph.cpp, metrics.cpp,
placement.cpp and topology.cpp compiled by oracle/Makefile — and records its
outputs on the reference's own fixtures (tests/testutil.hpp,
tests/test_placement.cpp, tests/acceptance.cpp) plus the BASELINE C1 graphs.
The GPU box never reads /root/reference; it reads this JSON.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, RefLib, build, topology_defaults  # noqa: E402
from tests.util import derive_stream, fig8_edges, random_edges  # noqa: E402


def hexs(a):
    return [f"{int(x):016x}" for x in np.ascontiguousarray(a, np.float64).view(np.uint64)]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def topo_dict(t):
    return {f: (list(getattr(t, f)) if f.startswith("link_") else getattr(t, f))
            for f, _ in t._fields_ if f != "_pad0"}


def five_features():  # test_placement.cpp:18-24
    return np.array([0.5, 0.4, 0.3, 0.2, 0.1])


def scenarios():
    """acceptance.cpp:183-268 (a)-(d) and test_placement.cpp:44-68."""
    a = dict(servers=1, numa_per_server=2, gpus_per_server=4, gpu_feature_capacity=1,
             host_feature_capacity=4, disk_feature_capacity=8, nvlink_within_numa=0, infiniband=0)
    b = dict(a, nvlink_within_numa=1)
    c = dict(servers=2, numa_per_server=1, gpus_per_server=1, gpu_feature_capacity=1,
             host_feature_capacity=1, disk_feature_capacity=3, nvlink_within_numa=0, infiniband=0)
    d = dict(c, infiniband=1)
    e = dict(b, servers=2, infiniband=1)  # test_placement.cpp:180-200
    return {"a": a, "b": b, "c": c, "d": d, "closest_replica": e}


def random_topologies():
    """test_placement.cpp:147-178 draws."""
    rng = derive_stream(103, 1)
    out = []
    for _ in range(40):
        n = 1 + rng.below(60)
        vals = [rng.uniform() for _ in range(n)]
        t = dict(servers=1 + rng.below(3), numa_per_server=1 + rng.below(2))
        t["gpus_per_server"] = t["numa_per_server"] * (1 + rng.below(2))
        t["gpu_feature_capacity"] = rng.below(4)
        t["host_feature_capacity"] = rng.below(10)
        t["disk_feature_capacity"] = 20 + rng.below(40)
        t["nvlink_within_numa"] = int(rng.below(2) == 0)
        t["infiniband"] = int(rng.below(2) == 0)
        out.append((vals, t))
    return out


def sampler_goldens(o, r):
    """batch_sample (sampler.cpp:114-149) on the fixtures of test_sampler.cpp."""
    def run(ro, col, ww, seeds, fan, rs):
        nodes, counts, uniq = r.batch_sample(ro, col, ww, np.array(seeds, np.uint64), fan, rs)
        return {"seeds": [int(x) for x in seeds], "fanouts": list(fan), "rng_seed": rs,
                "nodes": nodes.tolist(), "counts": counts.tolist(), "unique": uniq.tolist()}

    out = {}
    n, s, d, w = fig8_edges()
    ro, col, ww = o.build_csr(n, s, d, w)
    out["fig8_full"] = run(ro, col, ww, [4], [10, 10], 1)  # test_sampler.cpp:15-26
    rng = derive_stream(83, 3)  # test_sampler.cpp:109-111
    out["fig8_batch"] = run(ro, col, ww, [rng.below(n) for _ in range(100)], [2, 2], 7)
    out["fig8_dup"] = run(ro, col, ww, [0, 0, 3, 0], [2, 2], 7)
    out["fig8_empty"] = run(ro, col, ww, [], [2, 2], 5)
    ro, col, ww = o.build_csr(3, [0, 1], [1, 2], [1.0, 1.0])  # chain3, test_sampler.cpp:28-35
    out["chain3"] = run(ro, col, ww, [0], [1, 1], 99)
    ro, col, ww = o.build_csr(3, [0, 0, 0, 0], [1, 1, 1, 2], [1.0] * 4)  # :135-150
    out["parallel"] = [run(ro, col, ww, [0], [2], i) for i in range(50)]
    rnd = []
    rng = derive_stream(79, 2)  # test_sampler.cpp:57-80
    for it in range(20):
        n, s, d, w = random_edges(rng, 30, 300, True)
        ro, col, ww = o.build_csr(n, s, d, w)
        ent = run(ro, col, ww, [rng.below(n)], [2, 3], it)
        ent["edges"] = [n, s, d, w]
        rnd.append(ent)
    out["random"] = rnd
    c1 = {}
    for name, weighted in [("uniform", False), ("weighted", True)]:
        ro, col, ww = o.synthetic_graph(100_000, 1_000_000, 7, weighted, False)
        seeds = o.request_ids(11, 0, 100_000, 4096)  # tools/bench.cpp:89-94
        nodes, counts, uniq = r.batch_sample(ro, col, ww, seeds, [15, 10], 3)
        c1[name] = {"total": int(len(nodes)), "unique": int(len(uniq)), "nodes_sha256": digest(nodes),
                    "counts_sha256": digest(counts), "unique_sha256": digest(uniq)}
    out["c1_bench"] = c1
    return out


def main():
    build(ref=True)
    r = RefLib()
    o = Oracle()
    g = {"generator": "tests/golden/make_golden.py via oracle/_ref (unmodified reference)"}

    n, s, d, w = fig8_edges()
    ro, col, ww = o.build_csr(n, s, d, w)
    g["fig8"] = {str(L): hexs(r.access_prob(ro, col, ww, L)) for L in (1, 2, 3, 4)}

    c1 = {}
    for name, weighted, transposed, layers in [("uniform_L2", False, False, 2),
                                               ("uniform_L3", False, False, 3),
                                               ("weighted_L3", True, False, 3),
                                               ("transposed_L3", False, True, 3)]:
        ro, col, ww = o.synthetic_graph(100_000, 1_000_000, 7, weighted, transposed)
        p = r.access_prob(ro, col, ww, layers)
        c1[name] = {"sha256": digest(p), "graph_sha256": digest(np.concatenate(
            [ro.view(np.uint8), col.view(np.uint8), ww.view(np.uint8)])),
            "head": hexs(p[:16])}
        if name == "uniform_L2":
            t8 = topology_defaults(gpus_per_server=8, numa_per_server=1, nvlink_within_numa=1,
                                   gpu_feature_capacity=6_000, host_feature_capacity=100_000)
            lo, ids = r.plan_placement(p, t8)
            loc, off = r.build_lookup_table(lo, ids, t8, 0)
            req = o.request_ids(11, 0, 100_000, 4096)
            gl, gc, gt, oo = r.plan_reads(loc, off, req, 8)
            c1[name]["placement8"] = {"topology": topo_dict(t8), "plan_sha256": digest(
                np.concatenate([lo.view(np.uint8), ids.view(np.uint8)])),
                "lut_sha256": digest(np.concatenate([loc.view(np.uint8), off.view(np.uint8)])),
                "reads": {"group_loc": gl.tolist(), "group_count": gc.tolist(),
                          "group_transitions": gt.tolist(), "offsets_sha256": digest(oo)}}
    g["c1"] = c1

    # FAP (metrics.cpp:95-132): fig8 at K=1..3, uniform and seeded; C1 hashes
    n, s, d, w = fig8_edges()
    ro, col, ww = o.build_csr(n, s, d, w)
    seed = np.array([0.5, 0.1, 0.1, 0.1, 0.1, 0.1])
    g["fap_fig8"] = {str(K): hexs(r.compute_fap(ro, col, ww, K)) for K in (0, 1, 2, 3)}
    g["fap_fig8_seeded"] = {"seed": seed.tolist(),
                            "values": hexs(r.compute_fap(ro, col, ww, 2, seed))}
    fc1 = {}
    for name, weighted in [("uniform_K2", False), ("weighted_K3", True)]:
        ro, col, ww = o.synthetic_graph(100_000, 1_000_000, 7, weighted, False)
        fc1[name] = digest(r.compute_fap(ro, col, ww, 2 if not weighted else 3))
    g["fap_c1"] = fc1

    g["sampler"] = sampler_goldens(o, r)

    sc = {}
    for name, kw in scenarios().items():
        t = topology_defaults(**kw)
        lo, ids = r.plan_placement(five_features(), t)
        loc, off = r.build_lookup_table(lo, ids, t, 0)
        ent = {"topology": topo_dict(t), "loc_offsets": lo.tolist(), "loc_ids": ids.tolist(),
               "lut_loc": loc.tolist(), "lut_off": off.tolist()}
        gl, gc, gt, oo = r.plan_reads(loc, off, [4, 1, 0, 3, 1], 2)
        ent["reads_41031_p2"] = [gl.tolist(), gc.tolist(), gt.tolist(), oo.tolist()]
        sc[name] = ent
    g["scenarios"] = sc

    # reference export texts of scenario (b) (placement.cpp:406-459)
    import ctypes as C
    import tempfile

    L = r._lib
    u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
    i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
    L.qvr_placement_exports.argtypes = [u64p, i64p, C.c_uint64, C.c_void_p, C.c_char_p, C.c_char_p]
    L.qvr_lookup_exports.argtypes = [i64p, u64p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_char_p,
                                     C.c_char_p]
    tb = topology_defaults(**scenarios()["b"])
    lo, ids = r.plan_placement(five_features(), tb)
    loc, off = r.build_lookup_table(lo, ids, tb, 0)
    with tempfile.TemporaryDirectory() as d:
        pj, pc, lj, lc = (os.path.join(d, x) for x in ("p.json", "p.csv", "l.json", "l.csv"))
        L.qvr_placement_exports(lo, ids, len(lo) - 1, C.addressof(tb), pj.encode(), pc.encode())
        L.qvr_lookup_exports(loc, off, len(loc), 0, tb.gpus_per_server, lj.encode(), lc.encode())
        g["exports_b"] = {k: open(p).read() for k, p in
                          [("placement_json", pj), ("placement_csv", pc), ("lookup_json", lj),
                           ("lookup_csv", lc)]}

    # "short by 3" (test_placement.cpp:138-145)
    t = topology_defaults(**dict(scenarios()["c"], disk_feature_capacity=0, host_feature_capacity=1))
    try:
        r.plan_placement(five_features(), t)
        raise SystemExit("expected PlacementError")
    except Exception as e:  # noqa: BLE001
        g["short_by_3"] = {"code": getattr(e, "code", None), "msg": getattr(e, "msg", str(e)),
                           "topology": topo_dict(t)}

    rnd = []
    for vals, kw in random_topologies():
        t = topology_defaults(**kw)
        ent = {"values": vals, "topology": topo_dict(t)}
        try:
            lo, ids = r.plan_placement(np.array(vals), t)
            ent["loc_offsets"] = lo.tolist()
            ent["loc_ids"] = ids.tolist()
            homes = {}
            for home in range(t.servers):
                loc, off = r.build_lookup_table(lo, ids, t, home)
                homes[str(home)] = [loc.tolist(), off.tolist()]
            ent["luts"] = homes
        except Exception as e:  # noqa: BLE001
            ent["error"] = {"code": getattr(e, "code", None), "msg": getattr(e, "msg", str(e))}
        rnd.append(ent)
    g["random_placements"] = rnd

    g["page_transitions"] = [[[2, 10, 3, 11], 2, r.page_transitions([2, 10, 3, 11], 2)],
                             [[2, 3, 10, 11], 2, r.page_transitions([2, 3, 10, 11], 2)],
                             [[5], 2, r.page_transitions([5], 2)],
                             [[3, 1, 2, 0], 8, r.page_transitions([3, 1, 2, 0], 8)],
                             [[], 4, r.page_transitions([], 4)]]

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
