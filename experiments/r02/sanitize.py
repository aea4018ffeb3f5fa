"""Drives every kernel family of libqvb.so once on small inputs, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  K0 sampler (warp, CTA and large-row paths), K1 P(n,j) (sliced sweeps,
  first sweep over classes incl. exceptions, node-major code gathers +
  TMA-staged products, weighted layout), K2 rank, K3 lookup tables (mask and
  any-location paths), K4 read plans (host table, device table, store
  table), K5 gathers (flat, row-group, tier-split, planned, TMA and cp.async
  variants, host tier), FAP, in_adjacency, from_edges, transition_view.

Every result is also checked against the oracle, so a run that the tool
does not flag is a correct one.
    compute-sanitizer --tool memcheck --error-exitcode 9 python experiments/r02/sanitize.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from oracle.oracle import Oracle, topology_defaults  # noqa: E402
from paper_2305_10863_b200 import qvb  # noqa: E402


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def main():
    import torch

    o = Oracle()
    n, e = 30_000, 300_000
    for weighted in (False, True):
        ro, col, w = o.synthetic_graph(n, e, 7, weighted, False)
        for env in ({}, {"QVB_SEG_SOURCES": "7000"}, {"QVB_SEG_SOURCES": "7000", "QVB_SEG_LAYOUT": "slices"},
                    {"QVB_FIRST": "gather"}):
            os.environ.update(env)
            g = qvb.DeviceGraph.upload(ro, col, w if weighted else None)
            for layers in (2, 3):
                assert (bits(g.access_prob(layers)) == bits(o.access_prob(ro, col, w, layers))).all(), env
            g.close()
            for k in env:
                del os.environ[k]
        assert (bits(qvb.compute_fap(ro, col, w, 3).values) == bits(o.compute_fap(ro, col, w, 3))).all()
        tro, tcol, tw = qvb.in_adjacency(ro, col, w)
        a = o.in_adjacency(ro, col, w)
        assert (tro == a[0]).all() and (tcol == a[1]).all()
        rs, dist, par = qvb.transition_view(ro, col, w)
        assert (bits(rs) == bits(o.row_sums(ro, w))).all()
        # sampler
        s = qvb.Sampler.upload(ro, col, w if weighted else None) if hasattr(qvb.Sampler, "upload") else None
        if s is not None:
            seeds = o.request_ids(3, 1, n, 512)
            r = s.batch_sample(seeds, [15, 10], 3)
            got = r.arrays()
            exp = o.batch_sample(ro, col, w, seeds, [15, 10], 3)
            assert all((x == y).all() for x, y in zip(got, exp))
            r.close()
            s.close()
    src = np.array([1, 3, 3, 0, 2], np.uint64)
    dst = np.array([2, 0, 0, 1, 3], np.uint64)
    qvb.from_edges(4, src, dst, np.ones(5))

    # placement, tables, read plans
    v = np.random.default_rng(1).random(n)
    t = qvb.Topology.with_defaults(gpus_per_server=4, nvlink_within_numa=1, gpu_feature_capacity=n // 8,
                                   gpu_replicated_capacity=n // 32, host_feature_capacity=n)
    lo, ids = qvb.plan_placement(v, t)
    loc, off = qvb.build_lookup_table(lo, ids, t, 0, 1)
    os.environ["QVB_LUT_GENERAL"] = "1"
    loc2, off2 = qvb.build_lookup_table(lo, ids, t, 0, 1)
    del os.environ["QVB_LUT_GENERAL"]
    assert (loc == loc2).all() and (off == off2).all()
    req = o.request_ids(11, 0, n, 70_000)
    exp_plan = o.plan_reads(loc, off, req, 8)
    assert all((a == b).all() for a, b in zip(qvb.plan_reads(loc, off, req, 8), exp_plan))

    dim = 100
    x = o.features(n, dim)
    exp = o.gather(x, req)
    stores = [qvb.FeatureStore(lo, ids, dim, t, reader=r, device=0) for r in range(4)]
    for r, st in enumerate(stores):
        for p in range(4):
            if p != r:
                st.attach_local_peer(p, stores[p])
    st = stores[1]
    assert all((a == b).all() for a, b in zip(st.plan_reads(req, 8), exp_plan))
    d_ids = torch.from_numpy(req.view(np.int64)).cuda()
    out = torch.empty((len(req), dim), dtype=torch.float32, device="cuda")
    for env in ({}, {"QVB_HOST_SORT": "1"}, {"QVB_GATHER_SPLIT": "0"}, {"QVB_GATHER_SMALL": "1000000"}):
        os.environ.update(env)
        st.gather(d_ids, out)
        torch.cuda.synchronize()
        assert (out.cpu().numpy() == exp).all(), env
        assert (st.gather_host(req) == exp).all()
        for k in env:
            del os.environ[k]
    st.gather(d_ids, out, planned=True)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == exp).all()
    for st in stores:
        st.close()
    # device-only store, TMA / cp.async gather variants (process-wide switch)
    t1 = qvb.Topology.with_defaults(gpus_per_server=1, gpu_feature_capacity=n, host_feature_capacity=n)
    lo1, ids1 = qvb.plan_placement(v, t1)
    st = qvb.FeatureStore(lo1, ids1, 128, t1, reader=0)
    x = o.features(n, 128)
    assert (st.gather_host(req) == o.gather(x, req)).all()
    st.close()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
