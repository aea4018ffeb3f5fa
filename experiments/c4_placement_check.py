"""C4 at full size against the unmodified reference, placement side: P from
our device sweep (itself bit-identical to the reference, r01zh), then
plan_placement -> build_lookup_table -> plan_reads on 1M ids, ours (device
rank + the sequential planner, device lookup table, device read planner)
against the reference's own functions (oracle/_ref), compared byte for byte.
8 GPUs with NVLink, GPU capacity N/16, host capacity N (the reference has no
replicated-capacity mode, so that extension stays 0 here).

  python experiments/c4_placement_check.py   (GPU box)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle, RefLib, topology_defaults  # noqa: E402  (the checker)
from paper_2305_10863_b200 import qvb  # noqa: E402
from tests.util import CONFIGS  # noqa: E402

c = CONFIGS["C4"]
n = c["n"]
g = qvb.DeviceGraph.synthetic(n, c["e"], 7, False, False)
p = g.access_prob(c["layers"])
g.close()
kw = dict(gpus_per_server=8, nvlink_within_numa=1, gpu_feature_capacity=n // 16, host_feature_capacity=n)
t = qvb.Topology.with_defaults(**kw)
ot = topology_defaults()  # the same fields, link table included
for f, _ in t._fields_:
    if f.startswith("link_"):
        for i in range(7):
            getattr(ot, f)[i] = getattr(t, f)[i]
    else:
        setattr(ot, f, getattr(t, f))
ref = RefLib()
res = {"config": "C4", "features": n}
t0 = time.perf_counter()
lo, ids = qvb.plan_placement(p, t)
res["ours_plan_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
lo2, ids2 = ref.plan_placement(p, ot)
res["reference_plan_s"] = time.perf_counter() - t0
res["plan_identical"] = bool(len(lo) == len(lo2) and (lo == lo2).all() and len(ids) == len(ids2) and (ids == ids2).all())
t0 = time.perf_counter()
loc, off = qvb.build_lookup_table(lo, ids, t, 0)
res["ours_lut_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
loc2, off2 = ref.build_lookup_table(lo2, ids2, ot, 0)
res["reference_lut_s"] = time.perf_counter() - t0
res["lut_identical"] = bool((loc == loc2).all() and (off == off2).all())
req = Oracle().request_ids(11, 0, n, 1 << 20)
t0 = time.perf_counter()
a = qvb.plan_reads(loc, off, req, 8)
res["ours_reads_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
b = ref.plan_reads(loc2, off2, req, 8)
res["reference_reads_s"] = time.perf_counter() - t0
res["reads_identical"] = bool(all((x == y).all() for x, y in zip(a, b)))
print(json.dumps(res), flush=True)
