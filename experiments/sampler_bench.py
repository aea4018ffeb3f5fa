"""Times qvb batch_sample (device events) vs the reference's OpenMP batch_sample.
python experiments/sampler_bench.py [C1|C2|C3] [seeds...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_10863_b200 import qvb  # noqa: E402
from tests.util import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
batches = [int(x) for x in sys.argv[2:]] or [4096, 65536]
c = CONFIGS[cfg]
smp = qvb.Sampler.synthetic(c["n"], c["e"], 7, c["weighted"])
i = smp.info()
print(cfg, "build_ms", round(i.build_ms, 2), "cands", i.candidates, "max", i.max_candidates,
      "parallel", i.parallel_edges, "MB", i.device_bytes >> 20)
from oracle.oracle import Oracle, RefLib  # noqa: E402
o = Oracle()
for b in batches:
    seeds = o.request_ids(11, 0, c["n"], b)
    for _ in range(3):
        smp.batch_sample(seeds, [15, 10], 3).close()
    ms = []
    for _ in range(10):
        t0 = time.perf_counter()
        r = smp.batch_sample(seeds, [15, 10], 3)
        t1 = time.perf_counter()
        inf = r.info()
        ms.append((inf.device_ms, (t1 - t0) * 1e3, inf.total_instances, inf.unique_count))
        r.close()
    d = np.median([m[0] for m in ms]); w = np.median([m[1] for m in ms])
    print("  device_ms min/max", round(min(m[0] for m in ms), 3), round(max(m[0] for m in ms), 3))
    print(f"seeds={b} device_ms={d:.3f} wall_ms={w:.3f} instances={ms[0][2]} unique={ms[0][3]} "
          f"Minst/s={ms[0][2] / d / 1e3:.1f}")
if RefLib.available() and os.environ.get("REF", "1") == "1":
    ro, col, w = o.synthetic_graph(c["n"], c["e"], 7, c["weighted"], False)
    r = RefLib()
    for b in batches:
        seeds = o.request_ids(11, 0, c["n"], b)
        r.batch_sample(ro, col, w, seeds, [15, 10], 3)
        t = []
        for _ in range(3):
            r.batch_sample(ro, col, w, seeds, [15, 10], 3)
            t.append(r.last_ms)
        print(f"reference seeds={b} ms={np.median(t):.2f} threads={r.max_threads()}")
