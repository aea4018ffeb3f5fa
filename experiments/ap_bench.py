"""Sweep-time experiments for K1: python experiments/ap_bench.py C4 "QVB_PF_BLOCKS=0" "QVB_PF_BLOCKS=1024" ...
Each argument after the config is a space-separated list of env settings."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_10863_b200 import qvb  # noqa: E402
from tests.util import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1]]
g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, c["weighted"])
i = g.info()
print("build_ms", round(i.build_ms, 1), "eu", i.unique_edge_count, "MB", i.device_bytes >> 20, flush=True)
ref = None
for setting in sys.argv[2:] or [""]:
    for kv in setting.split():
        k, v = kv.split("=")
        os.environ[k] = v
    out = g.access_prob(c["layers"])
    ms, ph = [], []
    for _ in range(5):
        g.access_prob(c["layers"], out=out)
        ms.append(g.last_sweep_ms())
        ph.append(g.phase_ms())
    same = ref is None or bool((out.view(np.uint64) == ref.view(np.uint64)).all())
    ref = out.copy() if ref is None else ref
    print(f"{setting or 'default'}: sweeps_ms={min(ms):.3f} per_sweep={min(ms) / (c['layers'] - 1):.3f} "
          f"same_as_first={same}", flush=True)
    best = ph[int(np.argmin(ms))]
    print("   phases_ms", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in best.items()}, flush=True)
    for kv in setting.split():
        os.environ.pop(kv.split("=")[0], None)
