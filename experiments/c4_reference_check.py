"""C4 at full size against the unmodified reference: the reference's own
compute_access_prob_ie (oracle/_ref, built from /root/reference sources; 16
OpenMP threads, including its per-call transpose) and ours end to end from the
same host CSR, compared bit for bit over all 111M nodes.

  python experiments/c4_reference_check.py   (GPU box; ~90 GB host RAM)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import RefLib  # noqa: E402  (test infrastructure: the checker)
from paper_2305_10863_b200 import qvb  # noqa: E402
from tests.util import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ro, col, w = qvb.synthetic_csr(c["n"], c["e"], 7, c["weighted"], False, device=0)
wt = w if c["weighted"] else None
qvb.compute_access_prob_ie(ro, col, wt, c["layers"], device=0)  # warm-up (pins the staging slots)
tm = [0.0, 0.0, 0.0]
t0 = time.perf_counter()
p_gpu = qvb.compute_access_prob_ie(ro, col, wt, c["layers"], device=0, timings=tm).values
gpu_s = time.perf_counter() - t0
ref = RefLib()
threads = os.cpu_count() or 1
ref.set_threads(threads)
t0 = time.perf_counter()
p_ref = ref.access_prob(ro, col, w, c["layers"], parallel=True)
ref_s = time.perf_counter() - t0
same = p_gpu.view(np.uint64) == p_ref.view(np.uint64)
print(json.dumps({"config": sys.argv[1] if len(sys.argv) > 1 else "C4", "nodes": int(c["n"]), "edges": int(c["e"]), "layers": c["layers"],
                  "gpu_e2e_s": gpu_s, "gpu_phases_ms": tm, "reference_s": ref_s, "reference_threads": threads,
                  "speedup_e2e": ref_s / gpu_s, "bit_identical_nodes": int(same.sum()),
                  "all_bit_identical": bool(same.all())}), flush=True)
