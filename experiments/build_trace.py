"""Launch list of the C2 in-CSR build from a host out-CSR (the e2e P call's
build part): run under ncu --metrics gpu__time_duration.sum."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_10863_b200 import qvb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
from tests.util import CONFIGS  # noqa: E402

c = CONFIGS[cfg]
ro, col, w = qvb.synthetic_csr(c["n"], c["e"], 7, c["weighted"], False, device=0)
tm = [0.0, 0.0, 0.0]
for _ in range(2):
    qvb.compute_access_prob_ie(ro, col, w if c["weighted"] else None, c["layers"], device=0, timings=tm)
    print(tm, flush=True)
