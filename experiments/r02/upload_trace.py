"""Where the end-to-end P call from a host CSR spends its time at C4:
upload (column narrowing through pinned staging + H2D) vs the in-CSR build
vs the sweeps vs the download (QVB_TRACE_UPLOAD prints the first split)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["QVB_TRACE_UPLOAD"] = "1"
from paper_2305_10863_b200 import qvb  # noqa: E402

n, e = 111_000_000, 1_600_000_000
t0 = time.perf_counter()
ro, col, w = qvb.synthetic_csr(n, e, 7, False, False)
print("synthetic_csr (device generate + copy to host) %.2f s" % (time.perf_counter() - t0), flush=True)
for k in range(3):
    tm = [0.0, 0.0, 0.0]
    t0 = time.perf_counter()
    qvb.compute_access_prob_ie(ro, col, None, 3, timings=tm)
    print("call %d: wall %.3f s | upload+build %.1f ms, sweeps %.1f ms, download %.1f ms" %
          (k, time.perf_counter() - t0, *tm), flush=True)
for k in range(2):
    t0 = time.perf_counter()
    rs, dist, par, g = qvb.transition_view(ro, col, None, keep=True)
    t1 = time.perf_counter()
    g.access_prob(3)
    t2 = time.perf_counter()
    g.close()
    print("transition_view %.3f s + access_prob %.3f s" % (t1 - t0, t2 - t1), flush=True)
