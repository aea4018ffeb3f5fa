"""One warm batch_sample for ncu: python experiments/sampler_once.py C2 65536"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_10863_b200 import qvb  # noqa: E402
from tests.util import CONFIGS, derive_stream  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
b = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
smp = qvb.Sampler.synthetic(c["n"], c["e"], 7, c["weighted"])
st = derive_stream(11, 0x5EED)
import numpy as np  # noqa: E402
seeds = np.array([st.below(c["n"]) for _ in range(b)], np.uint64)
smp.batch_sample(seeds, [15, 10], 3).close()
r = smp.batch_sample(seeds, [15, 10], 3)
print("device_ms", r.info().device_ms)
