"""host_knobs.py — tier-split gather knobs on C4 at mid and large batches:
per host fraction h and batch B, the device time of one qvb_gather for
  default            (host list ordered when the tier is >= 4 GB)
  sort               QVB_HOST_SORT=1 (order the host list whatever the tier size)
  sort_bits12        ... with 2^12 offset buckets instead of 2^16
  flat               QVB_GATHER_SMALL above B (the flat mixed kernel, no class split)
    python experiments/r02/host_knobs.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2305_10863_b200 import dist as D  # noqa: E402
from paper_2305_10863_b200 import qvb  # noqa: E402

SETTINGS = {
    "default": {},
    "sort": {"QVB_HOST_SORT": "1"},
    "sort_bits12": {"QVB_HOST_SORT": "1", "QVB_HOST_BUCKET_BITS": "12"},
    "flat": {"QVB_GATHER_SMALL": str(1 << 21)},
}
if "--more" in sys.argv:  # host-list knobs of the class split
    SETTINGS.update({
        "unsorted": {"QVB_HOST_SORT": "0"},
        "group4": {"QVB_HOST_GROUP": "4"},
        "group1": {"QVB_HOST_GROUP": "1"},
        "mixed_rows": {"QVB_GATHER_SPLIT": "0"},
    })


def main():
    cfg = bench.CONFIGS["C4"]
    n, e, dim, layers = cfg["n"], cfg["e"], cfg["dim"], cfg["layers"]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream(dev)
    g = qvb.DeviceGraph.synthetic(n, e, 7, False, False, device=0, stream=st)
    p = torch.empty(n, dtype=torch.float64, device=dev)
    g.access_prob(layers, out=p, stream=st)
    ph = p.cpu().numpy()
    g.close()
    del p
    reps = 20
    req = torch.empty((reps + 2, 1 << 20), dtype=torch.int64, device=dev)
    for k in range(reps + 2):
        qvb.request_ids_synthetic(11, k, n, req[k], device=0, stream=st)
    if "--p-weighted" in sys.argv:  # ids drawn from the CDF of P (simulator.cpp:99-132)
        cdf = np.cumsum(ph)
        cdf /= cdf[-1]
        rng = np.random.default_rng(5)
        req = torch.from_numpy(np.searchsorted(cdf, rng.random((reps + 2, 1 << 20)), side="right")
                               .clip(0, n - 1).astype(np.int64)).to(dev)
    out = torch.empty((1 << 20, dim), dtype=torch.float32, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for h in ((0.05, 0.10) if "--p-weighted" in sys.argv else (0.05, 0.10, 0.25)):
        topo = D.topology_for(qvb, n, 1, 0.0, h)
        lo, ids = qvb.plan_placement(ph, topo, device=0)
        store = D.build_store(qvb, lo, ids, dim, topo, 0, 0)
        for b in ((1 << 18, 1 << 20) if "--p-weighted" in sys.argv else (1 << 16, 1 << 18, 1 << 20)):
            line = []
            for name, env in SETTINGS.items():
                for k, v in env.items():
                    os.environ[k] = v
                for k in range(2):
                    store.gather(req[k, :b], out[:b], stream=st)
                torch.cuda.synchronize()
                ev[0].record(st)
                for k in range(reps):
                    store.gather(req[k + 2, :b], out[:b], stream=st)
                ev[1].record(st)
                ev[1].synchronize()
                store.check_error()
                ms = ev[0].elapsed_time(ev[1]) / reps
                line.append(f"{name} {ms * 1e3:8.1f} us")
                for k in env:
                    os.environ.pop(k, None)
            print(f"h={h:.2f} B={b:8d}: " + " | ".join(line), flush=True)
        store.close()


if __name__ == "__main__":
    main()
