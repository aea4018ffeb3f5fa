"""gather_sweep.py — the SURVEY §8(d) C5 gather sweep, reduced to what one GPU
can show: batch size B in {1K, 4K, 16K, 64K, 256K, 1M} x host-resident
coldest fraction h in {0, 5, 10, 25}% x request stream (uniform ids, the
P-weighted stream of simulator.cpp:99-132,207-211: ids drawn from the CDF of
P(n,L), and — except on C4 — the sampler-derived stream: the unique nodes of
batch_sample batches for out-degree-weighted seeds, simulator.cpp:245-254). Replication needs peers and is not swept here (bench.py --gpus N
covers it under torchrun).

Per cell: mean device time of one qvb_gather launch (CUDA events over 20
launches on distinct resident batches, replayed from a CUDA graph; the
Python-loop time per call is reported beside it), payload GB/s, and the fraction of the
mixed HBM / PCIe roofline bench.py uses (24 B metadata + 2 row moves per
device row; host rows bounded by PCIe). One JSON object per cell on stdout.

  python experiments/gather_sweep.py [C2|C3|C4] [planned]

`planned` times qvb_gather_planned instead (requests bucketed by location
and sorted by shard offset before the copy, the K4 order).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2305_10863_b200 import dist as D  # noqa: E402
from paper_2305_10863_b200 import qvb  # noqa: E402


def main():
    cname = sys.argv[1] if len(sys.argv) > 1 else "C2"
    planned = len(sys.argv) > 2 and sys.argv[2] == "planned"
    cfg = bench.CONFIGS[cname]
    n, e, dim, layers = cfg["n"], cfg["e"], cfg["dim"], cfg["layers"]
    rb = 4 * dim
    pk = bench.peaks()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream(dev)
    g = qvb.DeviceGraph.synthetic(n, e, 7, cfg["weighted"], False, device=0, stream=st)
    p = torch.empty(n, dtype=torch.float64, device=dev)
    g.access_prob(layers, out=p, stream=st)
    ph = p.cpu().numpy()
    g.close()
    del p
    cdf = np.cumsum(ph)
    cdf /= cdf[-1]
    reps = 20
    bmax = 1 << 20
    rng = np.random.default_rng(5)
    streams = {}
    uni = torch.empty((reps + 2, bmax), dtype=torch.int64, device=dev)
    for k in range(reps + 2):
        qvb.request_ids_synthetic(11, k, n, uni[k], device=0, stream=st)
    streams["uniform"] = uni
    pw = np.searchsorted(cdf, rng.random((reps + 2, bmax)), side="right").clip(0, n - 1)
    streams["p_weighted"] = torch.from_numpy(pw.astype(np.int64)).to(dev)
    # sampler-derived requests (simulator.cpp:245-254): the
    # unique nodes of qv_bench-style batch_sample batches (fanouts 15/10) for
    # out-degree-weighted seeds; the C4 host CSR is too large to build here
    samp = {}
    if cname != "C4":
        ro, _, _ = qvb.synthetic_csr(n, e, 7, cfg["weighted"], False, device=0)
        dcdf = np.cumsum(np.diff(ro.astype(np.int64)).astype(np.float64))
        dcdf /= dcdf[-1]
        del ro
        sp = qvb.Sampler.synthetic(n, e, 7, cfg["weighted"], False, device=0)
        for ns in (256, 1024, 4096):
            lst = []
            for k in range(reps + 2):
                seeds = np.searchsorted(dcdf, rng.random(ns), side="right").clip(0, n - 1).astype(np.uint64)
                r = sp.batch_sample(seeds, [15, 10], 1000 + k)
                lst.append(torch.from_numpy(r.arrays()[2].view(np.int64).copy()).to(dev))
                r.close()
            samp[ns] = lst
        sp.close()
    for h in (0.0, 0.05, 0.10, 0.25):
        topo = D.topology_for(qvb, n, 1, 0.0, h)
        lo, ids = qvb.plan_placement(ph, topo, device=0)
        store = D.build_store(qvb, lo, ids, dim, topo, 0, 0)
        loc, _ = qvb.build_lookup_table(lo, ids, topo, 0, 0, device=0)
        host_mask = torch.from_numpy(loc == 1).to(dev)
        out = torch.empty((bmax, dim), dtype=torch.float32, device=dev)
        for sname, req in streams.items():
            for b in (1 << 10, 1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20):
                for k in range(2):
                    store.gather(req[k, :b], out[:b], stream=st, planned=planned)
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record(st)
                for k in range(reps):
                    store.gather(req[k + 2, :b], out[:b], stream=st, planned=planned)
                ev[1].record(st)
                ev[1].synchronize()
                store.check_error()
                ms_loop = ev[0].elapsed_time(ev[1]) / reps
                # the same launches replayed from a CUDA graph: no Python/ctypes
                # call overhead between them (small batches are otherwise host-bound)
                ms = ms_loop
                try:
                    cg = torch.cuda.CUDAGraph()
                    cs = torch.cuda.Stream()
                    with torch.cuda.graph(cg, stream=cs):
                        for k in range(reps):
                            store.gather(req[k + 2, :b], out[:b], stream=cs, planned=planned)
                    cg.replay()
                    torch.cuda.synchronize()
                    ev[0].record()
                    cg.replay()
                    ev[1].record()
                    ev[1].synchronize()
                    ms = ev[0].elapsed_time(ev[1]) / reps
                    del cg
                except Exception as ex:  # noqa: BLE001
                    print(json.dumps({"graph_capture_failed": str(ex)}), file=sys.stderr)
                store.check_error()
                f_h = float(host_mask[req[2:, :b]].float().mean())
                hbm = b * (bench.META_BYTES + rb * (2 - f_h)) / pk["hbm_gbs"] / 1e9
                pcie = b * rb * f_h / bench.PCIE_GBS / 1e9
                t_roof = max(hbm, pcie)
                print(json.dumps({
                    "config": cname, "planned": planned, "host_fraction": h, "stream": sname, "batch": b,
                    "host_rows": f_h, "us_per_launch": ms * 1e3, "us_per_call_python_loop": ms_loop * 1e3,
                    "payload_gbs": b * rb / (ms / 1e3) / 1e9,
                    "bound": "pcie" if pcie > hbm else "hbm",
                    "roofline_frac": t_roof / (ms / 1e3)}), flush=True)
        for ns, lst in samp.items():
            bmean = int(np.mean([len(u) for u in lst[2:]]))
            for k in range(2):
                store.gather(lst[k], out[: len(lst[k])], stream=st, planned=planned)
            torch.cuda.synchronize()
            cg = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            with torch.cuda.graph(cg, stream=cs):
                for k in range(reps):
                    u = lst[k + 2]
                    store.gather(u, out[: len(u)], stream=cs, planned=planned)
            cg.replay()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            cg.replay()
            ev[1].record()
            ev[1].synchronize()
            store.check_error()
            ms = ev[0].elapsed_time(ev[1]) / reps
            f_h = float(torch.cat([host_mask[u] for u in lst[2:]]).float().mean())
            hbm = bmean * (bench.META_BYTES + rb * (2 - f_h)) / pk["hbm_gbs"] / 1e9
            pcie = bmean * rb * f_h / bench.PCIE_GBS / 1e9
            print(json.dumps({
                "config": cname, "planned": planned, "host_fraction": h, "stream": f"sampler_{ns}_seeds",
                "batch": bmean, "host_rows": f_h, "us_per_launch": ms * 1e3,
                "payload_gbs": bmean * rb / (ms / 1e3) / 1e9, "bound": "pcie" if pcie > hbm else "hbm",
                "roofline_frac": max(hbm, pcie) / (ms / 1e3)}), flush=True)
            del cg
        store.close()


if __name__ == "__main__":
    main()
