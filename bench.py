#!/usr/bin/env python
"""bench.py — the north-star measurement of the B200 Quiver feature-store path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one collect call: gather one batch of B uniform request ids
(derive_stream(11, 0x5EED, batch).below(N)) from the placed
feature table. The workload at N=1 is the north-star configuration, BASELINE
configs[3] (C4, ogbn-papers100M-shaped: 111M nodes, 1.6B edges, 128-dim fp32,
3-layer P(n,j)), which fits one B200 (`--config C2` etc. run the others):
the graph is generated on the device, P(n,j) ranks the features, the
placement manager partitions them over the N GPUs (hot replication / host
fraction optional), every rank builds its store and lookup table and serves
its own batches (weak scaling; no data-path collective).

`value` = whole-job gathered payload GB/s with ids resident in HBM; `e2e` =
the same through the public C-ABI from pinned host buffers (H2D ids, gather,
D2H rows, sync) every step. The line also carries the P(n,j) pass
(`access_prob`: edges/s, its roofline and the reference CPU timing), the
request-ID producer upstream of the collect call (`sampler`: qv_bench's
batch_sample of 4096 seeds with fanouts {15, 10}, instances/s vs the
reference's OpenMP batch_sample), the `roofline` of the dominant gather
kernel and the `cpu_baseline`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gathered feature GB/s at 1/2/4/8 B200 and access-prob edges/s vs HBM roofline"
CONFIGS = {
    "C1": dict(n=100_000, e=1_000_000, dim=128, layers=2, weighted=False,
               desc="C1 synthetic power-law graph: 100K nodes, avg degree 10, 128-dim fp32"),
    "C2": dict(n=2_400_000, e=62_000_000, dim=100, layers=2, weighted=False,
               desc="C2 ogbn-products-shaped: 2.4M nodes, 62M edges, 100-dim fp32, 2-layer P"),
    "C3": dict(n=233_000, e=114_000_000, dim=602, layers=3, weighted=True,
               desc="C3 Reddit-shaped: 233K nodes, 114M edges, 602-dim fp32, 3-layer weighted P"),
    "C4": dict(n=111_000_000, e=1_600_000_000, dim=128, layers=3, weighted=False,
               desc="C4 ogbn-papers100M-shaped: 111M nodes, 1.6B edges, 128-dim fp32, 3-layer P"),
}
META_BYTES = 24  # 8 B id + 16 B reference-layout lookup row per request
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
D2H_GBS = 57.3  # measured: pinned 512 MB device->host copies (experiments/r02/pcie_copy.py, profiles/r02/r02ae_pcie_copy.txt)
PCIE_GBS = 56.9  # measured: 512-byte row reads of pinned host memory in offset order, the best PCIe read rate on the box (profiles/r02/r02o_host_vmm.txt; random rows: 51.3)


def bench_config(args, cfg, world: int) -> dict:
    """The line's `config`, built identically by both arms (--impl ours and
    --impl reference) so the driver can match them."""
    n, dim, B = cfg["n"], cfg["dim"], args.batch
    row_bytes = 4 * dim
    return {
        "workload": cfg["desc"] + f"; gather batches of {B} uniform ids per GPU",
        "config": args.config, "batch": B, "dim": dim, "n_features": n, "layers": cfg["layers"],
        "features_partitioned_over": world, "replicate_fraction": args.replicate,
        "host_fraction": args.host_frac,
        "l2": "inputs larger than L2 (feature table %.0f MB, %.0f MB of rows per step)" % (
            n * row_bytes / 1e6, B * row_bytes / 1e6),
        "parallelism": f"feature-partitioned x{world}, one process per GPU",
    }


def _max_rss_gb() -> float:
    import resource

    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6  # KiB -> GB (approx.)


def traffic_key(args, world: int) -> str:
    return f"{args.config}|b{args.batch}|r{args.replicate:g}|h{args.host_frac:g}|n{world}"


def load_traffic(key: str) -> dict:
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            ent = json.load(f).get(key, {})
        return {k: v["bytes_per_launch"] for k, v in ent.items()}
    except Exception:  # noqa: BLE001
        return {}


def peaks():
    p = {"hbm_gbs": 6549.4, "source": "measured"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p["hbm_gbs"] = float(json.load(f)["hbm_gbs"])
    except Exception:  # noqa: BLE001
        p = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}
    return p


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during a window."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.01):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.period = period_s
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.N = None

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.N:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def bytes_per_sweep(eu: int, n: int, weighted: bool) -> int:
    """uniform 12 B/edge + 32 B/node; weighted 20 B/edge + 24 B/node."""
    return eu * (20 if weighted else 12) + n * (24 if weighted else 32)


# measured random 4-byte gather rate from an L2-resident vector on this pool's
# B200s (experiments/die_split.cu, experiments/gather_paths.cu: 273-288 G/s):
# one L1 wavefront per random gather, ~1 per SM per clock
GATHER_CEILING = 286e9


def access_prob_line(cfg, info, layers, ap_call, ap_sweep, phases, pk):
    """The P(n,j) leg of the bench line. ``roofline`` is the call's dominant
    phase against its own algorithmic bytes; ``survey_model`` is the north-star
    statement (every sweep moves 12 B per coalesced edge and 32 B
    per node, T_roof = bytes / HBM peak) as the ratio T_roof / T_call. The
    first sweep streams 2-byte out-degree classes instead of gathering
    (P(s,1) is uniform), so it moves fewer bytes than that model assumes."""
    n, eu = cfg["n"], info.unique_edge_count
    sweeps = layers - 1
    ap_ms = statistics.mean(ap_call)
    sweep_ms = statistics.mean(ap_sweep)
    ph = {k: statistics.mean(p[k] for p in phases) for k in ("first", "gather", "products", "other")}
    launches = phases[-1]["launches"]
    later = sweeps - 1 if ph["first"] > 0 else sweeps
    cols = info.segment_columns
    nseg = info.segments
    # algorithmic bytes per phase (all sweeps of one call)
    alg = {
        # classes 2 B/slot, perm 4 B/node, P out 8 B/node; for a later sweep
        # also its 1/row_sum in and its 4-byte code out
        "first": info.first_slots * 2 + n * (4 + 8 + (12 if layers > 2 else 0)),
        # per later sweep: column in + code out per edge, plus the code
        # segment once (the gathers themselves are L2 hits)
        "gather": later * (cols * 8 + n * 4),
        # per later sweep: codes in, lens per pass, P(j-1) and 1/row_sum in,
        # P out (+ code out if another sweep follows)
        "products": sum(cols * 4 + n * nseg + n * 24 + (n * 4 if j < sweeps - 1 else 0)
                        for j in range(later)),
    }
    kernels = {}
    for k, name in (("first", "k_first"), ("gather", "k_codes"), ("products", "k_products")):
        if ph[k] > 0:
            a = alg[k] / (ph[k] / 1e3) / 1e9
            kernels[name] = {"ms_per_call": ph[k], "algorithmic_bytes": alg[k], "achieved_gbs": a,
                             "frac_hbm": a / pk["hbm_gbs"]}
    if ph["gather"] > 0:
        gps = later * cols / (ph["gather"] / 1e3)
        kernels["k_codes"].update({"gathers_per_s": gps, "gather_ceiling_per_s": GATHER_CEILING,
                                   "frac_gather_ceiling": gps / GATHER_CEILING})
    if ph["other"] > 0:
        kernels["k_sweep"] = {"ms_per_call": ph["other"]}
    survey_bytes = bytes_per_sweep(eu, n, info.layout == 1) * sweeps
    t_roof = survey_bytes / (pk["hbm_gbs"] * 1e9) * 1e3
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_call"]) if kernels else None
    if dom in ("k_first", "k_codes", "k_products"):
        d = kernels[dom]
        roof = {"bound": "hbm", "kernel": dom, "traffic": None, "algorithmic_bytes": d["algorithmic_bytes"],
                "achieved": d["achieved_gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": d["frac_hbm"], "per_launch_ms": d["ms_per_call"], "peak_source": pk["source"]}
    else:  # sliced sweeps: the SURVEY per-sweep model, except that a weighted
        # first sweep does not gather (P(s,1) is uniform): 12 B/edge there
        w = info.layout == 1
        sb = survey_bytes - (eu * 8 if w and sweeps >= 1 else 0)
        a = sb / (sweep_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": "k_sweep", "traffic": None, "algorithmic_bytes": sb,
                "achieved": a, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": a / pk["hbm_gbs"],
                "peak_source": pk["source"]}
    return {
        "metric": "access-prob edges/s (coalesced in-edges x sweeps / device time of the P call)",
        "value": eu * sweeps / (ap_ms / 1e3),
        "unit": "edges/s",
        "ms_per_call": ap_ms,
        "sweep_ms": sweep_ms,
        "layers": layers,
        "graph": {"nodes": n, "edges": cfg["e"], "unique_edges": eu,
                  "exceptions": info.exception_count,
                  "layout": "weighted" if info.layout else "compact",
                  "first_sweep_classes": info.classes, "source_segments": nseg,
                  "in_csr_build_ms": info.build_ms, "in_csr_build_note": "device generator + in-CSR build, first build in the process (includes growing the stream-ordered memory pool; a warm build at C4 takes ~0.23 s, see access_prob.e2e)", "device_bytes": info.device_bytes},
        "roofline": roof,
        "kernels": kernels,
        "survey_model": {"bytes": survey_bytes, "t_roof_ms": t_roof, "ms": ap_ms,
                         "frac": t_roof / ap_ms,
                         "note": "SURVEY §8(d) per-sweep bytes (12 B/edge + 32 B/node) at the HBM peak, "
                                 "over the measured call time: the north-star 'P pass vs HBM roofline'"},
        "gpu_launches": launches * len(ap_call),
    }


def run_ours(args):
    import numpy as np
    import torch

    from paper_2305_10863_b200 import dist as D
    from paper_2305_10863_b200 import qvb

    rank, world, local = D.init()
    local = D.device_index(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    cfg = CONFIGS[args.config]
    n, e, dim, layers = cfg["n"], cfg["e"], cfg["dim"], cfg["layers"]
    row_bytes = 4 * dim
    B = args.batch
    pk = peaks()

    # ---- P(n,j): graph on device, K timed passes ------------------------------
    g = qvb.DeviceGraph.synthetic(n, e, 7, cfg["weighted"], False, device=local, stream=stream)
    info = g.info()
    p_dev = torch.empty(n, dtype=torch.float64, device=dev)
    sharded = [False]

    def p_call():
        # N > 1: the sweeps split over the ranks by node chunks with one
        # in-place all-gather of P (and codes) per layer
        if world > 1:  # (QVB_SHARE_GPU: gloo exchange through host memory, function only)
            _, sharded[0] = D.sharded_access_prob(g, layers, local, out=p_dev, stream=stream)
        else:
            g.access_prob(layers, out=p_dev, stream=stream)

    for _ in range(args.warmup):
        p_call()
    torch.cuda.synchronize(dev)
    D.barrier()
    ap_call, ap_sweep, phases = [], [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(args.steps):
        ev[0].record(stream)
        p_call()
        ev[1].record(stream)
        ev[1].synchronize()
        ap_call.append(D.max_over_ranks(ev[0].elapsed_time(ev[1])))
        ap_sweep.append(g.last_sweep_ms())
        phases.append(g.phase_ms())
    p_host = p_dev.cpu().numpy()
    access_prob = access_prob_line(cfg, info, layers, ap_call, ap_sweep, phases, pk)
    access_prob["sharded_over_ranks"] = world if sharded[0] else 1
    if sharded[0]:  # the roofline of the whole job: world GPUs' HBM
        sm = access_prob["survey_model"]
        sm["t_roof_ms"] /= world
        sm["frac"] = sm["t_roof_ms"] / sm["ms"]
        sm["note"] += f"; sweeps split over {world} GPUs: T_roof / {world}"
    g.close()

    # ---- K0 sampler: qv_bench's batch_sample (tools/bench.cpp:89-94) ----------
    sampler, sample_first = (sampler_leg(args, qvb, cfg, local, stream, rank) if args.sample_seeds
                             else (None, None))

    # ---- placement + store ------------------------------------------------------
    topo = D.topology_for(qvb, n, world, args.replicate, args.host_frac)
    t0 = time.perf_counter()
    lo, ids = qvb.plan_placement(p_host, topo, device=local)
    plan_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    loc, off = qvb.build_lookup_table(lo, ids, topo, 0, rank, device=local)
    lut_s = time.perf_counter() - t0
    rank_ms = None
    if rank == 0:
        p_dev_rank = torch.empty(n, dtype=torch.int64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        qvb._check(qvb._lib().qvb_rank_desc(local, p_dev.data_ptr(), n, p_dev_rank.data_ptr(), 1,
                                             stream.cuda_stream))
        e1.record(stream)
        e1.synchronize()
        rank_ms = e0.elapsed_time(e1)
        del p_dev_rank
    planner = {"rank_desc_device_ms": rank_ms, "plan_placement_s": plan_s,
               "build_lookup_table_s": lut_s,
               "note": "plan_placement = device rank + the reference's sequential planner on the "
                       "host; build_lookup_table / plan_reads = C-ABI calls incl. host<->device "
                       "copies of their arguments and results"}
    f_l = float(np.mean(loc == rank))
    f_h = float(np.mean(loc == world))
    f_p = 1.0 - f_l - f_h
    store = D.build_store(qvb, lo, ids, dim, topo, rank, local)

    # request batches resident in HBM: (W + K) distinct batches per rank
    nb = args.warmup + args.steps
    req = torch.empty((nb, B), dtype=torch.int64, device=dev)
    for k in range(nb):
        qvb.request_ids_synthetic(11, rank * 1_000_003 + k, n, req[k], device=local, stream=stream)
    if rank == 0:  # K4 read planner on one batch, through the C-ABI
        req0 = req[0].cpu().numpy().view(np.uint64)
        qvb.plan_reads(loc, off, req0[:1024], 8)
        t0 = time.perf_counter()
        qvb.plan_reads(loc, off, req0, 8)
        planner["plan_reads_s"] = time.perf_counter() - t0
        planner["plan_reads_ids"] = int(len(req0))
    if rank == 0:  # K4 over the store's resident table: ids in HBM, plan to the host
        store.plan_reads(req[0], 8, stream=stream)
        ts = []
        for k in range(3):
            t0 = time.perf_counter()
            store.plan_reads(req[k], 8, stream=stream)
            ts.append(time.perf_counter() - t0)
        planner["store_plan_reads_s"] = min(ts)
        planner["store_plan_reads_note"] = ("qvb_store_plan_reads: the store's resident lookup "
                                            "table, device ids, flattened plan copied to the host")
    out = torch.empty((B, dim), dtype=torch.float32, device=dev)
    for k in range(args.warmup):
        store.gather(req[k], out, stream=stream, planned=args.planned)
    torch.cuda.synchronize(dev)
    store.check_error()

    clocks = ClockSampler(local)
    with clocks:
        # keep the clocks observable: ~1 s of the same gathers right before the
        # timed region (untimed), sampled together with it
        t_end = time.perf_counter() + args.clock_window
        while time.perf_counter() < t_end:
            for k in range(args.warmup):
                store.gather(req[k], out, stream=stream, planned=args.planned)
            torch.cuda.synchronize(dev)
        D.barrier()
        torch.cuda.synchronize(dev)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        evs[0].record(stream)
        for k in range(args.steps):
            store.gather(req[args.warmup + k], out, stream=stream, planned=args.planned)
            evs[k + 1].record(stream)
        torch.cuda.synchronize(dev)
        D.barrier()
    store.check_error()
    launch_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    total_ms = evs[0].elapsed_time(evs[-1])
    max_ms = D.max_over_ranks(total_ms)
    payload = world * args.steps * B * row_bytes
    value = payload / (max_ms / 1e3) / 1e9
    per_launch_ms = statistics.mean(launch_ms)
    # mixed local-HBM / NVLink / PCIe roofline: per id, HBM
    # moves the metadata, this GPU's reads and writes and the peers' reads of
    # this GPU's shard (symmetric partition); NVLink carries the peer rows;
    # PCIe the host rows. The slowest link bounds the launch.
    hbm_per_id = META_BYTES + row_bytes * (1 + f_l + f_p)
    links = {"hbm": (B * hbm_per_id, pk["hbm_gbs"], pk["source"]),
             "nvlink": (B * row_bytes * f_p, NVLINK_GBS, "measured peer copy (B200_PROFILING.md)"),
             "pcie": (B * row_bytes * f_h, PCIE_GBS, "measured offset-ordered row reads over PCIe, experiments/r02/host_vmm.cu")}
    bound = max(links, key=lambda k: links[k][0] / links[k][1])
    # the store buckets batches that leave its own shard by location class
    # (csrc/store.cu launch_split); batches <= 48K ids (and, with a host tier,
    # batches <= 256K ids expecting <= 16K host rows) take the flat kernel
    flat = B <= 49152 or (f_h > 0 and B <= 262144 and B * f_h <= 16384)  # store.cu launch_gather
    gather_kernel = ("k_gather" if flat else
                     "k_gather_classes" if (f_p > 0 or f_h > 0) and not args.planned else
                     "k_gather_sorted" if args.planned else "k_gather_rows")
    alg, link_peak, link_src = links[bound]
    achieved = alg / (per_launch_ms / 1e3) / 1e9

    # ---- e2e through the public API from pinned host buffers --------------------
    e2e = None
    if not args.no_e2e:
        host_ids = [req[args.warmup + k].cpu().pin_memory() for k in range(args.steps)]
        host_out = torch.empty((B, dim), dtype=torch.float32).pin_memory()
        store.gather_host(host_ids[0].numpy().view(np.uint64), host_out.numpy(), stream=stream)
        D.barrier()
        t0 = time.perf_counter()
        for k in range(args.steps):
            store.gather_host(host_ids[k].numpy().view(np.uint64), host_out.numpy(), stream=stream)
        e2e_s = D.max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": payload / e2e_s / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": B * 8, "d2h_bytes_per_step": B * row_bytes,
               # the rows leave over PCIe: the pinned D2H copy rate bounds the call
               "d2h_ceiling_GBps": D2H_GBS, "frac_of_d2h_ceiling": payload / e2e_s / 1e9 / D2H_GBS,
               "note": "qvb_gather_host per step: H2D ids (pinned) + gather + D2H rows (pinned) "
                       "+ stream sync; wall clock, max over ranks"}
    if not args.no_e2e and rank == 0:  # the P legs are per-rank replicas: rank 0 reports them
        # P(n,j) end to end: host out-CSR -> device -> in-CSR -> sweeps -> host P
        ro, col, w = qvb.synthetic_csr(n, e, 7, cfg["weighted"], False, device=local)
        tm = [0.0, 0.0, 0.0]
        # untimed calls first (warm-up, like the gather's W steps: the first
        # pins the upload's staging slots once per process, and the second
        # still pays some one-time costs)
        for _ in range(max(1, min(args.warmup, 3))):
            qvb.compute_access_prob_ie(ro, col, w if cfg["weighted"] else None, layers, device=local)
        t0 = time.perf_counter()
        qvb.compute_access_prob_ie(ro, col, w if cfg["weighted"] else None, layers, device=local,
                                   timings=tm)
        wall = time.perf_counter() - t0
        access_prob["e2e"] = {
            "value": info.unique_edge_count * (layers - 1) / wall, "unit": "edges/s",
            "wall_s": wall, "upload_build_ms": tm[0], "sweeps_ms": tm[1], "download_ms": tm[2],
            "h2d_bytes": int(ro.nbytes + col.nbytes + (w.nbytes if cfg["weighted"] else 0)),
            "d2h_bytes": n * 8,
            "note": "qvb_compute_access_prob_ie from a host qv::Graph-layout CSR (the reference "
                    "call, which rebuilds its transpose every call)"}
        # the drop-in's call pattern compute_access_prob_ie(g, transition_view(g), L):
        # one upload builds the view (row sums, distinct out-degrees) and the
        # device graph the sweeps then run on
        wv = w if cfg["weighted"] else None
        t0 = time.perf_counter()
        rs, dist_out, _par, vg = qvb.transition_view(ro, col, wv, device=local, keep=True)
        t1 = time.perf_counter()
        pv = vg.access_prob(layers)
        t2 = time.perf_counter()
        vg.close()
        access_prob["e2e_dropin"] = {
            "value": info.unique_edge_count * (layers - 1) / (t2 - t0), "unit": "edges/s",
            "wall_s": t2 - t0, "transition_view_s": t1 - t0, "compute_access_prob_ie_s": t2 - t1,
            "identical_to_device_call": bool((pv.view(np.uint64) == p_host.view(np.uint64)).all()),
            "note": "qv::compute_access_prob_ie(g, qv::transition_view(g), L) from a host CSR: "
                    "qvb_transition_view (upload, device row sums / distinct out-degrees, "
                    "in-CSR kept) + qvb_access_prob on it, P copied to the host"}
        del rs, dist_out, pv
    else:
        ro = col = w = None

    # ---- CPU baseline (rank 0, N=1) ---------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if sampler is not None:
            sampler["cpu_baseline"] = sampler_cpu(args, cfg, ro, col, w, sample_first)
        cpu, ap_cpu = cpu_baseline(
            args, cfg, p_host, (loc, off), ro, col, w, steps=min(args.steps, args.cpu_steps),
            req0_plan=lambda r: qvb.plan_reads(loc, off, r, 8))
        access_prob["cpu_baseline"] = ap_cpu
    ro = col = w = None

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32 rows copied bit-exact (P in fp64)",
        "data": "synthetic (bench.cpp generator seed 7; SURVEY §8(d) features and request streams)",
        "config": bench_config(args, cfg, world),
        "placement": {
            "fractions": {"local": f_l, "peer": f_p, "host": f_h}, "placement_s": plan_s,
            "l2_policy": "rows and outputs stream with L2 evict_first; the %.0f MB lookup table is%s "
                         "kept with evict_last" % (n * 8 / 1e6, "" if n * 8 <= (32 << 20) else " not"),
            **({"shared_gpu": "QVB_SHARE_GPU=1: every rank on one GPU to exercise the multi-rank "
                              "path (IPC peers, setup collectives); the ranks time-slice the GPU, "
                              "so these timings are not a performance measurement"}
               if D.shared_gpu() and world > 1 else {}),
        },
        "roofline": {"bound": bound, "kernel": gather_kernel, "achieved": achieved,
                     "peak": link_peak, "unit": "GB/s", "frac": achieved / link_peak,
                     "traffic": None, "algorithmic_bytes_per_id": hbm_per_id,
                     "algorithmic_bytes_per_launch": alg,
                     "per_launch_ms": per_launch_ms, "peak_source": link_src,
                     "link_times_ms": {k: v[0] / v[1] / 1e6 for k, v in links.items()}},
        "e2e": e2e,
        "gpu_launches": args.steps,
        "access_prob": access_prob,
        "sampler": sampler,
        "planner": planner,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    # ncu dram bytes per launch (profiles/make_traffic.py), only from a capture
    # of exactly this line's workload key; null otherwise
    tr = load_traffic(traffic_key(args, world))
    line["roofline"]["traffic"] = tr.get(gather_kernel)
    access_prob["roofline"]["traffic"] = tr.get(access_prob["roofline"]["kernel"])
    line["roofline"]["traffic_key"] = access_prob["roofline"]["traffic_key"] = traffic_key(args, world)
    store.close()
    line["host_max_rss_gb"] = _max_rss_gb()
    if rank == 0:
        print(json.dumps(line), flush=True)


SAMPLE_FANOUTS = [15, 10]  # tools/bench.cpp:66
SAMPLE_RNG = 3               # tools/bench.cpp:92


def sample_seeds(n, k, count):
    """Seed batch k: derive_stream(11, 0x5EED, k).below(n) — batch 0 is qv_bench's."""
    from tests.util import derive_stream
    import numpy as np

    st = derive_stream(11, 0x5EED, k)
    return np.array([st.below(n) for _ in range(count)], np.uint64)


def sampler_leg(args, qvb, cfg, local, stream, rank):
    import numpy as np

    S = args.sample_seeds
    smp = qvb.Sampler.synthetic(cfg["n"], cfg["e"], 7, cfg["weighted"], device=local, stream=stream)
    info = smp.info()
    batches = [sample_seeds(cfg["n"], rank * 1_000_003 + k, S) for k in range(args.warmup + args.steps)]
    for k in range(args.warmup):
        smp.batch_sample(batches[k], SAMPLE_FANOUTS, SAMPLE_RNG, stream=stream).close()
    dev_ms, wall_ms, inst, uniq = [], [], 0, 0
    first = None
    for k in range(args.steps):
        t0 = time.perf_counter()
        r = smp.batch_sample(batches[args.warmup + k], SAMPLE_FANOUTS, SAMPLE_RNG, stream=stream)
        u = r.arrays()[2] if k == 0 else None  # e2e of the first: unique ids back on the host
        wall_ms.append((time.perf_counter() - t0) * 1e3)
        i = r.info()
        dev_ms.append(i.device_ms)
        inst += i.total_instances
        uniq += i.unique_count
        if k == 0:
            first = (r.arrays(), u)
        r.close()
    smp.close()
    ms = statistics.mean(dev_ms)
    return {
        "metric": "sampled node instances/s (batch_sample, device time per call)",
        "value": inst / (sum(dev_ms) / 1e3), "unit": "instances/s",
        "ms_per_batch": ms, "seeds_per_batch": S, "fanouts": SAMPLE_FANOUTS,
        "rng_seed": SAMPLE_RNG, "instances_per_batch": inst / args.steps,
        "unique_per_batch": uniq / args.steps,
        "e2e": {"value": inst / (sum(wall_ms) / 1e3), "unit": "instances/s",
                "ms_per_batch": statistics.mean(wall_ms), "h2d_bytes_per_step": S * 8,
                "d2h_bytes_per_step": int(len(first[1]) * 8),
                "note": "qvb_batch_sample from host seeds (wall clock; first batch also copies "
                        "the sorted unique ids back)"},
        "candidates": {"count": info.candidates, "parallel_edges": bool(info.parallel_edges),
                       "max_row": info.max_candidates, "build_ms": info.build_ms,
                       "device_bytes": info.device_bytes},
        "gpu_launches_per_batch": 12 + 8 * len(SAMPLE_FANOUTS),
    }, first


def sampler_cpu(args, cfg, ro, col, w, first):
    """The reference's OpenMP batch_sample on the same graph and first batch."""
    from oracle.oracle import Oracle, RefLib

    ref = RefLib() if RefLib.available() else None
    lib = ref or Oracle()
    if ro is None:
        ro, col, w = Oracle().synthetic_graph(cfg["n"], cfg["e"], 7, cfg["weighted"], False)
    threads = os.cpu_count() or 1
    seeds = sample_seeds(cfg["n"], args.warmup, args.sample_seeds)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        res = lib.batch_sample(ro, col, w, seeds, SAMPLE_FANOUTS, SAMPLE_RNG)
        ts.append(ref.last_ms / 1e3 if ref else time.perf_counter() - t0)
    same = all((a == b).all() for a, b in zip(res, first[0]))
    s = min(ts)
    return {"value": len(res[0]) / s, "unit": "instances/s", "ms_per_batch": s * 1e3,
            "cores": threads if ref else 1, "kind": "reference" if ref else "port",
            "sample": f"qv::batch_sample({args.sample_seeds} seeds, {{15, 10}}, 3) on the "
                      f"{cfg['desc']} graph, best of 3 (transition_view excluded)",
            "identical_to_gpu": bool(same)}


def cpu_baseline(args, cfg, p_host, lut, ro, col, w, steps, req0_plan):
    """Reference CPU path on this host (rank 0, N=1): the reference's own
    compute_access_prob_ie on the full graph (OpenMP, all host threads; also a
    whole-graph bit-identity check of our P), and per collect step the
    reference's plan_reads (single-threaded, as written) on the same lookup
    table plus the row copy it only models (threaded memcpy restatement)."""
    import numpy as np

    from oracle.oracle import Oracle, RefLib

    o = Oracle()
    n, dim = cfg["n"], cfg["dim"]
    threads = os.cpu_count() or 1
    ref = RefLib() if RefLib.available() else None
    if ro is None:
        ro, col, w = o.synthetic_graph(n, cfg["e"], 7, cfg["weighted"], False, threads=threads)
    # P(n,j): the reference call itself (OpenMP, includes its transpose)
    if ref is not None:
        ref.set_threads(threads)
        t0 = time.perf_counter()
        p_ref = ref.access_prob(ro, col, w, cfg["layers"], parallel=True)
        ap_s = time.perf_counter() - t0
        kind = "reference"
    else:
        t0 = time.perf_counter()
        p_ref = o.access_prob(ro, col, w, cfg["layers"])
        ap_s = time.perf_counter() - t0
        kind = "port"
    ap = {"value": cfg["e"] * (cfg["layers"] - 1) / ap_s, "unit": "edges/s (input edges)",
          "cores": threads if kind == "reference" else 1, "kind": kind,
          "sample": f"one qv::compute_access_prob_ie call on the full {cfg['desc']} graph "
                    f"(L={cfg['layers']}, includes the reference's per-call transpose)",
          "seconds": ap_s,
          "bit_identical_nodes": int((p_ref.view(np.uint64) == p_host.view(np.uint64)).sum()),
          "bit_identical_to_gpu": bool((p_ref.view(np.uint64) == p_host.view(np.uint64)).all())}
    del p_ref
    # collect: the reference's read planner (placement.cpp:355-380) on each
    # batch of this rank's lookup table + the byte copy it only models
    loc, off = lut
    x = o.features(n, dim, threads=threads)
    plan_s = gather_s = 0.0
    b = args.batch
    same_plan = None
    for k in range(steps):
        req = o.request_ids(11, k, n, b)
        t0 = time.perf_counter()
        rp = (ref or o).plan_reads(loc, off, req, 8)
        t1 = time.perf_counter()
        o.gather(x, req, threads=threads)
        t2 = time.perf_counter()
        plan_s += t1 - t0
        gather_s += t2 - t1
        if k == 0 and req0_plan is not None:
            same_plan = all((u == v).all() for u, v in zip(rp, req0_plan(req)))
    del x
    payload = steps * b * 4 * dim
    cpu = {"value": payload / (plan_s + gather_s) / 1e9, "unit": "GB/s", "cores": threads,
           "kind": "reference" if ref is not None else "port",
           "sample": f"{steps} batches x {b} uniform ids on the {args.config} table: qv::plan_reads "
                     f"(the reference's collect call, 1 thread) + the row copy it only models "
                     f"(memcpy restatement, {threads} threads)",
           "plan_reads_s": plan_s, "memcpy_s": gather_s,
           "memcpy_only_GBps": payload / gather_s / 1e9,
           "read_plan_identical_to_gpu": same_plan}
    return cpu, ap


def run_reference(args):
    """--impl reference: the reference's own CPU path (oracle/_ref, the
    unmodified sources), rank 0 only, on this arm's workload: its
    compute_access_prob_ie on the full graph, its plan_placement and
    build_lookup_table for the 1-GPU table, then per step its plan_reads on
    a batch plus the row copy it only models (threaded memcpy restatement)."""
    from oracle.oracle import Oracle, RefLib, topology_defaults

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    n, dim, B = cfg["n"], cfg["dim"], args.batch
    o = Oracle()
    ref = RefLib() if RefLib.available() else None
    lib = ref or o
    threads = os.cpu_count() or 1
    if ref:
        ref.set_threads(threads)
    t0 = time.perf_counter()
    ro, col, w = o.synthetic_graph(n, cfg["e"], 7, cfg["weighted"], False, threads=threads)
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    p = ref.access_prob(ro, col, w, cfg["layers"], True) if ref else o.access_prob(ro, col, w, cfg["layers"])
    ap_s = time.perf_counter() - t0
    sampler = None
    if args.sample_seeds:  # qv_bench's batch_sample leg (tools/bench.cpp:89-94)
        seeds = sample_seeds(n, args.warmup, args.sample_seeds)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            res = lib.batch_sample(ro, col, w, seeds, SAMPLE_FANOUTS, SAMPLE_RNG)
            ts.append(ref.last_ms / 1e3 if ref else time.perf_counter() - t0)
        sampler = {"value": len(res[0]) / min(ts), "unit": "instances/s",
                   "ms_per_batch": min(ts) * 1e3, "seeds_per_batch": args.sample_seeds,
                   "cores": threads if ref else 1}
    del ro, col, w
    t = topology_defaults(gpus_per_server=1, gpu_feature_capacity=n, host_feature_capacity=n)
    t0 = time.perf_counter()
    lo, ids = lib.plan_placement(p, t)
    t1 = time.perf_counter()
    loc, off = lib.build_lookup_table(lo, ids, t, 0)
    t2 = time.perf_counter()
    plan_s, lut_s = t1 - t0, t2 - t1
    del lo, ids
    x = o.features(n, dim, threads=threads)
    reqs = [o.request_ids(11, k, n, B) for k in range(args.warmup + args.steps)]
    for k in range(args.warmup):
        lib.plan_reads(loc, off, reqs[k], 8)
        o.gather(x, reqs[k], threads=threads)
    t0 = time.perf_counter()
    for k in range(args.steps):
        lib.plan_reads(loc, off, reqs[args.warmup + k], 8)
        o.gather(x, reqs[args.warmup + k], threads=threads)
    el = time.perf_counter() - t0
    value = args.steps * B * 4 * dim / el / 1e9
    kind = "reference" if ref else "port"
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32 rows copied bit-exact (P in fp64)",
        "data": "synthetic (bench.cpp generator seed 7; SURVEY §8(d) features and request streams)",
        "config": bench_config(args, cfg, world),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": f"each step: qv::plan_reads on a {B}-id batch (reference "
                                   f"code, oracle/_ref, 1 thread as written) + the row copy it only "
                                   f"models (memcpy restatement, {threads} threads)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "access_prob": {"value": cfg["e"] * (cfg["layers"] - 1) / ap_s,
                        "unit": "edges/s (input edges)", "seconds": ap_s, "kind": kind,
                        "cores": threads},
        "planner": {"plan_placement_s": plan_s, "build_lookup_table_s": lut_s, "cores": 1,
                    "graph_generation_s": gen_s},
        "sampler": sampler,
        "host_max_rss_gb": _max_rss_gb(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(CONFIGS), default="C4",
                    help="workload (default: the north-star C4, which fits one B200)")
    ap.add_argument("--batch", type=int, default=1 << 20)
    ap.add_argument("--replicate", type=float, default=0.0)
    ap.add_argument("--host-frac", type=float, default=0.0)
    ap.add_argument("--clock-window", type=float, default=1.0)
    ap.add_argument("--cpu-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sample-seeds", type=int, default=4096,
                    help="seeds per batch_sample call of the sampler leg (0: skip)")
    ap.add_argument("--planned", action="store_true", help="location-bucketed, offset-sorted gather (K4 order)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
