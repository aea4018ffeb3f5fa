"""bench.py contract pieces that need no GPU: the default workload is the
north-star C4 config (BASELINE.json configs[3]), both arms build the same
`config`, traffic is keyed by the exact workload, and the P leg's roofline
arithmetic follows SURVEY §8(d)."""
import argparse
import json
import os
import types

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _args(**kw):
    a = dict(config="C4", batch=1 << 20, replicate=0.0, host_frac=0.0)
    a.update(kw)
    return argparse.Namespace(**a)


def test_default_workload_is_the_north_star_config():
    c4 = bench.CONFIGS["C4"]
    assert (c4["n"], c4["e"], c4["dim"], c4["layers"], c4["weighted"]) == (111_000_000, 1_600_000_000, 128, 3, False)
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert "111M nodes, 1.6B edges, 128-dim" in base["configs"][3]
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--config", choices=list(CONFIGS), default="C4"' in src


def test_both_arms_share_one_config_builder():
    a = bench.bench_config(_args(), bench.CONFIGS["C4"], 1)
    b = bench.bench_config(_args(), bench.CONFIGS["C4"], 1)
    assert a == b and a["workload"].startswith("C4 ogbn-papers100M-shaped")
    assert a["features_partitioned_over"] == 1 and a["batch"] == 1 << 20
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count("bench_config(args, cfg, world)") >= 2  # ours and the reference arm


def test_traffic_is_keyed_by_the_exact_workload():
    assert bench.traffic_key(_args(), 1) == "C4|b1048576|r0|h0|n1"
    assert bench.traffic_key(_args(host_frac=0.25), 1) == "C4|b1048576|r0|h0.25|n1"
    t = bench.load_traffic("C4|b1048576|r0|h0|n1")
    assert t and all(v > 0 for v in t.values())
    assert bench.load_traffic("C4|b1|r0|h0|n1") == {}  # never another workload's capture


def test_access_prob_roofline_arithmetic():
    n, eu, cols, nseg, slots = 1000, 14000, 14000, 2, 20000
    info = types.SimpleNamespace(unique_edge_count=eu, segment_columns=cols, segments=nseg,
                                 first_slots=slots, layout=0, exception_count=0, classes=10,
                                 build_ms=1.0, device_bytes=1)
    ph = {"first": 0.010, "gather": 0.040, "products": 0.020, "other": 0.0, "launches": 4}
    pk = {"hbm_gbs": 6500.0, "source": "test"}
    cfg = {"n": n, "e": eu}
    line = bench.access_prob_line(cfg, info, 3, [0.08, 0.08], [0.075], [ph], pk)
    t_roof = bench.bytes_per_sweep(eu, n, False) * 2 / (6500.0 * 1e9) * 1e3
    assert abs(line["survey_model"]["frac"] - t_roof / 0.08) < 1e-12
    assert line["roofline"]["kernel"] == "k_codes"  # the dominant phase
    k = line["kernels"]["k_codes"]
    assert abs(k["gathers_per_s"] - cols / 0.040e-3) < 1e-3 * k["gathers_per_s"]
    assert abs(k["frac_gather_ceiling"] - k["gathers_per_s"] / bench.GATHER_CEILING) < 1e-12
    assert abs(line["value"] - eu * 2 / 0.08e-3) < 1e-6 * line["value"]
