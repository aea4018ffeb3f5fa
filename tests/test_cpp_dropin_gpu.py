"""The qv:: C++ drop-in (what a reference user links) passes the reference's
own hot-path test cases (tests/cpp/test_dropin.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2305_10863_b200")


def build_test_binary():
    from oracle.oracle import build as build_oracle
    from paper_2305_10863_b200 import build

    build.build()
    build_oracle(ref=False)
    out = os.path.join(ROOT, "build", "test_dropin")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-o", out, src, "-L" + PKG, "-lqv_b200", "-lqvb",
           "-L" + os.path.join(ROOT, "oracle"), "-loracle",
           "-Wl,-rpath," + PKG + ":" + os.path.join(ROOT, "oracle")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_dropin_compiles_against_headers():
    build_test_binary()


@pytest.mark.gpu
def test_dropin_reference_cases(qvb, tmp_path):
    import json

    import numpy as np

    from paper_2305_10863_b200 import formats as F
    from tests.util import fig8_edges

    exe = build_test_binary()
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failed" in r.stdout
    # the C++ exports are byte-identical to the reference's own (golden texts)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["exports_b"]
    for name, key in [("placement_b.json", "placement_json"), ("placement_b.csv", "placement_csv"),
                      ("lookup_b.json", "lookup_json"), ("lookup_b.csv", "lookup_csv")]:
        assert open(tmp_path / name).read() == gold[key], name
    n, s, d, w = fig8_edges()
    ro, col, ww = F.from_edges(n, s, d, w)
    F.save_graph_csr(str(tmp_path / "py.qvcsr"), ro, col, ww)
    assert open(tmp_path / "py.qvcsr", "rb").read() == open(tmp_path / "fig8.qvcsr", "rb").read()
    tab = np.array([0.5, 1.0 / 3.0, 1e-300, 12345.678])
    F.save_table_binary(str(tmp_path / "py.qvtab"), tab, 2)
    F.save_table_csv(str(tmp_path / "py.csv"), tab)
    assert open(tmp_path / "py.qvtab", "rb").read() == open(tmp_path / "table.qvtab", "rb").read()
    assert open(tmp_path / "py.csv").read() == open(tmp_path / "table.csv").read()
