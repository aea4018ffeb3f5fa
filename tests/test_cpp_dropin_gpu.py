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
def test_dropin_reference_cases(qvb):
    exe = build_test_binary()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failed" in r.stdout
