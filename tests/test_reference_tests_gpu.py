"""The reference's OWN unit tests, compiled unchanged against the qv:: drop-in.

oracle/Makefile `reftests` compiles /root/reference/proj/tests/test_metrics.cpp,
test_placement.cpp, test_graph.cpp and test_sampler.cpp — unmodified — with
include shims that map qv/{graph,metrics,placement,sampler,topology,error}.hpp
to paper_2305_10863_b200/cpp/qv_b200.hpp and a minimal doctest stand-in
(oracle/reftests/doctest.h). The binary (oracle/_ref/reftests_dropin) is built
where the reference exists and travels to the GPU box; every drop-in call in
it runs on the B200.

Filtered out (outside the north-star path, see oracle/reftests/shim_stubs.cpp):
the pure-PSGS cases (they would test the shim's stand-in), topology JSON
round-trip (config parsing) and the Monte-Carlo oracle cases.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "reftests_dropin")
EXCLUDE = [
    "worked subgraph-size example*", "chain with unit fanouts*", "isolated node has subgraph size 1",
    "psgs values are at least 1", "sparse horner psgs*",
    "topology json round trips*",
    "tree-size oracle*", "walk oracle*",
]


def _need_binary():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/reftests_dropin not built (needs /root/reference at build time)")


def test_reference_test_binary_links():
    """CPU: the binary exists where the reference was present and resolves
    the in-tree drop-in libraries."""
    _need_binary()
    r = subprocess.run(["ldd", EXE], capture_output=True, text=True)
    assert "libqv_b200.so" in r.stdout and "not found" not in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_dropin(qvb):
    _need_binary()
    r = subprocess.run([EXE, "-tce=" + ",".join(EXCLUDE)], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-8000:])
    m = re.search(r"test cases: (\d+) passed, (\d+) failed, (\d+) skipped", r.stdout)
    assert m, r.stdout
    passed, failed, skipped = map(int, m.groups())
    assert failed == 0 and r.returncode == 0, r.stderr[-8000:]
    # 17 metrics + 19 placement + 12 graph + 14 sampler cases, 12 filtered out
    assert passed == 50 and skipped == 12, (passed, skipped)
