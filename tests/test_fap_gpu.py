"""FAP estimator on the GPU vs the oracle and the
reference goldens, bit for bit (metrics.cpp:95-132, test_metrics.cpp)."""
import hashlib
import json
import os

import numpy as np
import pytest

from tests.util import CONFIGS, bits, derive_stream, fig8_edges, random_edges

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def hexs(a):
    return [f"{int(x):016x}" for x in bits(a)]


def test_fap_fig8_golden(qvb, oracle):
    n, s, d, w = fig8_edges()
    ro, col, ww = oracle.build_csr(n, s, d, w)
    for K, gold in GOLD["fap_fig8"].items():
        assert hexs(qvb.compute_fap(ro, col, ww, int(K)).values) == gold
    sd = GOLD["fap_fig8_seeded"]
    assert hexs(qvb.compute_fap(ro, col, ww, 2, np.array(sd["seed"])).values) == sd["values"]


@pytest.mark.parametrize("weighted", [False, True])
def test_fap_random_bit_exact(qvb, oracle, weighted):
    rng = derive_stream(83, int(weighted))
    for it in range(30):
        n, s, d, w = random_edges(rng, 60, 400, weighted)
        ro, col, ww = oracle.build_csr(n, s, d, w)
        seed = None
        if it % 3 == 0:
            x = np.array([rng.uniform() for _ in range(n)])
            seed = x / x.sum()
        for hops in range(4):
            got = qvb.compute_fap(ro, col, ww if weighted else None, hops, seed).values
            exp = oracle.compute_fap(ro, col, ww, hops, seed)
            assert (bits(got) == bits(exp)).all(), (it, hops)


@pytest.mark.parametrize("name,weighted,transposed,hops", [("uniform_K2", False, False, 2),
                                                           ("weighted_K3", True, False, 3)])
def test_fap_c1_golden(qvb, oracle, name, weighted, transposed, hops):
    c = CONFIGS["C1"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, weighted, transposed)
    got = qvb.compute_fap(ro, col, w, hops).values
    assert hashlib.sha256(got.tobytes()).hexdigest() == GOLD["fap_c1"][name]


def test_fap_transposed_hubs_and_c2(qvb, oracle):
    c = CONFIGS["C1"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, True)  # in-degree hubs: long rows
    assert (bits(qvb.compute_fap(ro, col, w, 3).values) == bits(oracle.compute_fap(ro, col, w, 3))).all()
    c = CONFIGS["C2"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, False)
    assert (bits(qvb.compute_fap(ro, col, None, 2).values) == bits(oracle.compute_fap(ro, col, w, 2))).all()


def test_fap_errors(qvb, oracle):
    n, s, d, w = fig8_edges()
    ro, col, ww = oracle.build_csr(n, s, d, w)
    with pytest.raises(qvb.ValidationError, match="negative mass"):
        qvb.compute_fap(ro, col, ww, 2, -np.ones(6))
    with pytest.raises(qvb.ValidationError, match="does not sum to 1"):
        qvb.compute_fap(ro, col, ww, 2, np.ones(6))
    with pytest.raises(qvb.ValidationError, match="size"):
        qvb.compute_fap(ro, col, ww, 2, np.ones(3) / 3)
