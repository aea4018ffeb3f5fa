"""K1 fused passes (k_pass_fused, the opt-in QVB_PRODUCTS=fused A/B path; the
default decoupled sweep measured faster, profiles/r02/r02an_fused_passes.md):
one launch per source segment gathers the codes into shared memory and
multiplies each node's run into the running product carried between passes. Same factors in the same
order as the reference (metrics.cpp:152-168): bit-identical to the oracle and
to the decoupled k_codes + k_products_tma sweep."""
import numpy as np
import pytest

from tests.util import CONFIGS, bits, derive_stream, random_edges

pytestmark = pytest.mark.gpu


@pytest.fixture
def fused(monkeypatch):
    monkeypatch.setenv("QVB_PRODUCTS", "fused")
    monkeypatch.setenv("QVB_SEG_LAYOUT", "nm")
    return monkeypatch


@pytest.mark.parametrize("seg_sources", ["1", "7", "1000", "31337"])
def test_fused_segmented_bit_exact(qvb, oracle, fused, seg_sources):
    """Many source segments on small graphs (markers: C1's y exceed the code
    range; exceptions: parallel edges of the transposed generator)."""
    fused.setenv("QVB_SEG_SOURCES", seg_sources)
    if seg_sources in ("1", "7"):
        rng = derive_stream(83, int(seg_sources))
        for _ in range(10):
            n, s, d, w = random_edges(rng, 40 if seg_sources == "7" else 200, 250, True)
            if (n + int(seg_sources) - 1) // int(seg_sources) > 255:
                continue
            ro, col, ww = oracle.build_csr(n, s, d, w)
            g = qvb.DeviceGraph.upload(ro, col, None)
            for layers in (2, 3, 4):
                exp = oracle.access_prob(ro, col, np.ones_like(ww), layers)
                assert (bits(g.access_prob(layers)) == bits(exp)).all()
            g.close()
        return
    c = CONFIGS["C1"]
    for transposed in (False, True):
        ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, transposed)
        g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, transposed)
        for layers in (2, 3, 4):
            assert (bits(g.access_prob(layers)) == bits(oracle.access_prob(ro, col, w, layers))).all()
        g.close()


@pytest.mark.parametrize("cap", [None, "0", "700"])
def test_fused_c2_segments_bit_exact(qvb, oracle, fused, cap):
    """C2 in 4 MiB segments; cap forces chunks over it onto the unstaged path
    (0: every chunk; 700: a mix)."""
    c = CONFIGS["C2"]
    fused.setenv("QVB_SEG_MB", "4")
    if cap is not None:
        fused.setenv("QVB_FP_CAP", cap)
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, False)
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    for layers in (2, 3):
        assert (bits(g.access_prob(layers)) == bits(oracle.access_prob(ro, col, w, layers))).all()
    g.close()


def test_fused_equals_decoupled_c4(qvb, monkeypatch):
    """The north-star graph: fused and decoupled sweeps give the same bits."""
    c = CONFIGS["C4"]
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    monkeypatch.delenv("QVB_PRODUCTS", raising=False)
    exp = g.access_prob(c["layers"])
    monkeypatch.setenv("QVB_PRODUCTS", "fused")
    got = g.access_prob(c["layers"])
    g.close()
    assert (bits(got) == bits(exp)).all()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_sharded_c2_bit_exact(qvb, fused, world):
    """Row-sharded fused sweeps (ranks as threads on one GPU): every rank ends
    with the single-GPU answer."""
    from tests.test_sharded_p_gpu import run_threads
    c = CONFIGS["C2"]
    fused.setenv("QVB_SEG_MB", "4")
    fused.setenv("QVB_F1_WINDOW", "32")
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    exp = g.access_prob(3)
    g.close()
    out, flags = run_threads(qvb, lambda: qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False), 3, world)
    assert all(flags)
    for r in range(world):
        assert (bits(out[r]) == bits(exp)).all(), r
