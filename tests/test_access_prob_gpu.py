"""K1 parity: the device P(n,j) against the CPU oracle, bit for bit.

Mirrors the reference's own P(n,j) tests (tests/test_metrics.cpp:136-235,
acceptance.cpp:156-173) and adds the BASELINE configs. The bar is
bit-identical fp64 (north_star allows 1e-9 relative; SURVEY §0 shows only a
bit-exact P keeps the placement/LUT exact, so that is what we test).
"""
import os

import numpy as np
import pytest

from tests.util import c4_reference_enabled, CONFIGS, bits, derive_stream, fig8_edges, random_edges

pytestmark = pytest.mark.gpu

GOLD_FIG8 = {  # SURVEY §8(c), produced by the reference (tests/golden/golden.json)
    2: [0.30555555555555552, 0.16666666666666666, 0.30555555555555552, 0.36342592592592593,
        0.16666666666666666, 0.23611111111111113],
    3: [0.42129629629629622, 0.16666666666666666, 0.55793467078189296, 0.55056691529492463,
        0.16666666666666666, 0.35281635802469136],
}


def _csr(oracle, n, src, dst, w):
    return oracle.build_csr(n, src, dst, w)


def test_fig8_golden(qvb, oracle):
    ro, col, w = _csr(oracle, *fig8_edges())
    for layers, gold in GOLD_FIG8.items():
        p = qvb.compute_access_prob_ie(ro, col, w, layers).values
        assert (bits(p) == bits(np.array(gold))).all(), (layers, p.tolist())
    p1 = qvb.compute_access_prob_ie(ro, col, w, 1).values
    assert (p1 == 1.0 / 6).all()


def test_two_neighbor_parent(qvb, oracle):
    # test_metrics.cpp:143-152
    ro, col, w = _csr(oracle, 3, [1, 1], [0, 2], [1.0, 1.0])
    p = qvb.compute_access_prob_ie(ro, col, w, 2).values
    base = 1.0 / 3.0
    assert abs(p[0] - (base + (1.0 - base) * (base * 0.5))) < 1e-14
    assert (bits(p) == bits(oracle.access_prob(ro, col, w, 2))).all()


@pytest.mark.parametrize("weighted", [True, False])
def test_random_graphs_bit_exact(qvb, oracle, weighted):
    # test_metrics.cpp:154-175 draws; every layer count 1..4, bit-exact.
    rng = derive_stream(59, 5 if weighted else 6)
    for _ in range(40):
        n, s, d, w = random_edges(rng, 40, 250, weighted)
        ro, col, ww = _csr(oracle, n, s, d, w)
        g = qvb.DeviceGraph.upload(ro, col, ww if weighted else None)
        for layers in range(1, 5):
            got = g.access_prob(layers)
            exp = oracle.access_prob(ro, col, ww, layers)
            assert (bits(got) == bits(exp)).all(), (n, layers)
        g.close()


def test_star_and_properties(qvb, oracle):
    # star centre with 5 leaves (test_metrics.cpp:167-174); bounds/monotone (:177-193)
    ro, col, w = _csr(oracle, 6, [1, 2, 3, 4, 5], [0] * 5, [1.0] * 5)
    p = qvb.compute_access_prob_ie(ro, col, w, 2).values
    assert (bits(p) == bits(oracle.access_prob(ro, col, w, 2))).all()
    rng = derive_stream(61, 6)
    for _ in range(10):
        n, s, d, ww = random_edges(rng, 30, 200, True)
        ro, col, ww = _csr(oracle, n, s, d, ww)
        g = qvb.DeviceGraph.upload(ro, col, ww)
        prev = None
        for j in range(1, 5):
            v = g.access_prob(j)
            assert (v >= 0).all() and (v <= 1 + 1e-15).all()
            if prev is not None:
                assert (v >= prev - 1e-15).all()
            prev = v
        g.close()


def test_zero_edges_and_isolated(qvb, oracle):
    ro = np.zeros(5, np.uint64)
    p = qvb.compute_access_prob_ie(ro, np.zeros(0, np.uint64), None, 3).values
    assert (p == 0.25).all()


def test_errors(qvb, oracle):
    ro, col, w = _csr(oracle, *fig8_edges())
    with pytest.raises(qvb.ValidationError):
        qvb.compute_access_prob_ie(ro, col, w, 0)
    bad = col.copy()
    bad[2] = 99
    with pytest.raises(qvb.ValidationError, match="column index out of range at node 1"):
        qvb.compute_access_prob_ie(ro, bad, w, 2)
    neg = w.copy()
    neg[3] = -1.0
    with pytest.raises(qvb.ValidationError, match="negative or NaN edge weight at node 3"):
        qvb.compute_access_prob_ie(ro, col, neg, 2)
    zero = w.copy()
    zero[0] = zero[1] = 0.0
    with pytest.raises(qvb.ValidationError, match="node 0 has out-edges but all weights are zero"):
        qvb.compute_access_prob_ie(ro, col, zero, 2)
    with pytest.raises(qvb.ValidationError, match="empty graph"):
        qvb.compute_access_prob_ie(np.zeros(1, np.uint64), np.zeros(0, np.uint64), None, 2)
    nm = ro.copy()
    nm[1], nm[2] = nm[2], nm[1]
    with pytest.raises(qvb.ValidationError):
        qvb.compute_access_prob_ie(nm, col, w, 2)


@pytest.mark.parametrize("weighted,transposed,layers", [(False, False, 2), (False, False, 3),
                                                        (True, False, 3), (False, True, 3),
                                                        (True, True, 2)])
def test_c1_bit_exact(qvb, oracle, weighted, transposed, layers):
    c = CONFIGS["C1"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, weighted, transposed)
    exp = oracle.access_prob(ro, col, w, layers)
    got = qvb.compute_access_prob_ie(ro, col, w, layers).values
    assert (bits(got) == bits(exp)).all()
    # the device generator builds the identical graph
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, weighted, transposed)
    assert (bits(g.access_prob(layers)) == bits(exp)).all()
    info = g.info()
    assert info.edge_count == c["e"]
    g.close()


def test_c2_bit_exact(qvb, oracle):
    c = CONFIGS["C2"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, False)
    exp = oracle.access_prob(ro, col, w, 2)
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    assert (bits(g.access_prob(2)) == bits(exp)).all()
    g.close()


def test_concurrent_calls_on_one_graph(qvb):
    """qvb_access_prob from several threads, each on its own stream, into
    device buffers on one graph (it reuses its sweep buffers): every result
    equals the serial one bit for bit."""
    import threading

    import torch

    c = CONFIGS["C2"]
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    ref = g.access_prob(3)
    outs = {}

    def work(tid):
        s = torch.cuda.Stream()
        res = []
        for k in range(6):
            o = torch.empty(c["n"], dtype=torch.float64, device="cuda")
            g.access_prob(2 + (tid + k) % 2, out=o, stream=s)
            res.append((2 + (tid + k) % 2, o))
        s.synchronize()
        outs[tid] = res

    th = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    ref2 = g.access_prob(2)
    g.close()
    for res in outs.values():
        for layers, o in res:
            assert (bits(o.cpu().numpy()) == bits(ref if layers == 3 else ref2)).all()


def test_layouts_exercised(qvb, oracle):
    # unit weights with parallel edges -> compact layout with exceptions;
    # real weights -> weighted layout
    c = CONFIGS["C1"]
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    i = g.info()
    assert i.layout == 0 and i.exception_count > 0 and i.unique_edge_count < c["e"]
    g.close()
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, True, False)
    assert g.info().layout == 1
    g.close()


def test_unit_weights_mostly_parallel_take_weighted_layout(qvb, oracle):
    """Unit weights where most unique edges are coalesced parallel edges:
    too many exceptions for the compact layout, so the weighted layout is
    built from unit weights (single edges' R filled from 1/row_sum)."""
    rng = derive_stream(577, 1)
    n = 3000
    src, dst = [], []
    for _ in range(40000):
        s, d = rng.below(n), rng.below(n)
        for _ in range(1 + rng.below(3)):  # 1-3 parallel copies
            src.append(s)
            dst.append(d)
    ro, col, w = oracle.build_csr(n, src, dst, [1.0] * len(src))
    g = qvb.DeviceGraph.upload(ro, col, None)
    assert g.info().layout == 1
    for layers in (2, 3, 4):
        assert (bits(g.access_prob(layers)) == bits(oracle.access_prob(ro, col, w, layers))).all()
    g.close()


@pytest.mark.parametrize("layout", ["nm", "slices"])
@pytest.mark.parametrize("seg_sources", ["1", "7", "1000", "31337"])
def test_segmented_passes_bit_exact(qvb, oracle, seg_sources, layout, monkeypatch):
    """Force many source segments (passes carrying the running product in
    source order) on small graphs: results must stay bit-identical, for the
    node-major passes (default) and the per-pass degree-sorted slices."""
    monkeypatch.setenv("QVB_SEG_SOURCES", seg_sources)
    monkeypatch.setenv("QVB_SEG_LAYOUT", layout)
    rng = derive_stream(79, int(seg_sources))
    if seg_sources in ("1", "7"):  # <= 255 segments: tiny graphs only
        for _ in range(10):
            n, s, d, w = random_edges(rng, 40 if seg_sources == "7" else 200, 250, True)
            if (n + int(seg_sources) - 1) // int(seg_sources) > 255:
                continue
            ro, col, ww = _csr(oracle, n, s, d, w)
            for weighted in (True, False):
                g = qvb.DeviceGraph.upload(ro, col, ww if weighted else None)
                for layers in (2, 3, 4):
                    exp = oracle.access_prob(ro, col, ww if weighted else np.ones_like(ww), layers)
                    assert (bits(g.access_prob(layers)) == bits(exp)).all()
                g.close()
        return
    c = CONFIGS["C1"]
    for weighted, transposed in [(False, False), (True, False), (False, True)]:
        ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, weighted, transposed)
        g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, weighted, transposed)
        for layers in (2, 3):
            assert (bits(g.access_prob(layers)) == bits(oracle.access_prob(ro, col, w, layers))).all()
        g.close()


@pytest.mark.parametrize("weighted", [False, True])
def test_c2_node_major_segments_bit_exact(qvb, oracle, weighted, monkeypatch):
    """C2 split into several source segments (node-major passes). Unweighted
    P values straddle the 4-byte code range (y < 2^-22 coded, larger y
    gathered), so both operand paths run; weighted streams R per edge."""
    c = CONFIGS["C2"]
    monkeypatch.setenv("QVB_SEG_MB", "4")
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, weighted, False)
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, weighted, False)
    for layers in (2, 3):
        assert (bits(g.access_prob(layers)) == bits(oracle.access_prob(ro, col, w, layers))).all()
    g.close()


@pytest.mark.parametrize("bufw", ["160", "928"])
def test_products_small_staging_buffer(qvb, oracle, bufw, monkeypatch):
    """k_products_tma with a staging buffer smaller than most slices
    (QVB_PT_BUFW): slices that outgrow it take the global lock-step path,
    the rest the staged one; C2 node-major segments stay bit-exact."""
    c = CONFIGS["C2"]
    monkeypatch.setenv("QVB_SEG_MB", "4")
    monkeypatch.setenv("QVB_PT_BUFW", bufw)
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, False)
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    assert (bits(g.access_prob(3)) == bits(oracle.access_prob(ro, col, w, 3))).all()
    g.close()


def test_c3_weighted_bit_exact(qvb, oracle):
    """C3 (Reddit-shaped, 233K nodes, 114M edges, 3-layer edge-weighted) at full size."""
    c = CONFIGS["C3"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, True, False)
    exp = oracle.access_prob(ro, col, w, 3)
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, True, False)
    assert g.info().layout == 1
    assert (bits(g.access_prob(3)) == bits(exp)).all()
    g.close()


def test_c4_segmented_equals_single_pass(qvb, monkeypatch):
    """C4 (papers-shaped, 111M nodes, 1.6B edges): the source-segmented sweep
    (14 passes carrying the running products) and a single-pass sweep over
    the same device graph are bit-identical, and P obeys its invariants."""
    c = CONFIGS["C4"]
    monkeypatch.setenv("QVB_SEG_MB", "64")
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    p_seg = g.access_prob(3)
    g.close()
    monkeypatch.setenv("QVB_SEG_MB", "4096")
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    p_one = g.access_prob(3)
    p2 = g.access_prob(2)
    g.close()
    assert (bits(p_seg) == bits(p_one)).all()
    assert (p_one >= p2).all() and (p2 >= 1.0 / c["n"]).all() and (p_one <= 1.0).all()


@pytest.mark.parametrize("first", ["classes", "gather", "classes-w32"])
def test_first_sweep_paths_bit_exact(qvb, oracle, first, monkeypatch):
    """The first sweep streams 2-byte out-degree classes (P(s,1) is uniform,
    so a factor depends on its source only through 1/row_sum); QVB_FIRST=gather
    keeps the gathering first sweep. Both bit-identical to the oracle on
    random graphs with parallel edges (exceptions), unit weights given as a
    weight array, and C1 (uniform / transposed)."""
    if first == "gather":
        monkeypatch.setenv("QVB_FIRST", "gather")
    if first == "classes-w32":  # unsorted slices of 32 in node order (the large-graph layout)
        monkeypatch.setenv("QVB_F1_WINDOW", "32")
    rng = derive_stream(61, 1)
    for trial in range(30):
        n, s, d, w = random_edges(rng, 60, 300, False)
        ro, col, ww = _csr(oracle, n, s, d, w)
        g = qvb.DeviceGraph.upload(ro, col, None if trial % 2 else ww)
        info = g.info()
        assert (info.classes > 0) == (first != "gather" and info.layout == 0)
        for layers in (2, 3):
            assert (bits(g.access_prob(layers)) == bits(oracle.access_prob(ro, col, ww, layers))).all()
        g.close()
    c = CONFIGS["C1"]
    for transposed in (False, True):
        ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, transposed)
        g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, transposed)
        assert g.info().exception_count > 0
        for layers in (2, 3):
            assert (bits(g.access_prob(layers)) == bits(oracle.access_prob(ro, col, w, layers))).all()
        g.close()


def _coalesced_rows(oracle, ro, col, w, nodes):
    """The reference's per-node factor list (metrics.cpp:152-166): in-row of
    the transpose, parallel edges merged in order, R = w_sum / row_sum(s)."""
    tro, tcol, tw = oracle.in_adjacency(ro, col, w)
    rs = oracle.row_sums(ro, w)
    out = []
    for v in nodes:
        a, b = int(tro[v]), int(tro[v + 1])
        row, k = [], a
        while k < b:
            s, wt = int(tcol[k]), tw[k]
            k += 1
            while k < b and int(tcol[k]) == s:
                wt += tw[k]
                k += 1
            row.append((s, wt / rs[s]))
        out.append(row)
    return out


@pytest.mark.parametrize("weighted", [False, True])
def test_in_rows_match_reference_rows(qvb, oracle, weighted, monkeypatch):
    """qvb_graph_in_rows (the rows the node-major sweeps multiply) equals the
    reference's coalesced in-rows, sources and R bit for bit, on C1 forced
    into many source segments."""
    monkeypatch.setenv("QVB_SEG_SOURCES", "9000")
    c = CONFIGS["C1"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, weighted, False)
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, weighted, False)
    assert g.info().segments > 1
    rng = np.random.default_rng(5)
    nodes = np.unique(np.concatenate([rng.integers(0, c["n"], 3000), [0, c["n"] - 1]]))
    rp, src, R = g.in_rows(nodes)
    exp = _coalesced_rows(oracle, ro, col, w, nodes)
    for i, row in enumerate(exp):
        a, b = int(rp[i]), int(rp[i + 1])
        assert [int(x) for x in src[a:b]] == [s for s, _ in row]
        assert (bits(R[a:b]) == bits(np.array([r for _, r in row]))).all()
    g.close()


def test_c4_sampled_against_oracle(qvb, oracle):
    """C4 at full size (111M nodes, 1.6B edges, 3 layers) against the oracle's
    restatement on a sample of 20,000 nodes, layer by layer: P(v,2) from the
    uniform P(.,1), and P(v,3) from the device's P(.,2) (itself checked on the
    sample), each over the in-row the device multiplies — bit for bit. This
    checks the first sweep (class stream), the per-segment code gathers and
    the ordered products at the configuration they are built for."""
    c = CONFIGS["C4"]
    n = c["n"]
    g = qvb.DeviceGraph.synthetic(n, c["e"], 7, False, False)
    assert g.info().segments > 1 and g.info().classes > 0
    p2 = g.access_prob(2)
    p3 = g.access_prob(3)
    rng = np.random.default_rng(11)
    nodes = np.unique(np.concatenate([rng.integers(0, n, 20000), [0, 1, n // 2, n - 1]]))
    rp, src, R = g.in_rows(nodes)
    g.close()
    tro = np.zeros(n + 1, np.uint64)
    tro[nodes.astype(np.int64) + 1] = np.diff(rp)
    np.cumsum(tro, out=tro)
    assert int(tro[-1]) == len(src)
    ones = np.ones(n, np.float64)
    base = np.full(n, 1.0 / n)
    exp2 = oracle.sweep_nodes(tro, src.astype(np.uint64), R, ones, base, nodes)
    assert (bits(p2[nodes]) == bits(exp2)).all()
    exp3 = oracle.sweep_nodes(tro, src.astype(np.uint64), R, ones, p2, nodes)
    assert (bits(p3[nodes]) == bits(exp3)).all()


@pytest.mark.skipif(not c4_reference_enabled(),
                    reason="needs >= 150 GB host RAM (QVB_C4_REFERENCE=1 forces, =0 skips)")
def test_c4_full_against_reference():
    """All 111M C4 nodes against the unmodified reference's own
    compute_access_prob_ie (oracle/_ref, 16 threads), from one host CSR."""
    from oracle.oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    from paper_2305_10863_b200 import qvb

    c = CONFIGS["C4"]
    ro, col, w = qvb.synthetic_csr(c["n"], c["e"], 7, False, False)
    p = qvb.compute_access_prob_ie(ro, col, None, c["layers"]).values
    ref = RefLib()
    ref.set_threads(os.cpu_count() or 1)
    exp = ref.access_prob(ro, col, w, c["layers"], parallel=True)
    assert (bits(p) == bits(exp)).all()


def test_concurrent_uploads_and_downloads(qvb, oracle):
    """Several host threads upload graphs and copy P back at once (the staging
    pool gives each large copy its own pinned set): every result exact."""
    import threading

    c = CONFIGS["C2"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, False, False, threads=8)
    exp = oracle.access_prob(ro, col, w, 2)
    res, errs = {}, []

    def run(k):
        try:
            res[k] = qvb.compute_access_prob_ie(ro, col, None, 2).values
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)

    th = [threading.Thread(target=run, args=(k,)) for k in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(6):
        assert (bits(res[k]) == bits(exp)).all()
