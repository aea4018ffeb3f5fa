"""Graph construction, validation and transition_view on the device (the
drop-in's Graph::from_edges / Graph::validate / transition_view) against the
unmodified reference (oracle/_ref): same CSR bytes, same row sums, distinct
out-degrees and parallel-edge flag, same error messages (graph.cpp:16-93,
292-318); and the view's resident device graph gives the reference's P.
"""
import numpy as np
import pytest

from tests.util import derive_stream

pytestmark = pytest.mark.gpu


def random_edges(rng, n_max=60, e_max=400, weighted=True, parallel=True):
    n = 1 + rng.below(n_max)
    e = rng.below(e_max)
    src = np.array([rng.below(n) for _ in range(e)], np.uint64)
    dst = np.array([rng.below(n) for _ in range(e)], np.uint64)
    if parallel and e > 4:
        dst[: e // 4] = dst[e // 4: 2 * (e // 4)]
        src[: e // 4] = src[e // 4: 2 * (e // 4)]
    w = np.array([0.25 + rng.uniform() if weighted else 1.0 for _ in range(e)])
    return n, src, dst, w


def test_from_edges_view_and_p_match_reference(qvb, ref):
    rng = derive_stream(181, 1)
    for it in range(60):
        n, s, d, w = random_edges(rng, weighted=it % 2 == 0, parallel=it % 3 != 0)
        a = qvb.from_edges(n, s, d, w)
        b = ref.from_edges(n, s, d, w)
        assert all((x.view(np.uint64) == y.view(np.uint64)).all() for x, y in zip(a, b))
        ro, col, ww = b
        rs, dist, par = qvb.transition_view(ro, col, ww)
        rs2, dist2, par2 = ref.transition_view(ro, col, ww)
        assert (rs.view(np.uint64) == rs2.view(np.uint64)).all()
        assert (dist == dist2).all() and par == par2
        qvb.graph_validate(ro, col, ww)
        rs3, _, _, g = qvb.transition_view(ro, col, ww, keep=True)
        for layers in (1, 2, 3):
            p = g.access_prob(layers)
            assert (p.view(np.uint64) == ref.access_prob(ro, col, ww, layers).view(np.uint64)).all()
        g.close()


def test_c2_transition_view_matches_reference(qvb, ref):
    from tests.util import CONFIGS

    c = CONFIGS["C2"]
    ro, col, w = qvb.synthetic_csr(c["n"], c["e"], 7, False, False)
    rs, dist, par = qvb.transition_view(ro, col, w)
    rs2, dist2, par2 = ref.transition_view(ro, col, w)
    assert (rs == rs2).all() and (dist == dist2).all() and par == par2 and par


@pytest.mark.parametrize("case", ["endpoint", "weight", "nan"])
def test_from_edges_errors_match_reference(qvb, ref, case):
    n = 5
    s = np.array([0, 1, 2, 3], np.uint64)
    d = np.array([1, 2, 3, 4], np.uint64)
    w = np.array([1.0, 1.0, 1.0, 1.0])
    if case == "endpoint":
        d[2] = 9
        w[3] = -1.0  # a later bad weight must not win
    elif case == "weight":
        w[1] = -2.0
        d[3] = 7
    else:
        w[0] = np.nan
    with pytest.raises(qvb.ValidationError) as e1:
        qvb.from_edges(n, s, d, w)
    from oracle.oracle import OracleError

    with pytest.raises(OracleError) as e2:
        ref.from_edges(n, s, d, w)
    assert str(e1.value) == e2.value.msg


@pytest.mark.parametrize("case", ["mono", "col", "neg", "zero_row", "zero_before_bad"])
def test_validate_errors_match_reference(qvb, ref, case):
    from oracle.oracle import OracleError

    ro = np.array([0, 2, 3, 5, 6], np.uint64)
    col = np.array([1, 2, 0, 3, 1, 0], np.uint64)
    w = np.array([1.0, 2.0, 1.0, 0.5, 0.5, 1.0])
    if case == "mono":
        ro = np.array([0, 3, 2, 5, 6], np.uint64)
    elif case == "col":
        col[4] = 4
    elif case == "neg":
        w[3] = -0.5
    elif case == "zero_row":
        w[2] = 0.0
    else:
        w[2] = 0.0
        col[5] = 9
    with pytest.raises(qvb.ValidationError) as e1:
        qvb.graph_validate(ro, col, w)
    with pytest.raises(OracleError) as e2:
        ref.validate(ro, col, w)
    assert str(e1.value) == e2.value.msg
