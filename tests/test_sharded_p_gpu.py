"""Row-sharded P(n,j) (one exchange step per layer).

Ranks compute their node chunks of every sweep and exchange P_j (and the
codes the next sweep gathers) in place; the result must be bit-identical to
the single-GPU call. On a one-GPU box the ranks are threads, each with its
own copy of the device graph, and the exchange copies the other ranks'
chunks device to device behind a barrier — the same library entry point and
callback contract the NCCL exchange (paper_2305_10863_b200.dist) drives on a
multi-GPU node.
"""
import threading

import numpy as np
import pytest

from tests.util import CONFIGS, bits

pytestmark = pytest.mark.gpu


class _Dev:
    def __init__(self, ptr, count, ts):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": ts, "data": (ptr, False),
                                         "version": 3}


def run_threads(qvb, make_graph, layers, world):
    import torch

    graphs = [make_graph() for _ in range(world)]
    reg = [None] * world
    bar = threading.Barrier(world)
    out, flags, errs = [None] * world, [None] * world, []

    def exchange_for(rank):
        def ex(layer, p, codes, chunk, stream):
            torch.cuda.synchronize()  # this rank's sweep is done
            reg[rank] = (p, codes)
            bar.wait()
            for ptr_i, ts in ((0, "<f8"), (1, "<i4")):
                if reg[rank][ptr_i] is None or not reg[rank][ptr_i]:
                    continue
                mine = torch.as_tensor(_Dev(reg[rank][ptr_i], world * chunk, ts), device="cuda")
                for o in range(world):
                    if o != rank:
                        theirs = torch.as_tensor(_Dev(reg[o][ptr_i], world * chunk, ts), device="cuda")
                        mine[o * chunk:(o + 1) * chunk].copy_(theirs[o * chunk:(o + 1) * chunk])
            torch.cuda.synchronize()
            bar.wait()  # nobody overwrites a buffer another rank still reads
        return ex

    def work(rank):
        try:
            out[rank], flags[rank] = graphs[rank].access_prob_sharded(layers, rank, world, exchange_for(rank))
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for g in graphs:
        g.close()
    assert not errs, errs
    return out, flags


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_c2_node_major_bit_exact(qvb, monkeypatch, world):
    c = CONFIGS["C2"]
    monkeypatch.setenv("QVB_SEG_MB", "4")       # node-major segmented layout at C2 size
    monkeypatch.setenv("QVB_F1_WINDOW", "32")   # first-sweep slices in node order
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    exp = {L: g.access_prob(L) for L in (1, 2, 3)}
    g.close()
    for layers in (1, 2, 3):
        out, flags = run_threads(qvb, lambda: qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False),
                                 layers, world)
        for r in range(world):
            assert (bits(out[r]) == bits(exp[layers])).all(), (layers, r)
        assert all(flags) == (layers >= 2), flags  # split when there is a sweep


def test_sharded_falls_back_on_other_layouts(qvb, oracle):
    """Weighted or sliced layouts compute every node on every rank (no
    exchange); the answer is still the reference's."""
    c = CONFIGS["C1"]
    ro, col, w = oracle.synthetic_graph(c["n"], c["e"], 7, True, False)
    exp = oracle.access_prob(ro, col, w, 3)
    out, flags = run_threads(qvb, lambda: qvb.DeviceGraph.upload(ro, col, w), 3, 2)
    assert not any(flags)
    for r in range(2):
        assert (bits(out[r]) == bits(exp)).all()


def test_sharded_world_one_is_the_plain_call(qvb):
    c = CONFIGS["C1"]
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    p = g.access_prob(3)
    q, sharded = g.access_prob_sharded(3, 0, 1, None)
    assert (bits(p) == bits(q)).all() and not sharded
    with pytest.raises(qvb.ValidationError):
        g.access_prob_sharded(3, 2, 2, lambda *a: None)
    g.close()


def test_sharded_c4_full_size_bit_exact(qvb):
    """Papers scale (C4: 111M nodes, 1.6B edges, its default node-major
    layout): two ranks' sharded 3-layer pass equals the one-GPU pass on all
    111M nodes."""
    c = CONFIGS["C4"]
    g = qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False)
    exp = g.access_prob(3)
    g.close()
    out, flags = run_threads(qvb, lambda: qvb.DeviceGraph.synthetic(c["n"], c["e"], 7, False, False), 3, 2)
    assert all(flags)
    for r in range(2):
        assert (bits(out[r]) == bits(exp)).all(), r
