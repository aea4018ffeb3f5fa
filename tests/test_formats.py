"""CPU: on-disk formats are byte-compatible with the reference (SURVEY §8(f)
next row #3): QVCSR1 graphs, edge-list text, QVTAB1/CSV tables and the
placement / lookup-table JSON+CSV exports, compared with files written by the
unmodified reference (oracle/_ref)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.oracle import topology_defaults
from paper_2305_10863_b200 import formats as F
from paper_2305_10863_b200.qvb import ParseError, ValidationError
from tests.util import derive_stream, random_edges

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


@pytest.fixture(scope="module")
def rl(ref):
    L = ref._lib
    L.qvr_save_graph_csr.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, C.c_char_p]
    L.qvr_load_graph.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p]
    L.qvr_save_table_binary.argtypes = [C.c_char_p, f64p, C.c_uint64, C.c_uint64]
    L.qvr_save_table_csv.argtypes = [C.c_char_p, f64p, C.c_uint64]
    L.qvr_placement_exports.argtypes = [u64p, i64p, C.c_uint64, C.c_void_p, C.c_char_p, C.c_char_p]
    L.qvr_lookup_exports.argtypes = [i64p, u64p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_char_p,
                                     C.c_char_p]
    L.qvr_last_error.restype = C.c_char_p
    return L


def ref_load(rl, path, csr, remap=False):
    n, e = C.c_uint64(0), C.c_uint64(0)
    rc = rl.qvr_load_graph(path.encode(), int(csr), int(remap), C.byref(n), C.byref(e), None, None, None)
    if rc:
        return rl.qvr_last_error().decode()
    ro = np.zeros(n.value + 1, np.uint64)
    col = np.zeros(max(e.value, 1), np.uint64)
    w = np.zeros(max(e.value, 1), np.float64)
    rl.qvr_load_graph(path.encode(), int(csr), int(remap), C.byref(n), C.byref(e), ro.ctypes.data,
                      col.ctypes.data, w.ctypes.data)
    return ro, col[: e.value], w[: e.value]


def same_bytes(a, b):
    return open(a, "rb").read() == open(b, "rb").read()


def test_csr_binary_round_trip(rl, oracle, tmp_path):
    ro, col, w = oracle.synthetic_graph(5000, 40000, 7, True)
    ours, theirs = str(tmp_path / "a.qvcsr"), str(tmp_path / "b.qvcsr")
    F.save_graph_csr(ours, ro, col, w)
    rl.qvr_save_graph_csr(len(ro) - 1, len(col), ro, col, w, theirs.encode())
    assert same_bytes(ours, theirs)
    r2, c2, w2 = F.load_graph(theirs)
    assert (r2 == ro).all() and (c2 == col).all() and (w2.view(np.uint64) == w.view(np.uint64)).all()
    # truncated and bad-magic files fail like the reference
    data = open(ours, "rb").read()
    open(str(tmp_path / "t.qvcsr"), "wb").write(data[:-8])
    with pytest.raises(ParseError, match="truncated csr-binary file"):
        F.load_graph(str(tmp_path / "t.qvcsr"))
    assert "truncated" in ref_load(rl, str(tmp_path / "t.qvcsr"), True)
    open(str(tmp_path / "m.qvcsr"), "wb").write(b"XXCSR1" + data[6:])
    with pytest.raises(ParseError, match="bad magic"):
        F.load_graph(str(tmp_path / "m.qvcsr"))


EDGE_LISTS = {
    "plain": "0 1\n1 2 0.5\n# comment\n2 0 2\n\n",
    "remap": "10 30\n30 20 1.5\n",
    "bad_line": "0 1\nfoo\n",
    "bad_weight": "0 1 abc\n",
    "trailing": "0 1 1.0 9\n",
    "one_id": "0\n",
    "empty": "# nothing\n",
    "neg_weight": "0 1 -1\n1 0\n",
    "zero_row": "0 1 0\n1 0\n",
}


@pytest.mark.parametrize("name", list(EDGE_LISTS))
@pytest.mark.parametrize("remap", [False, True])
def test_edge_list_loader_matches_reference(rl, tmp_path, name, remap):
    p = str(tmp_path / f"{name}.txt")
    open(p, "w").write(EDGE_LISTS[name])
    theirs = ref_load(rl, p, False, remap)
    if isinstance(theirs, str):
        with pytest.raises((ParseError, ValidationError)) as ei:
            F.load_graph(p, "edge_list_text", remap)
        assert str(ei.value) == theirs
        return
    ro, col, w = F.load_graph(p, "edge_list_text", remap)
    assert (ro == theirs[0]).all() and (col == theirs[1]).all()
    assert (w.view(np.uint64) == theirs[2].view(np.uint64)).all()


def test_tables_match_reference(rl, tmp_path):
    rng = derive_stream(3, 3)
    v = np.array([rng.uniform() * 10 ** rng.below(12) for _ in range(1000)])
    for fn_ours, fn_ref, ext in [(lambda p: F.save_table_binary(p, v, 3),
                                  lambda p: rl.qvr_save_table_binary(p.encode(), v, len(v), 3), "qvtab"),
                                 (lambda p: F.save_table_csv(p, v),
                                  lambda p: rl.qvr_save_table_csv(p.encode(), v, len(v)), "csv")]:
        a, b = str(tmp_path / f"a.{ext}"), str(tmp_path / f"b.{ext}")
        fn_ours(a)
        fn_ref(b)
        assert same_bytes(a, b), ext
    back, k = F.load_table_binary(str(tmp_path / "b.qvtab"))
    assert k == 3 and (back.view(np.uint64) == v.view(np.uint64)).all()


def test_placement_and_lookup_exports_match_reference(rl, oracle, tmp_path):
    rng = derive_stream(17, 2)
    for it in range(6):
        n = 1 + rng.below(200)
        v = np.array([rng.uniform() for _ in range(n)])
        t = topology_defaults(servers=1 + rng.below(2), numa_per_server=1 + rng.below(2))
        t.gpus_per_server = t.numa_per_server * (1 + rng.below(3))
        t.gpu_feature_capacity = rng.below(20)
        t.host_feature_capacity = rng.below(50)
        t.disk_feature_capacity = n
        t.nvlink_within_numa = rng.below(2)
        t.infiniband = rng.below(2)
        lo, ids = oracle.plan_placement(v, t)
        loc, off = oracle.build_lookup_table(lo, ids, t, 0)
        rj, rc = str(tmp_path / "rp.json"), str(tmp_path / "rp.csv")
        rl.qvr_placement_exports(lo, ids, n, C.addressof(t), rj.encode(), rc.encode())
        assert F.placement_to_json_text(lo, ids, t) == open(rj).read()
        F.save_placement_csv(str(tmp_path / "op.csv"), lo, ids, t)
        assert same_bytes(str(tmp_path / "op.csv"), rc)
        lj, lc = str(tmp_path / "rl.json"), str(tmp_path / "rl.csv")
        rl.qvr_lookup_exports(loc, off, n, 0, t.gpus_per_server, lj.encode(), lc.encode())
        assert F.lookup_to_json_text(loc, off, 0, t.gpus_per_server) == open(lj).read()
        F.save_lookup_csv(str(tmp_path / "ol.csv"), loc, off)
        assert same_bytes(str(tmp_path / "ol.csv"), lc)


def test_from_edges_matches_oracle(oracle):
    rng = derive_stream(23, 1)
    for _ in range(20):
        n, s, d, w = random_edges(rng, 50, 300, True)
        a = F.from_edges(n, s, d, w)
        b = oracle.build_csr(n, s, d, w)
        assert all((x == y).all() for x, y in zip(a, b))
