"""On-disk / wire formats of the reference, byte-compatible (SURVEY §8(f) next
row #3) — host plumbing around the device path, so files move between
`qvserve` and this library unchanged:

* QVCSR1 graphs (graph.cpp:197-258) and the edge-list text loader
  (graph.cpp:112-195) with its ParseError/ValidationError messages;
* QVTAB1 tables and `node_id,value` CSV (metrics.cpp:203-250);
* placement / lookup-table JSON (nlohmann ordered_json dump(2)) and CSV
  (placement.cpp:406-459).
"""
from __future__ import annotations

import json
import os
import struct

import numpy as np

from .qvb import ParseError, ValidationError

CSR_MAGIC = b"QVCSR1"
TAB_MAGIC = b"QVTAB1"
TIER_NAMES = ("gpu", "host", "disk")


# ---- graphs ----------------------------------------------------------------------
def save_graph_csr(path: str, row_offsets, col, weights) -> None:
    """save_graph_csr (graph.cpp:248-258)."""
    ro = np.ascontiguousarray(row_offsets, "<u8")
    c = np.ascontiguousarray(col, "<u8")
    w = np.ascontiguousarray(weights, "<f8") if weights is not None else np.ones(len(c), "<f8")
    with open(path, "wb") as f:
        f.write(CSR_MAGIC)
        f.write(struct.pack("<QQ", len(ro) - 1, len(c)))
        f.write(ro.tobytes())
        f.write(c.tobytes())
        f.write(w.tobytes())


def validate_graph(n, row_offsets, col, weights) -> None:
    """Graph::validate (graph.cpp:58-93), messages included (vectorised)."""
    ro = np.asarray(row_offsets, np.uint64)
    c = np.asarray(col, np.uint64)
    w = np.asarray(weights, np.float64)
    e = len(c)
    if n == 0:
        raise ValidationError("empty graph: node count is zero")
    if len(ro) != n + 1:
        raise ValidationError("row_offsets size mismatch")
    if ro[0] != 0 or ro[-1] != e:
        raise ValidationError("row_offsets endpoints invalid")
    if len(w) != e:
        raise ValidationError("edge array size mismatch")
    bad = np.nonzero(ro[1:] < ro[:-1])[0]
    if len(bad):
        raise ValidationError(f"row_offsets not non-decreasing at node {bad[0]}")
    rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(ro).astype(np.int64))
    first = n
    msg = None
    badc = np.nonzero(c >= n)[0]
    badw = np.nonzero(~(w >= 0.0))[0]
    cand = []
    if len(badc):
        cand.append((int(badc[0]), 0))
    if len(badw):
        cand.append((int(badw[0]), 1))
    if cand:
        ei, kind = min(cand)
        first = int(rows[ei])
        msg = ("column index out of range at node " if kind == 0 else
               "negative or NaN edge weight at node ") + str(first)
    pos = np.zeros(n, bool)
    np.logical_or.at(pos, rows.astype(np.int64), w > 0.0)
    zero = np.nonzero((np.diff(ro) > 0) & ~pos)[0]
    if len(zero) and int(zero[0]) < first:
        raise ValidationError(f"node {int(zero[0])} has out-edges but all weights are zero")
    if msg:
        raise ValidationError(msg)


def _load_csr_binary(path: str):
    try:
        f = open(path, "rb")
    except OSError:
        raise ParseError("cannot open graph file: " + path) from None
    with f:
        data = f.read()
    if len(data) < 6:
        raise ParseError(path + ": truncated csr-binary file")
    if data[:6] != CSR_MAGIC:
        raise ParseError(path + ": bad magic, not a QVCSR1 file")
    if len(data) < 22:
        raise ParseError(path + ": truncated csr-binary file")
    n, e = struct.unpack_from("<QQ", data, 6)
    if n == 0:
        raise ValidationError("empty graph in " + path)
    need = 22 + 8 * (n + 1) + 16 * e
    if len(data) < need:
        raise ParseError(path + ": truncated csr-binary file")
    ro = np.frombuffer(data, "<u8", n + 1, 22).copy()
    col = np.frombuffer(data, "<u8", e, 22 + 8 * (n + 1)).copy()
    w = np.frombuffer(data, "<f8", e, 22 + 8 * (n + 1) + 8 * e).copy()
    validate_graph(n, ro, col, w)
    return ro, col, w


def _load_edge_list(path: str, remap_sparse_ids: bool):
    try:
        f = open(path)
    except OSError:
        raise ParseError("cannot open graph file: " + path) from None
    src, dst, wts = [], [], []
    with f:
        for line_no, raw in enumerate(f, 1):
            line = raw.rstrip("\n")
            if "#" in line:
                line = line[: line.index("#")]
            tok = line.split()
            if not tok:
                continue
            try:
                s = int(tok[0])
                if s < 0:
                    raise ValueError
            except ValueError:
                raise ParseError(f"{path}:{line_no}: malformed edge line: '{line}'") from None
            if len(tok) < 2:
                raise ParseError(f"{path}:{line_no}: malformed edge line: '{line}'")
            try:
                d = int(tok[1])
                if d < 0:
                    raise ValueError
            except ValueError:
                raise ParseError(f"{path}:{line_no}: malformed edge line: '{line}'") from None
            w = 1.0
            if len(tok) >= 3:
                try:
                    w = float(tok[2])
                except ValueError:
                    raise ParseError(f"{path}:{line_no}: malformed weight '{tok[2]}'") from None
                if len(tok) > 3:
                    raise ParseError(f"{path}:{line_no}: trailing tokens after weight: '{tok[3]}'")
            src.append(s)
            dst.append(d)
            wts.append(w)
    if not src:
        raise ValidationError("empty graph: no edges in " + path)
    s = np.array(src, np.uint64)
    d = np.array(dst, np.uint64)
    w = np.array(wts, np.float64)
    n = int(max(s.max(), d.max())) + 1
    present = np.zeros(n, bool)
    present[s.astype(np.int64)] = True
    present[d.astype(np.int64)] = True
    if not present.all():
        if not remap_sparse_ids:
            raise ValidationError(path + ": node ids are not contiguous 0..N-1 (use id remapping "
                                  "for sparse-id inputs)")
        remap = np.cumsum(present) - 1
        s = remap[s.astype(np.int64)].astype(np.uint64)
        d = remap[d.astype(np.int64)].astype(np.uint64)
        n = int(present.sum())
    return from_edges(n, s, d, w)


def from_edges(n: int, src, dst, weights):
    """Graph::from_edges / build_csr (graph.cpp:16-56): stable by source."""
    if n == 0:
        raise ValidationError("empty graph: node count is zero")
    s = np.asarray(src, np.uint64)
    d = np.asarray(dst, np.uint64)
    w = np.asarray(weights, np.float64)
    bad = np.nonzero((s >= n) | (d >= n))[0]
    if len(bad):
        i = int(bad[0])
        raise ValidationError(f"edge endpoint {max(int(s[i]), int(d[i]))} out of range for node "
                              f"count {n}")
    badw = np.nonzero(~(w >= 0.0))[0]
    if len(badw):
        i = int(badw[0])
        raise ValidationError(f"negative or NaN edge weight on edge {int(s[i])} -> {int(d[i])}")
    order = np.argsort(s, kind="stable")
    ro = np.zeros(n + 1, np.uint64)
    ro[1:] = np.cumsum(np.bincount(s.astype(np.int64), minlength=n))
    col, ww = d[order], w[order]
    validate_graph(n, ro, col, ww)
    return ro, col, ww


def load_graph(path: str, fmt: str = "csr_binary", remap_sparse_ids: bool = False):
    """load_graph (graph.cpp:237-246): fmt 'csr_binary' | 'edge_list_text'."""
    if fmt == "csr_binary":
        return _load_csr_binary(path)
    if fmt == "edge_list_text":
        return _load_edge_list(path, remap_sparse_ids)
    raise ValidationError("unknown graph format")


# ---- tables ------------------------------------------------------------------------
def save_table_binary(path: str, values, k: int) -> None:
    v = np.ascontiguousarray(values, "<f8")
    with open(path, "wb") as f:
        f.write(TAB_MAGIC)
        f.write(struct.pack("<QQ", len(v), k))
        f.write(v.tobytes())


def load_table_binary(path: str):
    """-> (values, k)"""
    try:
        f = open(path, "rb")
    except OSError:
        raise ParseError("cannot open table file: " + path) from None
    with f:
        data = f.read()
    if len(data) < 6 or data[:6] != TAB_MAGIC:
        raise ParseError(path + ": bad magic, not a QVTAB1 file")
    if len(data) < 22:
        raise ParseError(path + ": truncated table header")
    n, k = struct.unpack_from("<QQ", data, 6)
    if len(data) < 22 + 8 * n:
        raise ParseError(path + ": truncated table values")
    return np.frombuffer(data, "<f8", n, 22).copy(), k


def save_table_csv(path: str, values) -> None:
    with open(path, "w") as f:
        f.write("node_id,value\n")
        f.writelines("%d,%.17g\n" % (i, v) for i, v in enumerate(np.asarray(values, np.float64)))


# ---- placement / lookup exports --------------------------------------------------
def _decode(loc: int, gps: int):
    stride = gps + 2
    server, slot = divmod(int(loc), stride)
    if slot < gps:
        return server, 0, slot
    return server, (1 if slot == gps else 2), 0


def placement_to_json_text(loc_offsets, loc_ids, topo) -> str:
    """placement_to_json_text (placement.cpp:406-422): ordered_json dump(2)."""
    lo = np.asarray(loc_offsets, np.uint64)
    ids = np.asarray(loc_ids, np.int64)
    gps = int(topo.gpus_per_server)
    feats = []
    for f in range(len(lo) - 1):
        locs = []
        for k in range(int(lo[f]), int(lo[f + 1])):
            s, t, d = _decode(ids[k], gps)
            locs.append({"server": s, "tier": TIER_NAMES[t], "device": d,
                         "replica": k > int(lo[f])})
        feats.append({"id": f, "locations": locs})
    return json.dumps({"feature_count": len(lo) - 1, "features": feats}, indent=2) + "\n"


def save_placement_csv(path: str, loc_offsets, loc_ids, topo) -> None:
    lo = np.asarray(loc_offsets, np.uint64)
    ids = np.asarray(loc_ids, np.int64)
    gps = int(topo.gpus_per_server)
    with open(path, "w") as f:
        f.write("feature_id,server,tier,device,replica\n")
        for fi in range(len(lo) - 1):
            for k in range(int(lo[fi]), int(lo[fi + 1])):
                s, t, d = _decode(ids[k], gps)
                f.write(f"{fi},{s},{TIER_NAMES[t]},{d},{1 if k > int(lo[fi]) else 0}\n")


def lookup_to_json_text(location_ids, offsets, home_server: int, gpus_per_server: int) -> str:
    """lookup_to_json_text (placement.cpp:437-449)."""
    rows = [{"feature": f, "location": int(l), "offset": int(o)}
            for f, (l, o) in enumerate(zip(location_ids, offsets))]
    return json.dumps({"home_server": home_server, "gpus_per_server": gpus_per_server,
                       "rows": rows}, indent=2) + "\n"


def save_lookup_csv(path: str, location_ids, offsets) -> None:
    with open(path, "w") as f:
        f.write("feature_id,location_id,offset\n")
        f.writelines(f"{i},{int(l)},{int(o)}\n" for i, (l, o) in enumerate(zip(location_ids, offsets)))


def exists(path: str) -> bool:
    return os.path.exists(path)
