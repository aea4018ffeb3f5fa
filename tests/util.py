"""Test fixtures mirroring the reference's tests/testutil.hpp and rng.hpp.

RngStream / derive_stream follow include/qv/rng.hpp:10-57 exactly, so the
random graphs below are the same graphs the reference's own tests draw
(testutil.hpp:43-55 ``random_graph``) for the same stream keys.
"""
from __future__ import annotations

import os

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def splitmix64(x: int) -> int:
    x = (x + GAMMA) & M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class RngStream:
    def __init__(self, state: int):
        self.state = state & M64

    def next(self) -> int:
        self.state = (self.state + GAMMA) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        return (self.next() * n) >> 64


def derive_stream(master: int, a: int, b: int = 0, c: int = 0) -> RngStream:
    s = splitmix64(master ^ 0x6A09E667F3BCC909)
    s = splitmix64(s ^ splitmix64(a ^ 0xBB67AE8584CAA73B))
    s = splitmix64(s ^ splitmix64(b ^ 0x3C6EF372FE94F82B))
    s = splitmix64(s ^ splitmix64(c ^ 0xA54FF53A5F1D36F1))
    return RngStream(s)


def random_edges(rng: RngStream, max_nodes=50, max_edges=300, weighted=True):
    """testutil.hpp:43-55: (n, src, dst, w) in input order."""
    n = 2 + rng.below(max_nodes - 1)
    m = 1 + rng.below(max_edges)
    src, dst, w = [], [], []
    for _ in range(m):
        s = rng.below(n)
        d = rng.below(n)
        src.append(s)
        dst.append(d)
        w.append(0.25 + rng.uniform() if weighted else 1.0)
    return n, src, dst, w


def fig8_edges():
    """testutil.hpp:32-36"""
    return 6, [0, 0, 1, 3, 4], [3, 5, 3, 2, 0], [1.0] * 5


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


# BASELINE.json configs.
CONFIGS = {
    "C1": dict(n=100_000, e=1_000_000, weighted=False, layers=2, dim=128),
    "C2": dict(n=2_400_000, e=62_000_000, weighted=False, layers=2, dim=100),
    "C3": dict(n=233_000, e=114_000_000, weighted=True, layers=3, dim=602),
    "C4": dict(n=111_000_000, e=1_600_000_000, weighted=False, layers=3, dim=128),
}


def host_ram_gb() -> float:
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except (ValueError, OSError, AttributeError):
        return 0.0


def c4_reference_enabled() -> bool:
    """C4-vs-unmodified-reference checks: on by default where the host has
    the RAM (the B200 boxes: 196 GB); QVB_C4_REFERENCE=0 turns them off,
    =1 forces them."""
    v = os.environ.get("QVB_C4_REFERENCE")
    if v is not None:
        return v == "1"
    return host_ram_gb() >= 150
