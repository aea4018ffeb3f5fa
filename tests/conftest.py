import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build

    build(ref=True)
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference (oracle/_ref); skipped where it was not built."""
    from oracle.oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref/libqvref.so not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def qvb():
    """The product library; GPU tests only."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_10863_b200 import build, qvb as Q

    build.build()
    return Q
