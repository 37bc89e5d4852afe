import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def oracle():
    """C restatement of the reference (oracle/oracle.c) -- the checker."""
    from oracle.bind import Oracle
    return Oracle("oracle")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled from its sources (oracle/_ref)."""
    from oracle import bind
    if not bind.ref_available():
        try:
            bind.build(ref=True)
        except Exception:
            pass
    if not bind.ref_available():
        pytest.skip("reference library oracle/_ref/librsref.so unavailable (no /root/reference here)")
    return bind.Oracle("ref")


@pytest.fixture(scope="session")
def kat():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a CUDA device")
    import paper_2505_12663_b200 as P
    P.lib()
    return torch.device("cuda")
