import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and liblazypca_b200.so")


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ctx():
    """One lazypca_b200 context on cuda:0. On a GPU test run a missing library
    or device is an error, not a skip: the product has no CPU fallback."""
    from paper_1709_07175_b200 import Context
    c = Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref), built here from /root/reference or
    shipped prebuilt to the GPU box."""
    from oracle import refbind
    if not refbind.available():
        refbind.build_if_possible()
    if not refbind.available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return refbind


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    class G:
        omega = np.load(GOLDEN / "omega.npz")
        reducers = np.load(GOLDEN / "reducers.npz")
        kat = np.load(GOLDEN / "kat.npz")
    return G
