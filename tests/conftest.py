import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


requires_ref = pytest.mark.skipif(
    not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblp2d_ref.so")),
    reason="oracle/_ref (the compiled reference) not built")


def cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def O():
    import oracle_py

    oracle_py.oracle_lib()
    return oracle_py


@pytest.fixture(scope="session")
def P():
    import paper_1902_04995_b200 as P

    P.lp2d.N.lib()
    return P


def load_batch(name):
    import paper_1902_04995_b200 as P

    d = np.load(os.path.join(GOLDEN, f"batch_{name}.npz"))
    return P.PackedBatch(d["m"], d["offset"], d["ax"], d["ay"], d["b"], d["perm"], d["c"], d["M"])


def load_npz(name):
    return dict(np.load(os.path.join(GOLDEN, name)))
