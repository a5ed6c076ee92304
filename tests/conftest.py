import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def bitwise(a, b) -> bool:
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def product_vehicle(name):
    from paper_2503_09203_b200 import vehicles as pv
    import variants

    if name in variants.VARIANTS:
        return variants.build(name, pv, pv, pv, pv.load_vehicle("bluerov"))
    return pv.load_vehicle(name)


@pytest.fixture
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
