import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def golden_catalog():
    from oracle.scene import load_catalog_tuples
    with open(os.path.join(GOLDEN, "catalog.json")) as fh:
        return load_catalog_tuples(json.load(fh))


def scene_names():
    return sorted(f[6:-4] for f in os.listdir(GOLDEN) if f.startswith("scene_"))


@pytest.fixture(scope="session")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="session")
def catalog():
    return golden_catalog()
