"""Shared fixtures: golden vectors (generated from the reference by
tests/golden/make_golden.py) and graph reconstruction."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def graph_of(d, pfx):
    from paper_2304_13194_b200 import Graph
    return Graph(d[pfx + "offs"].astype(np.int64), d[pfx + "adj"].astype(np.int64),
                 d[pfx + "ew"].astype(np.int64), d[pfx + "vw"].astype(np.int64))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load(name)
        return cache[name]
    return get


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
