"""Boundary-only sweeps: after the first Jetlp sweep of a level,
the level kernel keeps every vertex's weighted external degree current and
sweeps only boundary rows; rebalance stats take interior candidates' weighted
degree without reading their adjacency. Both are exact restatements, so the
result must equal the full-sweep run (JET_FULL_SWEEPS=1) bit for bit -- in
both modes, on unit-weight and weighted levels (every coarse level is
weighted), and on a graph with hubs."""

import os

import numpy as np
import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen

pytestmark = pytest.mark.gpu


def _both(g, cfg):
    os.environ.pop("JET_FULL_SWEEPS", None)
    a = J.partition(g, cfg)
    os.environ["JET_FULL_SWEEPS"] = "1"
    try:
        b = J.partition(g, cfg)
    finally:
        os.environ.pop("JET_FULL_SWEEPS", None)
    return a, b


@pytest.mark.parametrize("det", [True, False])
@pytest.mark.parametrize("case", ["grid27_48", "rmat14"])
def test_boundary_sweeps_equal_full_sweeps(case, det):
    if case == "grid27_48":
        g, k = gen.grid27_graph(48), 32
    else:
        g, k = gen.rmat_graph(14, 16, 0), 16
    cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=1, deterministic=det)
    a, b = _both(g, cfg)
    assert a.state.cutsize == b.state.cutsize
    assert np.array_equal(np.asarray(a.state.parts), np.asarray(b.state.parts))
    assert a.metrics["balanced"] and b.metrics["balanced"]
