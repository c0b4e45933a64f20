"""Edge cases the reference's driver tests exercise (test_driver.py): k = 1,
k = n, k > n, infeasible balance, disconnected graphs, isolated vertices,
heavy vertex weights; both modes; results checked against the C oracle
(pinned to the reference) where the reference defines them."""

import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import oracle as O  # noqa: E402  test infrastructure: the checker


def _two_grids():
    """Two disconnected 12x12 grids plus three isolated vertices."""
    a = gen.grid_graph(12, 12)
    n1 = a.n
    offs = np.concatenate([a.row_offsets, a.row_offsets[1:] + a.row_offsets[-1]])
    adj = np.concatenate([a.adjacency, a.adjacency + n1])
    offs = np.concatenate([offs, np.full(3, offs[-1])])
    ew = np.ones(len(adj), np.int64)
    vw = np.ones(len(offs) - 1, np.int64)
    return J.Graph(offs.astype(np.int64), adj.astype(np.int64), ew, vw)


@pytest.mark.parametrize("det", [True, False])
def test_k1_and_k_equal_n(det):
    g = gen.grid_graph(8, 8)
    r = J.partition(g, J.RefinerConfig(k=1, deterministic=det))
    assert r.state.cutsize == 0 and set(np.unique(r.state.parts)) == {0}
    r = J.partition(g, J.RefinerConfig(k=g.n, imbalance=0.0, deterministic=det))
    assert len(np.unique(r.state.parts)) == g.n
    assert r.state.cutsize == J.cutsize(g, r.state.parts)


def test_k_above_n_and_infeasible_balance():
    g = gen.grid_graph(4, 4)
    with pytest.raises(ValueError):
        J.partition(g, J.RefinerConfig(k=17))
    heavy = J.Graph(g.row_offsets, g.adjacency, g.edge_weights,
                    np.where(np.arange(g.n) == 0, 100, 1).astype(np.int64))
    with pytest.raises(J.BalanceInfeasibleError):
        J.partition(heavy, J.RefinerConfig(k=4, imbalance=0.03))


@pytest.mark.parametrize("det", [True, False])
def test_disconnected_with_isolated_vertices(det):
    g = _two_grids()
    cfg = J.RefinerConfig(k=4, imbalance=0.03, seed=0, deterministic=det)
    r = J.partition(g, cfg)
    assert r.metrics["balanced"]
    assert r.state.cutsize == J.cutsize(g, r.state.parts)
    if det:
        ref = O.partition(g, k=4, imbalance=0.03, seed=0)
        assert r.state.cutsize == ref["cut"]
        assert np.array_equal(r.state.parts, ref["parts"])


@pytest.mark.parametrize("det", [True, False])
def test_weighted_graph(det):
    rng = np.random.default_rng(5)
    base = gen.grid_graph(20, 20)
    # symmetric random edge weights: weight of {u, v} = hash of the pair
    u = np.repeat(np.arange(base.n), np.diff(base.row_offsets))
    v = base.adjacency
    w = 1 + (np.minimum(u, v) * 7919 + np.maximum(u, v) * 104729) % 9
    vw = rng.integers(1, 4, size=base.n)
    g = J.Graph(base.row_offsets, base.adjacency, w.astype(np.int64), vw.astype(np.int64))
    cfg = J.RefinerConfig(k=6, imbalance=0.05, seed=2, deterministic=det)
    r = J.partition(g, cfg)
    assert r.state.cutsize == J.cutsize(g, r.state.parts)
    if det:
        ref = O.partition(g, k=6, imbalance=0.05, seed=2)
        assert r.state.cutsize == ref["cut"]
        assert np.array_equal(r.state.parts, ref["parts"])


def test_device_rgg_weighted_vs_oracle():
    """A device-generated geometric graph (2^15 points) given random integer
    edge and vertex weights on the host: deterministic mode equals the oracle."""
    g0 = gen.geometric_graph(1 << 15, 0.012, seed=4)
    u = np.repeat(np.arange(g0.n), np.diff(g0.row_offsets))
    v = g0.adjacency
    w = 1 + (np.minimum(u, v) * 31 + np.maximum(u, v) * 17) % 7
    vw = 1 + (np.arange(g0.n) * 13) % 3
    g = J.Graph(g0.row_offsets, g0.adjacency, w.astype(np.int64), vw.astype(np.int64))
    for k in (16, 100):
        r = J.partition(g, J.RefinerConfig(k=k, imbalance=0.03, seed=1, deterministic=True))
        ref = O.partition(g, k=k, imbalance=0.03, seed=1)
        assert r.state.cutsize == ref["cut"], (k, r.state.cutsize, ref["cut"])
        assert np.array_equal(r.state.parts, ref["parts"])
