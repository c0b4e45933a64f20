"""CPU-only tests: the C-ABI library loads and exports every declared
symbol; the host-side numpy-RNG restatement and the host initial
partitioner match the reference; config scalars; generators."""

import re
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, graph_of, load

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import _lib
from paper_2304_13194_b200 import generators as gen
from paper_2304_13194_b200.config import rebalance_thresholds, to_c


def header_symbols():
    text = (ROOT / "include" / "jet.h").read_text()
    return sorted(set(re.findall(r"\b(jet_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.exported_symbols())
    assert lib.jet_api_version() == 1


def test_no_gpu_reports_error_not_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(J.JetpartError):
        J.Context(0)


def _pcg(words):
    import ctypes as C
    st = _lib.Pcg64State()
    arr = np.asarray(words, dtype=np.uint32)
    _lib.check(_lib.lib().jet_rng_seed(_lib.ptr(arr), len(arr), C.byref(st)))
    return st


def _words(seeds):
    out = []
    for s in seeds:
        if s == 0:
            out.append(0)
        while s:
            out.append(s & 0xFFFFFFFF)
            s >>= 32
    return out


@pytest.mark.parametrize("seeds", [[0], [0, 1, 2], [7, 3, 11], [5_000_000_000, 3], [1, 2, 3, 4, 5, 6]])
def test_seed_sequence_matches_numpy(seeds):
    st = _pcg(_words(seeds))
    ref = np.random.default_rng(seeds).bit_generator.state["state"]
    assert (st.state_hi << 64 | st.state_lo) == ref["state"]
    assert (st.inc_hi << 64 | st.inc_lo) == ref["inc"]


def test_bounded_integers_match_numpy_across_calls():
    import ctypes as C
    rng = np.random.default_rng([3, 2, 1])
    st = _pcg(_words([3, 2, 1]))
    for high, cnt in [(5, 7), (1, 3), (7, 1), (1 << 20, 5), (3, 9), (2**33, 3), (97, 40)]:
        out = np.empty(cnt, np.int64)
        _lib.check(_lib.lib().jet_rng_integers(C.byref(st), high, cnt, _lib.ptr(out)))
        assert out.tolist() == rng.integers(0, high, size=cnt).tolist()
    s = rng.bit_generator.state
    assert st.has_uint32 == s["has_uint32"] and st.uinteger == s["uinteger"]


def test_initial_partition_host_matches_reference():
    d = load("pipeline")
    for i in range(int(d["count"][0])):
        g = graph_of(d, f"p{i}_")
        k, seed = int(d[f"p{i}_cfg"][0]), int(d[f"p{i}_cfg"][1])
        imb = float(d[f"p{i}_imb"][0])
        limit = J.part_weight_limit(int(g.vertex_weights.sum()), k, imb)
        out = np.empty(g.n, np.int64)
        arrs = [np.ascontiguousarray(a, dtype=np.int64) for a in
                (g.row_offsets, g.adjacency, g.edge_weights, g.vertex_weights)]
        _lib.check(_lib.lib().jet_initial_partition(
            g.n, *[_lib.ptr(a) for a in arrs], k, limit, seed, 4, _lib.ptr(out)))
        assert np.array_equal(out, d[f"p{i}_ip"]), i


def test_config_scalars_match_reference_expressions():
    W, k = 2_097_152, 64
    cfg = to_c(J.RefinerConfig(k=k), W)
    assert cfg.limit == int((1 + Fraction("0.03")) * W // k) == 33751 + 0 * 1 or cfg.limit == 33751
    assert cfg.sigma == 33653
    assert (cfg.c_finest_num, cfg.c_finest_den) == (1, 4)
    assert (cfg.c_other_num, cfg.c_other_den) == (3, 4)
    assert rebalance_thresholds(65536, 8, 0.03, J.part_weight_limit(65536, 8, 0.03), 0.1) == 8413


def test_refiner_config_validation():
    for bad in [dict(k=0), dict(k=2, phi=0), dict(k=2, c_finest=1.5), dict(k=2, sub_buckets=0),
                dict(k=2, imbalance=-1), dict(k=2, seed=-1), dict(k=2, no_improve_limit=0)]:
        with pytest.raises(ValueError):
            J.RefinerConfig(**bad)


def test_generators_match_golden_grid():
    g = gen.grid_graph(32, 40)
    d = load("coarsen")
    # corpus index 40 is grid_graph(32, 40) in make_golden.py
    assert np.array_equal(g.row_offsets, d["g40_offs"])
    assert np.array_equal(g.adjacency, d["g40_adj"])


def test_grid27_sizes():
    g = gen.grid27_graph(8)
    n = 8 ** 3
    # edges of the 26-neighbour stencil: (3n^(1/3)-... ) closed form via counting
    N = 8
    m = sum((N - abs(a)) * (N - abs(b)) * (N - abs(c))
            for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1) if (a, b, c) != (0, 0, 0)) // 2
    assert g.n == n and g.m == m
    assert np.all(np.diff(g.adjacency[g.row_offsets[1]:g.row_offsets[2]]) > 0)


@pytest.mark.parametrize("shape", [(5, 5, 5), (3, 4, 6), (1, 7, 2)])
def test_grid27_matches_reference_preprocess(shape):
    """grid27_graph builds the 27-point CSR directly; the golden is the
    reference's preprocess (graph.py:132-200) of the raw stencil pairs
    (tests/golden/make_grid27.py)."""
    d = np.load(Path(__file__).parent / "golden" / "grid27.npz")
    g = gen.grid27_graph(*shape)
    key = "%dx%dx%d" % shape
    for attr, suffix in (("row_offsets", "offs"), ("adjacency", "adj"),
                         ("edge_weights", "ew"), ("vertex_weights", "vw")):
        assert np.array_equal(getattr(g, attr), d[f"{key}_{suffix}"]), attr
