"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) applied
to the GPU path, in both modes where the criterion is about the pipeline:

  01  afterburner == sequential statement on 1,000 random graphs   (:95-113)
  02  exact-delta apply stays in sync over 100 random passes       (:116-140)
  03  the 120-run corpus is always balanced                        (:143-147)
  04  jet_refine never worsens a balanced input (500 inputs)       (:150-172)
  05  projection preserves the cut (pipeline and direct)           (:175-198)

The corpus is the reference's (:56-63): grid 64x64, cube 20^3, R-MAT 2^14
ef 8 seed 101 and RGG 2^14 r=0.0155 seed 202 (the latter two generated on the
device, bit-identical to the reference's generators, tests/test_generators.py),
k in {8, 32}, lambda in {1.01, 1.03, 1.10}, seeds 0-4."""

import numpy as np
import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen
from paper_2304_13194_b200 import ops

from helpers import (afterburner_sequential, brute_conn, gain_filter, random_graph,
                     random_partition)

pytestmark = pytest.mark.gpu

KS = (8, 32)
IMBALANCES = (0.01, 0.03, 0.10)
SEEDS = range(5)


def _host(dg):
    offs, adj, ew, vw = dg.download()
    dg.free()
    return J.Graph(offs, adj, ew, vw)


@pytest.fixture(scope="module")
def corpus():
    return {
        "grid64": gen.grid_graph(64, 64),
        "cube20": gen.cube_graph(20, 20, 20),
        "rmat14": _host(gen.rmat_device(14, 8, 101)),
        "rgg14": _host(gen.geometric_device(1 << 14, 0.0155, 202)),
    }


def _sweep(corpus, deterministic):
    runs = []
    for name, g in corpus.items():
        for k in KS:
            for imb in IMBALANCES:
                for seed in SEEDS:
                    cfg = J.RefinerConfig(k=k, imbalance=imb, seed=seed,
                                          deterministic=deterministic)
                    r = J.partition(g, cfg)
                    runs.append({"graph": name, "k": k, "imbalance": imb, "seed": seed,
                                 "cut": r.state.cutsize, "metrics": r.metrics,
                                 "parts": r.state.parts, "pw": r.state.part_weights})
    return runs


@pytest.fixture(scope="module", params=[True, False], ids=["deterministic", "throughput"])
def corpus_runs(request, corpus):
    return request.param, _sweep(corpus, request.param)


def test_01_afterburner_matches_sequential_statement():
    rng = np.random.default_rng(20230426)
    bad = 0
    for trial in range(1000):
        g = random_graph(rng, n_lo=8, n_hi=200)
        k = (2, 4, 8)[trial % 3]
        st = random_partition(rng, g, k)
        dest, gain, bnd, cs = J.select_destinations(g, st)
        cand = np.flatnonzero(gain_filter(gain, cs, 0.75, bnd, np.zeros(g.n, bool)))
        got = J.afterburner(g, cand, st.parts, dest, gain)
        want = afterburner_sequential(g, cand, st.parts, dest, gain)
        bad += int(not np.array_equal(got, want))
    assert bad == 0, f"{bad} of 1000 random graphs differ"


def test_02_apply_stays_in_sync():
    rng = np.random.default_rng(7)
    for trial in range(10):
        g = random_graph(rng, n_lo=40, n_hi=150, max_weight=4, max_vertex_weight=3)
        k = (2, 4, 8)[trial % 3]
        st = random_partition(rng, g, k)
        table = J.build_conn(g, st)
        for step in range(100):
            if step % 5 == 4:
                moves = J.jetlp_pass(g, st, table, c=0.75)
            else:
                cnt = int(rng.integers(1, max(2, g.n // 3)))
                verts = rng.choice(g.n, size=cnt, replace=False)
                dests = (st.parts[verts] + rng.integers(1, k, size=cnt)) % k
                moves = J.MoveList(verts, dests)
            table.apply(moves)
        fresh = J.PartitionState.from_parts(g, st.parts, k)
        assert st.cutsize == fresh.cutsize, trial
        assert np.array_equal(st.part_weights, fresh.part_weights), trial
        exp = brute_conn(g, st.parts)
        for v in range(0, g.n, 7):
            assert table.row_items(v) == exp[v], (trial, v)


def test_03_corpus_always_balanced(corpus_runs):
    det, runs = corpus_runs
    assert len(runs) == 120
    bad = [(r["graph"], r["k"], r["imbalance"], r["seed"]) for r in runs
           if not r["metrics"]["balanced"]]
    assert not bad, (det, bad)
    for r in runs:
        assert int(r["pw"].max()) <= r["metrics"]["part_weight_limit"]


def test_04_refinement_never_worsens_balanced_inputs():
    rng = np.random.default_rng(4)
    checked = violations = 0
    while checked < 500:
        g = random_graph(rng, n_lo=12, n_hi=80, max_weight=3)
        k = (2, 4, 8)[checked % 3]
        order = np.random.default_rng(checked).permutation(g.n)
        parts = np.zeros(g.n, np.int64)
        parts[order] = np.arange(g.n) % k
        st = J.PartitionState.from_parts(g, parts, k)
        if not J.is_balanced(st, 0.1):
            continue
        checked += 1
        cfg = J.RefinerConfig(k=k, imbalance=0.1, seed=checked)
        best, stats = J.jet_refine(g, st, cfg, finest=bool(checked % 2))
        if not stats["balanced"] or best.cutsize > st.cutsize or not J.is_balanced(best, 0.1):
            violations += 1
    assert violations == 0


def test_05_projection_preserves_cut(corpus, corpus_runs):
    det, runs = corpus_runs
    bad = 0
    for r in runs:
        lv = r["metrics"]["levels"]
        for above, below in zip(lv, lv[1:]):
            bad += int(below["cut_in"] != above["cut_out"])
    assert bad == 0, det
    rng = np.random.default_rng(5)
    for g in corpus.values():
        h = J.build_hierarchy(g, 200)
        h.validate()
        coarse = h.levels[-1]
        parts = rng.integers(0, 8, size=coarse.n if hasattr(coarse, "n") else len(coarse.row_offsets) - 1)
        expected = J.cutsize(coarse, parts)
        for level in range(len(h.levels) - 2, -1, -1):
            parts = parts[h.maps[level]]
            assert J.cutsize(h.levels[level], parts) == expected
