"""Pin the C oracle to the reference: every golden vector (produced by
running the reference itself, tests/golden/make_golden.py) must be
reproduced exactly. CPU only."""

import hashlib
import sys

import numpy as np
import pytest

from conftest import ROOT, graph_of, load

sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402


def n_cases(d):
    return int(d["count"][0])


def test_oracle_match_and_contract():
    d = load("coarsen")
    for i in range(n_cases(d)):
        g = graph_of(d, f"g{i}_")
        m = O.match(g)
        assert np.array_equal(m, d[f"g{i}_match"]), i
        (off, adj, ew, vw), vmap = O.contract(g, m)
        assert np.array_equal(vmap, d[f"g{i}_vmap"]), i
        assert np.array_equal(off, d[f"g{i}_c_offs"]), i
        assert np.array_equal(adj, d[f"g{i}_c_adj"]), i
        assert np.array_equal(ew, d[f"g{i}_c_ew"]), i
        assert np.array_equal(vw, d[f"g{i}_c_vw"]), i


def test_oracle_gains_afterburner_jetlp():
    d = load("refine")
    for i in range(n_cases(d)):
        g = graph_of(d, f"r{i}_")
        k = int(d[f"r{i}_k"][0])
        parts = d[f"r{i}_parts"]
        dest, gain, bnd, cs = O.select_destinations(g, parts, k)
        assert np.array_equal(dest, d[f"r{i}_dest"]) and np.array_equal(gain, d[f"r{i}_gain"]), i
        assert np.array_equal(bnd, d[f"r{i}_bnd"]) and np.array_equal(cs, d[f"r{i}_cs"]), i
        f2 = O.afterburner(g, d[f"r{i}_cand"], parts, dest, gain)
        assert np.array_equal(f2, d[f"r{i}_f2"]), i
        assert O.cutsize(g, parts) == int(d[f"r{i}_cut"][0])
        for ab in (1, 0):
            for lk in (1, 0):
                mv, md, mg, locks = O.jetlp_pass(g, parts, k, d[f"r{i}_locks"], float(d[f"r{i}_c"][0]),
                                                 bool(ab), bool(lk))
                tag = f"r{i}_lp{ab}{lk}_"
                assert np.array_equal(mv, d[tag + "v"]) and np.array_equal(md, d[tag + "d"]), (i, ab, lk)
                assert np.array_equal(mg, d[tag + "g"]), (i, ab, lk)
                if lk:
                    assert np.array_equal(locks, d[tag + "locks"]), i


def test_oracle_rebalance():
    d = load("rebalance")
    for i in range(n_cases(d)):
        g = graph_of(d, f"b{i}_")
        k = int(d[f"b{i}_k"][0])
        limit, sigma, rho = (int(x) for x in d[f"b{i}_lim"])
        for strong in (0, 1):
            rng = np.random.default_rng([i, strong, 99])
            mv, md, mg = O.rebalance_pass(g, d[f"b{i}_parts"], k, d[f"b{i}_pw"], limit, sigma, rng,
                                          rho, bool(strong))
            tag = f"b{i}_s{strong}_"
            assert np.array_equal(mv, d[tag + "v"]), (i, strong)
            assert np.array_equal(md, d[tag + "d"]), (i, strong)
            assert np.array_equal(mg, d[tag + "g"]), (i, strong)
            s = rng.bit_generator.state
            exp = d[tag + "rng"]
            assert (s["state"]["state"] >> 64, s["state"]["state"] & (2**64 - 1)) == \
                (int(exp[0]), int(exp[1])), i
            assert (s["has_uint32"], s["uinteger"]) == (int(exp[2]), int(exp[3])), i


def test_oracle_refine_initpart_partition():
    d = load("pipeline")
    for i in range(n_cases(d)):
        g = graph_of(d, f"p{i}_")
        k, seed, ab, lk = (int(x) for x in d[f"p{i}_cfg"])
        imb = float(d[f"p{i}_imb"][0])
        kw = dict(imbalance=imb, seed=seed, afterburner=bool(ab), locking=bool(lk))
        p, st = O.refine(g, d[f"p{i}_rparts_in"], k, finest=True, level=0, **kw)
        exp = d[f"p{i}_rstats"].tolist()
        assert [st["iterations"], st["lp_passes"], st["weak_passes"], st["strong_passes"],
                st["cut"], int(st["balanced"])] == exp, i
        assert np.array_equal(p, d[f"p{i}_rparts"]), i
        assert np.array_equal(O.initial_partition(g, k, imb, seed=seed, restarts=4), d[f"p{i}_ip"]), i
        r = O.partition(g, k, **kw)
        assert r["cut"] == int(d[f"p{i}_cut"][0]), i
        assert np.array_equal(r["parts"], d[f"p{i}_parts"]), i
        assert r["iterations"] == d[f"p{i}_iters"].tolist(), i


def test_oracle_known_answer_grid256():
    """grid 256x256, k=8, imbalance 0.03, seed 0 -> cut 1183."""
    from paper_2304_13194_b200 import generators as gen
    d = load("oracle_grid256")
    g = gen.grid_graph(256, 256)
    r = O.partition(g, 8, imbalance=0.03, seed=0)
    assert r["cut"] == 1183
    assert r["iterations"] == d["iters"].tolist()
    text = "".join(f"{int(p)}\n" for p in r["parts"]).encode()
    assert hashlib.md5(text).hexdigest() == "c4d3683a3bbddffbc66147f6a0beb53b"
