"""GPU parity: every hot-path kernel against the reference's own outputs
(golden vectors from tests/golden/make_golden.py), bit-exact."""

import numpy as np
import pytest

from conftest import graph_of

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import ops

pytestmark = pytest.mark.gpu


def n_cases(d):
    return int(d["count"][0])


def test_cutsize_and_part_weights(golden):
    d = golden("refine")
    for i in range(n_cases(d)):
        g = graph_of(d, f"r{i}_")
        k = int(d[f"r{i}_k"][0])
        st = J.PartitionState.from_parts(g, d[f"r{i}_parts"], k)
        assert st.cutsize == int(d[f"r{i}_cut"][0]), i
        assert np.array_equal(st.part_weights, d[f"r{i}_pw"]), i


def test_match_vertices(golden):
    d = golden("coarsen")
    for i in range(n_cases(d)):
        g = graph_of(d, f"g{i}_")
        got = J.match_vertices(g)
        assert np.array_equal(got, d[f"g{i}_match"]), (i, np.flatnonzero(got != d[f"g{i}_match"])[:10])


def test_contract(golden):
    d = golden("coarsen")
    for i in range(n_cases(d)):
        g = graph_of(d, f"g{i}_")
        cg, vmap = J.contract(g, d[f"g{i}_match"])
        assert np.array_equal(vmap, d[f"g{i}_vmap"]), i
        assert np.array_equal(cg.row_offsets, d[f"g{i}_c_offs"]), i
        assert np.array_equal(cg.adjacency, d[f"g{i}_c_adj"]), i
        assert np.array_equal(cg.edge_weights, d[f"g{i}_c_ew"]), i
        assert np.array_equal(cg.vertex_weights, d[f"g{i}_c_vw"]), i


def test_build_hierarchy(golden):
    d = golden("coarsen")
    for i in range(n_cases(d)):
        g = graph_of(d, f"g{i}_")
        h = J.build_hierarchy(g, 40)
        assert [lv.n if hasattr(lv, "n") else len(lv.row_offsets) - 1 for lv in h.levels] == \
            d[f"g{i}_hier_n"].tolist(), i
        for j, mp in enumerate(h.maps):
            assert np.array_equal(mp, d[f"g{i}_hier_map{j}"]), (i, j)


def test_select_destinations(golden):
    d = golden("refine")
    for i in range(n_cases(d)):
        g = graph_of(d, f"r{i}_")
        k = int(d[f"r{i}_k"][0])
        st = J.PartitionState(d[f"r{i}_parts"], k, d[f"r{i}_pw"], int(d[f"r{i}_cut"][0]))
        dest, gain, bnd, cs = J.select_destinations(g, st)
        assert np.array_equal(dest, d[f"r{i}_dest"]), i
        assert np.array_equal(gain, d[f"r{i}_gain"]), i
        assert np.array_equal(bnd, d[f"r{i}_bnd"]), i
        assert np.array_equal(cs, d[f"r{i}_cs"]), i


def test_afterburner(golden):
    d = golden("refine")
    for i in range(n_cases(d)):
        g = graph_of(d, f"r{i}_")
        got = J.afterburner(g, d[f"r{i}_cand"], d[f"r{i}_parts"], d[f"r{i}_dest"], d[f"r{i}_gain"])
        assert np.array_equal(got, d[f"r{i}_f2"]), i


@pytest.mark.parametrize("ab,lk", [(1, 1), (1, 0), (0, 1), (0, 0)])
def test_jetlp_pass(golden, ab, lk):
    d = golden("refine")
    for i in range(n_cases(d)):
        g = graph_of(d, f"r{i}_")
        k = int(d[f"r{i}_k"][0])
        st = J.PartitionState(d[f"r{i}_parts"], k, d[f"r{i}_pw"], int(d[f"r{i}_cut"][0]))
        table = ops.LockTable(g, st)
        table.locks[:] = d[f"r{i}_locks"]
        mv = J.jetlp_pass(g, st, table, float(d[f"r{i}_c"][0]), use_afterburner=bool(ab),
                          use_locks=bool(lk))
        tag = f"r{i}_lp{ab}{lk}_"
        assert np.array_equal(mv.vertices, d[tag + "v"]), (i, len(mv), len(d[tag + "v"]))
        assert np.array_equal(mv.dests, d[tag + "d"]), i
        assert np.array_equal(mv.gains, d[tag + "g"]), i
        if lk:
            assert np.array_equal(table.locks, d[tag + "locks"]), i


@pytest.mark.parametrize("strong", [0, 1])
def test_rebalance_pass(golden, strong):
    d = golden("rebalance")
    for i in range(n_cases(d)):
        g = graph_of(d, f"b{i}_")
        k = int(d[f"b{i}_k"][0])
        limit, sigma, rho = (int(x) for x in d[f"b{i}_lim"])
        st = J.PartitionState(d[f"b{i}_parts"], k, d[f"b{i}_pw"], 0)
        rng = np.random.default_rng([i, strong, 99])
        fn = J.strong_rebalance_pass if strong else J.weak_rebalance_pass
        mv = fn(g, st, None, limit, sigma, rng, rho)
        tag = f"b{i}_s{strong}_"
        assert np.array_equal(mv.vertices, d[tag + "v"]), (i, mv.vertices[:10], d[tag + "v"][:10])
        assert np.array_equal(mv.dests, d[tag + "d"]), i
        assert np.array_equal(np.asarray(mv.gains, np.float64), d[tag + "g"]), i
        s = rng.bit_generator.state
        exp = d[tag + "rng"]
        assert (s["state"]["state"] >> 64, s["state"]["state"] & (2**64 - 1)) == (int(exp[0]), int(exp[1])), i
        assert (s["has_uint32"], s["uinteger"]) == (int(exp[2]), int(exp[3])), i


def test_jet_refine(golden):
    d = golden("pipeline")
    for i in range(n_cases(d)):
        g = graph_of(d, f"p{i}_")
        k, seed, ab, lk = (int(x) for x in d[f"p{i}_cfg"])
        cfg = J.RefinerConfig(k=k, imbalance=float(d[f"p{i}_imb"][0]), seed=seed,
                              afterburner=bool(ab), locking=bool(lk), deterministic=True)
        st = J.PartitionState.from_parts(g, d[f"p{i}_rparts_in"], k)
        out, stats = J.jet_refine(g, st, cfg, finest=True, seed_path=(0,))
        exp = d[f"p{i}_rstats"].tolist()
        got = [stats["iterations"], stats["lp_passes"], stats["weak_passes"],
               stats["strong_passes"], out.cutsize, int(stats["balanced"])]
        assert got == exp, (i, got, exp)
        assert np.array_equal(out.parts, d[f"p{i}_rparts"]), i


def test_partition_pipeline(golden):
    d = golden("pipeline")
    for i in range(n_cases(d)):
        g = graph_of(d, f"p{i}_")
        k, seed, ab, lk = (int(x) for x in d[f"p{i}_cfg"])
        cfg = J.RefinerConfig(k=k, imbalance=float(d[f"p{i}_imb"][0]), seed=seed,
                              afterburner=bool(ab), locking=bool(lk), deterministic=True)
        res = J.partition(g, cfg)
        assert [lv["iterations"] for lv in res.metrics["levels"]] == d[f"p{i}_iters"].tolist(), i
        assert res.state.cutsize == int(d[f"p{i}_cut"][0]), i
        assert np.array_equal(res.state.parts, d[f"p{i}_parts"]), i


def test_oracle_config_grid256(golden):
    """BASELINE configs[0]: the reference's known answer, bit-exact."""
    import hashlib
    from paper_2304_13194_b200 import generators as gen
    d = golden("oracle_grid256")
    g = gen.grid_graph(256, 256)
    assert np.array_equal(J.match_vertices(g), d["match"].astype(np.int64))
    res = J.partition(g, J.RefinerConfig(k=8, imbalance=0.03, seed=0, deterministic=True))
    assert res.state.cutsize == 1183 == int(d["cut"][0])
    assert res.state.part_weights.tolist() == d["pw"].tolist()
    assert [lv["iterations"] for lv in res.metrics["levels"]] == d["iters"].tolist()
    text = "".join(f"{int(p)}\n" for p in res.state.parts).encode()
    assert hashlib.md5(text).hexdigest() == bytes(d["md5"]).decode() == "c4d3683a3bbddffbc66147f6a0beb53b"
