"""Generate golden vectors by running the REFERENCE (`jetpart`) itself.

Run in the build container, where /root/reference exists:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
The GPU box has no /root/reference; the committed .npz files are what the
parity tests compare against there. Every case stores its inputs and the
reference's outputs; graphs are stored as CSR arrays.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from jetpart import coarsen, conn, driver, generators, graph as G, initpart, rebalance, refine  # noqa: E402

OUT = Path(__file__).resolve().parent
I64 = np.int64


def put_graph(d, pfx, g):
    d[pfx + "offs"] = g.row_offsets.astype(I64)
    d[pfx + "adj"] = g.adjacency.astype(np.int32)
    d[pfx + "ew"] = g.edge_weights.astype(np.int32)
    d[pfx + "vw"] = g.vertex_weights.astype(np.int32)


def random_graph(rng, n_lo, n_hi, p=None, max_weight=1, max_vertex_weight=1):
    n = int(rng.integers(n_lo, n_hi + 1))
    p = min(1.0, 3.0 / n) if p is None else p
    while True:
        iu, ju = np.triu_indices(n, k=1)
        mask = rng.random(len(iu)) < p
        if not mask.any():
            continue
        w = rng.integers(1, max_weight + 1, size=int(mask.sum()))
        vw = rng.integers(1, max_vertex_weight + 1, size=n)
        g, _ = G.preprocess(np.stack([iu[mask], ju[mask], w], axis=1), n, vw)
        if g.n >= 4:
            return g


def graph_corpus(seed=7, count=40):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        mw = [1, 1, 5, 50][i % 4]
        mvw = [1, 3, 1, 4][i % 4]
        dense = i % 5 == 0
        g = random_graph(rng, 20, 400, p=(0.3 if dense else None), max_weight=mw,
                         max_vertex_weight=mvw)
        out.append(g)
    # structured graphs
    out.append(generators.grid_graph(32, 40))
    out.append(generators.cube_graph(9, 10, 11))
    out.append(generators.rmat_graph(11, 8, seed=3))
    out.append(generators.geometric_graph(2**11, 0.04, seed=5))
    out.append(generators.gnp_graph(300, 0.05, seed=9, max_weight=7, max_vertex_weight=3))
    # star: exercises two-hop matching and a hub row
    star_edges = [(0, i) for i in range(1, 3000)] + [(i, i + 1) for i in range(1, 100)]
    out.append(G.preprocess(np.array(star_edges), 3000)[0])
    return out


def coarsening_cases():
    d = {}
    for i, g in enumerate(graph_corpus()):
        put_graph(d, f"g{i}_", g)
        m = coarsen.match_vertices(g)
        d[f"g{i}_match"] = m
        cg, vmap = coarsen.contract(g, m)
        put_graph(d, f"g{i}_c_", cg)
        d[f"g{i}_vmap"] = vmap
        h = coarsen.build_hierarchy(g, 40)
        d[f"g{i}_hier_n"] = np.array([lv.n for lv in h.levels], I64)
        d[f"g{i}_hier_m"] = np.array([lv.m for lv in h.levels], I64)
        for j, mp in enumerate(h.maps):
            d[f"g{i}_hier_map{j}"] = mp
    d["count"] = np.array([len(graph_corpus())])
    np.savez_compressed(OUT / "coarsen.npz", **d)


def refine_cases():
    """select_destinations / filter / afterburner / jetlp_pass on random partitions."""
    d = {}
    rng = np.random.default_rng(11)
    corpus = graph_corpus(seed=8, count=30)
    for i, g in enumerate(corpus):
        k = int(rng.integers(2, 17))
        parts = rng.integers(0, k, size=g.n)
        st = G.PartitionState.from_parts(g, parts, k)
        table = conn.build_conn(g, st)
        put_graph(d, f"r{i}_", g)
        d[f"r{i}_k"] = np.array([k])
        d[f"r{i}_parts"] = parts.astype(I64)
        d[f"r{i}_pw"] = st.part_weights
        d[f"r{i}_cut"] = np.array([st.cutsize])
        dest, gain, bnd, cs = refine.select_destinations(g, st, table)
        d[f"r{i}_dest"], d[f"r{i}_gain"], d[f"r{i}_bnd"], d[f"r{i}_cs"] = dest, gain, bnd, cs
        c = [0.25, 0.75, 0.3, 0.5][i % 4]
        locks = rng.random(g.n) < 0.1
        d[f"r{i}_c"] = np.array([c])
        d[f"r{i}_locks"] = locks
        cand = np.flatnonzero(refine.gain_ratio_filter(gain, cs, c, bnd, locks))
        d[f"r{i}_cand"] = cand
        d[f"r{i}_f2"] = refine.afterburner(g, cand, st.parts, dest, gain)
        for ab in (True, False):
            for lk in (True, False):
                t2 = conn.build_conn(g, st.copy())
                t2.locks[:] = locks
                mv = refine.jetlp_pass(g, st, t2, c, use_afterburner=ab, use_locks=lk)
                tag = f"r{i}_lp{int(ab)}{int(lk)}_"
                d[tag + "v"], d[tag + "d"], d[tag + "g"] = mv.vertices, mv.dests, mv.gains
                d[tag + "locks"] = t2.locks.copy()
    d["count"] = np.array([len(corpus)])
    np.savez_compressed(OUT / "refine.npz", **d)


def rebalance_cases():
    d = {}
    rng = np.random.default_rng(12)
    corpus = graph_corpus(seed=9, count=40)
    idx = 0
    for i, g in enumerate(corpus):
        for rep in range(2):
            k = int(rng.integers(2, 12))
            skew = rng.random(k) + 0.2
            skew[rng.integers(0, k)] *= 3 + rep * 3
            parts = rng.choice(k, size=g.n, p=skew / skew.sum())
            st = G.PartitionState.from_parts(g, parts, k)
            W = g.total_vertex_weight
            imb = [0.03, 0.05, 0.1][idx % 3]
            limit = G.part_weight_limit(W, k, imb)
            sigma = rebalance.rebalance_thresholds(W, k, imb, limit, 0.1)
            if not np.any(st.part_weights > limit) or not np.any(st.part_weights < sigma):
                continue
            rho = [32, 32, 4, 1, 7][idx % 5]
            put_graph(d, f"b{idx}_", g)
            d[f"b{idx}_k"] = np.array([k])
            d[f"b{idx}_parts"] = parts.astype(I64)
            d[f"b{idx}_pw"] = st.part_weights
            d[f"b{idx}_lim"] = np.array([limit, sigma, rho])
            for strong in (0, 1):
                r = np.random.default_rng([idx, strong, 99])
                fn = rebalance.strong_rebalance_pass if strong else rebalance.weak_rebalance_pass
                mv = fn(g, st, conn.build_conn(g, st.copy()), limit, sigma, r, rho)
                tag = f"b{idx}_s{strong}_"
                d[tag + "v"], d[tag + "d"] = mv.vertices, mv.dests
                d[tag + "g"] = np.asarray(mv.gains, dtype=np.float64)
                s = r.bit_generator.state
                d[tag + "rng"] = np.array([s["state"]["state"] >> 64, s["state"]["state"] & (2**64 - 1),
                                           s["has_uint32"], s["uinteger"]], dtype=np.uint64)
            idx += 1
    d["count"] = np.array([idx])
    np.savez_compressed(OUT / "rebalance.npz", **d)


def pipeline_cases():
    d = {}
    rng = np.random.default_rng(13)
    corpus = graph_corpus(seed=10, count=24)
    idx = 0
    for i, g in enumerate(corpus):
        k = int(rng.integers(2, 9))
        if k > g.n:
            continue
        imb = [0.03, 0.1, 0.01][i % 3]
        cfg = refine.RefinerConfig(k=k, imbalance=imb, seed=int(rng.integers(0, 5)),
                                   afterburner=(i % 7 != 3), locking=(i % 11 != 5))
        try:
            res = driver.partition(g, cfg)
        except Exception as e:  # BalanceInfeasible on tiny weighted graphs
            print("skip", i, type(e).__name__)
            continue
        put_graph(d, f"p{idx}_", g)
        d[f"p{idx}_cfg"] = np.array([k, cfg.seed, int(cfg.afterburner), int(cfg.locking)])
        d[f"p{idx}_imb"] = np.array([imb])
        d[f"p{idx}_parts"] = res.state.parts
        d[f"p{idx}_cut"] = np.array([res.state.cutsize])
        d[f"p{idx}_iters"] = np.array([lv["iterations"] for lv in res.metrics["levels"]])
        # jet_refine on a random start (level 0, finest) and initial partition
        parts = rng.integers(0, k, size=g.n)
        st = G.PartitionState.from_parts(g, parts, k)
        out, stats = refine.jet_refine(g, st, cfg, finest=True, seed_path=(0,))
        d[f"p{idx}_rparts_in"] = parts.astype(I64)
        d[f"p{idx}_rparts"] = out.parts
        d[f"p{idx}_rstats"] = np.array([stats["iterations"], stats["lp_passes"], stats["weak_passes"],
                                        stats["strong_passes"], out.cutsize, int(stats["balanced"])])
        ip = initpart.initial_partition(g, k, imb, seed=cfg.seed, restarts=4)
        d[f"p{idx}_ip"] = ip.parts
        idx += 1
    d["count"] = np.array([idx])
    np.savez_compressed(OUT / "pipeline.npz", **d)


def oracle_config():
    """BASELINE configs[0]: grid 256x256, k=8, imbalance 0.03, seed 0."""
    g = generators.grid_graph(256, 256)
    res = driver.partition(g, refine.RefinerConfig(k=8, imbalance=0.03, seed=0))
    parts = res.state.parts
    text = "".join(f"{int(p)}\n" for p in parts).encode()
    d = {
        "parts": parts.astype(np.int8),
        "cut": np.array([res.state.cutsize]),
        "pw": res.state.part_weights,
        "iters": np.array([lv["iterations"] for lv in res.metrics["levels"]]),
        "hier_n": np.array([lv["n"] for lv in res.metrics["levels"]][::-1]),
        "md5": np.frombuffer(hashlib.md5(text).hexdigest().encode(), dtype=np.uint8),
    }
    # one Jetlp step on parts = default_rng(0).integers(0, 8, n)
    p0 = np.random.default_rng(0).integers(0, 8, g.n)
    st = G.PartitionState.from_parts(g, p0, 8)
    t = conn.build_conn(g, st)
    dest, gain, bnd, cs = refine.select_destinations(g, st, t)
    mv = refine.jetlp_pass(g, st, conn.build_conn(g, st), 0.25)
    d.update({"step_cut": np.array([st.cutsize]), "step_dest": dest, "step_gain": gain,
              "step_bnd": bnd, "step_nmoves": np.array([len(mv)]), "step_mv": mv.vertices,
              "step_md": mv.dests})
    m = coarsen.match_vertices(g)
    d["match"] = m.astype(np.int32)
    np.savez_compressed(OUT / "oracle_grid256.npz", **d)
    print("grid256 cut", res.state.cutsize, hashlib.md5(text).hexdigest())


if __name__ == "__main__":
    which = sys.argv[1:] or ["coarsen", "refine", "rebalance", "pipeline", "oracle"]
    if "coarsen" in which:
        coarsening_cases()
    if "refine" in which:
        refine_cases()
    if "rebalance" in which:
        rebalance_cases()
    if "pipeline" in which:
        pipeline_cases()
    if "oracle" in which:
        oracle_config()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
