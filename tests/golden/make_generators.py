"""Golden outputs of the reference's own generators (generators.py:32-97,
preprocess graph.py:132-200), for the on-device generators' parity tests.

Run in the build container (imports /root/reference read-only):
    python tests/golden/make_generators.py   # writes tests/golden/generators.npz
"""
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
from jetpart import generators  # noqa: E402

CASES = [
    ("rmat_a", "rmat", dict(scale=10, edge_factor=8, seed=0)),
    ("rmat_b", "rmat", dict(scale=12, edge_factor=16, seed=3)),
    ("rmat_c", "rmat", dict(scale=9, edge_factor=4, seed=1, probs=(0.45, 0.15, 0.15, 0.25))),
    ("rgg_a", "rgg", dict(n=4096, radius=0.03, seed=0)),
    ("rgg_b", "rgg", dict(n=3000, radius=0.025, seed=2)),
    ("rgg_c", "rgg", dict(n=20000, radius=float(np.sqrt(12 / (np.pi * 20000))), seed=0)),
]

if __name__ == "__main__":
    d = {}
    for name, kind, kw in CASES:
        if kind == "rmat":
            g = generators.rmat_graph(**kw)
            probs = kw.get("probs", (0.57, 0.19, 0.19, 0.05))
            d[name + "_args"] = np.array([kw["scale"], kw["edge_factor"], kw["seed"]], np.int64)
            d[name + "_probs"] = np.array(probs, np.float64)
        else:
            g = generators.geometric_graph(**kw)
            d[name + "_args"] = np.array([kw["n"], kw["seed"]], np.int64)
            d[name + "_radius"] = np.array([kw["radius"]], np.float64)
        d[name + "_offs"] = g.row_offsets.astype(np.int64)
        d[name + "_adj"] = g.adjacency.astype(np.int32)
        d[name + "_ew"] = g.edge_weights.astype(np.int32)
        d[name + "_vw"] = g.vertex_weights.astype(np.int32)
        print(name, g.n, g.m, flush=True)
    np.savez_compressed(Path(__file__).parent / "generators.npz", **d)
