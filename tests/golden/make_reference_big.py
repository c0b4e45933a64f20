"""Golden answers for the benchmarked configs, produced by running the Python
REFERENCE itself (imported read-only from /root/reference/pkg/src), not the C
oracle. Build-container only (the GPU box has no /root/reference). Slow:
128^3 ~3 min, RGG 2^24 and R-MAT 2^22 much longer; run once per case:

    python tests/golden/make_reference_big.py grid27_128 rgg16m rmat22

For each case it records the cut, the md5 of the part vector (little-endian
int64, the dtype of the reference's PartitionState.parts), the part weights,
the per-level (n, m, iterations, cut_out) report of metrics["levels"]
(driver.py:96-114) and the reference's own wall time. The 27-point grid is
built with the reference's `preprocess` (graph.py:132-200) from a raw
26-neighbour edge list, and the md5 of its CSR is recorded too, so the
package's `grid27_graph` is checked against the reference's preprocessing.
Merges into tests/golden/reference_big.json."""
import hashlib
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

OUT = Path(__file__).parent / "reference_big.json"

CASES = {
    "grid27_128": (("grid27", 128), 64),
    "rgg16m": (("rgg", 1 << 24, math.sqrt(12 / (math.pi * (1 << 24))), 0), 256),
    "rmat22": (("rmat", 22, 16, 0), 64),
    # small cases to exercise the script quickly
    "grid27_32": (("grid27", 32), 64),
}


def md5_i64(a):
    return hashlib.md5(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def raw_grid27(N):
    """Raw 26-neighbour edge list (each undirected edge once, u < v)."""
    idx = np.arange(N ** 3, dtype=np.int64).reshape(N, N, N)
    us, vs = [], []
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            for c in (-1, 0, 1):
                if (a, b, c) <= (0, 0, 0):
                    continue
                src = idx[max(0, -a):N - max(0, a), max(0, -b):N - max(0, b), max(0, -c):N - max(0, c)]
                dst = idx[max(0, a):N - max(0, -a) or None, max(0, b):N - max(0, -b) or None,
                          max(0, c):N - max(0, -c) or None]
                us.append(src.ravel())
                vs.append(dst.ravel())
    return np.stack([np.concatenate(us), np.concatenate(vs)], axis=1)


def build(spec):
    from jetpart import generators
    from jetpart.graph import preprocess
    if spec[0] == "grid27":
        N = spec[1]
        g, _ = preprocess(raw_grid27(N), N ** 3)
        return g
    if spec[0] == "rmat":
        return generators.rmat_graph(spec[1], spec[2], spec[3])
    return generators.geometric_graph(spec[1], spec[2], spec[3])


def run(name):
    from jetpart.driver import partition
    from jetpart.refine import RefinerConfig
    spec, k = CASES[name]
    t = time.time()
    g = build(spec)
    tg = time.time() - t
    print(name, "n", g.n, "m", g.m, "gen", round(tg, 1), "s", flush=True)
    t = time.perf_counter()
    r = partition(g, RefinerConfig(k=k, imbalance=0.03, seed=0))
    tp = time.perf_counter() - t
    st = r.state
    levels = [[int(L["level"]), int(L["n"]), int(L["m"]), int(L["iterations"]), int(L["cut_out"])]
              for L in r.metrics["levels"]]
    rec = {
        "spec": list(spec), "k": k, "imbalance": 0.03, "seed": 0,
        "n": int(g.n), "m": int(g.m),
        "csr_md5": {"row_offsets": md5_i64(g.row_offsets), "adjacency": md5_i64(g.adjacency),
                    "edge_weights": md5_i64(g.edge_weights)},
        "cut": int(st.cutsize), "parts_md5": md5_i64(st.parts),
        "part_weights": [int(x) for x in st.part_weights],
        "balanced": bool(r.metrics["balanced"]), "n_levels": int(r.metrics["n_levels"]),
        "levels": levels,
        "reference_seconds": {kk: round(float(v), 2) for kk, v in r.metrics["times"].items()},
        "host": {"cpu_count": os.cpu_count(), "threads_used": 1},
    }
    print(name, "cut", rec["cut"], "md5", rec["parts_md5"], "t", round(tp, 1), flush=True)
    d = json.loads(OUT.read_text()) if OUT.exists() else {}
    d[name] = rec
    OUT.write_text(json.dumps(d, indent=1) + "\n")


if __name__ == "__main__":
    for name in sys.argv[1:] or ["grid27_128"]:
        run(name)
