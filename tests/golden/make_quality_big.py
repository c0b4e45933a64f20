"""Reference cutsizes for BASELINE configs 3-4 (seed 0), from the reference's
own generators (imported read-only from /root/reference) and the C oracle
(oracle/, pinned against the reference). Slow (minutes); run once:
    python tests/golden/make_quality_big.py [rmat22|rgg16m]
Merges into tests/golden/quality.json."""
import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "oracle"))

CASES = {
    "rmat22": (("rmat", 22, 16, 0), 64),
    "rgg16m": (("rgg", 1 << 24, math.sqrt(12 / (math.pi * (1 << 24))), 0), 256),
}

if __name__ == "__main__":
    import oracle as O
    from jetpart import generators
    names = sys.argv[1:] or list(CASES)
    f = Path(__file__).parent / "quality.json"
    for name in names:
        spec, k = CASES[name]
        t = time.time()
        g = generators.rmat_graph(spec[1], spec[2], spec[3]) if spec[0] == "rmat" else \
            generators.geometric_graph(spec[1], spec[2], spec[3])
        tg = time.time() - t
        t = time.time()
        r = O.partition(g, k=k, imbalance=0.03, seed=0)
        tp = time.time() - t
        print(name, g.n, g.m, "gen", round(tg, 1), "s partition", round(tp, 1), "s cut", r["cut"], flush=True)
        d = json.loads(f.read_text())
        d[name] = {"spec": list(spec), "k": k, "imbalance": 0.03, "cuts": {"0": int(r["cut"])},
                   "n": int(g.n), "m": int(g.m), "oracle_partition_s": round(tp, 1)}
        f.write_text(json.dumps(d, indent=1) + "\n")
