"""Reference cutsizes for BASELINE configs 3-4 (partition seeds 0-4 on the
seed-0 graph), from the reference's own generators (imported read-only from
/root/reference) and the C oracle (oracle/, pinned against the reference).
Slow (minutes per seed; seeds run in parallel processes); run once:
    python tests/golden/make_quality_big.py [rmat22|rgg16m] [--seeds 0,1,2,3,4]
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

_G = None
_K = None


def _init(g, k):
    global _G, _K
    sys.path.insert(0, str(ROOT / "oracle"))
    _G, _K = g, k


def _one(seed):
    import oracle as O
    t = time.time()
    r = O.partition(_G, k=_K, imbalance=0.03, seed=seed)
    return seed, int(r["cut"]), round(time.time() - t, 1)


if __name__ == "__main__":
    import multiprocessing as mp
    from jetpart import generators
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    seeds = [0]
    if "--seeds" in sys.argv:
        seeds = [int(x) for x in sys.argv[sys.argv.index("--seeds") + 1].split(",")]
        args = [a for a in args if a != sys.argv[sys.argv.index("--seeds") + 1]]
    names = args or list(CASES)
    f = Path(__file__).parent / "quality.json"
    for name in names:
        spec, k = CASES[name]
        t = time.time()
        g = generators.rmat_graph(spec[1], spec[2], spec[3]) if spec[0] == "rmat" else \
            generators.geometric_graph(spec[1], spec[2], spec[3])
        tg = time.time() - t
        globals()["_G"], globals()["_K"] = g, k
        if len(seeds) == 1 or "--serial" in sys.argv:
            res = [_one(sd) for sd in seeds]
        else:  # spawn, not fork: the oracle's OpenMP runtime does not survive a fork
            with mp.get_context("spawn").Pool(min(len(seeds), 4), initializer=_init,
                                              initargs=(g, k)) as pool:
                res = pool.map(_one, seeds)
        for seed, cut, tp in res:
            print(name, g.n, g.m, "gen", round(tg, 1), "s seed", seed, "partition", tp, "s cut", cut,
                  flush=True)
        d = json.loads(f.read_text())
        rec = d.get(name, {"spec": list(spec), "k": k, "imbalance": 0.03, "cuts": {},
                           "n": int(g.n), "m": int(g.m)})
        for seed, cut, tp in res:
            rec["cuts"][str(seed)] = cut
            if seed == 0:
                rec["oracle_partition_s"] = tp
        d[name] = rec
        f.write_text(json.dumps(d, indent=1) + "\n")
