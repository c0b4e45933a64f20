import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import graph_of
import paper_2304_13194_b200 as J
d = dict(np.load('tests/golden/pipeline.npz'))
i = int(sys.argv[1])
g = graph_of(d, f"p{i}_")
k, seed, ab, lk = (int(x) for x in d[f"p{i}_cfg"])
cfg = J.RefinerConfig(k=k, imbalance=float(d[f"p{i}_imb"][0]), seed=seed, afterburner=bool(ab), locking=bool(lk))
res = J.partition(g, cfg)
print("iters", [lv["iterations"] for lv in res.metrics["levels"]], "ref", d[f"p{i}_iters"].tolist(), "cut", res.state.cutsize, d[f"p{i}_cut"][0])
