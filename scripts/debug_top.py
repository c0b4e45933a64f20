import sys, hashlib, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import graph_of
import paper_2304_13194_b200 as J
d = dict(np.load('tests/golden/pipeline.npz'))
i = int(sys.argv[1])
g = graph_of(d, f"p{i}_")
k, seed, ab, lk = (int(x) for x in d[f"p{i}_cfg"])
imb = float(d[f"p{i}_imb"][0])
cfg = J.RefinerConfig(k=k, imbalance=imb, seed=seed, afterburner=bool(ab), locking=bool(lk))
h = J.build_hierarchy(g, max(200, 2 * k, 32))
top = len(h.levels) - 1
gc = h.levels[top]
st = J.initial_partition(gc, k, imb, seed=seed, restarts=8)
print("init pw", st.part_weights.tolist(), "limit", J.part_weight_limit(int(np.sum(gc.vertex_weights)), k, imb))
out, stats = J.jet_refine(gc, st, cfg, finest=False, seed_path=(top,))
print("top", top, "pw", out.part_weights.tolist(), "cut", out.cutsize, stats["iterations"], stats["balanced"],
      hashlib.md5(out.parts.tobytes()).hexdigest()[:12])
