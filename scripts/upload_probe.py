import os, sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen
print("cpus", os.cpu_count())
g = gen.grid27_graph(128)
cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=True)
for th in ["4", "8", "16", "32"]:
    os.environ["JET_UPLOAD_THREADS"] = th
    J.partition(g, cfg)
    ts = []
    for _ in range(3):
        t = time.perf_counter(); r = J.partition(g, cfg); ts.append(time.perf_counter() - t)
    print(th, [round(x*1e3,1) for x in ts], {k: round(v*1e3, 1) for k, v in r.metrics["times"].items()})
