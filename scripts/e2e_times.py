"""Median upload / device / download split of partition() from host int64
arrays (headline workload, throughput mode); JET_UPLOAD_THREADS picks the
host staging threads."""
import os, sys, statistics
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen
g = gen.grid27_graph(128)
cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=False)
J.partition(g, cfg)
rows = []
for _ in range(7):
    r = J.partition(g, cfg)
    t = r.metrics["times"]
    rows.append((t["total"], t["upload"], t["device_pipeline"], t["download"]))
med = [statistics.median(x[i] for x in rows) * 1e3 for i in range(4)]
print(f"threads={os.environ.get('JET_UPLOAD_THREADS', '16')} cpus={os.cpu_count()} total={med[0]:.2f} "
      f"upload={med[1]:.2f} device={med[2]:.2f} download={med[3]:.2f} ms cut={r.state.cutsize}")
