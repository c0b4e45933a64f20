"""Median CUDA-event time of the device-resident headline partition (L2 flushed
before each), throughput mode unless JET_MODE=det; for A/B of builds (JET_LIB)."""
import os, statistics, sys
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
g = gen.grid27_graph(128)
cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=os.environ.get("JET_MODE") == "det")
ctx = _lib.Context(0)
dg = _lib.DeviceGraph.upload(g, ctx)
for _ in range(3):
    partition_resident(dg, g, cfg, want_parts=False)
ts = []
for _ in range(10):
    ctx.flush_l2()
    ctx.synchronize()
    ctx.timer_start()
    partition_resident(dg, g, cfg, want_parts=False)
    ts.append(ctx.timer_stop())
print("median %.2f ms min %.2f max %.2f" % (statistics.median(ts), min(ts), max(ts)))
