"""Per-step device-timed partitions (bench-like loop) to see step-to-step jitter."""
import sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
g = gen.grid27_graph(128)
cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=False)
ctx = _lib.Context(0)
dg = _lib.DeviceGraph.upload(g, ctx)
for _ in range(3):
    partition_resident(dg, g, cfg, want_parts=False)
for flush in (True, False):
    ts = []
    for _ in range(12):
        if flush:
            ctx.flush_l2()
        ctx.timer_start()
        partition_resident(dg, g, cfg, want_parts=False)
        ts.append(round(ctx.timer_stop(), 1))
    print("flush" if flush else "noflush", ts, flush=True)
