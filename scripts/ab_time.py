"""A/B timing helper: median device time of partitions of one workload in
both modes (L2 flushed before each), the cut, and (JET_PHASES=1) nothing
else. Variants are chosen by environment (JET_LIB, JET_LV_* knobs).
  python scripts/ab_time.py [grid N | rmat S | rgg LOG2N] [k] [reps]"""
import os, sys, statistics
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
kind = sys.argv[1] if len(sys.argv) > 1 else "grid"
size = int(sys.argv[2]) if len(sys.argv) > 2 else 128
k = int(sys.argv[3]) if len(sys.argv) > 3 else 64
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 7
ctx = _lib.Context(0)
if kind == "grid":
    g = gen.grid27_graph(size); dg = _lib.DeviceGraph.upload(g, ctx)
elif kind == "rmat":
    g = None; dg = gen.rmat_device(size, 16, 0, ctx=ctx)
else:
    import math
    g = None; n = 1 << size; dg = gen.geometric_device(n, math.sqrt(12 / (math.pi * n)), 0, ctx=ctx)
out = []
for det in (False, True):
    cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=det)
    for _ in range(2):
        partition_resident(dg, g, cfg, want_parts=False)
    ts = []
    for _ in range(reps):
        ctx.flush_l2(); ctx.timer_start()
        _, pw, st = partition_resident(dg, g, cfg, want_parts=False)
        ts.append(ctx.timer_stop())
    out.append(f"{'det' if det else 'fast'} {statistics.median(ts):.2f} ms (min {min(ts):.2f}) cut={st.cutsize} bal={st.balanced}")
print(" | ".join(out), flush=True)
