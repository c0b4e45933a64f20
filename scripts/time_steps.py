"""Device-event step times of the headline partition under bench-like
conditions (L2 flush, profiling on/off) -- to find timing artefacts."""
import sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
g = gen.grid27_graph(128)
cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=True)
ctx = _lib.Context(0)
dg = _lib.DeviceGraph.upload(g, ctx)
for i in range(3):
    partition_resident(dg, g, cfg, want_parts=False)
for flush in (False, True):
    for prof in (False, True):
        ctx.profile(prof)
        ctx.profile_only("refine_level" if prof else None)
        ctx.profile_reset()
        ts, ws = [], []
        for _ in range(4):
            if flush:
                ctx.flush_l2()
            ctx.synchronize()
            w = time.perf_counter()
            ctx.timer_start()
            partition_resident(dg, g, cfg, want_parts=False)
            ts.append(ctx.timer_stop())
            ws.append(1e3 * (time.perf_counter() - w))
        print(f"flush={flush} prof={prof}: event ms {[round(t,1) for t in ts]} wall ms {[round(t,1) for t in ws]}", flush=True)
