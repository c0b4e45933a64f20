"""Per-run event time and host-side stage times of the device-resident headline
partition (throughput mode), to locate timing outliers."""
import sys
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
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    ctx.flush_l2()
    ctx.synchronize()
    ctx.timer_start()
    _, _, st = partition_resident(dg, g, cfg, want_parts=False)
    t = ctx.timer_stop()
    print(f"{i:2d} event {t:6.1f} ms  coarsen {st.t_coarsen*1e3:6.1f} init {st.t_initial*1e3:5.1f} "
          f"unc {st.t_uncoarsen*1e3:6.1f} total {st.t_total*1e3:6.1f}", flush=True)
