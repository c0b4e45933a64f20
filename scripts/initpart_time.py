"""t_initial (host vs device initial partitioning) on a few workloads."""
import math, sys, statistics
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
ctx = _lib.Context(0)
for name, mk, k in (("grid27_128", lambda: _lib.DeviceGraph.upload(gen.grid27_graph(128), ctx), 64),
                    ("rmat22", lambda: gen.rmat_device(22, 16, 0, ctx=ctx), 64),
                    ("rmat20_k1024", lambda: gen.rmat_device(20, 16, 0, ctx=ctx), 1024),
                    ("rgg24", lambda: gen.geometric_device(1 << 24, math.sqrt(12 / (math.pi * (1 << 24))), 0, ctx=ctx), 256)):
    dg = mk()
    out = []
    for dev in (False, True):
        cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=False, device_initial_partition=dev)
        ts, tot = [], []
        for _ in range(3):
            _, _, st = partition_resident(dg, None, cfg, want_parts=False)
            ts.append(st.t_initial * 1e3); tot.append(st.t_total * 1e3)
        out.append(f"{'device' if dev else 'host'} init {statistics.median(ts):.2f} ms total {statistics.median(tot):.1f} ms cut {st.cutsize}")
    print(name, " | ".join(out), flush=True)
    dg.free()
