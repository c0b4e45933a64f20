"""Initial-partitioning cost at large k: RGG 2^20, k=1024."""
import math, sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
ctx = _lib.Context.default()
n = 1 << 20
dg = gen.geometric_device(n, math.sqrt(12 / (math.pi * n)), 0, ctx=ctx)
for k in (256, 1024):
    cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=True)
    for rep in range(2):
        t = time.perf_counter()
        _, pw, st = partition_resident(dg, None, cfg, want_parts=False)
        print(f"k={k} rep{rep}: total {time.perf_counter()-t:.3f}s coarsen {st.t_coarsen:.3f} "
              f"init {st.t_initial:.3f} unc {st.t_uncoarsen:.3f} cut {st.cutsize} bal {st.balanced} "
              f"levels {st.n_levels}", flush=True)
