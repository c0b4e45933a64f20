import sys
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
ctx = _lib.Context.default()
dg = gen.rmat_device(int(sys.argv[1]), 16, 0, ctx=ctx)
cfg = J.RefinerConfig(k=int(sys.argv[2]), imbalance=0.03, seed=0, deterministic=True)
_, pw, st = partition_resident(dg, None, cfg, want_parts=False)
for i in range(st.n_levels):
    L = st.levels[i]
    print(f"   L{L.level}: n={L.n} m={L.m} iters={L.iterations} lp={L.lp_passes} w={L.weak_passes} s={L.strong_passes} {L.seconds*1e3:.1f}ms", flush=True)
