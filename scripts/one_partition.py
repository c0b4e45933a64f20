"""One device-resident partition of a 27-point grid (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import os
import paper_2304_13194_b200 as J
DET = os.environ.get('JET_MODE', 'det') == 'det'
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = gen.grid27_graph(N)
ctx = _lib.Context.default()
dg = _lib.DeviceGraph.upload(g, ctx)
cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=DET)
for _ in range(reps):
    parts, pw, st = partition_resident(dg, g, cfg, want_parts=False)
print("cut", st.cutsize, "launches", st.kernel_launches)
