"""Per-level x per-kernel event profile of one partition."""
import sys, collections
sys.path.insert(0, '.')
import os
import paper_2304_13194_b200 as J
DET = os.environ.get('JET_MODE', 'det') == 'det'
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = gen.grid27_graph(N)
ctx = _lib.Context.default()
dg = _lib.DeviceGraph.upload(g, ctx)
cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=DET)
partition_resident(dg, g, cfg, want_parts=False)
ctx.profile(True); ctx.profile_only("@levels"); ctx.profile_reset()
parts, pw, st = partition_resident(dg, g, cfg, want_parts=False)
rep = ctx.profile_report()
lv = collections.defaultdict(dict)
for name, v in rep.items():
    if ':' not in name: continue
    l, kname = name.split(':', 1)
    lv[l][kname] = v
def order(l):
    return -1 if l == 'coarsen' else int(l[1:])
for l in sorted(lv, key=order):
    tot = sum(v['ms'] for v in lv[l].values())
    n = sum(v['launches'] for v in lv[l].values())
    top = sorted(lv[l].items(), key=lambda x: -x[1]['ms'])[:7]
    print(f"{l:8s} {tot:7.2f}ms {n:5d}L | " + "  ".join(f"{k}:{v['launches']}x{1e3*v['ms']/v['launches']:.0f}us" for k, v in top))
print("cut", st.cutsize)
