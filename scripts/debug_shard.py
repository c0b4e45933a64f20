import sys, threading, traceback, os
sys.path.insert(0, '.')
import numpy as np
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import _lib, generators as gen
from paper_2304_13194_b200.driver import partition_resident
g = gen.grid27_graph(32)
cfg = J.RefinerConfig(k=16, imbalance=0.03, seed=1, deterministic=True)
ref = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
print("ref cut", ref[2].cutsize, flush=True)
size = 2
group = _lib.LocalGroup(size)
ctxs = [_lib.Context(0) for _ in range(size)]
dgs = []
for r, c in enumerate(ctxs):
    c.attach_local(group, r)
    c.set_shard_min_vertices(2000)
    dgs.append(_lib.DeviceGraph.upload(g, c))
out = [None] * size
def work(r):
    try:
        out[r] = partition_resident(dgs[r], g, cfg)
        print("rank", r, "cut", out[r][2].cutsize, flush=True)
    except Exception:
        print("rank", r, "ERROR", traceback.format_exc(), flush=True)
ths = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(size)]
for t in ths: t.start()
for t in ths: t.join(timeout=60)
print("alive", [t.is_alive() for t in ths], flush=True)
os._exit(0)
