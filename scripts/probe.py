"""Quick performance probe: one partition of a named workload with the
per-kernel-class CUDA-event profile."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
import os
import paper_2304_13194_b200 as J
DET = os.environ.get('JET_MODE', 'det') == 'det'
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
t = time.perf_counter(); g = gen.grid27_graph(N); print("gen", time.perf_counter() - t, g.n, g.m, flush=True)
ctx = _lib.Context.default()
dg = _lib.DeviceGraph.upload(g, ctx)
cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=DET)
for rep in range(3):
    ctx.profile(rep == 2)
    ctx.profile_reset()
    t = time.perf_counter()
    parts, pw, st = partition_resident(dg, g, cfg)
    el = time.perf_counter() - t
    print(f"rep {rep}: {el:.3f}s cut={st.cutsize} bal={st.balanced} levels={st.n_levels} "
          f"coarsen={st.t_coarsen:.3f} init={st.t_initial:.3f} unc={st.t_uncoarsen:.3f} launches={st.kernel_launches}", flush=True)
rep = ctx.profile_report()
tot = sum(v['ms'] for k_, v in rep.items() if k_ != '__total__')
for name, v in sorted(rep.items(), key=lambda x: -x[1]['ms']):
    if name == '__total__': continue
    gbs = v['bytes'] / (v['ms'] * 1e-3) / 1e9 if v['ms'] > 0 else 0
    print(f"{name:20s} launches={v['launches']:6d} ms={v['ms']:9.3f} ({100*v['ms']/tot:5.1f}%) GB/s={gbs:8.1f}")
print("total device ms", tot)
for i in range(st.n_levels):
    L = st.levels[i]
    print(f"  L{L.level}: n={L.n} m={L.m} iters={L.iterations} lp={L.lp_passes} w={L.weak_passes} s={L.strong_passes} cut {L.cut_in}->{L.cut_out} {L.seconds*1e3:.1f}ms")
t = time.perf_counter()
res = J.partition(g, cfg)
print("e2e partition", time.perf_counter() - t, res.state.cutsize, res.metrics['times'])
