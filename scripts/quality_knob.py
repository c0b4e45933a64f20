"""Throughput-mode time and cut on 128^3 (seeds 0-4) and configs 3-4 (seed 0)
under the current environment (knob experiments)."""
import math, os, statistics, sys, json
CPV = int(os.environ.get('CPV', '4')); CPF = int(os.environ.get('CPF', '0')); CT = int(os.environ.get('CT', '200'))
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
q = json.load(open('tests/golden/quality.json'))
ctx = _lib.Context(0)
out = []
g2 = gen.grid_graph(256, 256); d2 = _lib.DeviceGraph.upload(g2, ctx)
r2 = []
for seed in range(5):
    cfg = J.RefinerConfig(k=8, imbalance=0.03, seed=seed, deterministic=False, throughput_patience=CPV, patience_from_level=CPF, coarse_target=CT)
    _, pw, st = partition_resident(d2, g2, cfg, want_parts=False)
    r2.append(st.cutsize / q['grid2d_256x256']['cuts'][str(seed)])
geo2 = math.exp(sum(map(math.log, r2)) / 5)
out.append(f"geo256={geo2:.4f}")
d2.free()
g = gen.grid27_graph(128); dg = _lib.DeviceGraph.upload(g, ctx)
rat = []
for seed in range(5):
    cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=seed, deterministic=False, throughput_patience=CPV, patience_from_level=CPF, coarse_target=CT)
    partition_resident(dg, g, cfg, want_parts=False)
    ts = []
    for _ in range(3):
        ctx.flush_l2(); ctx.timer_start(); _, pw, st = partition_resident(dg, g, cfg, want_parts=False); ts.append(ctx.timer_stop())
    rat.append(st.cutsize / q['grid27_128']['cuts'][str(seed)])
    out.append(f"g128 s{seed} {statistics.median(ts):.2f}ms r={rat[-1]:.4f} bal={st.balanced}")
geo = math.exp(sum(map(math.log, rat)) / 5)
dg.free()
for name, k in (("rmat22", 64), ("rgg16m", 256)):
    dg = gen.rmat_device(22, 16, 0, ctx=ctx) if name == "rmat22" else gen.geometric_device(1 << 24, math.sqrt(12 / (math.pi * (1 << 24))), 0, ctx=ctx)
    cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=False, throughput_patience=CPV, patience_from_level=CPF, coarse_target=CT)
    partition_resident(dg, None, cfg, want_parts=False)
    ts = []
    for _ in range(2):
        ctx.flush_l2(); ctx.timer_start(); _, pw, st = partition_resident(dg, None, cfg, want_parts=False); ts.append(ctx.timer_stop())
    out.append(f"{name} {min(ts):.1f}ms r={st.cutsize / q[name]['cuts']['0']:.4f} bal={st.balanced}")
    dg.free()
print(f"geo128={geo:.4f} | " + " | ".join(out), flush=True)
