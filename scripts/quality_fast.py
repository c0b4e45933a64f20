"""Throughput mode vs the reference's cuts (tests/golden/quality.json): every
recorded case and seed, time, cut ratio, balance."""
import json, math, sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
q = json.load(open('tests/golden/quality.json'))
ctx = _lib.Context.default()
for name, case in q.items():
    spec = case["spec"]
    if spec[0] == "grid":
        g = gen.grid_graph(spec[1], spec[2]); dg = _lib.DeviceGraph.upload(g, ctx)
    elif spec[0] == "grid27":
        g = gen.grid27_graph(spec[1]); dg = _lib.DeviceGraph.upload(g, ctx)
    elif spec[0] == "rmat":
        g = None; dg = gen.rmat_device(spec[1], spec[2], spec[3], ctx=ctx)
    else:
        g = None; dg = gen.geometric_device(spec[1], spec[2], spec[3], ctx=ctx)
    ratios = []
    for seed, ref in case["cuts"].items():
        for det in (True, False):
            cfg = J.RefinerConfig(k=case["k"], imbalance=0.03, seed=int(seed), deterministic=det)
            partition_resident(dg, g, cfg, want_parts=False)
            t = time.perf_counter()
            _, pw, st = partition_resident(dg, g, cfg, want_parts=False)
            el = time.perf_counter() - t
            if not det:
                ratios.append(st.cutsize / ref)
            print(f"{name} seed {seed} {'det ' if det else 'fast'}: {el*1e3:8.1f} ms cut {st.cutsize} "
                  f"ratio {st.cutsize/ref:.4f} bal {st.balanced}", flush=True)
    print(f"{name}: fast geomean ratio {math.exp(sum(map(math.log, ratios))/len(ratios)):.4f}", flush=True)
