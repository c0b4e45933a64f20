"""Partition BASELINE configs 3-4 on the device: R-MAT 2^22 ef16 k=64 and
RGG 2^24 (mean degree ~12) k=256, generated on the device. Prints generation
and partition times, cut, balance, levels."""
import math, os, sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident

which = sys.argv[1:] or ["rmat22", "rgg16m"]
mode = os.environ.get("JET_MODE", "det") == "det"
ctx = _lib.Context.default()
for name in which:
    t = time.perf_counter()
    if name.startswith("rmat"):
        scale = int(name[4:])
        dg = gen.rmat_device(scale, 16, 0, ctx=ctx)
        k = 64
    else:
        n = 1 << 24 if name == "rgg16m" else int(name[3:])
        dg = gen.geometric_device(n, math.sqrt(12 / (math.pi * n)), 0, ctx=ctx)
        k = 256
    ctx.synchronize()
    tg = time.perf_counter() - t
    n, nnz, W = dg.info()
    cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=mode)
    for rep in range(3):
        ctx.profile(rep == 2)
        ctx.profile_reset()
        t = time.perf_counter()
        parts, pw, st = partition_resident(dg, None, cfg, want_parts=False)
        tp = time.perf_counter() - t
        print(f"{name}: n={n} m={nnz//2} gen={tg:.3f}s rep{rep} partition={tp:.3f}s "
              f"(coarsen {st.t_coarsen:.3f} init {st.t_initial:.3f} unc {st.t_uncoarsen:.3f}) "
              f"cut={st.cutsize} balanced={st.balanced} levels={st.n_levels} "
              f"launches={st.kernel_launches}", flush=True)
    rp = ctx.profile_report()
    tot = sum(v['ms'] for k_, v in rp.items() if k_ != '__total__')
    for nm, v in sorted(rp.items(), key=lambda x: -x[1]['ms'])[:14]:
        if nm != '__total__':
            print(f"   {nm:20s} launches={v['launches']:6d} ms={v['ms']:9.3f} ({100*v['ms']/tot:5.1f}%)")
    for i in range(st.n_levels):
        L = st.levels[i]
        print(f"   L{L.level}: n={L.n} m={L.m} iters={L.iterations} lp={L.lp_passes} w={L.weak_passes} "
              f"s={L.strong_passes} cut {L.cut_in}->{L.cut_out} {L.seconds*1e3:.1f}ms", flush=True)
    dg.free()
