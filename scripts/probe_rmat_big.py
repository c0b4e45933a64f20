"""BASELINE configs[4] shape on one GPU: R-MAT scale S (default 27), edge
factor 16, k=1024, generated on the device; one partition per mode with
per-level stats. python scripts/probe_rmat_big.py [scale] [modes]"""
import os, sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fast", "det"]
ctx = _lib.Context.default()
t = time.perf_counter()
dg = gen.rmat_device(scale, 16, 0, ctx=ctx)
n, nnz, W = dg.info()
print(f"rmat {scale}: n={n} m={nnz // 2} gen {time.perf_counter() - t:.2f}s", flush=True)
for mode in modes:
    cfg = J.RefinerConfig(k=int(os.environ.get("JET_K", "1024")), imbalance=0.03, seed=0,
                          deterministic=(mode == "det"))
    for rep in range(2 if len(sys.argv) > 3 else 1):
        ctx.timer_start()
        t = time.perf_counter()
        _, pw, st = partition_resident(dg, None, cfg, want_parts=False)
        ms = ctx.timer_stop()
        print(f"{mode} rep{rep}: device {ms / 1e3:.3f}s wall {time.perf_counter() - t:.3f}s "
              f"coarsen {st.t_coarsen:.3f} init {st.t_initial:.3f} unc {st.t_uncoarsen:.3f} "
              f"cut {st.cutsize} bal {st.balanced} levels {st.n_levels} "
              f"edges/s {nnz / 2 / (ms / 1e3):.3e}", flush=True)
        for i in range(st.n_levels):
            L = st.levels[i]
            print(f"  L{L.level}: n={L.n} m={L.m} it={L.iterations} lp={L.lp_passes} "
                  f"w={L.weak_passes} s={L.strong_passes} cut {L.cut_in}->{L.cut_out} "
                  f"{L.seconds * 1e3:.1f}ms", flush=True)
