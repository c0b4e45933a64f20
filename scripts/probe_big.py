"""Largest R-MAT the single-GPU path takes today (config 5 shape, smaller
scale): R-MAT 2^25 ef16, k=1024, both modes."""
import sys, time
sys.path.insert(0, '.')
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, _lib
from paper_2304_13194_b200.driver import partition_resident
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 25
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ctx = _lib.Context.default()
t = time.perf_counter()
dg = gen.rmat_device(scale, 16, 0, ctx=ctx)
ctx.synchronize()
n, nnz, W = dg.info()
print(f"rmat{scale}: n={n} m={nnz//2} gen={time.perf_counter()-t:.2f}s", flush=True)
for det in (False, True):
    cfg = J.RefinerConfig(k=k, imbalance=0.03, seed=0, deterministic=det)
    for rep in range(2):
        t = time.perf_counter()
        _, pw, st = partition_resident(dg, None, cfg, want_parts=False)
        el = time.perf_counter() - t
        print(f"  {'det ' if det else 'fast'} rep{rep}: {el:.3f}s coarsen {st.t_coarsen:.3f} init {st.t_initial:.3f} "
              f"unc {st.t_uncoarsen:.3f} cut {st.cutsize} bal {st.balanced} levels {st.n_levels} "
              f"edges/s {(nnz//2)/el:.3e}", flush=True)
