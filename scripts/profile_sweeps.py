"""Isolate the refinement sweeps for ncu (run under --profile-from-start off):
one Jetlp pass and one weak/strong rebalance pass on L0 and L1 of the 128^3
27-point grid, starting from the final partition (projected to L1)."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen, ops

cu = ctypes.CDLL("libcuda.so.1")
g = gen.grid27_graph(128)
cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=True)
res = J.partition(g, cfg)
p0 = res.state.parts.copy()
h = J.build_hierarchy(g, 128)
g1, vmap = h.levels[1], h.maps[0]
p1 = np.zeros(g1.n if hasattr(g1, "n") else len(g1.row_offsets) - 1, np.int64)
p1[vmap] = p0


def unbalance(graph, parts, k):
    # push 2% of part 0..7's neighbours' weight into parts 0..7: a weak pass then has work
    parts = parts.copy()
    n = len(parts)
    rng = np.random.default_rng(1)
    idx = rng.choice(n, size=n // 50, replace=False)
    parts[idx] = parts[idx] % 8
    return parts


for name, gg, pp in (("L0", g, p0), ("L1", g1, p1)):
    st = J.PartitionState.from_parts(gg, pp, 64)
    ub = J.PartitionState.from_parts(gg, unbalance(gg, pp, 64), 64)
    W = int(np.sum(gg.vertex_weights))
    lim = int((1 + 0.03) * W // 64)
    sigma = lim - max(1, int(0.1 * 0.03 * W / 64))
    ops.select_destinations(gg, st)  # warm (uploads the graph)
    cu.cuProfilerStart()
    ops.select_destinations(gg, st)
    ops.jetlp_pass(gg, st, None, 0.25)
    ops.weak_rebalance_pass(gg, ub, None, lim, sigma, np.random.default_rng([0, 0, 1]))
    ops.strong_rebalance_pass(gg, ub, None, lim, sigma, np.random.default_rng([0, 0, 1]))
    cu.cuProfilerStop()
    print(name, "done", flush=True)
