"""Golden CSR of the 27-point stencil built through the reference's own
`preprocess` (graph.py:132-200) on a raw pair list, for the host generator's
parity test (grid27_graph builds the CSR directly, without preprocess).

Run in the build container (imports /root/reference read-only):
    python tests/golden/make_grid27.py   # writes tests/golden/grid27.npz
"""
import itertools
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
from jetpart.graph import preprocess  # noqa: E402

SHAPES = [(5, 5, 5), (3, 4, 6), (1, 7, 2)]

if __name__ == "__main__":
    d = {}
    for (nx, ny, nz) in SHAPES:
        idx = np.arange(nx * ny * nz, dtype=np.int64).reshape(nx, ny, nz)
        pairs = []
        for a, b, c in itertools.product((-1, 0, 1), repeat=3):
            if (a, b, c) == (0, 0, 0):
                continue
            sx = slice(max(0, -a), nx - max(0, a))
            sy = slice(max(0, -b), ny - max(0, b))
            sz = slice(max(0, -c), nz - max(0, c))
            src = idx[sx, sy, sz].ravel()
            dst = idx[max(0, a):nx + min(0, a), max(0, b):ny + min(0, b), max(0, c):nz + min(0, c)].ravel()
            pairs.append(np.stack([src, dst], axis=1))
        g, _ = preprocess(np.concatenate(pairs), nx * ny * nz)
        key = f"{nx}x{ny}x{nz}"
        d[key + "_offs"] = g.row_offsets
        d[key + "_adj"] = g.adjacency
        d[key + "_ew"] = g.edge_weights
        d[key + "_vw"] = g.vertex_weights
    np.savez_compressed(Path(__file__).with_name("grid27.npz"), **d)
    print("wrote", sorted(d))
