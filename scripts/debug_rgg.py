import os, sys
sys.path.insert(0, '.')
import numpy as np
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components
from paper_2304_13194_b200 import generators as gen
n, r, seed = 3000, 0.025, 2
os.environ["JET_GEN_NO_LCC"] = "1"
g = gen.geometric_graph(n, r, seed)
pts = np.random.default_rng([seed, n]).random((n, 2))
d = pts[:, None, :] - pts[None, :, :]
close = (d * d).sum(axis=2) <= r * r
np.fill_diagonal(close, False)
deg = close.sum(1)
print("nnz dev", len(g.adjacency), "ref", close.sum())
bad = np.flatnonzero(np.diff(g.row_offsets) != deg)
print("rows with wrong degree", len(bad), bad[:10], np.diff(g.row_offsets)[bad[:10]], deg[bad[:10]])
A = csr_matrix(close)
nc, lab = connected_components(A, directed=False)
sz = np.bincount(lab)
print("components", nc, "largest", sz.max())
os.environ["JET_GEN_NO_LCC"] = "0"
g2 = gen.geometric_graph(n, r, seed)
print("lcc n", g2.n, "nnz", len(g2.adjacency), "offs tail", g2.row_offsets[-5:])
