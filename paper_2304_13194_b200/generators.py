"""Benchmark / test inputs (host numpy). Graph generation is outside the
partitioner's hot path; these build the same CSR the
reference's generators produce for lattices, without its preprocess pass
(a lattice is connected and already clean, so preprocess is the identity).
"""

from __future__ import annotations

import numpy as np

from .graph import Graph


def _stencil_graph(dims, offsets, dtype=np.int64) -> Graph:
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    coords = np.indices(dims, dtype=np.int32).reshape(len(dims), -1)
    strides = np.array([int(np.prod(dims[i + 1:])) for i in range(len(dims))], dtype=np.int64)
    # offsets in ascending id order give rows sorted by neighbour id
    offsets = sorted(offsets, key=lambda o: int(np.dot(o, strides)))
    nbr = np.full((n, len(offsets)), -1, dtype=np.int64)
    ids = np.arange(n, dtype=np.int64)
    for j, off in enumerate(offsets):
        ok = np.ones(n, dtype=bool)
        for a, d in enumerate(off):
            c = coords[a] + d
            ok &= (c >= 0) & (c < dims[a])
        nbr[ok, j] = ids[ok] + int(np.dot(off, strides))
    valid = nbr >= 0
    deg = valid.sum(axis=1)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=offs[1:])
    adj = nbr[valid].astype(dtype)
    return Graph(offs, adj, np.ones(len(adj), dtype=dtype), np.ones(n, dtype=dtype))


def grid_graph(rows: int, cols: int, dtype=np.int64) -> Graph:
    """4-neighbour lattice, id = r*cols + c (generators.py:11-18)."""
    return _stencil_graph((rows, cols), [(-1, 0), (0, -1), (0, 1), (1, 0)], dtype)


def cube_graph(nx: int, ny: int, nz: int, dtype=np.int64) -> Graph:
    """6-neighbour cubic mesh (generators.py:21-29)."""
    offs = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    return _stencil_graph((nx, ny, nz), offs, dtype)


def grid27_graph(nx: int, ny: int | None = None, nz: int | None = None, dtype=np.int64) -> Graph:
    """3D 27-point stencil (26 neighbours), id = (x*ny + y)*nz + z."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
            if (a, b, c) != (0, 0, 0)]
    return _stencil_graph((nx, ny, nz), offs, dtype)
