"""Benchmark / test inputs. Graph generation is outside the partitioner's
hot path. Lattices are built on the host (numpy): the
same CSR the reference's generators produce, without its preprocess pass (a
lattice is connected and already clean, so preprocess is the identity).
R-MAT and random geometric graphs are generated on the device (csrc/gen.cu),
bit-identical to the reference's rmat_graph / geometric_graph + preprocess.
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


# ---------------------------------------------------------------------------
# Random inputs, generated on the device (csrc/gen.cu): the same graphs the
# reference's rmat_graph / geometric_graph + preprocess produce
# (generators.py:32-97, graph.py:132-200), replayed from numpy's PCG64 stream.

def rmat_device(scale: int, edge_factor: int = 8, seed: int = 0,
                probs=(0.57, 0.19, 0.19, 0.05), ctx=None):
    """R-MAT graph (largest component) resident on the device."""
    import ctypes as C
    from . import _lib
    ctx = ctx or _lib.Context.default()
    pr = np.ascontiguousarray(probs, dtype=np.float64)
    if pr.shape != (4,):
        raise ValueError("probs must have four entries")
    h = C.c_void_p()
    _lib.check(_lib.lib().jet_generate_rmat(ctx.handle, int(scale), int(edge_factor),
                                            int(seed), _lib.ptr(pr), C.byref(h)))
    return _lib.DeviceGraph(ctx, h)


def geometric_device(n: int, radius: float, seed: int = 0, ctx=None):
    """Random geometric graph on the unit square (largest component), on the device."""
    import ctypes as C
    from . import _lib
    ctx = ctx or _lib.Context.default()
    h = C.c_void_p()
    _lib.check(_lib.lib().jet_generate_geometric(ctx.handle, int(n), float(radius), int(seed),
                                                 C.byref(h)))
    return _lib.DeviceGraph(ctx, h)


def _host(dg) -> Graph:
    offs, adj, ew, vw = dg.download()
    return Graph(offs, adj, ew, vw)


def rmat_graph(scale: int, edge_factor: int = 8, seed: int = 0,
               probs=(0.57, 0.19, 0.19, 0.05)) -> Graph:
    """The reference's rmat_graph (generators.py:32-55), generated on the device."""
    dg = rmat_device(scale, edge_factor, seed, probs)
    try:
        return _host(dg)
    finally:
        dg.free()


def geometric_graph(n: int, radius: float, seed: int = 0) -> Graph:
    """The reference's geometric_graph (generators.py:58-97), generated on the device."""
    dg = geometric_device(n, radius, seed)
    try:
        return _host(dg)
    finally:
        dg.free()
