"""CSR graph container, partition state and metrics.

Mirrors the hot-path part of jetpart/graph.py: `Graph` (:17-62),
`from_edge_arrays` (:103-116), `part_weight_limit` (:203-212), `cutsize`
(:215-221), `PartitionState` (:224-258), `is_balanced` (:261-266),
`imbalance_of` (:269-273). Metrics over a whole graph run on the GPU.
Any object exposing row_offsets / adjacency / edge_weights / vertex_weights
(including the reference's own Graph) is accepted wherever a Graph is.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction
from functools import cached_property

import numpy as np

from . import _lib


@dataclass(eq=False)
class Graph:
    """Undirected weighted graph in CSR form; every edge stored twice."""

    row_offsets: np.ndarray
    adjacency: np.ndarray
    edge_weights: np.ndarray
    vertex_weights: np.ndarray

    @property
    def n(self) -> int:
        return len(self.row_offsets) - 1

    @property
    def m(self) -> int:
        return len(self.adjacency) // 2

    @cached_property
    def total_vertex_weight(self) -> int:
        return int(np.asarray(self.vertex_weights).sum())

    @cached_property
    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def neighbors(self, v):
        lo, hi = self.row_offsets[v], self.row_offsets[v + 1]
        return self.adjacency[lo:hi], self.edge_weights[lo:hi]

    @property
    def entry_rows(self) -> np.ndarray:
        """Row (source vertex) of every adjacency entry."""
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_offsets))

    def validate(self) -> None:
        """The reference's structural invariants (graph.py:64-100): CSR
        shape, id and weight ranges, no self loops or duplicate neighbours,
        symmetric entries with equal weights. Raises ValueError."""
        n, offs = self.n, np.asarray(self.row_offsets)
        adj, ew, vw = (np.asarray(a) for a in (self.adjacency, self.edge_weights,
                                                self.vertex_weights))
        checks = [
            (n >= 1, "graph must have at least one vertex"),
            (offs[0] == 0 and bool(np.all(offs[1:] >= offs[:-1])),
             "row_offsets must be non-decreasing from 0"),
            (offs[-1] == len(adj), "row_offsets[n] must equal adjacency length"),
            (len(ew) == len(adj), "edge_weights length mismatch"),
            (len(vw) == n, "vertex_weights length mismatch"),
            (len(adj) == 0 or (adj.min() >= 0 and adj.max() < n), "neighbor id out of range"),
            (bool(np.all(vw >= 1)), "vertex weights must be >= 1"),
            (bool(np.all(ew >= 1)), "edge weights must be >= 1"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        src = self.entry_rows
        if np.any(src == adj):
            raise ValueError("self-loop present")
        fwd = src * n + adj
        fo = np.argsort(fwd, kind="stable")
        if np.any(fwd[fo][1:] == fwd[fo][:-1]):
            raise ValueError("duplicate neighbor within a row")
        rev = adj * n + src
        ro = np.argsort(rev, kind="stable")
        if not (np.array_equal(fwd[fo], rev[ro]) and np.array_equal(ew[fo], ew[ro])):
            raise ValueError("adjacency is not symmetric with equal weights")


def graph_n(graph) -> int:
    return len(graph.row_offsets) - 1


def total_weight(graph) -> int:
    w = getattr(graph, "total_vertex_weight", None)
    return int(w) if w is not None else int(np.asarray(graph.vertex_weights).sum())


def from_edge_arrays(n, u, v, w, vertex_weights=None) -> Graph:
    """CSR from clean directed entry arrays, rows sorted by neighbour id."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.int64)
    order = np.lexsort((v, u))
    u, v, w = u[order], v[order], w[order]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(u, minlength=n), out=offsets[1:])
    if vertex_weights is None:
        vertex_weights = np.ones(n, dtype=np.int64)
    return Graph(offsets, v, w, np.asarray(vertex_weights, dtype=np.int64))


def part_weight_limit(total_weight: int, k: int, imbalance: float) -> int:
    """floor((1 + imbalance) * W / k) in exact rational arithmetic."""
    if imbalance < 0:
        raise ValueError("imbalance must be >= 0")
    factor = Fraction(1) + Fraction(str(imbalance))
    return int(factor * total_weight // k)


def _device_graph(graph, ctx=None):
    dg = getattr(graph, "_jet_device_graph", None)
    if dg is not None and dg.ctx is (ctx or _lib.Context.default()):
        return dg
    return _lib.DeviceGraph.upload(graph, ctx)


def cutsize(graph, parts) -> int:
    """Total weight of cut edges (GPU)."""
    if isinstance(parts, PartitionState):
        parts = parts.parts
    parts = _lib.as_i64(parts)
    dg = _device_graph(graph)
    out = C.c_int64()
    _lib.check(_lib.lib().jet_cutsize(dg.ctx.handle, dg.handle, _lib.ptr(parts), C.byref(out)))
    return int(out.value)


def part_weights(graph, parts, k) -> np.ndarray:
    parts = _lib.as_i64(parts)
    dg = _device_graph(graph)
    out = np.zeros(k, dtype=np.int64)
    _lib.check(_lib.lib().jet_part_weights(dg.ctx.handle, dg.handle, _lib.ptr(parts), k,
                                           _lib.ptr(out)))
    return out


@dataclass(eq=False)
class PartitionState:
    """A k-way partition with cached part weights and cutsize."""

    parts: np.ndarray
    k: int
    part_weights: np.ndarray
    cutsize: int

    @classmethod
    def from_parts(cls, graph, parts, k: int) -> "PartitionState":
        parts = np.asarray(parts, dtype=np.int64)
        if len(parts) != graph_n(graph):
            raise ValueError("partition length must equal vertex count")
        if len(parts) and (parts.min() < 0 or parts.max() >= k):
            raise ValueError("part id out of range")
        return cls(parts.copy(), k, part_weights(graph, parts, k), cutsize(graph, parts))

    def copy(self) -> "PartitionState":
        return PartitionState(self.parts.copy(), self.k, self.part_weights.copy(), self.cutsize)

    def check(self, graph) -> None:
        """Verify the cached part weights and cutsize (graph.py:250-258)."""
        fresh = PartitionState.from_parts(graph, self.parts, self.k)
        if not np.array_equal(fresh.part_weights, self.part_weights):
            raise ValueError("cached part weights are stale")
        if fresh.cutsize != self.cutsize:
            raise ValueError("cached cutsize is stale")
        if int(np.asarray(self.part_weights).sum()) != total_weight(graph):
            raise ValueError("part weights do not sum to total vertex weight")


def is_balanced(state, imbalance: float, total_weight=None) -> bool:
    if total_weight is None:
        total_weight = int(state.part_weights.sum())
    limit = part_weight_limit(total_weight, state.k, imbalance)
    return bool(np.all(state.part_weights <= limit))


def imbalance_of(state, total_weight=None) -> float:
    if total_weight is None:
        total_weight = int(state.part_weights.sum())
    return float(state.part_weights.max()) * state.k / total_weight
