"""Test-side graph builders and sequential checkers (test infrastructure, not
product code). The random-graph recipe follows the reference's test fixture
(pkg/tests/conftest.py:43-58: G(n, p) with p = min(1, 3/n), largest
component); the checkers restate reference semantics literally, one loop per
definition, so the GPU results are compared against an independent statement."""

from __future__ import annotations

import numpy as np
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components

from paper_2304_13194_b200 import Graph, PartitionState, from_edge_arrays


def graph_from_edges(edges, n, vertex_weights=None) -> Graph:
    t = [(e[0], e[1], e[2] if len(e) == 3 else 1) for e in edges]
    u = np.array([a for a, _, _ in t] + [b for _, b, _ in t], dtype=np.int64)
    v = np.array([b for _, b, _ in t] + [a for a, _, _ in t], dtype=np.int64)
    w = np.array([c for _, _, c in t] * 2, dtype=np.int64)
    return from_edge_arrays(n, u, v, w, vertex_weights)


def random_graph(rng, n_lo=8, n_hi=60, p=None, max_weight=1, max_vertex_weight=1) -> Graph:
    """Connected random graph: G(n, p), largest component (ties: lowest id),
    vertices renumbered in ascending order (graph.py:132-200 semantics)."""
    n = int(rng.integers(n_lo, n_hi + 1))
    if p is None:
        p = min(1.0, 3.0 / n)
    while True:
        iu, ju = np.triu_indices(n, k=1)
        mask = rng.random(len(iu)) < p
        if not mask.any():
            continue
        u, v = iu[mask].astype(np.int64), ju[mask].astype(np.int64)
        w = rng.integers(1, max_weight + 1, size=len(u)).astype(np.int64)
        vw = rng.integers(1, max_vertex_weight + 1, size=n).astype(np.int64)
        adj = csr_matrix((np.ones(len(u)), (u, v)), shape=(n, n))
        nc, lab = connected_components(adj, directed=False)
        sizes = np.bincount(lab, minlength=nc)
        first = np.array([np.flatnonzero(lab == c)[0] for c in range(nc)])
        best = min(range(nc), key=lambda c: (-sizes[c], first[c]))
        keep = lab == best
        if keep.sum() < 4:
            continue
        newid = np.full(n, -1, np.int64)
        newid[keep] = np.arange(int(keep.sum()))
        e = keep[u]
        uu, vv, ww = newid[u[e]], newid[v[e]], w[e]
        return from_edge_arrays(int(keep.sum()), np.concatenate([uu, vv]),
                                np.concatenate([vv, uu]), np.concatenate([ww, ww]), vw[keep])


def random_partition(rng, graph, k) -> PartitionState:
    return PartitionState.from_parts(graph, rng.integers(0, k, size=graph.n), k)


def brute_conn(graph, parts):
    """Per-vertex {part: weight} rows by direct summation (conn(v, p))."""
    out = []
    for v in range(graph.n):
        row = {}
        lo, hi = graph.row_offsets[v], graph.row_offsets[v + 1]
        for u, w in zip(graph.adjacency[lo:hi].tolist(), graph.edge_weights[lo:hi].tolist()):
            p = int(parts[u])
            row[p] = row.get(p, 0) + int(w)
        out.append(row)
    return out


def brute_cutsize(graph, parts) -> int:
    total = 0
    for v in range(graph.n):
        lo, hi = graph.row_offsets[v], graph.row_offsets[v + 1]
        for u, w in zip(graph.adjacency[lo:hi].tolist(), graph.edge_weights[lo:hi].tolist()):
            if parts[v] != parts[u]:
                total += int(w)
    return total // 2


def afterburner_sequential(graph, cand, parts, dests, gain):
    """refine.py:127-156 read literally: candidates ordered by (higher gain,
    lower id); each candidate sees the earlier ones as already moved."""
    cand = [int(c) for c in cand]
    in_c = set(cand)
    key = {v: (-int(gain[v]), v) for v in cand}
    out = []
    for v in cand:
        f = 0
        lo, hi = graph.row_offsets[v], graph.row_offsets[v + 1]
        for u, w in zip(graph.adjacency[lo:hi].tolist(), graph.edge_weights[lo:hi].tolist()):
            pu = int(dests[u]) if (u in in_c and key[u] < key[v]) else int(parts[u])
            if pu == int(dests[v]):
                f += w
            elif pu == int(parts[v]):
                f -= w
        out.append(f)
    return np.array(out, dtype=np.int64)


def gain_filter(gain, conn_self, c, boundary, locks):
    """refine.py:108-124: boundary, unlocked, -F < floor(conn_self * c)."""
    from fractions import Fraction
    fr = Fraction(str(c))
    lim = (np.asarray(conn_self, dtype=object) * fr.numerator) // fr.denominator
    ok = np.array([-int(g) < int(l) for g, l in zip(gain, lim)], dtype=bool)
    return np.asarray(boundary, bool) & ~np.asarray(locks, bool) & ok
