"""Per-kernel entry points with the reference's names and argument meaning.

Each function runs the corresponding sm_100a kernels through the C-ABI:
  match_vertices        coarsen.py:47-107
  contract              coarsen.py:110-138
  build_hierarchy       coarsen.py:141-161
  select_destinations   refine.py:78-105
  afterburner           refine.py:127-156
  jetlp_pass            refine.py:159-183
  weak_rebalance_pass   rebalance.py:139-183
  strong_rebalance_pass rebalance.py:186-240
  jet_refine            refine.py:190-294
  initial_partition     initpart.py:70-94 (host C++ inside libjet)
The reference threads a ConnectivityTable through these calls; on the GPU the
conn(v, p) rows are rebuilt on chip in every pass, so the table object holds
the lock bits and answers content queries (`get_many`, `row_items`,
`nonzero_triples`) and `apply` with GPU kernels (csrc/conn.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import RefinerConfig, ratio_parts, to_c
from .graph import Graph, PartitionState, _device_graph, graph_n, total_weight
from .moves import MoveList


class ConnectivityTable:
    """The reference's ConnectivityTable (conn.py:29-262) over the GPU.

    conn(v, p) is never stored on the device: every refinement pass rebuilds
    the rows on chip from the CSR, and this object does the same on demand
    (`jet_conn_triples`). What the reference exposes of its table -- the
    nonzero (row, part, weight) contents, the locks and the exact-delta
    `apply` -- behaves identically; the open-addressing layout is not
    modelled (only the nonzero contents are observable).
    `row_capacity` is the Eq. 9 bound min(deg v, k)."""

    def __init__(self, graph, state):
        self.graph = graph
        self.state = state
        self.k = state.k
        self.locks = np.zeros(graph_n(graph), dtype=bool)

    # -- sizing (a virtual layout: the rows live on chip, per pass) ---------
    @property
    def allocated_slots(self) -> int:
        deg = np.diff(np.asarray(self.graph.row_offsets))
        return 2 * int(np.minimum(deg, self.k).sum())

    @property
    def slack_slots(self) -> int:
        return 0

    def row_capacity(self, v: int) -> int:
        lo, hi = self.graph.row_offsets[v], self.graph.row_offsets[v + 1]
        return int(min(hi - lo, self.k))

    # -- contents ------------------------------------------------------------
    def _triples(self, rows=None):
        dg = _device_graph(self.graph)
        parts = _lib.as_i64(self.state.parts)
        r = None if rows is None else _lib.as_i64(rows)
        nr = graph_n(self.graph) if r is None else len(r)
        L = _lib.lib()
        cnt = C.c_int64()
        _lib.check(L.jet_conn_triples(dg.ctx.handle, dg.handle, _lib.ptr(parts), int(self.k),
                                      _lib.ptr(r), nr, None, None, None, 0, C.byref(cnt)))
        m = cnt.value
        out = [np.empty(m, np.int64) for _ in range(3)]
        _lib.check(L.jet_conn_triples(dg.ctx.handle, dg.handle, _lib.ptr(parts), int(self.k),
                                      _lib.ptr(r), nr, *[_lib.ptr(a) for a in out], m,
                                      C.byref(cnt)))
        return out

    def get_many(self, rows, parts) -> np.ndarray:
        """conn(rows[i], parts[i]) for every i (conn.py:70-93)."""
        rows = np.asarray(rows, dtype=np.int64)
        parts = np.asarray(parts, dtype=np.int64)
        if len(rows) == 0:
            return np.zeros(0, dtype=np.int64)
        uniq = np.unique(rows)
        tr, tp, tw = self._triples(uniq)
        key = tr * self.k + tp
        want = rows * self.k + parts
        if len(key) == 0:
            return np.zeros(len(rows), dtype=np.int64)
        pos = np.minimum(np.searchsorted(key, want), len(key) - 1)
        return np.where(key[pos] == want, tw[pos], 0).astype(np.int64)

    def conn(self, v: int, p: int) -> int:
        return int(self.get_many(np.array([v]), np.array([p]))[0])

    def row_items(self, v: int) -> dict:
        _, tp, tw = self._triples(np.array([v]))
        return {int(p): int(w) for p, w in zip(tp, tw)}

    def nonzero_triples(self):
        """All nonzero (row, part, weight) entries in canonical order."""
        return tuple(self._triples())

    def same_contents(self, other) -> bool:
        return all(np.array_equal(x, y)
                   for x, y in zip(self.nonzero_triples(), other.nonzero_triples()))

    # -- locks ---------------------------------------------------------------
    def reset_locks(self) -> None:
        self.locks[:] = False

    def set_locks(self, vertices) -> None:
        self.locks[vertices] = True

    # -- updates -------------------------------------------------------------
    def apply(self, moves) -> None:
        """Apply a move list to the bound state by exact deltas on the GPU
        (conn.py:215-254): part weights, parts and the cut. A move to the
        current part raises AssertionError, as in the reference."""
        if len(moves) == 0:
            return
        st = self.state
        dg = _device_graph(self.graph)
        parts = np.ascontiguousarray(st.parts, dtype=np.int64)
        pw = np.ascontiguousarray(st.part_weights, dtype=np.int64)
        cut = C.c_int64(int(st.cutsize))
        mv, md = _lib.as_i64(moves.vertices), _lib.as_i64(moves.dests)
        _lib.check(_lib.lib().jet_apply_moves(
            dg.ctx.handle, dg.handle, _lib.ptr(parts), int(st.k), _lib.ptr(pw), C.byref(cut),
            _lib.ptr(mv), _lib.ptr(md), len(mv)))
        st.parts[:] = parts
        st.part_weights[:] = pw
        st.cutsize = int(cut.value)

    def rebuild_row(self, v: int) -> None:
        """conn.py:143-163 recomputes a row from the graph and the state; here
        every query already rebuilds the rows it reads from the CSR."""
        if not 0 <= int(v) < graph_n(self.graph):
            raise IndexError("row out of range")

    def check(self) -> None:
        """The GPU rebuilds rows from the CSR and the bound state, so the
        contents are in sync by construction; verify the state's cached part
        weights and cut against a recount (conn.py:256-262)."""
        fresh = PartitionState.from_parts(self.graph, self.state.parts, self.k)
        if fresh.cutsize != self.state.cutsize or \
                not np.array_equal(fresh.part_weights, self.state.part_weights):
            raise ValueError("connectivity table out of sync")


LockTable = ConnectivityTable  # round-1 name


def build_conn(graph, state) -> ConnectivityTable:
    """Construct the connectivity table for a partition (conn.py:265-267)."""
    return ConnectivityTable(graph, state)


def update_conn(table: ConnectivityTable, moves) -> None:
    """Apply a move list to the table and its bound state (conn.py:270-272)."""
    table.apply(moves)


def _ctx():
    return _lib.Context.default()


def match_vertices(graph, seed: int = 0) -> np.ndarray:
    del seed  # the reference ignores it too (coarsen.py:58)
    dg = _device_graph(graph)
    out = np.empty(graph_n(graph), dtype=np.int64)
    _lib.check(_lib.lib().jet_match(dg.ctx.handle, dg.handle, _lib.ptr(out)))
    return out


def _graph_from_device(dg) -> Graph:
    offs, adj, ew, vw = dg.download()
    return Graph(offs, adj, ew, vw)


def contract(graph, matching):
    dg = _device_graph(graph)
    partner = _lib.as_i64(matching)
    vmap = np.empty(graph_n(graph), dtype=np.int64)
    h = C.c_void_p()
    _lib.check(_lib.lib().jet_contract(dg.ctx.handle, dg.handle, _lib.ptr(partner),
                                       C.byref(h), _lib.ptr(vmap)))
    cg = _lib.DeviceGraph(dg.ctx, h)
    try:
        coarse = _graph_from_device(cg)
    finally:
        cg.free()
    return coarse, vmap


@dataclass
class Hierarchy:
    """Coarse graphs plus fine-to-coarse maps (coarsen.py:19-44)."""

    levels: list = field(default_factory=list)
    maps: list = field(default_factory=list)

    def __len__(self):
        return len(self.levels)

    def validate(self) -> None:
        """The reference's structural checks (coarsen.py:33-44)."""
        total = total_weight(self.levels[0])
        for i, vmap in enumerate(self.maps):
            fine, coarse = self.levels[i], self.levels[i + 1]
            if len(vmap) != graph_n(fine):
                raise ValueError("map length mismatch")
            if graph_n(coarse) >= graph_n(fine):
                raise ValueError("coarse level must be strictly smaller")
            if len(np.unique(vmap)) != graph_n(coarse):
                raise ValueError("map must be surjective onto coarse vertices")
            if total_weight(coarse) != total:
                raise ValueError("vertex weight not conserved")


def build_hierarchy(graph, target: int, seed: int = 0) -> Hierarchy:
    del seed
    dg = _device_graph(graph)
    h = C.c_void_p()
    L = _lib.lib()
    _lib.check(L.jet_hierarchy_build(dg.ctx.handle, dg.handle, int(target), C.byref(h)))
    try:
        out = Hierarchy([graph], [])
        nl = L.jet_hierarchy_levels(h)
        for i in range(nl - 1):
            fine_n = graph_n(out.levels[-1])
            vmap = np.empty(fine_n, dtype=np.int64)
            _lib.check(L.jet_hierarchy_map(dg.ctx.handle, h, i, _lib.ptr(vmap)))
            view = _lib.DeviceGraph(dg.ctx, L.jet_hierarchy_level(h, i + 1), owner=h)
            out.levels.append(_graph_from_device(view))
            out.maps.append(vmap)
    finally:
        L.jet_hierarchy_free(h)
    return out


def select_destinations(graph, state, table=None):
    dg = _device_graph(graph)
    n = graph_n(graph)
    parts = _lib.as_i64(state.parts)
    dest = np.empty(n, np.int64)
    gain = np.empty(n, np.int64)
    bnd = np.empty(n, np.uint8)
    cs = np.empty(n, np.int64)
    _lib.check(_lib.lib().jet_select_destinations(
        dg.ctx.handle, dg.handle, _lib.ptr(parts), int(state.k), _lib.ptr(dest), _lib.ptr(gain),
        _lib.ptr(bnd), _lib.ptr(cs)))
    return dest, gain, bnd.astype(bool), cs


def afterburner(graph, cand, parts, dests, gain) -> np.ndarray:
    dg = _device_graph(graph)
    cand = _lib.as_i64(cand)
    parts, dests, gain = _lib.as_i64(parts), _lib.as_i64(dests), _lib.as_i64(gain)
    out = np.empty(len(cand), np.int64)
    _lib.check(_lib.lib().jet_afterburner(
        dg.ctx.handle, dg.handle, _lib.ptr(cand), len(cand), _lib.ptr(parts),
        _lib.ptr(dests), _lib.ptr(gain), _lib.ptr(out)))
    return out


def jetlp_pass(graph, state, table, c: float, use_afterburner: bool = True,
               use_locks: bool = True) -> MoveList:
    dg = _device_graph(graph)
    n = graph_n(graph)
    num, den, use_float = ratio_parts(c)
    locks = np.ascontiguousarray(table.locks, dtype=np.uint8) if table is not None else \
        np.zeros(n, np.uint8)
    mv = np.empty(n, np.int64)
    md = np.empty(n, np.int64)
    mg = np.empty(n, np.int64)
    cnt = C.c_int64()
    parts = _lib.as_i64(state.parts)
    _lib.check(_lib.lib().jet_jetlp_pass(
        dg.ctx.handle, dg.handle, _lib.ptr(parts), int(state.k),
        _lib.ptr(locks), num, den, float(c), use_float, int(bool(use_afterburner)),
        int(bool(use_locks)), _lib.ptr(mv), _lib.ptr(md), _lib.ptr(mg), C.byref(cnt)))
    m = cnt.value
    if use_locks and table is not None:
        table.locks[:] = locks.astype(bool)
    return MoveList(mv[:m].copy(), md[:m].copy(), mg[:m].copy())


def _rng_to_c(rng) -> _lib.Pcg64State:
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("the GPU path replays numpy's PCG64 stream only")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return _lib.Pcg64State(s >> 64, s & m, inc >> 64, inc & m, st["has_uint32"], st["uinteger"])


def _rng_from_c(rng, c: _lib.Pcg64State) -> None:
    st = rng.bit_generator.state
    st["state"]["state"] = (c.state_hi << 64) | c.state_lo
    st["state"]["inc"] = (c.inc_hi << 64) | c.inc_lo
    st["has_uint32"] = c.has_uint32
    st["uinteger"] = c.uinteger
    rng.bit_generator.state = st


def _rebalance(graph, state, limit, sigma, rng, sub_buckets, strong) -> MoveList:
    dg = _device_graph(graph)
    n = graph_n(graph)
    cstate = _rng_to_c(rng)
    mv = np.empty(n, np.int64)
    md = np.empty(n, np.int64)
    mg = np.empty(n, np.float64)
    cnt = C.c_int64()
    parts, pw = _lib.as_i64(state.parts), _lib.as_i64(state.part_weights)
    _lib.check(_lib.lib().jet_rebalance_pass(
        dg.ctx.handle, dg.handle, _lib.ptr(parts), int(state.k),
        _lib.ptr(pw), int(limit), int(sigma), int(sub_buckets),
        int(strong), C.byref(cstate), _lib.ptr(mv), _lib.ptr(md), _lib.ptr(mg), C.byref(cnt)))
    _rng_from_c(rng, cstate)
    m = cnt.value
    gains = mg[:m].copy() if strong else mg[:m].astype(np.int64)
    return MoveList(mv[:m].copy(), md[:m].copy(), gains)


def weak_rebalance_pass(graph, state, table, limit, sigma, rng, sub_buckets: int = 32) -> MoveList:
    return _rebalance(graph, state, limit, sigma, rng, sub_buckets, False)


def strong_rebalance_pass(graph, state, table, limit, sigma, rng, sub_buckets: int = 32) -> MoveList:
    return _rebalance(graph, state, limit, sigma, rng, sub_buckets, True)


def jet_refine(graph, state, config: RefinerConfig, finest: bool = True, seed_path=()):
    if len(seed_path) > 1:
        raise ValueError("seed_path holds at most the level index")
    dg = _device_graph(graph)
    n = graph_n(graph)
    cfg = to_c(config, total_weight(graph))
    parts = np.empty(n, np.int64)
    pw = np.empty(config.k, np.int64)
    cut = C.c_int64()
    st = _lib.LevelStats()
    level = int(seed_path[0]) if seed_path else -1
    parts_in = _lib.as_i64(state.parts)
    cap = 4096
    tr = np.empty(4 * cap, np.int64)
    ntr = C.c_int64()
    _lib.check(_lib.lib().jet_refine_trace(
        dg.ctx.handle, dg.handle, _lib.ptr(parts_in), C.byref(cfg),
        int(bool(finest)), level, _lib.ptr(parts), _lib.ptr(pw), C.byref(cut), C.byref(st),
        _lib.ptr(tr), cap, C.byref(ntr)))
    out = PartitionState(parts, config.k, pw, int(cut.value))
    kinds = {1: "lp", 2: "weak", 3: "strong"}
    trace = [(kinds[int(a)], int(b), int(c_), int(d)) for a, b, c_, d in
             tr[:4 * min(ntr.value, cap)].reshape(-1, 4)]
    stats = {
        "iterations": st.iterations, "lp_passes": st.lp_passes,
        "weak_passes": st.weak_passes, "strong_passes": st.strong_passes,
        "moves": st.moves, "rebalance_stuck": bool(st.rebalance_stuck),
        "trace": trace, "balanced": bool(st.balanced),
        "best_cut": int(cut.value) if st.balanced else None,
    }
    return out, stats


def initial_partition(graph, k: int, imbalance: float, seed: int = 0,
                      restarts: int = 8) -> PartitionState:
    from .graph import part_weight_limit
    if k < 1:
        raise ValueError("k must be >= 1")
    n = graph_n(graph)
    if k > n:
        raise ValueError(f"k={k} exceeds vertex count {n}")
    limit = part_weight_limit(total_weight(graph), k, imbalance)
    out = np.empty(n, np.int64)
    arrs = [_lib.as_i64(a) for a in (graph.row_offsets, graph.adjacency, graph.edge_weights,
                                     graph.vertex_weights)]
    _lib.check(_lib.lib().jet_initial_partition(
        n, *[_lib.ptr(a) for a in arrs], k, limit, seed, restarts, _lib.ptr(out)))
    return PartitionState.from_parts(graph, out, k)
