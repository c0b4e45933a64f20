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
conn(v, p) rows are rebuilt on chip in every pass, so the table reduces to
the lock bits (`LockTable`).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import RefinerConfig, ratio_parts, to_c
from .graph import Graph, PartitionState, _device_graph, graph_n, total_weight
from .moves import MoveList


class LockTable:
    """Lock bits of the reference's ConnectivityTable (conn.py:125-129)."""

    def __init__(self, graph, state=None):
        self.graph = graph
        self.state = state
        self.k = state.k if state is not None else None
        self.locks = np.zeros(graph_n(graph), dtype=bool)

    def reset_locks(self) -> None:
        self.locks[:] = False

    def set_locks(self, vertices) -> None:
        self.locks[vertices] = True

    def apply(self, moves) -> None:
        """Apply a move list to the bound state (parts, weights, cut)."""
        if len(moves) == 0:
            return
        st = self.state
        assert np.all(st.parts[moves.vertices] != moves.dests), "move to current part"
        parts = st.parts.copy()
        parts[moves.vertices] = moves.dests
        fresh = PartitionState.from_parts(self.graph, parts, st.k)
        st.parts[:] = fresh.parts
        st.part_weights[:] = fresh.part_weights
        st.cutsize = fresh.cutsize


def build_conn(graph, state) -> LockTable:
    return LockTable(graph, state)


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
    levels: list = field(default_factory=list)
    maps: list = field(default_factory=list)

    def __len__(self):
        return len(self.levels)


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
    _lib.check(_lib.lib().jet_refine(
        dg.ctx.handle, dg.handle, _lib.ptr(parts_in), C.byref(cfg),
        int(bool(finest)), level, _lib.ptr(parts), _lib.ptr(pw), C.byref(cut), C.byref(st)))
    out = PartitionState(parts, config.k, pw, int(cut.value))
    stats = {
        "iterations": st.iterations, "lp_passes": st.lp_passes,
        "weak_passes": st.weak_passes, "strong_passes": st.strong_passes,
        "moves": st.moves, "rebalance_stuck": bool(st.rebalance_stuck),
        "trace": [], "balanced": bool(st.balanced),
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
