"""End-to-end multilevel partitioning (mirror of jetpart/driver.py:24-160).

`partition(graph, config)` is the drop-in entry point: one C-ABI call runs
coarsening, initial partitioning, projection and Jet refinement on the GPU
(initial partitioning of the <= max(200, 2k)-vertex coarsest level runs on
the host inside libjet, as in the reference). Checks and the metrics
dictionary follow the reference exactly.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import RefinerConfig, to_c
from .errors import BalanceInfeasibleError
from .graph import PartitionState, graph_n, part_weight_limit, total_weight


@dataclass
class PartitionResult:
    state: PartitionState
    metrics: dict = field(default_factory=dict)


def project(coarse_state: PartitionState, vmap, fine_graph) -> PartitionState:
    """Pull a coarse partition down one level (driver.py:32-45)."""
    vmap = _lib.as_i64(vmap)
    n = graph_n(fine_graph)
    if len(vmap) != n:
        raise ValueError("map length must equal fine vertex count")
    cparts = _lib.as_i64(coarse_state.parts)
    out = np.empty(n, np.int64)
    ctx = _lib.Context.default()
    _lib.check(_lib.lib().jet_project(ctx.handle, len(cparts), _lib.ptr(cparts), n,
                                      _lib.ptr(vmap), _lib.ptr(out)))
    return PartitionState.from_parts(fine_graph, out, coarse_state.k)


def _prepare(graph, config: RefinerConfig):
    n = graph_n(graph)
    if config.k < 1:
        raise ValueError("k must be >= 1")
    if config.k > n:
        raise ValueError(f"k={config.k} exceeds vertex count {n}")
    W = total_weight(graph)
    limit = part_weight_limit(W, config.k, config.imbalance)
    heaviest = int(np.asarray(graph.vertex_weights).max())
    if heaviest > limit:
        raise BalanceInfeasibleError(
            f"vertex weight {heaviest} exceeds the part weight limit {limit}")
    if config.k * limit < W:
        raise BalanceInfeasibleError(
            f"k * limit = {config.k * limit} cannot hold the total vertex weight {W}")
    return n, W, limit


def _arrays(graph):
    return _lib.csr_arrays(graph)


def partition(graph, config: RefinerConfig, ctx: _lib.Context | None = None) -> PartitionResult:
    """Partition a graph into config.k balanced parts, minimising the cut."""
    n, W, limit = _prepare(graph, config)
    (offs, adj, ew, vw), codes = _arrays(graph)
    ctx = ctx or _lib.Context.default()
    t0 = time.perf_counter()
    cfg = to_c(config, W)
    parts = np.empty(n, np.int64)
    pw = np.empty(config.k, np.int64)
    st = _lib.RunStats()
    _lib.check(_lib.lib().jet_partition(
        ctx.handle, n, _lib.ptr(offs), _lib.ptr(adj), codes[0], _lib.ptr(ew), codes[1],
        _lib.ptr(vw), codes[2], C.byref(cfg), _lib.ptr(parts), _lib.ptr(pw), C.byref(st)))
    total = time.perf_counter() - t0
    state = PartitionState(parts, config.k, pw, int(st.cutsize))
    return PartitionResult(state, build_metrics(graph, config, state, st, total, W, limit))


def build_metrics(graph, config, state, st, total, W, limit) -> dict:
    """The reference's metrics dict (driver.py:106-120, 129-160) + GPU extras."""
    levels = []
    if config.k > 1:
        for i in range(st.n_levels):
            L = st.levels[i]
            levels.append({
                "level": L.level, "n": L.n, "m": L.m, "cut_in": L.cut_in,
                "cut_out": L.cut_out, "balanced_in": bool(L.balanced_in),
                "balanced": bool(L.balanced), "iterations": L.iterations,
                "lp_passes": L.lp_passes, "weak_passes": L.weak_passes,
                "strong_passes": L.strong_passes, "rebalance_stuck": bool(L.rebalance_stuck),
                "seconds": L.seconds,
            })
        times = {"coarsen": st.t_coarsen, "initial": st.t_initial,
                 "uncoarsen": st.t_uncoarsen, "total": total}
    else:
        times = {"total": total}
    times["device_pipeline"] = st.t_total
    times["upload"] = st.t_upload
    times["download"] = st.t_download
    return {
        "n": graph_n(graph),
        "m": len(graph.adjacency) // 2,
        "k": config.k,
        "seed": config.seed,
        "cutsize": state.cutsize,
        "imbalance": float(state.part_weights.max()) * state.k / W,
        "balanced": bool(np.all(state.part_weights <= limit)),
        "part_weight_limit": limit,
        "levels": levels,
        "n_levels": st.n_levels if config.k > 1 else 1,
        "times": times,
        "kernel_launches": int(st.kernel_launches),
        "config": {
            "k": config.k, "imbalance": config.imbalance, "c_finest": config.c_finest,
            "c_other": config.c_other, "phi": config.phi,
            "no_improve_limit": config.no_improve_limit, "sub_buckets": config.sub_buckets,
            "deadzone_fraction": config.deadzone_fraction, "seed": config.seed,
            "deterministic": config.deterministic, "coarse_target": config.coarse_target,
            "restarts": config.restarts, "afterburner": config.afterburner,
            "locking": config.locking,
            "throughput_patience": getattr(config, "throughput_patience", 0),
            "patience_from_level": getattr(config, "patience_from_level", 0),
            "patience_min_k": getattr(config, "patience_min_k", 0),
        },
    }


class _DeviceGraphInfo:
    """What _prepare reads, from a device-resident graph (unit vertex weights
    are recognised from W == n without a download)."""

    def __init__(self, dgraph):
        n, _, W = dgraph.info()
        self.row_offsets = np.empty(n + 1, np.int8)
        self.total_vertex_weight = W
        self.vertex_weights = np.ones(1, np.int64) if W == n else dgraph.download()[3]


def partition_resident(dgraph: _lib.DeviceGraph, graph, config: RefinerConfig,
                       want_parts: bool = True):
    """Partition a graph already resident in HBM (device-timed benchmark leg).

    `graph` supplies the host-side checks (vertex weights); `dgraph` is its
    uploaded copy. `graph` may be None for a device-generated graph: the
    checks then read the device copy. Returns (parts or None, part_weights,
    RunStats)."""
    if graph is None:
        graph = _DeviceGraphInfo(dgraph)
    n, W, limit = _prepare(graph, config)
    cfg = to_c(config, W)
    parts = np.empty(n, np.int64) if want_parts else None
    pw = np.empty(config.k, np.int64)
    st = _lib.RunStats()
    _lib.check(_lib.lib().jet_partition_graph(
        dgraph.ctx.handle, dgraph.handle, C.byref(cfg),
        _lib.ptr(parts) if want_parts else None, _lib.ptr(pw), C.byref(st)))
    return parts, pw, st
