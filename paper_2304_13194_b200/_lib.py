"""ctypes binding of libjet.so (the C-ABI declared in include/jet.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2304_13194_b200/csrc``). There is no fallback: if the library
or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (
    BalanceInfeasibleError,
    JetpartError,
    RebalanceInfeasibleError,
)

LIB_PATH = Path(__file__).resolve().parent / "libjet.so"
if os.environ.get("JET_LIB"):  # alternative build of the same library (experiments)
    LIB_PATH = Path(os.environ["JET_LIB"]).resolve()

JET_OK, JET_EINVAL, JET_EBALANCE, JET_ECUDA, JET_ENOMEM, JET_EREBALANCE = 0, 1, 2, 3, 4, 5
JET_EINTERNAL, JET_EUNSUPPORTED, JET_EASSERT = 6, 7, 8
JET_I32, JET_I64 = 4, 8
MAX_LEVELS = 64

i64 = C.c_int64
i32 = C.c_int32
P = C.c_void_p


class Pcg64State(C.Structure):
    _fields_ = [
        ("state_hi", C.c_uint64), ("state_lo", C.c_uint64),
        ("inc_hi", C.c_uint64), ("inc_lo", C.c_uint64),
        ("has_uint32", i32), ("uinteger", C.c_uint32),
    ]


class JetConfig(C.Structure):
    _fields_ = [
        ("k", i32), ("imbalance", C.c_double), ("limit", i64), ("sigma", i64),
        ("c_finest_num", i64), ("c_finest_den", i64),
        ("c_other_num", i64), ("c_other_den", i64),
        ("c_finest", C.c_double), ("c_other", C.c_double),
        ("c_finest_float", i32), ("c_other_float", i32),
        ("phi", C.c_double), ("no_improve_limit", i32), ("sub_buckets", i32),
        ("seed", C.c_uint64), ("coarse_target", i32), ("restarts", i32),
        ("afterburner", i32), ("locking", i32), ("deterministic", i32),
        ("verbose", i32), ("throughput_patience", i32), ("patience_from_level", i32),
        ("patience_min_k", i32), ("initpart_device", i32),
    ]


class LevelStats(C.Structure):
    _fields_ = [
        ("level", i32), ("n", i64), ("m", i64), ("cut_in", i64), ("cut_out", i64),
        ("balanced_in", i32), ("balanced", i32), ("iterations", i32),
        ("lp_passes", i32), ("weak_passes", i32), ("strong_passes", i32),
        ("rebalance_stuck", i32), ("moves", i64), ("seconds", C.c_double),
        ("distributed", i32),
    ]


class RunStats(C.Structure):
    _fields_ = [
        ("t_upload", C.c_double), ("t_coarsen", C.c_double), ("t_initial", C.c_double),
        ("t_uncoarsen", C.c_double), ("t_total", C.c_double), ("t_download", C.c_double),
        ("n_levels", i32), ("cutsize", i64), ("balanced", i32),
        ("max_part_weight", i64), ("kernel_launches", i64),
        ("levels", LevelStats * MAX_LEVELS),
    ]


_SIGS = {
    "jet_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "jet_destroy": (None, [P]),
    "jet_last_error": (C.c_char_p, []),
    "jet_api_version": (C.c_int, []),
    "jet_profile_enable": (C.c_int, [P, C.c_int]),
    "jet_profile_reset": (C.c_int, [P]),
    "jet_profile_report": (C.c_int, [P, C.c_char_p, i64]),
    "jet_synchronize": (C.c_int, [P]),
    "jet_profile_filter": (C.c_int, [P, C.c_char_p]),
    "jet_timer_start": (C.c_int, [P]),
    "jet_timer_stop": (C.c_int, [P, C.POINTER(C.c_double)]),
    "jet_flush_l2": (C.c_int, [P]),
    "jet_graph_upload": (C.c_int, [P, i64, P, P, C.c_int, P, C.c_int, P, C.c_int, C.POINTER(P)]),
    "jet_graph_upload_block": (C.c_int, [P, i64, P, P, C.c_int, P, C.c_int, P, C.c_int, i64, i64,
                                         C.POINTER(P)]),
    "jet_graph_block": (C.c_int, [P, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
    "jet_graph_info": (C.c_int, [P, P, P, P]),
    "jet_graph_download": (C.c_int, [P, P, P, P, P, P]),
    "jet_graph_free": (None, [P]),
    "jet_generate_rmat": (C.c_int, [P, i32, i32, C.c_uint64, P, C.POINTER(P)]),
    "jet_comm_nccl_id": (C.c_int, [P]),
    "jet_comm_attach_nccl": (C.c_int, [P, P, i32, i32]),
    "jet_comm_local_group": (C.c_int, [i32, C.POINTER(P)]),
    "jet_comm_local_group_free": (None, [P]),
    "jet_comm_attach_local": (C.c_int, [P, P, i32]),
    "jet_comm_detach": (C.c_int, [P]),
    "jet_set_shard_min_vertices": (C.c_int, [P, i64]),
    "jet_generate_geometric": (C.c_int, [P, i64, C.c_double, C.c_uint64, C.POINTER(P)]),
    "jet_cutsize": (C.c_int, [P, P, P, P]),
    "jet_part_weights": (C.c_int, [P, P, P, i32, P]),
    "jet_conn_triples": (C.c_int, [P, P, P, i32, P, i64, P, P, P, i64, P]),
    "jet_apply_moves": (C.c_int, [P, P, P, i32, P, P, P, P, i64]),
    "jet_match": (C.c_int, [P, P, P]),
    "jet_contract": (C.c_int, [P, P, P, C.POINTER(P), P]),
    "jet_hierarchy_build": (C.c_int, [P, P, i64, C.POINTER(P)]),
    "jet_hierarchy_levels": (C.c_int, [P]),
    "jet_hierarchy_level": (P, [P, C.c_int]),
    "jet_hierarchy_map": (C.c_int, [P, P, C.c_int, P]),
    "jet_hierarchy_free": (None, [P]),
    "jet_project": (C.c_int, [P, i64, P, i64, P, P]),
    "jet_select_destinations": (C.c_int, [P, P, P, i32, P, P, P, P]),
    "jet_afterburner": (C.c_int, [P, P, P, i64, P, P, P, P]),
    "jet_jetlp_pass": (C.c_int, [P, P, P, i32, P, i64, i64, C.c_double, i32, i32, i32,
                                 P, P, P, P]),
    "jet_rebalance_pass": (C.c_int, [P, P, P, i32, P, i64, i64, i32, i32, P, P, P, P, P]),
    "jet_refine": (C.c_int, [P, P, P, P, i32, i32, P, P, P, P]),
    "jet_refine_trace": (C.c_int, [P, P, P, P, i32, i32, P, P, P, P, P, i64, P]),
    "jet_initial_partition": (C.c_int, [i64, P, P, P, P, i32, i64, C.c_uint64, i32, P]),
    "jet_partition": (C.c_int, [P, i64, P, P, C.c_int, P, C.c_int, P, C.c_int, P, P, P, P]),
    "jet_partition_graph": (C.c_int, [P, P, P, P, P, P]),
    "jet_rng_seed": (C.c_int, [P, i32, P]),
    "jet_rng_integers": (C.c_int, [P, i64, i64, P]),
}

_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load libjet.so once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise JetpartError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'`"
                )
            h = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int) -> None:
    if status == JET_OK:
        return
    msg = lib().jet_last_error().decode("utf-8", "replace")
    if status == JET_EINVAL:
        raise ValueError(msg)
    if status == JET_EBALANCE:
        raise BalanceInfeasibleError(msg)
    if status == JET_EREBALANCE:
        raise RebalanceInfeasibleError(msg)
    if status == JET_ENOMEM:
        raise MemoryError(msg)
    if status == JET_EASSERT:
        raise AssertionError(msg)
    raise JetpartError(f"[jet status {status}] {msg}")


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def as_i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int64)


class Context:
    """One CUDA device + stream; a process-wide default per device."""

    _defaults: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0):
        self.device = device
        h = P()
        check(lib().jet_create(device, C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().jet_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def default(cls) -> "Context":
        dev = int(os.environ.get("JET_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        with cls._lock:
            ctx = cls._defaults.get(dev)
            if ctx is None:
                ctx = cls(dev)
                cls._defaults[dev] = ctx
            return ctx

    # profiling ------------------------------------------------------------
    def profile(self, on: bool = True):
        check(lib().jet_profile_enable(self.handle, 1 if on else 0))

    def profile_reset(self):
        check(lib().jet_profile_reset(self.handle))

    def profile_report(self) -> dict:
        n = lib().jet_profile_report(self.handle, None, 0)
        if n < 0:
            check(-n)
        buf = C.create_string_buffer(n + 1)
        lib().jet_profile_report(self.handle, buf, n + 1)
        out = {}
        for line in buf.value.decode().splitlines():
            name, launches, ms, nbytes = line.split("\t")
            out[name] = {"launches": int(launches), "ms": float(ms), "bytes": float(nbytes)}
        return out

    def synchronize(self):
        check(lib().jet_synchronize(self.handle))

    def profile_only(self, name: str | None):
        check(lib().jet_profile_filter(self.handle, (name or "").encode()))

    def timer_start(self):
        check(lib().jet_timer_start(self.handle))

    def timer_stop(self) -> float:
        ms = C.c_double()
        check(lib().jet_timer_stop(self.handle, C.byref(ms)))
        return ms.value

    def flush_l2(self):
        check(lib().jet_flush_l2(self.handle))

    # 1D vertex sharding (include/jet.h) ------------------------------------
    def attach_local(self, group: "LocalGroup", rank: int):
        check(lib().jet_comm_attach_local(self.handle, group.handle, int(rank)))
        self._group = group  # keep the group alive while attached

    def attach_nccl(self, nccl_id: bytes, rank: int, size: int):
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        check(lib().jet_comm_attach_nccl(self.handle, buf, int(rank), int(size)))

    def detach(self):
        check(lib().jet_comm_detach(self.handle))
        self._group = None

    def set_shard_min_vertices(self, n: int):
        check(lib().jet_set_shard_min_vertices(self.handle, int(n)))


class LocalGroup:
    """`size` virtual ranks (one context + host thread each) in one process."""

    def __init__(self, size: int):
        h = P()
        check(lib().jet_comm_local_group(int(size), C.byref(h)))
        self.handle, self.size = h, int(size)

    def __del__(self):  # pragma: no cover
        try:
            if self.handle:
                lib().jet_comm_local_group_free(self.handle)
                self.handle = None
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().jet_comm_nccl_id(buf))
    return buf.raw


def csr_arrays(graph):
    """The four CSR arrays of a Graph-like object as C-contiguous int64 (int32
    arrays are passed through), with their dtype codes. The C ABI derives the
    entry count from row_offsets[n] and reads that many adjacency and weight
    entries, so the lengths are checked here, before any native call."""
    offs = as_i64(graph.row_offsets)
    if len(offs) < 1:
        raise ValueError("row_offsets must have n + 1 >= 1 entries")
    n = len(offs) - 1
    out, codes = [offs], []
    for a in (graph.adjacency, graph.edge_weights, graph.vertex_weights):
        a = np.asarray(a)
        if a.ndim != 1:
            raise ValueError("graph arrays must be one-dimensional")
        if a.dtype == np.int32 and a.flags.c_contiguous:
            out.append(a)
            codes.append(JET_I32)
        else:
            out.append(as_i64(a))
            codes.append(JET_I64)
    nnz = int(offs[-1])
    if len(out[1]) != nnz:
        raise ValueError(f"adjacency has {len(out[1])} entries but row_offsets[n] = {nnz}")
    if len(out[2]) != len(out[1]):
        raise ValueError("edge_weights must align with adjacency")
    if len(out[3]) != n:
        raise ValueError(f"vertex_weights has {len(out[3])} entries for n = {n}")
    return out, codes


class DeviceGraph:
    """A device-resident CSR level (owning unless created as a view)."""

    def __init__(self, ctx: Context, handle, owner=None):
        self.ctx = ctx
        self.handle = handle
        self._owner = owner  # keeps a hierarchy alive for level views

    @classmethod
    def upload(cls, graph, ctx: Context | None = None) -> "DeviceGraph":
        ctx = ctx or Context.default()
        (offs, *arrays), codes = csr_arrays(graph)
        n = len(offs) - 1
        h = P()
        check(lib().jet_graph_upload(
            ctx.handle, n, ptr(offs), ptr(arrays[0]), codes[0], ptr(arrays[1]), codes[1],
            ptr(arrays[2]), codes[2], C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def upload_block(cls, graph, lo: int, hi: int, ctx: Context | None = None) -> "DeviceGraph":
        """This rank's block [lo, hi) of a 1D-distributed graph: complete
        row offsets and vertex weights, only the block's adjacency/weights
        (include/jet.h jet_graph_upload_block). Attach the communicator first."""
        ctx = ctx or Context.default()
        (offs, *arrays), codes = csr_arrays(graph)
        n = len(offs) - 1
        e0, e1 = int(offs[lo]), int(offs[hi])
        adj = np.ascontiguousarray(arrays[0][e0:e1])
        ew = np.ascontiguousarray(arrays[1][e0:e1])
        h = P()
        check(lib().jet_graph_upload_block(
            ctx.handle, n, ptr(offs), ptr(adj), codes[0], ptr(ew), codes[1],
            ptr(arrays[2]), codes[2], int(lo), int(hi), C.byref(h)))
        return cls(ctx, h)

    def block(self):
        """(row_lo, row_hi, entries stored on this rank)."""
        lo, hi, e = i64(), i64(), i64()
        check(lib().jet_graph_block(self.handle, C.byref(lo), C.byref(hi), C.byref(e)))
        return lo.value, hi.value, e.value

    def info(self):
        n, nnz, w = i64(), i64(), i64()
        check(lib().jet_graph_info(self.handle, C.byref(n), C.byref(nnz), C.byref(w)))
        return n.value, nnz.value, w.value

    def download(self):
        n, nnz, _ = self.info()
        offs = np.empty(n + 1, np.int64)
        adj = np.empty(nnz, np.int64)
        ew = np.empty(nnz, np.int64)
        vw = np.empty(n, np.int64)
        check(lib().jet_graph_download(self.ctx.handle, self.handle, ptr(offs), ptr(adj),
                                       ptr(ew), ptr(vw)))
        return offs, adj, ew, vw

    def free(self):
        if self.handle and self._owner is None:
            lib().jet_graph_free(self.handle)
        self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass
