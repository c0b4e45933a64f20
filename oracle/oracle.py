"""TEST INFRASTRUCTURE ONLY — ctypes front end of the C oracle
(oracle/jet_oracle.c), a sequential CPU restatement of the reference
partitioner. Used by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm as the checker; never by the product package.

Pinned: tests/test_oracle.py compares it with every golden vector produced
by running the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from fractions import Fraction
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_LIB = None
P = C.c_void_p
i64 = C.c_int64


def lib():
    global _LIB
    if _LIB is None:
        so = HERE / "liboracle.so"
        if not so.exists():
            subprocess.run(["make", "-C", str(HERE)], check=True)
        L = C.CDLL(str(so))
        sig = {
            "oracle_match": (None, [i64, P, P, P, P]),
            "oracle_contract": (None, [i64, P, P, P, P, P, P, P, P, P, P, P]),
            "oracle_select_destinations": (None, [i64, P, P, P, P, i64, P, P, P, P]),
            "oracle_afterburner": (None, [i64, P, P, P, P, i64, P, P, P, P]),
            "oracle_jetlp_pass": (i64, [i64, P, P, P, P, i64, P, i64, i64, C.c_double, C.c_int,
                                        C.c_int, C.c_int, P, P, P]),
            "oracle_rebalance_pass": (i64, [i64, P, P, P, P, P, i64, P, i64, i64, i64, C.c_int,
                                            P, P, P, P]),
            "oracle_refine": (None, [i64, P, P, P, P, P, P, P, C.c_int, i64, P]),
            "oracle_initial_partition": (None, [i64, P, P, P, P, i64, i64, i64, i64, P]),
            "oracle_partition": (i64, [i64, P, P, P, P, P, P, P, P, P, i64]),
            "oracle_cutsize": (i64, [i64, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _a(x):
    return np.ascontiguousarray(np.asarray(x), dtype=np.int64)


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _g(graph):
    return [_a(graph.row_offsets), _a(graph.adjacency), _a(graph.edge_weights),
            _a(graph.vertex_weights)]


def limit_of(W, k, imbalance):
    """graph.py:203-212"""
    return int((Fraction(1) + Fraction(str(imbalance))) * W // k)


def sigma_of(W, k, imbalance, limit, deadzone=0.1):
    """rebalance.py:26-32"""
    return limit - max(1, int(deadzone * imbalance * W / k))


def _ratio(c):
    r = Fraction(str(c))
    return (r.numerator, r.denominator, 0) if r.denominator <= 10**6 else (1, 1, 1)


def config(graph, k, imbalance=0.03, seed=0, c_finest=0.25, c_other=0.75, phi=0.999,
           no_improve_limit=12, sub_buckets=32, deadzone=0.1, coarse_target=200, restarts=8,
           afterburner=True, locking=True):
    W = int(np.asarray(graph.vertex_weights).sum())
    limit = limit_of(W, k, imbalance)
    sigma = sigma_of(W, k, imbalance, limit, deadzone)
    fn, fd, ff = _ratio(c_finest)
    on, od, of = _ratio(c_other)
    icfg = np.array([k, limit, sigma, fn, fd, on, od, ff, of, no_improve_limit, sub_buckets, seed,
                     coarse_target, restarts, int(afterburner), int(locking)], dtype=np.int64)
    dcfg = np.array([c_finest, c_other, phi], dtype=np.float64)
    return icfg, dcfg


def match(graph):
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    out = np.empty(n, np.int64)
    lib().oracle_match(n, _p(off), _p(adj), _p(ew), _p(out))
    return out


def contract(graph, partner):
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    partner = _a(partner)
    vmap = np.empty(n, np.int64)
    cn = i64()
    c_off = np.empty(n + 1, np.int64)
    c_adj = np.empty(max(len(adj), 1), np.int64)
    c_ew = np.empty(max(len(adj), 1), np.int64)
    c_vw = np.empty(n, np.int64)
    lib().oracle_contract(n, _p(off), _p(adj), _p(ew), _p(vw), _p(partner), _p(vmap), C.byref(cn),
                          _p(c_off), _p(c_adj), _p(c_ew), _p(c_vw))
    m = cn.value
    e = c_off[m]
    return (c_off[:m + 1].copy(), c_adj[:e].copy(), c_ew[:e].copy(), c_vw[:m].copy()), vmap


def select_destinations(graph, parts, k):
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    parts = _a(parts)
    dest, gain, cs = (np.empty(n, np.int64) for _ in range(3))
    bnd = np.empty(n, np.uint8)
    lib().oracle_select_destinations(n, _p(off), _p(adj), _p(ew), _p(parts), k, _p(dest),
                                     _p(gain), _p(bnd), _p(cs))
    return dest, gain, bnd.astype(bool), cs


def afterburner(graph, cand, parts, dests, gain):
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    cand, parts, dests, gain = _a(cand), _a(parts), _a(dests), _a(gain)
    out = np.empty(len(cand), np.int64)
    lib().oracle_afterburner(n, _p(off), _p(adj), _p(ew), _p(cand), len(cand), _p(parts),
                             _p(dests), _p(gain), _p(out))
    return out


def jetlp_pass(graph, parts, k, locks, c, use_afterburner=True, use_locks=True):
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    parts = _a(parts)
    lk = np.ascontiguousarray(locks, dtype=np.uint8)
    num, den, fl = _ratio(c)
    mv, md, mg = (np.empty(n, np.int64) for _ in range(3))
    m = lib().oracle_jetlp_pass(n, _p(off), _p(adj), _p(ew), _p(parts), k, _p(lk), num, den,
                                float(c), fl, int(use_afterburner), int(use_locks), _p(mv), _p(md),
                                _p(mg))
    return mv[:m].copy(), md[:m].copy(), mg[:m].copy(), lk.astype(bool)


def rebalance_pass(graph, parts, k, pw, limit, sigma, rng, sub_buckets=32, strong=False):
    """rng: numpy Generator (PCG64), advanced in place like numpy would."""
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    parts, pw = _a(parts), _a(pw)
    st = rng.bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    M = (1 << 64) - 1
    rs = np.array([s >> 64, s & M, inc >> 64, inc & M, st["has_uint32"], st["uinteger"]],
                  dtype=np.uint64)
    mv, md = np.empty(n, np.int64), np.empty(n, np.int64)
    mg = np.empty(n, np.float64)
    m = lib().oracle_rebalance_pass(n, _p(off), _p(adj), _p(ew), _p(vw), _p(parts), k, _p(pw),
                                    limit, sigma, sub_buckets, int(strong), _p(rs), _p(mv), _p(md),
                                    _p(mg))
    if m < 0:
        raise RuntimeError("RebalanceInfeasibleError")
    st["state"]["state"] = (int(rs[0]) << 64) | int(rs[1])
    st["has_uint32"] = int(rs[4])
    st["uinteger"] = int(rs[5])
    rng.bit_generator.state = st
    return mv[:m].copy(), md[:m].copy(), mg[:m].copy()


def refine(graph, parts, k, finest=True, level=0, **kw):
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    icfg, dcfg = config(graph, k, **kw)
    p = _a(parts).copy()
    stats = np.zeros(8, np.int64)
    lib().oracle_refine(n, _p(off), _p(adj), _p(ew), _p(vw), _p(p), _p(icfg), _p(dcfg),
                        int(finest), level, _p(stats))
    return p, {"iterations": int(stats[0]), "lp_passes": int(stats[1]),
               "weak_passes": int(stats[2]), "strong_passes": int(stats[3]),
               "cut": int(stats[4]), "balanced": bool(stats[5]), "stuck": bool(stats[6])}


def initial_partition(graph, k, imbalance, seed=0, restarts=8):
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    W = int(vw.sum())
    out = np.empty(n, np.int64)
    lib().oracle_initial_partition(n, _p(off), _p(adj), _p(ew), _p(vw), k,
                                   limit_of(W, k, imbalance), seed, restarts, _p(out))
    return out


def partition(graph, k, max_levels=-1, **kw):
    """Full multilevel partition. max_levels >= 0 refines only that many
    levels (top first) — the bounded CPU-baseline sample."""
    off, adj, ew, vw = _g(graph)
    n = len(off) - 1
    icfg, dcfg = config(graph, k, **kw)
    parts = np.empty(n, np.int64)
    iters = np.zeros(64, np.int64)
    nl = i64()
    cut = lib().oracle_partition(n, _p(off), _p(adj), _p(ew), _p(vw), _p(icfg), _p(dcfg),
                                 _p(parts), _p(iters), C.byref(nl), max_levels)
    L = nl.value
    done = L if max_levels < 0 else min(L, max_levels)
    return {"parts": parts, "cut": int(cut), "n_levels": L,
            "iterations": iters[:done].tolist()}


def cutsize(graph, parts):
    off, adj, ew, vw = _g(graph)
    parts = _a(parts)
    return int(lib().oracle_cutsize(len(off) - 1, _p(off), _p(adj), _p(ew), _p(parts)))
