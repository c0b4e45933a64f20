"""1D vertex-sharded refinement through the real sharded code
path with a local group: `size` contexts in one process, one host thread
each, on one GPU (the NCCL transport needs one GPU per rank). Every rank
must return the unsharded partition bit for bit."""

import threading

import numpy as np
import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import _lib
from paper_2304_13194_b200 import generators as gen
from paper_2304_13194_b200.driver import partition_resident

pytestmark = pytest.mark.gpu


def _run_sharded(g, cfg, size, shard_min):
    group = _lib.LocalGroup(size)
    ctxs = [_lib.Context(0) for _ in range(size)]
    ctxs[0].profile(True)
    dgs = []
    for r, c in enumerate(ctxs):
        c.attach_local(group, r)
        c.set_shard_min_vertices(shard_min)
        dgs.append(_lib.DeviceGraph.upload(g, c))
    out, errs = [None] * size, []

    def work(r):
        try:
            out[r] = partition_resident(dgs[r], g, cfg, want_parts=True)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert not any(t.is_alive() for t in th), "a rank did not finish"
    rep = ctxs[0].profile_report()
    assert rep.get("shard_pack", {}).get("launches", 0) > 0, "sharded path not taken"
    assert rep.get("rb_evict_ids", {}).get("launches", 0) + rep.get("rb_collect", {}).get(
        "launches", 0) > 0, "no sharded rebalancing pass"
    for c in ctxs:
        c.detach()
    return out


@pytest.mark.parametrize("size", [2, 3])
def test_sharded_equals_unsharded(size):
    g = gen.grid27_graph(32)
    cfg = J.RefinerConfig(k=16, imbalance=0.03, seed=1, deterministic=True)
    ref_parts, ref_pw, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    res = _run_sharded(g, cfg, size, shard_min=2000)
    for parts, pw, st in res:
        assert st.cutsize == ref_st.cutsize
        assert np.array_equal(parts, ref_parts)
        assert np.array_equal(pw, ref_pw)


def test_sharded_throughput_mode():
    """Throughput mode is deterministic run to run, so sharding reproduces it too."""
    g = gen.grid27_graph(32)
    cfg = J.RefinerConfig(k=16, imbalance=0.03, seed=3, deterministic=False)
    ref_parts, _, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    for parts, pw, st in _run_sharded(g, cfg, 2, shard_min=2000):
        assert st.cutsize == ref_st.cutsize
        assert np.array_equal(parts, ref_parts)


def test_sharded_skewed_rmat():
    """Skewed degrees (hub rows, block-per-row tiers) through the sharded path."""
    g = gen.rmat_graph(13, 16, 2)
    cfg = J.RefinerConfig(k=32, imbalance=0.03, seed=0, deterministic=True)
    ref_parts, ref_pw, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    for parts, pw, st in _run_sharded(g, cfg, 2, shard_min=500):
        assert st.cutsize == ref_st.cutsize
        assert np.array_equal(parts, ref_parts)


def test_sharded_pipeline_goldens(golden):
    """The reference's own answers on the pipeline cases, sharded over 2."""
    from conftest import graph_of
    d = golden("pipeline")
    for i in range(min(6, int(d["count"][0]))):
        g = graph_of(d, f"p{i}_")
        k, seed, ab, lk = (int(x) for x in d[f"p{i}_cfg"])
        if not ab:
            continue
        cfg = J.RefinerConfig(k=k, imbalance=float(d[f"p{i}_imb"][0]), seed=seed,
                              afterburner=True, locking=bool(lk), deterministic=True)
        for parts, pw, st in _run_sharded(g, cfg, 2, shard_min=1):
            assert st.cutsize == int(d[f"p{i}_cut"][0]), i
            assert np.array_equal(parts, d[f"p{i}_parts"]), i


def test_nccl_transport_single_rank(monkeypatch):
    """The NCCL transport (libnccl opened at run time) with one rank and the
    sharded path forced: exercises id creation, communicator setup and the
    all-gathers on one GPU."""
    monkeypatch.setenv("JET_SHARD_SINGLE", "1")
    g = gen.grid27_graph(24)
    cfg = J.RefinerConfig(k=8, imbalance=0.03, seed=0, deterministic=True)
    ref_parts, _, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    ctx = _lib.Context(0)
    ctx.attach_nccl(_lib.nccl_unique_id(), 0, 1)
    ctx.set_shard_min_vertices(1000)
    ctx.profile(True)
    parts, _, st = partition_resident(_lib.DeviceGraph.upload(g, ctx), g, cfg)
    assert ctx.profile_report().get("shard_pack", {}).get("launches", 0) > 0
    ctx.detach()
    assert st.cutsize == ref_st.cutsize
    assert np.array_equal(parts, ref_parts)


def test_sharded_rmat24_equals_unsharded():
    """Power-law input at scale (R-MAT 2^24 ef16, k=64, deterministic): two
    local ranks over the sharded path (levels >= 2^20 vertices sharded)
    return the unsharded partition bit for bit."""
    g = gen.rmat_graph(24, 16, 0)
    cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=True)
    ref_parts, ref_pw, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    res = _run_sharded(g, cfg, 2, shard_min=1 << 20)
    for parts, pw, st in res:
        assert st.cutsize == ref_st.cutsize
        assert np.array_equal(pw, ref_pw)
        assert np.array_equal(parts, ref_parts)


def _run_distributed(g, cfg, size, shard_min=None):
    """Each local rank uploads only its row block (DeviceGraph.upload_block):
    the finest level's matching, contraction and refinement run distributed
    (and those of every coarse level of >= shard_min vertices)."""
    from paper_2304_13194_b200 import dist as jd
    group = _lib.LocalGroup(size)
    ctxs = [_lib.Context(0) for _ in range(size)]
    b = jd.shard_bounds(g.row_offsets, size)
    out, blocks, errs = [None] * size, [None] * size, []

    def work(r):
        try:
            ctxs[r].attach_local(group, r)
            if shard_min is not None:
                ctxs[r].set_shard_min_vertices(shard_min)
            dg = _lib.DeviceGraph.upload_block(g, int(b[r]), int(b[r + 1]), ctxs[r])
            blocks[r] = dg.block()
            out[r] = partition_resident(dg, g, cfg, want_parts=True)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert not any(t.is_alive() for t in th), "a rank did not finish"
    for c in ctxs:
        c.detach()
    return out, blocks, b


@pytest.mark.parametrize("name,size,smin", [("grid27_32", 2, None), ("grid27_32", 3, None),
                                            ("rmat16", 2, None), ("grid27_32", 3, 1000),
                                            ("rmat16", 3, 1000)])
def test_distributed_levels_equal_replicated(name, size, smin):
    """Throughput mode on a 1D-distributed graph (every rank stores only its
    rows; with smin=1000 the coarse levels above 4096 vertices stay
    distributed too): same partition as the replicated run, bit for bit, and
    each rank holds only its block's entries."""
    g = gen.grid27_graph(32) if name.startswith("grid") else gen.rmat_graph(16, 16, 0)
    cfg = J.RefinerConfig(k=16, imbalance=0.03, seed=0, deterministic=False)
    ref_parts, ref_pw, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    res, blocks, b = _run_distributed(g, cfg, size, smin)
    offs = np.asarray(g.row_offsets)
    for r, ((parts, pw, st), (lo, hi, ent)) in enumerate(zip(res, blocks)):
        dist_levels = [st.levels[i].level for i in range(st.n_levels) if st.levels[i].distributed]
        assert 0 in dist_levels
        if smin is not None:
            assert len(dist_levels) >= 2, dist_levels
        assert (lo, hi) == (b[r], b[r + 1])
        assert ent == offs[hi] - offs[lo] < offs[-1]
        assert st.cutsize == ref_st.cutsize
        assert np.array_equal(pw, ref_pw)
        assert np.array_equal(parts, ref_parts)


def test_nccl_transport_distributed_single_rank():
    """The distributed path (block upload, halo exchanges, coarse gathers)
    over the NCCL transport with one rank holding the whole block."""
    g = gen.grid27_graph(24)
    cfg = J.RefinerConfig(k=8, imbalance=0.03, seed=0, deterministic=False)
    ref_parts, _, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    ctx = _lib.Context(0)
    ctx.attach_nccl(_lib.nccl_unique_id(), 0, 1)
    ctx.set_shard_min_vertices(1000)
    dg = _lib.DeviceGraph.upload_block(g, 0, g.n, ctx)
    parts, _, st = partition_resident(dg, g, cfg)
    assert st.levels[st.n_levels - 1].distributed == 1  # L0 (uncoarsened last)
    dg.free()
    ctx.detach()
    assert st.cutsize == ref_st.cutsize
    assert np.array_equal(parts, ref_parts)


def test_distributed_rmat24_equals_replicated():
    """R-MAT 2^24 ef16, k=64, throughput mode, two local ranks each storing
    half the rows (levels >= 2^20 vertices distributed)."""
    g = gen.rmat_graph(24, 16, 0)
    cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=False)
    ref_parts, ref_pw, ref_st = partition_resident(_lib.DeviceGraph.upload(g), g, cfg)
    res, blocks, b = _run_distributed(g, cfg, 2)
    for (parts, pw, st), (lo, hi, ent) in zip(res, blocks):
        assert ent < int(np.asarray(g.row_offsets)[-1])
        assert st.cutsize == ref_st.cutsize
        assert np.array_equal(pw, ref_pw)
        assert np.array_equal(parts, ref_parts)
