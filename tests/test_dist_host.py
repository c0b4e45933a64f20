"""Host side of the multi-GPU path on CPU (gloo, world_size 2): the NCCL id
bootstrap broadcast and the vertex block split."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_13194_b200 import dist as jd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=size)
    try:
        nid = jd.broadcast_id(lambda: bytes(range(128)), rank)
        q.put((rank, nid))
    finally:
        dist.destroy_process_group()


def test_broadcast_id_gloo():
    size, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(size))
    for p in ps:
        p.join(timeout=60)
    assert got[0] == got[1] == bytes(range(128))


@pytest.mark.parametrize("size", [1, 2, 3, 8])
def test_shard_bounds_cover_and_balance(size):
    rng = np.random.default_rng(0)
    deg = rng.integers(0, 50, size=1000)
    offs = np.concatenate([[0], np.cumsum(deg)])
    b = jd.shard_bounds(offs, size)
    assert b[0] == 0 and b[-1] == 1000 and np.all(np.diff(b) >= 0)
    per = np.diff(offs[b])
    assert per.max() - offs[-1] / size <= deg.max()
