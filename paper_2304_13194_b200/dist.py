"""Multi-GPU plumbing for the 1D vertex-sharded refinement.

One process per GPU under torchrun. torch.distributed is only the bootstrap:
rank 0 creates the NCCL unique id, every rank receives it through a
broadcast and attaches its context to the communicator; the exchange steps
then run inside libjet over NCCL (csrc/comm.cu). Every rank computes the same
partition. `shard_bounds` is the block split (balanced by entries, as
csrc/refine.cu k_shard_bounds): rank r uploads rows [b_r, b_{r+1}) with
`_lib.DeviceGraph.upload_block` for a distributed partition.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def shard_bounds(row_offsets, size: int) -> np.ndarray:
    """Vertex block boundaries [b_0 = 0, ..., b_size = n]: rank r owns
    [b_r, b_r+1), the first vertex whose row starts at or after r/size of the
    entries (balanced by entries, as csrc/refine.cu k_shard_bounds)."""
    offs = np.asarray(row_offsets, dtype=np.int64)
    n, nnz = len(offs) - 1, int(offs[-1])
    b = np.empty(size + 1, np.int64)
    for r in range(size + 1):
        if r == 0:
            b[r] = 0
        elif r == size:
            b[r] = n
        else:
            b[r] = int(np.searchsorted(offs[:n], (nnz * r) // size, side="left"))
    return b


def broadcast_id(make_id, rank: int, device=None) -> bytes:
    """Rank 0's make_id() (128 bytes) on every rank (torch.distributed)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(make_id()), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())


def attach_nccl(ctx: "_lib.Context", shard_min_vertices: int | None = None) -> None:
    """Attach `ctx` to an NCCL communicator over the current torch.distributed
    group (one rank per GPU)."""
    import torch
    import torch.distributed as dist
    rank, size = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", ctx.device) if dist.get_backend() == "nccl" else None
    nid = broadcast_id(_lib.nccl_unique_id, rank, dev)
    ctx.attach_nccl(nid, rank, size)
    if shard_min_vertices is not None:
        ctx.set_shard_min_vertices(shard_min_vertices)
