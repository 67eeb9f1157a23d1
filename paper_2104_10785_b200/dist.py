"""Multi-GPU plumbing: one process per GPU, NCCL communicator inside libksvd.

torch.distributed (any backend; gloo works) is used only to broadcast the
NCCL unique id from rank 0.  After `init_distributed()` every entry point
row-shards A with `linops.row_partition`; the only collectives on the GK
path are NCCL all-reduces of the length-n partial A^T q and of the small
CGS dot vectors / norms of the left basis (issued inside libksvd on the
context stream).
"""

from __future__ import annotations

import os

from . import _lib
from .linops import row_partition  # noqa: F401  (re-export)


def broadcast_uid(uid: bytes | None, rank: int) -> bytes:
    """Rank 0's NCCL unique id, delivered to every rank over torch.distributed."""
    import torch.distributed as dist

    obj = [uid if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out = obj[0]
    if not isinstance(out, (bytes, bytearray)) or len(out) != _lib.NCCL_UID_BYTES:
        raise RuntimeError("bad NCCL unique id broadcast")
    return bytes(out)


PX_SLOT = 1 << 17  # doubles per sender slot of the peer exchange (1 MB)


def open_peer_exchange(ctx: _lib.Context, slot: int = PX_SLOT) -> bool:
    """Map every rank's receive area over CUDA IPC (handles all-gathered over
    torch.distributed) so the GK step's all-reduces run as one NVLink kernel
    (csrc/peer.cuh) instead of ncclAllReduce.  Collective; returns whether
    the exchange passed its self-test on every rank (NCCL stays otherwise)."""
    import torch.distributed as dist

    mine = ctx.px_export(slot)
    allh = [None] * ctx.nranks
    dist.all_gather_object(allh, mine)
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != _lib.PX_HANDLE_BYTES
           for h in allh):
        raise RuntimeError("bad peer-exchange handle all-gather")
    return ctx.px_open(b"".join(bytes(h) for h in allh))


def init_distributed(device: int | None = None,
                     peer_exchange: bool | None = None) -> _lib.Context:
    """Create this rank's context (NCCL communicator when world > 1) and make
    it the process default.  Requires torch.distributed to be initialised
    when WORLD_SIZE > 1.  peer_exchange (default: env KSVD_P2P=1) maps the
    NVLink peer exchange for the step all-reduces."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(), dist.get_world_size()
    else:
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world > 1:
            raise RuntimeError("init torch.distributed before init_distributed()")
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", str(rank)))
    uid = None
    if world > 1:
        uid = broadcast_uid(_lib.nccl_unique_id() if rank == 0 else None, rank)
    ctx = _lib.Context(device=device, rank=rank, nranks=world, uid=uid)
    _lib.set_context(ctx)
    if peer_exchange is None:
        peer_exchange = os.environ.get("KSVD_P2P") == "1"
    if world > 1 and peer_exchange:
        open_peer_exchange(ctx)
    return ctx
