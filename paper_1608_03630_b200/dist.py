"""Host-side plumbing of the slab-decomposed path: one process per GPU, launched by
torchrun; torch.distributed only carries the NCCL unique id (and, in tests, gathers results).  Every
exchange of the hot path itself runs inside libdiffreg.so (NCCL grouped send/recv on the context
stream).  Argument marshalling only: no step of the method runs here."""
from __future__ import annotations

import os

import torch

from .diffreg import Comm, Config, dr_slab, nccl_unique_id


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 rank when absent)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def broadcast_uid(uid: bytes | None, rank: int) -> bytes:
    """Rank 0's NCCL unique id, delivered to every rank of the default torch.distributed group."""
    import torch.distributed as dist
    obj = [uid if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out = obj[0]
    assert isinstance(out, (bytes, bytearray)) and len(out) == 128, "bad NCCL unique id"
    return bytes(out)


def make_comm(rank: int, world: int) -> Comm | None:
    """NCCL communicator of the library for this rank (None with one rank).  Requires an initialised
    default torch.distributed process group (any backend) to broadcast the unique id."""
    if world == 1:
        return None
    uid = broadcast_uid(nccl_unique_id() if rank == 0 else None, rank)
    return Comm.nccl(uid, rank, world)


def slab_of(x: torch.Tensor, cfg: Config, nranks: int, rank: int) -> torch.Tensor:
    """This rank's x3 slab of a global scalar (N3, N2, N1) or vector (3, N3, N2, N1) field, contiguous."""
    z0, nz = dr_slab(cfg, nranks, rank)
    return x.narrow(x.dim() - 3, z0, nz).contiguous()


def assemble(slabs: list[torch.Tensor]) -> torch.Tensor:
    """Inverse of slab_of over all ranks (concatenation along x3)."""
    return torch.cat(slabs, dim=slabs[0].dim() - 3)


def map_peers(ctx) -> None:
    """Fused ghost exchange across processes (DR_PEER_GHOSTS=1): every rank exports its workspace's
    CUDA IPC handle, the handles are all-gathered over the default torch.distributed group, and each
    rank maps its two x3 neighbours' workspaces (dr_peer_import).  Collective."""
    import torch.distributed as dist
    mine = ctx.peer_export()
    allh = [None] * ctx.nranks
    dist.all_gather_object(allh, mine)
    ctx.peer_import([h for h, _ in allh], [o for _, o in allh])
