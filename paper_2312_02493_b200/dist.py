"""One-process-per-GPU plumbing: torch.distributed (gloo, host side only) to
ship NCCL's unique id from rank 0, to barrier, and to take the max of a
timing over ranks.  The data path itself never touches torch.distributed:
the library's NCCL communicators carry the collectives over NVLink."""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional


@dataclass
class DistEnv:
    world: int
    rank: int
    local_rank: int
    pg: Optional[object] = None  # torch.distributed module when world > 1

    def barrier(self) -> None:
        if self.pg is not None:
            self.pg.barrier()

    def max_over_ranks(self, x: float) -> float:
        if self.pg is None:
            return float(x)
        import torch

        t = torch.tensor([float(x)], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def broadcast_bytes(self, payload: Optional[bytes], src: int = 0) -> bytes:
        if self.pg is None:
            assert payload is not None
            return payload
        obj = [payload]
        self.pg.broadcast_object_list(obj, src=src)
        return obj[0]

    def gather_arrays(self, arr, dst: int = 0):
        """numpy array from every rank -> list on rank `dst` (None elsewhere)."""
        if self.pg is None:
            return [arr]
        out = [None] * self.world if self.rank == dst else None
        self.pg.gather_object(arr, out, dst=dst)
        return out

    def close(self) -> None:
        if self.pg is not None:
            self.pg.barrier()
            self.pg.destroy_process_group()
            self.pg = None


def init_from_env(backend: str = "gloo") -> DistEnv:
    """Reads WORLD_SIZE / RANK / LOCAL_RANK (torchrun) and, for world > 1,
    initialises a host-side process group (MASTER_ADDR defaults to 127.0.0.1)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world <= 1:
        return DistEnv(1, 0, local, None)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group(backend, rank=rank, world_size=world)
    return DistEnv(world, rank, local, dist)


def share_nccl_uid(env: DistEnv) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank receives the same bytes."""
    uid = None
    if env.rank == 0:
        from .flexcomm import get_unique_id

        uid = get_unique_id()
    return env.broadcast_bytes(uid, src=0)
