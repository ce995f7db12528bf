"""One-process-per-GPU plumbing: rank discovery, NCCL unique-id exchange, cube setup.

torch.distributed is used only to agree on the NCCL unique id (the reference's
run_spmd has no equivalent: its ranks are threads, cube3d/transport.hpp:378-398)
and for host-side barriers / max-over-ranks timing reductions. All data-path
collectives run inside libc3d on the per-axis NCCL communicators.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

from . import cube3d as c3


def env_ranks() -> Tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init_process_group(backend: str = "nccl"):
    import torch
    import torch.distributed as dist
    rank, world, local = env_ranks()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def exchange_uid(rank: int, world: int, uid_fn=None) -> Optional[bytes]:
    """Rank 0 creates the NCCL unique id; every rank receives the same 128 bytes."""
    if world == 1:
        return None
    import torch.distributed as dist
    obj = [(uid_fn or c3.Cube.unique_id)() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def make_cube(dims=None) -> c3.Cube:
    rank, world, local = env_ranks()
    dims = dims or c3.grid_for(world)
    if dims[0] * dims[1] * dims[2] != world:
        raise ValueError(f"grid {dims} does not have {world} ranks")
    uid = exchange_uid(rank, world)
    return c3.Cube(dims, rank, local, uid)


def max_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def destroy():
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()
