"""Multi-process plumbing (one process per GPU, torch.distributed for rendezvous only).

The data path's exchange runs inside libdc (dc_cct_merge_ranks over its own NCCL
communicator). Here: rank/world from the torchrun environment, the NCCL unique-id broadcast,
max-over-ranks of device timings, and the shard assignment of SURVEY §8(d) config 5.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank_world() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: str = "nccl", device: int | None = None):
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        kw = {}
        if backend == "nccl" and device is not None:
            kw["device_id"] = torch.device(f"cuda:{device}")
        dist.init_process_group(backend, **kw)
    return rank, world, local


def _dev(backend_device: str | None):
    if backend_device:
        return torch.device(backend_device)
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float, device: str | None = None) -> float:
    """Max of a per-rank scalar (device timings are taken as the max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def broadcast_bytes(b: bytes | None, src: int = 0, n: int = 128, device: str | None = None) -> bytes:
    """Broadcast a fixed-size byte string (the 128-byte ncclUniqueId) from src."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return bytes(b)
    t = torch.zeros(n, dtype=torch.uint8, device=_dev(device))
    if dist.get_rank() == src:
        t.copy_(torch.frombuffer(bytearray(b), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().numpy().tobytes())


def make_comm(ctx, world: int, rank: int):
    """libdc NCCL communicator: rank 0 creates the unique id, torch.distributed broadcasts it."""
    import paper_2411_02797_b200 as dc
    uid = dc.dc_nccl_unique_id() if rank == 0 else bytes(128)
    uid = broadcast_bytes(uid, 0)
    return dc.dc_comm_create(ctx, uid, world, rank)


def shards_for_rank(n_shards: int, rank: int, world: int) -> list[int]:
    """Config 5: rank p builds shards {s : s mod P == p}."""
    return [s for s in range(n_shards) if s % world == rank]
