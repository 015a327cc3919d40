"""Batch sharding across ranks (one process per GPU, torch.distributed).

Independent multiplications shard with no data-path collective (SURVEY.md
§8(e)): rank r owns a contiguous range of pairs.  Collectives are used only
for timing (max over ranks), counting (sum of certified pairs) and the
optional gather of products/flags to rank 0 (the north star's NCCL use).
Works with any backend (nccl on GPUs, gloo on CPU for the tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """(first pair, number of pairs) of rank's contiguous share of `batch`."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def _ready() -> bool:
    return dist.is_available() and dist.is_initialized()


def max_over_ranks(x: float, device=None) -> float:
    if not _ready():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not _ready():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_to_root(prod: torch.Tensor, cert: torch.Tensor, root: int = 0):
    """Gather equal-size shards [B_r][2n] u8 and [B_r] u8 onto `root`.

    Returns (products [world*B_r][2n], flags [world*B_r]) on root, (None, None)
    elsewhere.  Uses all_gather_into_tensor (supported by nccl and gloo)."""
    if not _ready():
        return prod, cert
    world, rank = dist.get_world_size(), dist.get_rank()
    out_p = torch.empty((world * prod.shape[0],) + tuple(prod.shape[1:]), dtype=prod.dtype,
                        device=prod.device)
    out_c = torch.empty((world * cert.shape[0],), dtype=cert.dtype, device=cert.device)
    dist.all_gather_into_tensor(out_p, prod.contiguous())
    dist.all_gather_into_tensor(out_c, cert.contiguous())
    if rank == root:
        return out_p, out_c
    return None, None
