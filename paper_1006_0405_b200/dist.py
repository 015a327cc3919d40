"""Batch sharding across ranks (one process per GPU, torch.distributed).

Independent multiplications shard with no data-path collective (SURVEY.md
§8(e)): rank r owns a contiguous range of pairs.  Collectives are used only
for timing (max over ranks), the summary of a step (certified pairs summed,
max radius maxed: ``summary_allreduce``) and the optional gather of products
and flags to the root (the north star's NCCL use), which
``multiply_gather`` pipelines with the multiplications: the shard is cut into
chunks, and chunk k's point-to-point sends to the root run on NCCL's stream
while chunk k+1 is multiplied on the compute stream.  Unequal shards need no
padding: every rank derives every rank's chunk plan from ``shard``.

``spawn`` re-launches a script under torch.distributed.run (one process per
GPU, rendezvous on 127.0.0.1), which is how ``bench.py --gpus N`` starts its
ranks when it was not itself started by torchrun.

Works with any backend (nccl on GPUs, gloo on CPU for the tests).
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from typing import Callable

import torch
import torch.distributed as dist


def shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """(first pair, number of pairs) of rank's contiguous share of `batch`."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def chunk_plan(batch: int, world: int, chunks: int) -> list[list[tuple[int, int]]]:
    """plan[r][k] = (first pair, count) of chunk k of rank r's shard, as global
    pair indices; chunks of one shard are contiguous and nearly equal (some
    are empty when the shard has fewer than `chunks` pairs)."""
    if chunks < 1:
        raise ValueError("chunks must be >= 1")
    plan = []
    for r in range(world):
        s0, c = shard(batch, r, world)
        plan.append([(s0 + o, k) for o, k in (shard(c, j, chunks) for j in range(chunks))])
    return plan


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


def summary_allreduce(cert: torch.Tensor, max_radius: torch.Tensor | None = None) -> tuple[int, float]:
    """(certified pairs over all ranks, max radius over all ranks) of one step:
    a local count / max on the device, then ONE all-gather of the two numbers
    (one collective for a SUM and a MAX).  max_radius None -> radius nan."""
    dev = cert.device
    loc = torch.stack([cert.to(torch.float64).sum(),
                       max_radius.to(torch.float64).max() if max_radius is not None and max_radius.numel()
                       else torch.tensor(float("nan"), dtype=torch.float64, device=dev)])
    if not _ready():
        return int(loc[0].item()), float(loc[1].item())
    world = dist.get_world_size()
    allv = torch.empty(2 * world, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(allv, loc)
    allv = allv.view(world, 2).cpu()
    rad = allv[:, 1]
    return int(allv[:, 0].sum().item()), float(rad.max().item()) if not torch.isnan(rad).all() else float("nan")


def multiply_gather(compute: Callable[[int, int], None], prod: torch.Tensor, cert: torch.Tensor, batch: int,
                    chunks: int = 4, root: int = 0, out_prod: torch.Tensor | None = None,
                    out_cert: torch.Tensor | None = None):
    """Multiply this rank's shard chunk by chunk and gather every chunk to `root`.

    compute(lo, cnt) must enqueue the multiplication of the local pairs
    [lo, lo + cnt) of this rank's shard into prod[lo:lo+cnt], cert[lo:lo+cnt]
    on the current stream (prod [shard][2n], cert [shard] are this rank's
    buffers).  After chunk k is enqueued, its sends (non-root) or receives
    (root, from every other rank) are posted as one batch of P2P operations;
    with NCCL they run on NCCL's stream after chunk k's work, so chunk k+1
    computes while chunk k travels.  Returns (products [batch][2n], flags
    [batch]) on root (the root's own chunks copied in), (None, None) elsewhere.
    Without an initialised process group it is a single-rank multiply."""
    world = dist.get_world_size() if _ready() else 1
    rank = dist.get_rank() if _ready() else 0
    plan = chunk_plan(batch, world, chunks)
    s0 = plan[rank][0][0]
    if rank == root:
        if out_prod is None:
            out_prod = torch.empty((batch,) + tuple(prod.shape[1:]), dtype=prod.dtype, device=prod.device)
        if out_cert is None:
            out_cert = torch.empty((batch,), dtype=cert.dtype, device=cert.device)
    pending = []
    for k in range(chunks):
        g0, cnt = plan[rank][k]
        if cnt:
            compute(g0 - s0, cnt)
        ops = []
        if rank == root:
            if cnt:
                out_prod[g0:g0 + cnt].copy_(prod[g0 - s0:g0 - s0 + cnt], non_blocking=True)
                out_cert[g0:g0 + cnt].copy_(cert[g0 - s0:g0 - s0 + cnt], non_blocking=True)
            for r in range(world):
                if r == root:
                    continue
                q0, qc = plan[r][k]
                if qc:
                    ops.append(dist.P2POp(dist.irecv, out_prod[q0:q0 + qc], r))
                    ops.append(dist.P2POp(dist.irecv, out_cert[q0:q0 + qc], r))
        elif cnt:
            ops.append(dist.P2POp(dist.isend, prod[g0 - s0:g0 - s0 + cnt], root))
            ops.append(dist.P2POp(dist.isend, cert[g0 - s0:g0 - s0 + cnt], root))
        if ops:
            pending.extend(dist.batch_isend_irecv(ops))
    for w in pending:
        w.wait()
    if rank == root:
        return out_prod, out_cert
    return None, None


def gather_to_root(prod: torch.Tensor, cert: torch.Tensor, batch: int | None = None, root: int = 0):
    """Gather already-computed shards (contiguous, shard() sizes, possibly
    unequal) of [B_r][2n] products and [B_r] flags onto `root` with
    point-to-point receives (no all-gather: only the root receives).
    batch: the whole job's pair count (default: world * local shard)."""
    if not _ready():
        return prod, cert
    world = dist.get_world_size()
    if batch is None:
        batch = world * prod.shape[0]
    return multiply_gather(lambda lo, cnt: None, prod, cert, batch, chunks=1, root=root)


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn(nprocs: int, script: str, args: list[str], env: dict | None = None, timeout: float | None = None) -> int:
    """Run `script args` as nprocs ranks of one node under torch.distributed.run
    (rendezvous on 127.0.0.1, a free port); returns the launcher's exit code.
    NCCL's INIT logging goes to stderr (ranks, transports, NVLS) unless the
    caller set NCCL_DEBUG."""
    e = dict(os.environ)
    e.setdefault("NCCL_DEBUG", "INFO")
    e.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    e.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if env:
        e.update(env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nprocs}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *args]
    return subprocess.run(cmd, env=e, timeout=timeout).returncode
