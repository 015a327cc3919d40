"""Host-side multi-rank logic on CPU (gloo, world_size 2): sharding, max/sum
over ranks, and the gather of products/flags to rank 0."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1006_0405_b200 import dist as ivd
from paper_1006_0405_b200 import inputs


def test_shard_covers_batch_disjointly():
    for batch in (1, 2, 7, 4096, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            seen = np.zeros(batch, int)
            for r in range(world):
                s, c = ivd.shard(batch, r, world)
                seen[s:s + c] += 1
            assert (seen == 1).all()
            counts = [ivd.shard(batch, r, world)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1


def test_shard_rejects_bad_args():
    with pytest.raises(ValueError):
        ivd.shard(10, 2, 2)


def test_chunk_plan_covers_every_shard():
    for batch in (1, 7, 100, 65536, 65537):
        for world in (1, 2, 3, 8):
            for chunks in (1, 3, 8):
                plan = ivd.chunk_plan(batch, world, chunks)
                seen = np.zeros(batch, int)
                for r in range(world):
                    s0, c = ivd.shard(batch, r, world)
                    pos = s0
                    for g0, cnt in plan[r]:
                        assert g0 == pos  # contiguous, in order
                        seen[g0:g0 + cnt] += 1
                        pos += cnt
                    assert pos == s0 + c
                assert (seen == 1).all()


@pytest.mark.parametrize("batch,chunks", [(7, 3), (3, 4)])
def test_spawned_two_ranks_gather_and_summary(batch, chunks):
    """dist.spawn (the bench.py --gpus N launch) with world size 2 on gloo:
    unequal shards (batch 7), chunks, more chunks than pairs (batch 3); the
    root's gathered products equal the oracle's long multiplication in pair
    order, the summary is the exact count / max, and the plain gather agrees."""
    import json
    import subprocess
    import sys
    import oracle
    n = 40
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dist_worker.py")
    cmd = [sys.executable, "-c",
           "import sys; sys.path.insert(0, %r); from paper_1006_0405_b200 import dist as d; "
           "sys.exit(d.spawn(2, %r, %r, env={'OMP_NUM_THREADS': '1'}))"
           % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), worker, [str(n), str(batch), str(chunks)])]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    a, b = inputs.pair_digits(0xD157, np.arange(batch), n, "uniform")
    want = oracle.long_multiply(a, b)
    o = oracle.ivmul(a, b)
    assert out["world"] == 2
    assert np.array_equal(np.array(out["prod"], np.uint8), want)
    assert out["cert"] == [1] * batch
    assert out["total"] == batch and out["maxrad"] == o["max_radius"].max()
    assert out["prod2_equal"] and out["cert2_equal"] and out["tmax"] == 2.5
    assert sum(c for _, c in out["calls"]) == ivd.shard(batch, 0, 2)[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank "multiplies" its shard: here the digits of its pairs stand in
        n, batch = 8, 6
        s, c = ivd.shard(batch, rank, world)
        a = torch.from_numpy(inputs.digits(11, np.arange(s, s + c), 0, 2 * n, "uniform"))
        cert = torch.full((c,), rank + 1, dtype=torch.uint8)
        t = ivd.max_over_ranks(1.5 + rank)
        tot = ivd.sum_over_ranks(c)
        gp, gc = ivd.gather_to_root(a, cert)
        if rank == 0:
            q.put((t, tot, gp.numpy().copy(), gc.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_max_sum_gather():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    t, tot, gp, gc = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.5 and tot == 6
    want = inputs.digits(11, np.arange(6), 0, 16, "uniform")
    assert np.array_equal(gp, want)
    assert gc.tolist() == [1, 1, 1, 2, 2, 2]
