"""A rank of the world-size-2 gloo test of the multi-rank host logic
(tests/test_dist.py), started through paper_1006_0405_b200.dist.spawn, i.e. the
same torch.distributed.run launch bench.py --gpus N uses.  The per-chunk
"multiply" is the CPU oracle (test side): what is tested is the launch,
sharding, chunked gather to the root and the summary all-reduce."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1006_0405_b200 import dist as ivd  # noqa: E402
from paper_1006_0405_b200 import inputs  # noqa: E402


def main():
    n, batch, chunks = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    s0, cnt = ivd.shard(batch, rank, world)
    a, b = inputs.pair_digits(0xD157, np.arange(s0, s0 + cnt), n, "uniform")
    prod = torch.zeros((cnt, 2 * n), dtype=torch.uint8)
    cert = torch.zeros((cnt,), dtype=torch.uint8)
    rad = torch.zeros((cnt,), dtype=torch.float64)
    calls = []

    def compute(lo, c):
        r = oracle.ivmul(a[lo:lo + c], b[lo:lo + c])
        prod[lo:lo + c] = torch.from_numpy(r["prod"])
        cert[lo:lo + c] = torch.from_numpy(r["cert"].astype(np.uint8))
        rad[lo:lo + c] = torch.from_numpy(r["max_radius"])
        calls.append((lo, c))

    gp, gc = ivd.multiply_gather(compute, prod, cert, batch, chunks=chunks)
    total, maxrad = ivd.summary_allreduce(cert, rad)
    gp2, gc2 = ivd.gather_to_root(prod, cert, batch)
    t = ivd.max_over_ranks(1.5 + rank)
    if rank == 0:
        print(json.dumps({"world": world, "total": total, "maxrad": maxrad, "tmax": t, "calls": calls,
                          "prod": gp.numpy().tolist(), "cert": gc.numpy().tolist(),
                          "prod2_equal": bool(torch.equal(gp, gp2)), "cert2_equal": bool(torch.equal(gc, gc2))}),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
