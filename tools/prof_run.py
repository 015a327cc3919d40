"""Dev tool: a few batched multiplications at (n, batch) for ncu captures.

    python tools/prof_run.py N BATCH [disc]     (disc: the circular-set kernel)
"""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, paper_1006_0405_b200 as ivm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
ctx = ivm.Context(0)
a = ctx.generate_digits(n, B, 1, 0); b = ctx.generate_digits(n, B, 1, 1)
disc = len(sys.argv) > 3 and sys.argv[3] == "disc"
for _ in range(3):
    if disc:
        ctx.multiply_disc(a, b)
    else:
        ctx.multiply(a, b)
torch.cuda.synchronize()
