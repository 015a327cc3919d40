"""A/B device timing of two builds of libivm.so on the same GPU (dev tool).

    python tools/ab.py ab/libivm_base.so ab/libivm_new.so [--n 4096] [--batch 4096] [--rounds 5]
    python tools/ab.py lib.so lib.so@IVM_KERNEL=v5      # same build, environment overrides
    AB_FN=disc python tools/ab.py ...                   # time ivm_multiply_disc instead

Alternates the two builds in fresh subprocesses (one library per process) and
prints the median ms per batch of each (CUDA events, L2 flushed between reps).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, torch
sys.path.insert(0, %r)
import paper_1006_0405_b200 as ivm
ctx = ivm.Context(0)
n, B, reps = %d, %d, %d
a = ctx.generate_digits(n, B, 1, 0); b = ctx.generate_digits(n, B, 1, 1)
out = torch.empty((B, 2 * n), dtype=torch.uint8, device="cuda"); cert = torch.empty((B,), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
import os
if os.environ.get("AB_FN") == "disc":
    mul = lambda: ctx.multiply_disc(a, b, out=out, cert=cert, want_radius=False)
else:
    mul = lambda: ctx.multiply(a, b, out=out, cert=cert)
for _ in range(3): mul()
ts = []
for _ in range(reps):
    flush.zero_(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); mul(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps(sorted(ts)[len(ts) // 2]))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    res = {l: [] for l in dict.fromkeys(args.libs)}
    for _ in range(args.rounds):
        for lib in args.libs:
            path, *kv = lib.split("@")
            env = dict(os.environ, IVM_LIB=os.path.abspath(path), **dict(x.split("=", 1) for x in kv))
            o = subprocess.run([sys.executable, "-c", CHILD % (ROOT, args.n, args.batch, args.reps)], env=env,
                               capture_output=True, text=True, check=True)
            res[lib].append(json.loads(o.stdout.strip().splitlines()[-1]))
    for lib, v in res.items():
        print(f"{lib}: median {statistics.median(v):.4f} ms  all {['%.4f' % x for x in v]}")


if __name__ == "__main__":
    main()
