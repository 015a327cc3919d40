"""Randomized soak test (dev tool, GPU): random sizes over every kernel family,
random batch sizes, digit kinds and precisions; every certified product is
checked against Python's exact integer product (a sample of pairs at large n),
every uncertified product must be all zeros.  Intended to catch intermittent
synchronization bugs (mbarrier phases, cluster / group barriers) that a fixed
test set may miss.

    python tools/soak.py [--seconds 180] [--seed 1]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=180)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import inputs
    rng = np.random.default_rng(args.seed)
    ctx = ivm.Context(0)
    big = lambda d: int.from_bytes(bytes(d), "little")
    t0 = time.time()
    runs = checked = fails = 0
    while time.time() - t0 < args.seconds:
        lg = int(rng.integers(0, 18))  # n ~ 2^lg .. 2^(lg+1)
        n = int(rng.integers(1 << lg, (2 << lg) if lg < 17 else 131073))
        n = min(n, 131072)
        if n >= 16 and rng.random() < 0.5:
            n -= n % 16  # 16-byte aligned rows: the throughput kernel variants
        maxb = max(1, min(600, 4_000_000 // n))
        B = int(rng.integers(1, maxb + 1))
        prec = ivm.F32 if (n <= 4096 and rng.random() < 0.2) else ivm.F64
        kinds = rng.integers(0, 4, B)
        a, b = inputs.pair_digits(int(rng.integers(1 << 30)), np.arange(B), n, kinds)
        if prec == ivm.F64 and rng.random() < 0.15:  # circular containment sets (every kernel family of theirs)
            out, cert, _ = ctx.multiply_disc(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), want_radius=False)
        else:
            out, cert = ctx.multiply(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), prec=prec)
        o, c = out.cpu().numpy(), cert.cpu().numpy().astype(bool)
        sample = np.arange(B) if n * B <= 400_000 else rng.choice(B, min(B, 4), replace=False)
        for p in sample:
            if c[p]:
                ok = big(o[p]) == big(a[p]) * big(b[p])
            else:
                ok = not o[p].any()
            checked += 1
            if not ok:
                fails += 1
                print(f"FAIL n={n} B={B} prec={prec} pair={p} kind={kinds[p]} cert={c[p]}", flush=True)
        if prec == ivm.F64 and not c.all():
            print(f"note: fp64 uncertified n={n} B={B}: {int((~c).sum())} pairs", flush=True)
        runs += 1
    print(f"soak: {runs} calls, {checked} products checked, {fails} failures, {time.time() - t0:.0f} s", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
