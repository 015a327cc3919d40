#!/usr/bin/env python3
"""GPU disc max radius / disc-oracle max radius per pair (R15; bar: within 2x),
for the radix-8 disc kernels (ivm_d3 / d4 / d7) at one size per kernel family and digit kind.

    python tools/disc_oracle_ratios.py [--out profiles/r02/disc_oracle_ratios.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import oracle
    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import inputs
    ctx = ivm.Context(0)
    rows = []
    for n, B in [(512, 16), (1000, 16), (4096, 16), (8192, 8), (16384, 8), (32768, 4), (75000, 4), (131072, 2)]:
        for kind, name in [(0, "uniform"), (1, "all255"), (2, "sparse")]:
            a, b = inputs.pair_digits(0xD0 + n, np.arange(B), n, np.full(B, kind))
            p, c, r = ctx.multiply_disc(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
            torch.cuda.synchronize()
            ref = oracle.disc_mul(a, b)
            ratio = np.maximum(r.cpu().numpy(), 1e-30) / np.maximum(ref["max_radius"], 1e-30)
            row = {"n": n, "m": ivm.fft_length(n), "kind": name, "pairs": B,
                   "gpu_certified": int(c.sum().item()), "oracle_certified": int(ref["cert"].sum()),
                   "ratio_min": float(ratio.min()), "ratio_max": float(ratio.max()),
                   "gpu_max_radius": float(r.max().item()), "oracle_max_radius": float(ref["max_radius"].max())}
            rows.append(row)
            print(row, flush=True)
    if args.out:
        json.dump({"about": "GPU disc radius / disc oracle radius per pair (bar: <= 2)", "library": ivm.lib().ivm_version().decode()
                   if hasattr(ivm.lib().ivm_version(), "decode") else "ivm", "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
