"""The paper's naive fixed-precision SS on B200: error rate
of the punctual round-to-nearest multiplication against exact products, next
to the certified interval path's certified fraction and the speeds.

    python tools/naive_errors.py [--out profiles/r01/naive_errors.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--ns", default="16,32,64,96,120,160,256,512,1024,2048,4096")
    ap.add_argument("--batch", type=int, default=1024)
    args = ap.parse_args()
    import torch
    import paper_1006_0405_b200 as ivm
    ctx = ivm.Context(0)
    rows = []
    for n in [int(x) for x in args.ns.split(",")]:
        B = args.batch
        a = ctx.generate_digits(n, B, 0x0A1E, 0)
        b = ctx.generate_digits(n, B, 0x0A1E, 1)
        exact = ctx.long_multiply(a, b)
        row = {"n": n, "pairs": B}
        for name, prec in (("f32", ivm.F32), ("f64", ivm.F64)):
            nv = ctx.multiply_naive(a, b, prec=prec)
            row[f"naive_{name}_wrong_fraction"] = float((nv != exact).any(dim=1).float().mean().item())
            row[f"naive_{name}_ms"] = timed(lambda: ctx.multiply_naive(a, b, prec=prec, out=nv))
            out, cert = ctx.multiply(a, b, prec=prec)
            row[f"certified_{name}_fraction"] = float(cert.float().mean().item())
            certb = cert.bool()
            row[f"certified_{name}_wrong"] = int((out[certb] != exact[certb]).any(dim=1).sum().item())
            row[f"certified_{name}_ms"] = timed(lambda: ctx.multiply(a, b, prec=prec, out=out, cert=cert))
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": "naive (punctual RN) SS vs certified interval SS, uniform digits, B200", "rows": rows},
                      f, indent=1)


if __name__ == "__main__":
    main()
