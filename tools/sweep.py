"""Perf sweep over FFT lengths (dev tool): device time per multiply batch,
fraction of the nominal FP64 roofline W(m) / (148*64*f).

    python tools/sweep.py [--prec f64|f32] [--ns 500,1000,2000,4096] [--batch 4096]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def W(m):
    L = int(math.log2(m))
    return 24 * m * L - 28 * m + 48


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="f64")
    ap.add_argument("--ns", default="128,256,500,1000,2000,4096")
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_1006_0405_b200 as ivm
    ctx = ivm.Context(0)
    prec = ivm.F64 if args.prec == "f64" else ivm.F32
    peak = 148 * 64 * 1965e6 * (2 if prec == ivm.F32 else 1)
    for n in [int(x) for x in args.ns.split(",")]:
        B = args.batch
        a = ctx.generate_digits(n, B, 1, 0)
        b = ctx.generate_digits(n, B, 1, 1)
        out = torch.empty((B, 2 * n), dtype=torch.uint8, device="cuda")
        cert = torch.empty((B,), dtype=torch.uint8, device="cuda")
        ctx.reserve(n, B, prec)
        for _ in range(2):
            ctx.multiply(a, b, prec=prec, out=out, cert=cert)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            ctx.multiply(a, b, prec=prec, out=out, cert=cert)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        m = ivm.fft_length(n)
        frac = W(m) * B / (ms / 1e3) / peak
        print(json.dumps({"n": n, "m": m, "batch": B, "ms": round(ms, 4), "cert": int(cert.sum()),
                          "digits_per_s": n * int(cert.sum()) / (ms / 1e3), "frac_W": round(frac, 4),
                          "us_per_mult": round(ms * 1e3 / B, 3)}), flush=True)


if __name__ == "__main__":
    main()
