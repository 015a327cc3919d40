"""The paper's comparison (its figure's lines) on B200: exact long
multiplication vs the certified fp64 interval FFT multiplication, in
certified (resp. exact) digits per second, for a range of operand lengths.
Uniform digits; batches sized for ~50 ms of work; CUDA-event device times.

    python tools/long_vs_fft.py [--out profiles/r01/long_vs_fft.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps):
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
    ap.add_argument("--ns", default="16,32,64,128,256,512,1000,2048,4096,8192,16384,32768,75000")
    args = ap.parse_args()
    import torch
    import paper_1006_0405_b200 as ivm
    ctx = ivm.Context(0)
    rows = []
    for n in [int(x) for x in args.ns.split(",")]:
        B = max(1, min(65536, int(2e9 / (n * max(n, 64)))))  # ~n^2 B bounded
        B = max(B, 148 if n <= 20000 else 16)
        a = ctx.generate_digits(n, B, 0x5EED, 0)
        b = ctx.generate_digits(n, B, 0x5EED, 1)
        out = torch.empty((B, 2 * n), dtype=torch.uint8, device="cuda")
        cert = torch.empty((B,), dtype=torch.uint8, device="cuda")
        t_fft = timed(lambda: ctx.multiply(a, b, prec=ivm.F64, out=out, cert=cert), 5)
        ncert = int(cert.sum().item())
        ref = out.clone()
        t_long = timed(lambda: ctx.long_multiply(a, b, out=out), 3)
        agree = bool(torch.equal(out[cert.bool()], ref[cert.bool()]))
        row = {"n": n, "batch": B, "fft_ms": t_fft, "long_ms": t_long, "fft_certified": ncert,
               "fft_certified_digits_per_s": ncert * n / (t_fft / 1e3), "long_digits_per_s": B * n / (t_long / 1e3),
               "products_agree": agree}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": "exact long multiplication vs certified fp64 interval FFT, uniform digits, B200",
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
