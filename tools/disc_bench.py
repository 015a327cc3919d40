"""Circular vs rectangular containment sets (R15), measured.

GPU part (needs a B200): device throughput of ivm_multiply_disc and of the
rectangular path (ivm_multiply_batched) on the same seeded inputs (up to the
C3 workload), CUDA events, L2 flushed between reps; and the largest radius of
each over uniform and all-255 pairs, n = 32 .. 131072.  CPU part (--oracle):
the two oracles' radii (n up to 131072).

    python tools/disc_bench.py [--out gpurun_out/disc.json]
    python tools/disc_bench.py --oracle [--out profiles/r01/disc_oracle_radii.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gpu(args):
    import torch
    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import inputs
    ctx = ivm.Context(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {"throughput": [], "radius": []}

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return sorted(ts)[len(ts) // 2]

    for n, B in ((1000, 4096), (4096, 4096), (16384, 2048), (75000, 64)):
        if n == 75000:  # config C3: half uniform, half all-255
            kinds = torch.from_numpy(inputs.class_of_pairs("C3", B).astype(np.uint8)).cuda()
            a = ctx.generate_digits(n, B, inputs.config_seed(3), 0, kind=kinds)
            b = ctx.generate_digits(n, B, inputs.config_seed(3), 1, kind=kinds)
        else:
            a = ctx.generate_digits(n, B, 1, 0)
            b = ctx.generate_digits(n, B, 1, 1)
        t_d = timed(lambda: ctx.multiply_disc(a, b, want_radius=False))
        t_r = timed(lambda: ctx.multiply(a, b))
        _, cd, _ = ctx.multiply_disc(a, b, want_radius=False)
        _, cr = ctx.multiply(a, b)
        res["throughput"].append({
            "n": n, "batch": B, "disc_ms": t_d, "rect_ms": t_r,
            "disc_digits_per_s": n * B / (t_d / 1e3), "rect_digits_per_s": n * B / (t_r / 1e3),
            "disc_certified": float(cd.float().mean()), "rect_certified": float(cr.float().mean())})
        print(res["throughput"][-1], flush=True)
    for n in (32, 256, 1000, 4096, 16384, 75000, 131072):
        for kind in ("uniform", "all255"):
            a, b = inputs.pair_digits(0xD15E + n, np.arange(64 if n <= 16384 else 8), n, kind)
            ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
            _, cd, rd = ctx.multiply_disc(ta, tb)
            rr = ctx.multiply_diag(ta, tb)
            res["radius"].append({"n": n, "kind": kind, "disc_max_radius": float(rd.max()),
                                  "rect_max_radius": float(rr["max_radius"].max()),
                                  "disc_over_rect": float(rd.max() / rr["max_radius"].max()),
                                  "disc_certified": float(cd.float().mean()),
                                  "rect_certified": float(rr["cert"].float().mean())})
            print(res["radius"][-1], flush=True)
    return res


def cpu():
    import oracle
    from paper_1006_0405_b200 import inputs
    out = []
    for n in (1000, 4096, 16384, 75000, 131072):
        for kind in ("uniform", "all255"):
            a, b = inputs.pair_digits(0xD15F + n, np.arange(2), n, kind)
            d = oracle.disc_mul(a, b)
            r = oracle.ivmul(a, b)
            out.append({"n": n, "kind": kind, "disc_max_radius": float(d["max_radius"].max()),
                        "rect_max_radius": float(r["max_radius"].max()),
                        "disc_over_rect": float(d["max_radius"].max() / r["max_radius"].max()),
                        "disc_certified": bool(d["cert"].all()), "rect_certified": bool(r["cert"].all())})
            print(out[-1], flush=True)
    return {"oracle_radii": out, "note": "oracle/ivm_oracle.c (rectangles) vs oracle/ivm_oracle_disc.c (discs), "
                                         "the paper's radix-2 FFT in both; 2 pairs per row"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = cpu() if args.oracle else gpu(args)
    out = args.out or os.path.join(ROOT, "gpurun_out", "disc_oracle.json" if args.oracle else "disc.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
