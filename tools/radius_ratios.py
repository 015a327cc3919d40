#!/usr/bin/env python3
"""GPU / oracle max-radius ratio distributions per config.

For every pair of C1, C2, C3 and C5 (C5: all 65,536 pairs unless --c5-pairs),
the GPU's max coefficient radius (ivm_multiply_batched_diag) is divided by the
oracle's (oracle.ivmul, R10), and the distribution is written per
digit kind.  The north-star bar is ratio <= 2 for every pair.

    python tools/radius_ratios.py [--out profiles/r02/radius_ratios.json] [--c5-pairs N]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1006_0405_b200 import inputs  # noqa: E402

KIND_NAMES = {0: "uniform", 1: "all255", 2: "sparse", 3: "uniform_msd"}


def summarize(ratio, gpu, ora):
    q = np.quantile(ratio, [0, 0.5, 0.9, 0.99, 1.0])
    return {"pairs": int(len(ratio)), "ratio_min": float(q[0]), "ratio_p50": float(q[1]),
            "ratio_p90": float(q[2]), "ratio_p99": float(q[3]), "ratio_max": float(q[4]),
            "gpu_max_radius": float(gpu.max()), "oracle_max_radius": float(ora.max()),
            "pairs_over_2x": int((ratio > 2).sum()), "pairs_over_1x": int((ratio > 1).sum())}


def run_config(ctx, name, pairs=None, chunk=4096):
    import torch
    import paper_1006_0405_b200 as ivm
    n, B = {"C1": (1000, 1), "C2": (4096, 4096), "C3": (75000, 64), "C5": (16384, 65536)}[name]
    if pairs is None:
        pairs = np.arange(B)
    kinds_all = inputs.class_of_pairs(name, B) if name in ("C3", "C5") else np.full(B, 3 if name == "C1" else 0)
    seed = inputs.config_seed(int(name[1:]))
    g_rad, o_rad, o_cert, g_cert = [], [], [], []
    t_gpu = t_ora = 0.0
    for i0 in range(0, len(pairs), chunk):
        pp = pairs[i0:i0 + chunk]
        kinds = kinds_all[pp]
        a, b = inputs.pair_digits(seed, pp, n, kinds)
        t0 = time.perf_counter()
        r = ctx.multiply_diag(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), prec=ivm.F64, coeffs=False)
        torch.cuda.synchronize()
        t_gpu += time.perf_counter() - t0
        g_rad.append(r["max_radius"].cpu().numpy())
        g_cert.append(r["cert"].cpu().numpy().astype(bool))
        t0 = time.perf_counter()
        o = oracle.ivmul(a, b)
        t_ora += time.perf_counter() - t0
        o_rad.append(o["max_radius"])
        o_cert.append(o["cert"])
    g, o = np.concatenate(g_rad), np.concatenate(o_rad)
    gc, oc = np.concatenate(g_cert), np.concatenate(o_cert)
    ratio = g / o
    kinds = kinds_all[pairs]
    out = {"n": n, "pairs": int(len(pairs)), "of": B, "gpu_certified": int(gc.sum()), "oracle_certified": int(oc.sum()),
           "all": summarize(ratio, g, o), "oracle_seconds": round(t_ora, 2), "gpu_seconds": round(t_gpu, 2)}
    for k in np.unique(kinds):
        sel = kinds == k
        out[KIND_NAMES[int(k)]] = summarize(ratio[sel], g[sel], o[sel])
    # histogram of the ratio over [0, 2] in 0.05 bins
    h, edges = np.histogram(ratio, bins=40, range=(0, 2))
    out["histogram"] = {"bin_edges_start": 0.0, "bin_width": 0.05, "counts": h.tolist(),
                        "above_2": int((ratio > 2).sum())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "radius_ratios.json"))
    ap.add_argument("--c5-pairs", type=int, default=65536)
    ap.add_argument("--configs", default="C1,C2,C3,C5")
    args = ap.parse_args()
    import paper_1006_0405_b200 as ivm
    ctx = ivm.Context(0)
    res = {"about": "GPU max radius / oracle max radius per pair (DESIGN.md R10); north-star bar: <= 2",
           "oracle_threads": oracle.max_threads(), "library": ivm.lib().ivm_version().decode()}
    for name in args.configs.split(","):
        pairs = None
        if name == "C5" and args.c5_pairs < 65536:
            pairs = np.linspace(0, 65535, args.c5_pairs).astype(np.int64)
        res[name] = run_config(ctx, name, pairs)
        a = res[name]["all"]
        print(f"{name}: pairs {res[name]['pairs']} ratio p50 {a['ratio_p50']:.3f} max {a['ratio_max']:.3f} "
              f"over2 {a['pairs_over_2x']} ({res[name]['oracle_seconds']} s oracle)", flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
