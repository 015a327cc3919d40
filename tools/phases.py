#!/usr/bin/env python3
"""Per-phase cycle breakdown of the hot kernels (experiment build, -DIVM_PHASES).

Thread 0 of every CTA adds the SM cycles since its previous mark to a per-CTA,
per-phase counter (csrc/ivm_phase.cuh); a phase includes the CTA barrier that
ends it.  The product library compiles the marks out.

    python tools/phases.py --build                     # CPU: ab/libivm_phases.so
    IVM_LIB=ab/libivm_phases.so python tools/phases.py --config C3 [--reps 3] [--out f.json]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {
    "v3": ["first pass a", "passes a", "first pass b", "passes b + pointwise + inv0", "inverse passes + emit",
           "cert flush", "carry + store"],
    "v4": ["cross a (+cluster wait)", "passes a", "cross b", "passes b + pointwise + inv0", "inverse local passes",
           "cluster sync 1", "last pass: emit", "cluster sync 3", "cert read", "carry scan",
           "cluster sync 4", "carry emit", "last pass: DSMEM loads + table wait",
           "last pass: twiddles + DFT (load stalls)"],
    "v5": ["cross a", "passes a", "cross b", "passes b + pointwise + inv0", "inverse local passes + xch",
           "group barrier 1", "last pass (L2) + emit", "boundary + group barrier 2", "cert + prev fetch",
           "carry scan", "group barrier 3", "carry emit + tail"],
    "v7": ["L: cross a", "L: passes a", "L: cross b", "L: passes b + pointwise + inv0",
           "L: inverse local passes + xch", "A: wait", "A: last pass (L2) + emit", "A: chunk carry + publish",
           "Cs: wait", "Cs: resolve + digits", "(unused)", "(unused)", "L: ring wait"],
}
KERNEL = {"C1": "v3", "C2": "v3", "C3": "v7" if os.environ.get("IVM_V7", "1") != "0" else "v5", "C5": "v4"}


def build():
    import paper_1006_0405_b200.build as b
    b.NVFLAGS = b.NVFLAGS + ["-DIVM_PHASES"]
    b.OUT = os.path.join(ROOT, "ab", "libivm_phases.so")
    b.OBJ = os.path.join(ROOT, "ab", "obj_phases")
    b.build(force=True)
    print(b.OUT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.build:
        return build()
    import torch
    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import inputs
    sys.path.insert(0, ROOT)
    import bench
    assert "phases" in ivm.LIB_PATH, "run with IVM_LIB=ab/libivm_phases.so"
    L = ivm.lib()
    L.ivm_phases_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    n, batch, _, kind, text = bench.CONFIGS[args.config]
    ctx = ivm.Context(0)
    seed = inputs.config_seed(int(args.config[1:]))
    dev = torch.device("cuda:0")
    if isinstance(kind, str):
        kinds_np = inputs.class_of_pairs(kind, batch).astype(np.uint8)
        kind = torch.from_numpy(kinds_np).to(dev)
    a = ctx.generate_digits(n, batch, seed, 0, kind=kind)
    b = ctx.generate_digits(n, batch, seed, 1, kind=kind)
    out = torch.empty((batch, 2 * n), dtype=torch.uint8, device=dev)
    cert = torch.empty((batch,), dtype=torch.uint8, device=dev)
    ctx.multiply(a, b, out=out, cert=cert)
    buf = np.zeros(2048 * 16, dtype=np.uint64)
    L.ivm_phases_read(buf.ctypes.data, buf.size)  # clears
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.reps):
        ctx.multiply(a, b, out=out, cert=cert)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.reps
    assert int(cert.sum()) == batch
    r = L.ivm_phases_read(buf.ctypes.data, buf.size)
    assert r == 0, r
    ph = buf.reshape(2048, 16).astype(np.float64) / args.reps
    res = {"config": args.config, "workload": text, "ms_per_call": ms, "kernels": {}}
    for part, sl in (("main", slice(0, 1024)), ("corun", slice(1024, 2048))):
        blk = ph[sl]
        used = blk.sum(axis=1) > 0
        if not used.any():
            continue
        blk = blk[used]
        kname = KERNEL[args.config] if part == "main" else "v5"
        names = NAMES[kname]
        tot = blk.sum(axis=1)
        mean = blk.mean(axis=0)
        rows = []
        for k, nm in enumerate(names):
            rows.append({"phase": nm, "mcycles_mean": mean[k] / 1e6, "share": float(mean[k] / tot.mean()),
                         "max_over_ctas": float(blk[:, k].max() / 1e6)})
        res["kernels"][part] = {"kernel": kname, "ctas": int(used.sum()), "mcycles_per_cta_mean": float(tot.mean() / 1e6),
                                "mcycles_per_cta_max": float(tot.max() / 1e6), "phases": rows}
        print(f"{part} ({kname}, {int(used.sum())} CTAs): {tot.mean() / 1e6:.3f} Mcycles/CTA "
              f"(max {tot.max() / 1e6:.3f}); {ms:.3f} ms per call")
        for row in rows:
            print(f"  {row['phase']:<34s} {row['mcycles_mean']:8.4f} Mcyc  {100 * row['share']:5.1f} %")
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
