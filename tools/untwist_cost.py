#!/usr/bin/env python3
"""How much of the odd-frequency kernels' coefficient width is the final untwist
(R13)?  Needs an experiment build of the library with
-DIVM_DUMP_PREROT (tools/untwist_cost.py --build writes ab/libivm_prerot.so),
whose interval dump also carries, in the otherwise-NaN imaginary slots of
coefficients k and k + m/2, the real and imaginary part of the packed value
BEFORE the output-side rotation (scaled by 2/m).

Per config size and digit kind it reports, over the used coefficients:
  rot = max width(c) / max width(pre-rotation part)   (<= sqrt 2: the untwist's factor)
  gpu_over_oracle = GPU max radius / oracle max radius (R10)

    python tools/untwist_cost.py --build        # CPU: compile the experiment library
    IVM_LIB=ab/libivm_prerot.so python tools/untwist_cost.py [--out profiles/r02/untwist_cost.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build():
    import paper_1006_0405_b200.build as b
    b.NVFLAGS = b.NVFLAGS + ["-DIVM_DUMP_PREROT"]
    b.OUT = os.path.join(ROOT, "ab", "libivm_prerot.so")
    b.OBJ = os.path.join(ROOT, "ab", "obj_prerot")
    b.build(force=True)
    import shutil
    shutil.rmtree(b.OBJ, ignore_errors=True)
    print(b.OUT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "untwist_cost.json"))
    args = ap.parse_args()
    if args.build:
        return build()
    import torch
    import oracle
    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import inputs
    assert "prerot" in ivm.LIB_PATH, "run with IVM_LIB=ab/libivm_prerot.so"
    ctx = ivm.Context(0)
    res = {"about": __doc__.split("\n\n")[0]}
    for n in (1000, 2048, 4096, 16384, 75000):
        for kind in ("uniform", "all255"):
            a, b = inputs.pair_digits(0x0D + n, np.arange(2), n, kind)
            r = ctx.multiply_diag(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), dump_pairs=[0, 1],
                                  coeffs=False)
            torch.cuda.synchronize()
            iv = r["intervals"].cpu().numpy()
            m = iv.shape[1]
            o = oracle.ivmul(a, b)
            rows = []
            for p in range(2):
                used = iv[p, :2 * n - 1]
                wc = used[:, 1] - used[:, 0]
                wpre = iv[p, :, 3] - iv[p, :, 2]
                wp = wpre[:2 * n - 1]
                rows.append({"rot": float(wc.max() / wp.max()),
                             "gpu_over_oracle": float(r["max_radius"][p].item() / o["max_radius"][p]),
                             "median_coeff_rot": float(np.median(wc / np.maximum(wp, 1e-300)))})
            res[f"n{n}_{kind}"] = {"m": m, "pairs": rows}
            print(n, kind, rows, flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
