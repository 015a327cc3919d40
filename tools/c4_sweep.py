"""C4 report (BASELINE.json configs[3]): fp32 interval precision-limit sweep.

For every C4 size (32, 64, 96, 120, 160, 256 digits; 1,024 pairs, half uniform,
half all-255) this runs the GPU path (fp32 interval FFT) and the oracle (the
paper's fp32 interval SS, plain C on the host) on ALL pairs and reports the
certified fraction per class side by side, the GPU/oracle flag agreement, the
max radii, and the GPU throughput.  Certified GPU products are checked
bit-exact against long multiplication.

    python tools/c4_sweep.py [--out profiles/r01/c4_sweep.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import oracle
    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import inputs
    ctx = ivm.Context(0)
    rows = []
    for n in inputs.CONFIGS["C4"][0]:
        a, b, kinds = inputs.config_inputs("C4", n=n)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        r = ctx.multiply_diag(ta, tb, prec=ivm.F32)
        torch.cuda.synchronize()
        cert = r["cert"].cpu().numpy().astype(bool)
        rad = r["max_radius"].cpu().numpy()
        prod = r["prod"].cpu().numpy()
        want = oracle.long_multiply(a, b)
        wrong = int(sum(1 for p in range(len(a)) if cert[p] and not np.array_equal(prod[p], want[p])))
        t0 = time.time()
        o = oracle.ivmul(a, b, prec="f32")
        t_oracle = time.time() - t0
        ocert = o["cert"].astype(bool)
        # device time per batch (CUDA events, warm)
        out = torch.empty((len(a), 2 * n), dtype=torch.uint8, device="cuda")
        cf = torch.empty((len(a),), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            ctx.multiply(ta, tb, prec=ivm.F32, out=out, cert=cf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            ctx.multiply(ta, tb, prec=ivm.F32, out=out, cert=cf)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        row = {"n": n, "m": ivm.fft_length(n), "pairs": int(len(a))}
        for name, k in (("uniform", 0), ("all255", 1)):
            sel = kinds == k
            row[f"gpu_certified_{name}"] = float(cert[sel].mean())
            row[f"oracle_certified_{name}"] = float(ocert[sel].mean())
            row[f"gpu_max_radius_{name}"] = float(np.max(rad[sel]))
            row[f"oracle_max_radius_{name}"] = float(np.max(o["max_radius"][sel]))
        margin = ocert & (o["max_radius"] < 0.25)
        row["flag_agreement"] = float((cert == ocert).mean())
        row["oracle_margin_pairs_not_certified_by_gpu"] = int((margin & ~cert).sum())
        row["gpu_certified_but_wrong"] = wrong
        row["gpu_ms_per_batch"] = ms
        row["gpu_certified_digits_per_s"] = float(cert.sum() * n / (ms / 1e3))
        row["oracle_s_per_batch"] = t_oracle
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"config": "C4", "precision": "fp32 rectangular complex intervals", "rows": rows}, f,
                      indent=1)


if __name__ == "__main__":
    main()
