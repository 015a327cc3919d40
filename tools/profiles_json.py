"""Dev tool: turn the CSVs written by tools/ncu_metrics.sh (gpurun_out/metrics_<cfg>.csv)
into the committed summaries bench.py reads: profiles/<round>/ncu_counters.json
(SURVEY §8(d.4) counters) and the DRAM-traffic entries of ncu_traffic.json.

    python tools/profiles_json.py [--round r01] [--src gpurun_out]
"""
import argparse
import csv
import json
import math
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIG = {"C1": (1000, 1), "C2": (4096, 4096), "C3": (75000, 64), "C5": (16384, 65536)}


def W_ops(m):
    L = int(math.log2(m))
    return 24 * m * L - 28 * m + 48


def read(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    if not rows:
        return None
    kernel = rows[0][4]
    v = {r[12]: r[14].replace(",", "") for r in rows if r[4] == kernel and r[0] == rows[0][0]}
    return kernel, {k: float(x) for k, x in v.items() if x.replace(".", "", 1).isdigit()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    out_dir = os.path.join(ROOT, "profiles", args.round)
    cpath, tpath = os.path.join(out_dir, "ncu_counters.json"), os.path.join(out_dir, "ncu_traffic.json")
    counters = json.load(open(cpath)) if os.path.exists(cpath) else {}
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for cfg, (n, batch) in CONFIG.items():
        f = os.path.join(args.src, f"metrics_{cfg}.csv")
        if not os.path.exists(f):
            continue
        got = read(f)
        if not got:
            continue
        kernel, v = got
        m = 1 << max(1, (2 * n - 1 - 1).bit_length())
        fp64 = (v.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
                + v.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
                + v.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0))
        dram = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
        counters[cfg] = {
            "kernel": kernel, "batch": batch, "fft_length": m,
            "executed_fp64_thread_ops_per_mult": fp64 / batch,
            "credited_W_per_mult": W_ops(m),
            "executed_over_W": fp64 / batch / W_ops(m),
            "fp64_pipe_active_pct": v.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": v.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "dram_bytes": dram,
            "dram_throughput_pct": v.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_bytes": v.get("lts__t_bytes.sum"),
            "smem_wavefronts": v.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "registers_per_thread": v.get("launch__registers_per_thread"),
            "warps_active_pct": v.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "grid": v.get("launch__grid_size"), "block": v.get("launch__block_size"),
            "time_ns": v.get("gpu__time_duration.sum"),
            "source": f"tools/ncu_metrics.sh (ncu --metrics ..., one launch of bench.py --config {cfg})",
        }
        t = traffic.get(cfg, {})
        t.update({"kernel": kernel.replace("void ", "").replace("(KParams)", "").replace("(KParams, Group5)", ""),
                  "capture": f"tools/ncu_metrics.sh: ncu --metrics ... -c 1 --launch-skip 3, python bench.py --config {cfg} "
                             f"--steps 1 --warmup 3 (profiles/{args.round}/metrics_{cfg}.csv)",
                  "dram_bytes_read": int(v.get("dram__bytes_read.sum", 0)),
                  "dram_bytes_write": int(v.get("dram__bytes_write.sum", 0)),
                  "dram_bytes_per_launch": int(dram)})
        traffic[cfg] = t
        print(cfg, kernel, f"{v.get('gpu__time_duration.sum', 0) / 1e3:.1f} us", f"dram {dram / 1e6:.1f} MB")
    json.dump(counters, open(cpath, "w"), indent=1)
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
