#!/usr/bin/env python3
"""Summarise one kernel of an `ncu --set full --import-source on` report for
profiles/<round>/: SOL and pipe counters, warp-stall reasons per issue, and the
executed SASS instruction mix (FP64 share), read with `ncu -i ... --page raw /
--page source --csv`.

    python tools/ncu_summary.py gpurun_out/c2_full_r02.ncu-rep > profiles/r02/ncu_full_c2_summary.txt
"""
import collections
import csv
import io
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    raw = ncu_csv(rep, "--page", "raw")
    d = dict(zip(raw[0], raw[2]))
    print(f"report: {rep}")
    print(f"kernel: {d.get('Kernel Name')}  grid {d.get('launch__grid_size')} block {d.get('launch__block_size')}  "
          f"registers {d.get('launch__registers_per_thread')}")
    keys = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
            "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k]}")
    print("warp stalls per issued instruction:")
    st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
          for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("ratio")}
    for k, v in sorted(st.items(), key=lambda x: -x[1]):
        if v >= 0.01:
            print(f"  {k:22s} {v:.3f}")
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hdr, data = src[1], src[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    E, S = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
    ops, samp = collections.Counter(), collections.Counter()
    for r in data:
        tok = r[ix["Source"]].strip().split()
        op = (tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]
        ops[op] += int(r[E])
        samp[op] += int(r[S])
    te, ts = sum(ops.values()), sum(samp.values())
    fp = sum(ops[o] for o in ("DADD", "DMUL", "DFMA"))
    print(f"executed warp instructions {te}, FP64 share {100 * fp / te:.1f} %, SASS instructions {len(data)}")
    for op, c in ops.most_common(16):
        print(f"  {op:8s} exec {100 * c / te:5.1f} %  stall samples {100 * samp[op] / ts:5.1f} %")


if __name__ == "__main__":
    main()
