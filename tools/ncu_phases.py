"""Dev tool: per-phase stall / instruction breakdown of one kernel in an ncu report.

    python tools/ncu_phases.py report.ncu-rep [kernel-substring]

Phases are delimited by CTA barriers (BAR.SYNC); prints, per phase, the share of
warp-stall samples (~ time) and of executed warp instructions, plus the top
stall reasons, and the instruction mix of the whole kernel."""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kname = sys.argv[2] if len(sys.argv) > 2 else None
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kname:
        cmd += ["-k", "regex:" + kname]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[1]
    rows = [x for x in r[2:] if len(x) == len(h)]
    src, ie, st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    ts = sum(int(x[st]) for x in rows) or 1
    te = sum(int(x[ie]) for x in rows) or 1
    print(f"total warp instrs {te}, stall samples {ts}")
    ops = collections.Counter()
    for x in rows:
        t = x[src].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += int(x[ie])
    print("mix:", ", ".join(f"{k} {100 * v / te:.1f}" for k, v in ops.most_common(16)))
    fp64 = sum(v for k, v in ops.items() if k in ("DADD", "DMUL", "DFMA"))
    print(f"FP64 share {100 * fp64 / te:.1f}%")
    start = 0
    phases = []
    for i, x in enumerate(rows):
        if "BAR.SYNC" in x[src] or i == len(rows) - 1:
            phases.append((start, i + 1))
            start = i + 1
    print(f"{'phase':>11} {'time%':>6} {'exec%':>6}  top stalls")
    for a, b in phases:
        s = sum(int(x[st]) for x in rows[a:b])
        e = sum(int(x[ie]) for x in rows[a:b])
        if s / ts < 0.01 and e / te < 0.01:
            continue
        red = sorted(((sum(int(x[h.index(k)]) for x in rows[a:b]), k) for k in keys), reverse=True)[:4]
        print(f"{a:5d}-{b:5d} {100 * s / ts:6.1f} {100 * e / te:6.1f}  " +
              ", ".join(f"{k[6:]} {100 * v / ts:.1f}" for v, k in red))


if __name__ == "__main__":
    main()
