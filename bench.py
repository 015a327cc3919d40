#!/usr/bin/env python3
"""Benchmark: certified base-256 digits multiplied per second (fp64 interval FFT).

Default workload = BASELINE.json configs[1]: a batch of 4,096
independent multiplications of 4,096-digit base-256 integers, uniform digits,
FFT length 8,192, binary64 rectangular complex interval containment sets.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one ivm_multiply_batched call over the whole batch (forward interval
FFTs, pointwise product, inverse FFT, round-and-certify, carry), inputs already
resident in HBM (generated on the device by the seeded generator).  L2 is
flushed (a 256 MiB write) between timed steps, outside the timed events.
Under torchrun every rank multiplies its own batch shard (weak scaling) and
rank 0 prints one JSON line with the max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "certified base-256 digits multiplied/sec (fp64 interval FFT); % of roofline"
UNIT = "digits/s"

CONFIGS = {
    # name: (n, batch, prec, kind (int, or "C3"/"C5" per-pair classes), workload text)
    "C1": (1000, 1, "f64", 3, "C1: one multiplication of two 1,000-digit base-256 integers, fp64, m=2048"),
    "C2": (4096, 4096, "f64", 0, "C2: 4,096 multiplications of 4,096-digit base-256 integers, uniform digits, fp64 intervals, m=8,192"),
    "C3": (75000, 64, "f64", "C3", "C3: 64 multiplications of 75,000-digit base-256 integers (the paper's limit), half uniform / half all-255, fp64, m=262,144"),
    "C5": (16384, 65536, "f64", "C5", "C5: 65,536 multiplications of 16,384-digit integers, 1/3 uniform, 1/3 all-255, 1/3 sparse, fp64, m=32,768; batch sharded across ranks"),
}
# per-rank batch: C5's batch is the whole job (strong scaling); the others are per rank (weak)
STRONG = {"C5"}


def W_ops(m: int) -> int:
    """nominal directed FP64 ops of the paper's radix-2
    algorithm per multiplication, W(m) = 24 m log2 m - 28 m + 48."""
    L = int(math.log2(m))
    return 24 * m * L - 28 * m + 48


def load_profile(config: str):
    """The committed ncu record of this config's dominant kernel (latest round
    under profiles/), else None."""
    try:
        rounds = sorted(d for d in os.listdir(os.path.join(ROOT, "profiles")) if d.startswith("r"))
        for r in reversed(rounds):
            f = os.path.join(ROOT, "profiles", r, "ncu_traffic.json")
            if os.path.exists(f):
                t = json.load(open(f)).get(config)
                if t:
                    return dict(t, file=f"profiles/{r}/ncu_traffic.json")
    except Exception:
        pass
    return None


def load_counters(config: str):
    """SURVEY §8(d.4) ncu counters of this config's dominant kernel (committed)."""
    try:
        rounds = sorted(d for d in os.listdir(os.path.join(ROOT, "profiles")) if d.startswith("r"))
        for r in reversed(rounds):
            f = os.path.join(ROOT, "profiles", r, "ncu_counters.json")
            if os.path.exists(f):
                t = json.load(open(f)).get(config)
                if t:
                    return dict(t, file=f"profiles/{r}/ncu_counters.json")
    except Exception:
        pass
    return None


def load_traffic(config: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    t = load_profile(config)
    return t["dram_bytes_per_launch"] if t else None


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML,
    every 10 ms; falls back to nvidia-smi)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for k, bit in self.REASONS.items():
            if r & bit:
                self.reasons.add(k)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                              "clocks_event_reasons.hw_thermal_slowdown,"
                              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if out:
            f = [x.strip() for x in out.split(",")]
            self.sm.append(float(f[0]))
            self.mx.append(float(f[1]))
            for k, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], f[2:]):
                if v.lower() == "active":
                    self.reasons.add(k)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.01 if self._nvml else 0.1)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.sm:
            return None
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(a, b, n, prec, budget_s=12.0):
    """The oracle as it stands (oracle/, plain C, OpenMP over pairs) on the host
    cores, on a bounded sample of the same workload."""
    import numpy as np
    import oracle
    cores = oracle.max_threads()
    B = a.shape[0]
    oracle.ivmul(a[:1], b[:1], prec=prec)  # builds the twiddle table (mpmath) outside the timing
    k = min(B, max(cores, 1))
    t0 = time.perf_counter()
    r = oracle.ivmul(a[:k], b[:k], prec=prec)
    dt = time.perf_counter() - t0
    per = dt / k
    k2 = int(min(B, max(k, budget_s / max(per, 1e-9))))
    if k2 > k:
        t0 = time.perf_counter()
        r = oracle.ivmul(a[:k2], b[:k2], prec=prec)
        dt = time.perf_counter() - t0
        k = k2
    certified = int(np.asarray(r["cert"]).sum())
    return {"value": certified * n / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"first {k} of {B} pairs of the same workload ({certified} certified), {dt:.2f} s wall"}


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    import numpy as np
    from paper_1006_0405_b200 import inputs
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n, batch, prec, kind, text = CONFIGS[args.config]
    import oracle
    cores = oracle.max_threads()
    k = max(cores, 8) if n < 20000 else max(2, cores // 4)
    pairs = np.arange(k)
    kinds = inputs.class_of_pairs(args.config, batch)[:k] if isinstance(kind, str) else np.full(k, kind)
    a, b = inputs.pair_digits(inputs.config_seed(int(args.config[1:])), pairs, n, kinds)
    for _ in range(args.warmup):
        oracle.ivmul(a[:cores], b[:cores], prec=prec)
    times, cert = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = oracle.ivmul(a, b, prec=prec)
        times.append(time.perf_counter() - t0)
        cert = int(r["cert"].sum())
    dt = sum(times) / len(times)
    value = cert * n / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.config in STRONG else "weak",
            "vs_baseline": None, "dtype": prec, "data": "synthetic (seeded SplitMix64 digits)",
            "impl": "reference",
            "config": {"workload": text, "n": n, "batch": batch, "fft_length": 1 << math.ceil(math.log2(2 * n - 1)),
                       "step_sample": f"{k} pairs per step (bounded sample of the {batch}-pair batch)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"{k} of {batch} pairs per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def time_config(ctx, cfg, steps, flush, dev):
    """Device time of one other config on this rank (N = 1 runs): the same
    protocol as the main measurement (inputs resident, L2 flushed outside the
    events, warm-up first); returns its summary for the line's other_configs.
    "<cfg>-disc": the same workload with circular containment sets (P:290,
    ivm_multiply_disc) instead of the rectangular ones."""
    import numpy as np
    import torch
    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import inputs
    disc = cfg.endswith("-disc")
    cfg = cfg[:-5] if disc else cfg
    n, batch, prec_s, kind, _ = CONFIGS[cfg]
    seed = inputs.config_seed(int(cfg[1:]))
    if isinstance(kind, str):
        kind = torch.from_numpy(inputs.class_of_pairs(kind, batch).astype(np.uint8)).to(dev)
    a = ctx.generate_digits(n, batch, seed, 0, kind=kind)
    b = ctx.generate_digits(n, batch, seed, 1, kind=kind)
    out = torch.empty((batch, 2 * n), dtype=torch.uint8, device=dev)
    cert = torch.empty((batch,), dtype=torch.uint8, device=dev)
    if disc:
        mul = lambda: ctx.multiply_disc(a, b, out=out, cert=cert, want_radius=False)
    else:
        mul = lambda: ctx.multiply(a, b, out=out, cert=cert)
    for _ in range(3):
        mul()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ms = []
    sampler = ClockSampler(dev.index if dev.index is not None else 0)
    sampler.start()
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        mul()
        e1.record(s)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    t = sum(ms) / len(ms)
    ncert = int(cert.sum().item())
    m = ivm.fft_length(n)
    peaks = load_peaks()
    peak_ops = 148 * 64 * peaks.get("sm_max_mhz", 1965.0) * 1e6
    r = {"workload": CONFIGS[cfg][4] + (" -- circular containment sets (P:290)" if disc else ""), "ms_per_step": t, "steps": steps, "value": ncert * n / (t / 1e3),
         "unit": UNIT, "certified_pairs": ncert, "batch": batch,
         "roofline_frac": W_ops(m) * batch / (t / 1e3) / peak_ops, "gpu_launches_per_step": ctx.last_launch_count,
         "clocks": clocks}
    del a, b, out, cert
    torch.cuda.empty_cache()
    return r


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1006_0405_b200 as ivm
    from paper_1006_0405_b200 import dist as ivd
    from paper_1006_0405_b200 import inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world} ranks were launched")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    n, batch, prec_s, kind, text = CONFIGS[args.config]
    prec = ivm.F64 if prec_s == "f64" else ivm.F32
    m = ivm.fft_length(n)
    seed = inputs.config_seed(int(args.config[1:]))
    ctx = ivm.Context(local)
    s = torch.cuda.current_stream()
    if args.config in STRONG:  # the whole job's batch is sharded across ranks
        pair0, batch = ivd.shard(batch, rank, world)
    else:  # weak scaling: each rank its own batch
        pair0 = rank * batch
    if isinstance(kind, str):
        kinds_np = inputs.class_of_pairs(kind, CONFIGS[kind][1])[pair0:pair0 + batch].astype(np.uint8)
        kind = torch.from_numpy(kinds_np).to(dev)
    a = ctx.generate_digits(n, batch, seed, 0, kind=kind, pair0=pair0)
    b = ctx.generate_digits(n, batch, seed, 1, kind=kind, pair0=pair0)
    out = torch.empty((batch, 2 * n), dtype=torch.uint8, device=dev)
    cert = torch.empty((batch,), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ctx.reserve(n, batch, prec)
    for _ in range(max(args.warmup, 0)):
        ctx.multiply(a, b, prec=prec, out=out, cert=cert)
    torch.cuda.synchronize()
    launches_per_step = ctx.last_launch_count
    sampler = ClockSampler(local)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(s)
        ctx.multiply(a, b, prec=prec, out=out, cert=cert)
        evs[i][1].record(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    tot_ms = sum(step_ms)
    ncert = int(cert.sum().item())
    tot_ms = ivd.max_over_ranks(tot_ms, device=dev)
    total_cert = ivd.sum_over_ranks(ncert, device=dev)
    gather = None
    if args.gather:
        # the same step with the products and flags gathered to rank 0, chunk k's
        # NCCL sends overlapping chunk k+1's multiplication (dist.multiply_gather)
        # the job: world x the per-rank batch (weak scaling), C5's whole batch (strong)
        job_batch = batch * world if args.config not in STRONG else CONFIGS[args.config][1]
        root_p = torch.empty((job_batch, 2 * n), dtype=torch.uint8, device=dev) if rank == 0 else None
        root_c = torch.empty((job_batch,), dtype=torch.uint8, device=dev) if rank == 0 else None

        def compute(lo, cnt):
            ctx.multiply(a[lo:lo + cnt], b[lo:lo + cnt], prec=prec, out=out[lo:lo + cnt], cert=cert[lo:lo + cnt])

        for _ in range(max(args.warmup, 1)):
            ivd.multiply_gather(compute, out, cert, job_batch, chunks=args.gather_chunks, out_prod=root_p,
                                out_cert=root_c)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        gms = []
        for _ in range(args.steps):
            flush.zero_()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(s)
            ivd.multiply_gather(compute, out, cert, job_batch, chunks=args.gather_chunks, out_prod=root_p,
                                out_cert=root_c)
            g1.record(s)
            torch.cuda.synchronize()
            gms.append(g0.elapsed_time(g1))
        g_ms = ivd.max_over_ranks(sum(gms) / len(gms), device=dev)
        gcert = int(root_c.sum().item()) if rank == 0 else 0
        gather = {"ms_per_step": g_ms, "value": gcert * n / (g_ms / 1e3) if rank == 0 else None,
                  "chunks": args.gather_chunks, "bytes_to_root_per_step": (2 * n + 1) * job_batch,
                  "method": "per-chunk NCCL isend/irecv to rank 0 overlapped with the next chunk's multiply"}
    ms_per_step = tot_ms / args.steps
    value = total_cert * n / (ms_per_step / 1e3)
    # one step's summary over the ranks: certified pairs (SUM) and, from a
    # diagnostic multiply, the max coefficient radius (MAX) -- one collective
    rad = ctx.multiply_diag(a, b, prec=prec, coeffs=False)["max_radius"]
    summ_cert, summ_rad = ivd.summary_allreduce(cert, rad)

    # ---- the other configs, same protocol, so the driver's run records them too ----
    others = None
    if world == 1 and args.other_configs:
        others = {}
        for cfg in [c for c in args.other_configs.split(",") if c and c != args.config]:
            others[cfg] = time_config(ctx, cfg, max(3, min(args.steps, 10)), flush, dev)

    # ---- end-to-end through the host-pointer C ABI (pinned host buffers) ----
    ha = a.cpu().pin_memory()
    hb = b.cpu().pin_memory()
    hout = torch.empty((batch, 2 * n), dtype=torch.uint8, pin_memory=True)
    hcert = torch.empty((batch,), dtype=torch.uint8, pin_memory=True)
    for _ in range(max(args.warmup, 3)):  # the host path warms up over a few calls (pinned pages, DMA)
        ctx.multiply_host(ha, hb, prec=prec, out=hout, cert=hcert)
    e2e_steps = max(1, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(e2e_steps):
        ctx.multiply_host(ha, hb, prec=prec, out=hout, cert=hcert)
    e1.record(s)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    e2e_ms = ivd.max_over_ranks(e2e_ms, device=dev)
    e2e_cert = int(hcert.sum().item()) * world
    e2e_value = e2e_cert * n / (e2e_ms / 1e3)

    if rank == 0:
        peaks = load_peaks()
        sm_max = peaks.get("sm_max_mhz", 1965.0)
        peak_ops = 148 * 64 * sm_max * 1e6  # directed FP64 instr/s (FMA = 1 op), nominal lanes
        kernel_s = ms_per_step / 1e3
        achieved = W_ops(m) * batch / kernel_s  # rank 0's share; ranks run the same shape
        # measured directed-FMA rate (probe), for context
        probe = None
        try:
            sink = torch.empty(148 * 1024 * 2, dtype=torch.float64, device=dev)
            ctx.peak_probe(0, 64, sink)
            torch.cuda.synchronize()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(s)
            cnt = ctx.peak_probe(0, 2048, sink)
            p1.record(s)
            torch.cuda.synchronize()
            probe = cnt / (p0.elapsed_time(p1) / 1e3)
        except Exception:
            pass
        import numpy as np
        ha_np, hb_np = ha.numpy(), hb.numpy()
        cb = None
        if not args.no_cpu_baseline:
            cb = cpu_baseline(ha_np, hb_np, n, prec_s)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.config in STRONG else "weak", "vs_baseline": None, "dtype": prec_s,
            "data": "synthetic (seeded SplitMix64 digits generated on device)",
            "config": {"workload": text, "n": n, "batch_per_gpu": batch, "fft_length": m,
                       "seed": seed,
                       "parallelism": f"batch-sharded x{world} (no data-path collective)",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "certified_pairs_per_step": total_cert,
                       "summary_allreduce": {"certified_pairs": summ_cert, "max_radius": summ_rad},
                       "with_gather_to_rank0": gather},
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12,
                         "unit": "Top/s (directed FP64 DADD/DMUL/DFMA, FMA = 1 op)",
                         "frac": achieved / peak_ops, "traffic": load_traffic(args.config),
                         "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                         "hw_counters": ({k: load_counters(args.config)[k] for k in
                                          ("kernel", "executed_fp64_thread_ops_per_mult", "credited_W_per_mult",
                                           "executed_over_W", "fp64_pipe_active_pct", "issue_active_pct",
                                           "dram_bytes", "registers_per_thread", "warps_active_pct", "file")
                                          if k in load_counters(args.config)}
                                         if load_counters(args.config) else None),
                         "frac_vs_probe": (achieved / probe) if probe else None,
                         "note": "W credits the paper's full complex FFT; the half-spectrum kernels execute about "
                                 "0.5 W FP64 instructions, so the hardware FP64 pipe is about half as busy as frac (hw_counters)",
                         "work_per_unit": f"W(m) = 24 m log2 m - 28 m + 48 = {W_ops(m)} ops per multiplication (SURVEY.md 8(d.1))",
                         "peak_basis": f"148 SM x 64 FP64 lanes x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz); directed-DFMA probe measured {probe/1e12 if probe else float('nan'):.2f} Top/s",
                         "kernel_ms": ms_per_step},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * n * batch * world,
                    "d2h_bytes_per_step": (2 * n + 1) * batch * world},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "cpu_baseline": cb,
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather", action="store_true",
                    help="also time the step with the products gathered to rank 0 (pipelined NCCL sends)")
    ap.add_argument("--gather-chunks", type=int, default=4)
    ap.add_argument("--other-configs", default="C1,C3,C5,C2-disc,C3-disc,C5-disc",
                    help="at N = 1 also time these configs (same protocol) into the line's other_configs; '' for none")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not started by torchrun: launch the N ranks (one process per GPU) ourselves
        from paper_1006_0405_b200 import dist as ivd
        sys.exit(ivd.spawn(args.gpus, os.path.abspath(__file__), sys.argv[1:]))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
