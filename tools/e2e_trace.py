"""Timeline of the chunked host pipeline (dev tool): the same copy-in /
multiply / copy-out chunks as ivm_multiply_batched_host, issued from Python
with torch streams and timed with events, so the overlap of the two copy
directions and the kernels can be read per chunk.

    python tools/e2e_trace.py [--chunks 8] [--order inputs_first|interleaved]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=8)
    ap.add_argument("--order", default="inputs_first")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=4096)
    args = ap.parse_args()
    import torch
    import paper_1006_0405_b200 as ivm
    ctx = ivm.Context(0)
    n, B = args.n, args.batch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    chunk = -(-B // args.chunks)
    chunk = -(-chunk // sms) * sms
    a = ctx.generate_digits(n, B, 1, 0).cpu().pin_memory()
    b = ctx.generate_digits(n, B, 1, 1).cpu().pin_memory()
    out = torch.empty((B, 2 * n), dtype=torch.uint8, pin_memory=True)
    da, db = torch.empty((B, n), dtype=torch.uint8, device="cuda"), torch.empty((B, n), dtype=torch.uint8, device="cuda")
    dp = torch.empty((B, 2 * n), dtype=torch.uint8, device="cuda")
    dc = torch.empty((B,), dtype=torch.uint8, device="cuda")
    s_in, s_out, s = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()
    ranges = [(p0, min(B, p0 + chunk)) for p0 in range(0, B, chunk)]

    def run(trace):
        ev = lambda: torch.cuda.Event(enable_timing=True)
        t0 = ev()
        t0.record(s)
        s_in.wait_stream(s)
        marks = []
        ins = []
        if args.order == "inputs_first":
            for p0, p1 in ranges:
                with torch.cuda.stream(s_in):
                    e_a = ev(); e_a.record(s_in)
                    da[p0:p1].copy_(a[p0:p1], non_blocking=True)
                    db[p0:p1].copy_(b[p0:p1], non_blocking=True)
                    e_b = ev(); e_b.record(s_in)
                ins.append((e_a, e_b))
        for k, (p0, p1) in enumerate(ranges):
            if args.order != "inputs_first":
                with torch.cuda.stream(s_in):
                    e_a = ev(); e_a.record(s_in)
                    da[p0:p1].copy_(a[p0:p1], non_blocking=True)
                    db[p0:p1].copy_(b[p0:p1], non_blocking=True)
                    e_b = ev(); e_b.record(s_in)
                ins.append((e_a, e_b))
            s.wait_event(ins[k][1])
            k0 = ev(); k0.record(s)
            ctx.multiply(da[p0:p1], db[p0:p1], out=dp[p0:p1], cert=dc[p0:p1])
            k1 = ev(); k1.record(s)
            s_out.wait_event(k1)
            with torch.cuda.stream(s_out):
                o0 = ev(); o0.record(s_out)
                out[p0:p1].copy_(dp[p0:p1], non_blocking=True)
                o1 = ev(); o1.record(s_out)
            marks.append((k0, k1, o0, o1))
        s.wait_stream(s_out)
        t1 = ev()
        t1.record(s)
        torch.cuda.synchronize()
        if trace:
            for k, ((i0, i1), (k0, k1, o0, o1)) in enumerate(zip(ins, marks)):
                f = lambda e: t0.elapsed_time(e)
                print(f"chunk {k}: in {f(i0):7.3f}-{f(i1):7.3f}  kernel {f(k0):7.3f}-{f(k1):7.3f}  "
                      f"out {f(o0):7.3f}-{f(o1):7.3f} ms")
        return t0.elapsed_time(t1)

    for _ in range(3):
        run(False)
    ts = [run(False) for _ in range(5)]
    print("total ms", [round(t, 3) for t in ts], "Gdig/s", round(B * n / (min(ts) / 1e3) / 1e9, 2))
    run(True)


if __name__ == "__main__":
    main()
