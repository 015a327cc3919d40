import sys, time, torch
sys.path.insert(0, '.')
import paper_1006_0405_b200 as ivm
ctx = ivm.Context(0)
n, B = 4096, 4096
a = ctx.generate_digits(n, B, 1, 0).cpu().pin_memory(); b = ctx.generate_digits(n, B, 1, 1).cpu().pin_memory()
out = torch.empty((B, 2 * n), dtype=torch.uint8, pin_memory=True); cert = torch.empty((B,), dtype=torch.uint8, pin_memory=True)
for _ in range(3): ctx.multiply_host(a, b, out=out, cert=cert)
s = torch.cuda.current_stream()
for rep in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s); ctx.multiply_host(a, b, out=out, cert=cert); e1.record(s); torch.cuda.synchronize()
    print("e2e ms", round(e0.elapsed_time(e1), 4), "Gdig/s", round(B * n / e0.elapsed_time(e1) / 1e6, 2))
# pure copy bandwidth
x = torch.empty(33554432, dtype=torch.uint8, pin_memory=True); d = torch.empty(33554432, dtype=torch.uint8, device="cuda")
for _ in range(2): d.copy_(x, non_blocking=True); torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("H2D GB/s", round(33554432 / e0.elapsed_time(e1) / 1e6, 1))
e0.record(); x.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("D2H GB/s", round(33554432 / e0.elapsed_time(e1) / 1e6, 1))
