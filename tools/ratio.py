import numpy as np, torch, os, sys
sys.path.insert(0, '/root/repo')
import oracle, paper_1006_0405_b200 as ivm
from paper_1006_0405_b200 import inputs
ctx = ivm.Context(0)
for n in [17, 100, 300, 513, 1000, 2000, 4096]:
    kinds = np.array([0, 1, 2, 0])
    a, b = inputs.pair_digits(77 + n, np.arange(4), n, kinds)
    r = ctx.multiply_diag(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), coeffs=False)
    torch.cuda.synchronize()
    g = r["max_radius"].cpu().numpy()
    o = oracle.ivmul(a, b)["max_radius"]
    print(os.environ.get("IVM_KERNEL", "v3"), n, ivm.fft_length(n), np.round(g / o, 3))
