import numpy as np, sys, torch
sys.path.insert(0, '.')
import paper_1006_0405_b200 as ivm
from paper_1006_0405_b200 import inputs
ctx = ivm.Context(0)
for n in [100000, 131072]:
    a, b = inputs.pair_digits(0x77 + n, np.arange(3), n, np.array([0, 1, 2]))
    r = ctx.multiply_diag(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    print(n, "cert", r["cert"].cpu().numpy(), "maxrad", r["max_radius"].cpu().numpy(), flush=True)
