import numpy as np, sys, time
sys.path.insert(0, '.')
import torch
import paper_1006_0405_b200 as ivm
import oracle
from paper_1006_0405_b200 import inputs
ctx = ivm.Context(0)
for n in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['4097', '8193', '20000'])]:
    a, b = inputs.pair_digits(7 + n, np.arange(3), n, np.array([0, 1, 2]))
    out, cert = ctx.multiply(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    want = oracle.long_multiply(a, b)
    o = out.cpu().numpy(); c = cert.cpu().numpy()
    print(n, "cert", c, "exact", [bool(np.array_equal(o[p], want[p])) for p in range(3)],
          "first diff", [int(np.argmax(o[p] != want[p])) if not np.array_equal(o[p], want[p]) else -1 for p in range(3)], flush=True)
