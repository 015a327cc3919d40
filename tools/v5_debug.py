import numpy as np, sys
sys.path.insert(0, '.')
import torch
import paper_1006_0405_b200 as ivm
import oracle
from paper_1006_0405_b200 import inputs
ctx = ivm.Context(0)
for n in [40000]:
    a, b = inputs.pair_digits(7 + n, np.arange(3), n, np.array([0, 1, 2]))
    r = ctx.multiply_diag(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), dump_pairs=[1])
    torch.cuda.synchronize()
    co = r["coeffs"].cpu().numpy()
    ex = oracle.coefficients(a[1:2], b[1:2])[0]
    bad = np.nonzero(co[1] != ex)[0]
    print("n", n, "bad coeff count", len(bad), bad[:20], "cert", r["cert"].cpu().numpy())
    if len(bad):
        print("gpu", co[1][bad[:5]], "exact", ex[bad[:5]])
    iv = r["intervals"].cpu().numpy()[0]
    print("intervals at bad", iv[bad[:5]])
    prod = r["prod"].cpu().numpy()[1]
    want = oracle.long_multiply(a[1:2], b[1:2])[0]
    d = np.nonzero(prod != want)[0]
    print("digit diffs", len(d), d[:10], prod[d[:6]], want[d[:6]])
