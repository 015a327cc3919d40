"""Single-process multi-GPU C API (ivm_multi_*) on the devices
present: shards multiplied independently and gathered to the root in shard
order; identical to the single-context path.  (The box has one GPU, so the
NCCL gather runs with ngpu = 1 -- the root copy path; the per-rank NCCL
launch model is covered by bench.py and tests/test_dist.py.)"""
import ctypes

import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs

pytestmark = pytest.mark.gpu


def test_multi_api_matches_single_context():
    import torch
    import paper_1006_0405_b200 as ivm
    L = ivm.lib()
    ngpu = torch.cuda.device_count()
    devs = (ctypes.c_int * ngpu)(*range(ngpu))
    h = ctypes.c_void_p()
    st = L.ivm_multi_create(ctypes.byref(h), ngpu, devs)
    if st == -5:
        pytest.skip("NCCL not loadable in this process")
    assert st == 0, st
    try:
        n, bpg = 1500, 24
        a, b = inputs.pair_digits(0x3A1, np.arange(ngpu * bpg), n, "uniform")
        ta = [torch.from_numpy(a[g * bpg:(g + 1) * bpg]).to(f"cuda:{g}") for g in range(ngpu)]
        tb = [torch.from_numpy(b[g * bpg:(g + 1) * bpg]).to(f"cuda:{g}") for g in range(ngpu)]
        tp = [torch.empty((bpg, 2 * n), dtype=torch.uint8, device=f"cuda:{g}") for g in range(ngpu)]
        tc = [torch.empty((bpg,), dtype=torch.uint8, device=f"cuda:{g}") for g in range(ngpu)]
        rp = torch.empty((ngpu * bpg, 2 * n), dtype=torch.uint8, device="cuda:0")
        rc = torch.empty((ngpu * bpg,), dtype=torch.uint8, device="cuda:0")
        arr = lambda ts: (ctypes.c_void_p * ngpu)(*[t.data_ptr() for t in ts])
        st = L.ivm_multi_multiply(h, arr(ta), arr(tb), n, bpg, arr(tp), arr(tc), ivm.F64, 1,
                                  ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(rc.data_ptr()))
        assert st == 0, st
        assert rc.cpu().numpy().all()
        assert np.array_equal(rp.cpu().numpy(), oracle.long_multiply(a, b))
        for g in range(ngpu):
            assert np.array_equal(tp[g].cpu().numpy(), rp[g * bpg:(g + 1) * bpg].cpu().numpy())
        # the summary all-reduce: certified pairs summed, max radius maxed
        ctxs = [ivm.Context(g) for g in range(ngpu)]
        rads = [ctxs[g].multiply_diag(ta[g], tb[g], coeffs=False)["max_radius"] for g in range(ngpu)]
        torch.cuda.synchronize()
        tot, mr = ctypes.c_uint64(), ctypes.c_double()
        st = L.ivm_multi_summary(h, arr(tc), arr(rads), bpg, ctypes.byref(tot), ctypes.byref(mr))
        assert st == 0, st
        assert tot.value == ngpu * bpg
        assert mr.value == max(float(r.max().item()) for r in rads) and mr.value > 0
        tc[0][3] = 0  # one uncertified flag
        st = L.ivm_multi_summary(h, arr(tc), None, bpg, ctypes.byref(tot), ctypes.byref(mr))
        assert st == 0 and tot.value == ngpu * bpg - 1 and np.isnan(mr.value)
    finally:
        assert L.ivm_multi_destroy(h) == 0


def test_multi_api_argument_errors():
    import paper_1006_0405_b200 as ivm
    L = ivm.lib()
    h = ctypes.c_void_p()
    assert L.ivm_multi_create(ctypes.byref(h), 0, None) == -1
    bad = (ctypes.c_int * 1)(999)
    assert L.ivm_multi_create(ctypes.byref(h), 1, bad) == -1
    assert L.ivm_multi_multiply(None, None, None, 4, 1, None, None, 0, 0, None, None) == -1
    assert L.ivm_multi_destroy(None) == 0
