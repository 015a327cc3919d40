"""The seeded digit generator (paper_1006_0405_b200/inputs.py) and its device
twin (ivm_generate_digits): determinism, distributions, bit equality."""
import numpy as np
import pytest

from paper_1006_0405_b200 import inputs


def test_deterministic_and_seed_sensitive():
    a1 = inputs.digits(1, np.arange(4), 0, 100, "uniform")
    a2 = inputs.digits(1, np.arange(4), 0, 100, "uniform")
    a3 = inputs.digits(2, np.arange(4), 0, 100, "uniform")
    assert np.array_equal(a1, a2) and not np.array_equal(a1, a3)
    b = inputs.digits(1, np.arange(4), 1, 100, "uniform")
    assert not np.array_equal(a1, b)


def test_distributions():
    u = inputs.digits(7, np.arange(64), 0, 4096, "uniform")
    assert abs(u.mean() - 127.5) < 1.0
    assert set(np.unique(inputs.digits(7, np.arange(4), 0, 50, "all255"))) == {255}
    s = inputs.digits(7, np.arange(64), 0, 4096, "sparse")
    frac0 = (s == 0).mean()
    assert 0.89 < frac0 < 0.91
    m = inputs.digits(7, np.arange(5000), 0, 3, "msd")
    assert (m[:, -1] != 0).all()


def test_config_classes():
    k = inputs.class_of_pairs("C5", 9)
    assert k.tolist() == [0, 1, 2] * 3
    k3 = inputs.class_of_pairs("C3", 64)
    assert (k3[:32] == 0).all() and (k3[32:] == 1).all()
    a, b, kinds = inputs.config_inputs("C1")
    assert a.shape == (1, 1000) and a[0, -1] != 0


@pytest.mark.gpu
def test_device_generator_bit_equal():
    import torch
    import paper_1006_0405_b200 as ivm
    ctx = ivm.Context(0)
    for kind in (0, 1, 2, 3):
        for n in (1, 7, 1000):
            for operand in (0, 1):
                d = ctx.generate_digits(n, 33, seed=0x10060405 + 3, operand=operand, kind=kind, pair0=5)
                torch.cuda.synchronize()
                want = inputs.digits(0x10060405 + 3, np.arange(5, 38), operand, n,
                                     list(inputs.KINDS)[kind])
                assert np.array_equal(d.cpu().numpy(), want), (kind, n, operand)
    kinds = torch.tensor([0, 1, 2] * 4, dtype=torch.uint8, device="cuda")
    d = ctx.generate_digits(64, 12, seed=99, operand=1, kind=kinds)
    want = inputs.digits(99, np.arange(12), 1, 64, np.array([0, 1, 2] * 4))
    assert np.array_equal(d.cpu().numpy(), want)
