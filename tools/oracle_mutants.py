#!/usr/bin/env python3
"""Mutation check of the oracle's pins (CPU only).

Copies oracle/, tests/ and the package's Python files into a scratch tree,
applies one mutation at a time to oracle/ivm_oracle.c, rebuilds liboracle.so
there and runs the oracle pins (-m "not gpu").  Every mutation must make at
least one pin fail; the script exits 1 if one survives.

    python tools/oracle_mutants.py
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RAD = "double r = (iv[2 * i + 1] - iv[2 * i]) / 2.0;"
MUTANTS = {
    "radius / 4": (RAD, "double r = (iv[2 * i + 1] - iv[2 * i]) / 4.0;"),
    "width instead of radius": (RAD, "double r = (iv[2 * i + 1] - iv[2 * i]);"),
    "radius rounded down": (RAD, "double r = -((iv[2 * i] - iv[2 * i + 1]) / 2.0);"),
    "imaginary radius dropped": ("for (size_t i = 0; i < 2 * len; i++) {\n        double r",
                                 "for (size_t i = 0; i < 2 * len; i += 2) {\n        double r"),
    "imaginary certify rule dropped": ("int unique = (cl == fh) && (il == 0.0) && (ih == 0.0);",
                                       "int unique = (cl == fh) && (il == il) && (ih == ih);"),
    "certify: floor/ceil swapped": ("double cl = ceil(iv[4 * i]), fh = floor(iv[4 * i + 1]);",
                                    "double cl = floor(iv[4 * i]), fh = ceil(iv[4 * i + 1]);"),
    "certify over 2n-2 coefficients": ("size_t used = 2 * n - 1; ", "size_t used = 2 * n - 2; "),
    "imag product term sign": ("r.im = iadd_##S(imul_##S(z.re, w.im), imul_##S(z.im, w.re));",
                               "r.im = isub_##S(imul_##S(z.re, w.im), imul_##S(z.im, w.re));"),
    "no conjugate in the inverse": ("if (inverse) w = cconj_##S(w);", "(void)0;"),
    "mul: max of 3 products": ("if (h4 > hi) hi = h4;", "(void)h4;"),
}
PINS = ["tests/test_oracle_exact_ss.py", "tests/test_oracle_intervals.py",
        "tests/test_oracle_multiply.py", "tests/test_oracle_fft.py"]


def main() -> int:
    src = open(os.path.join(ROOT, "oracle", "ivm_oracle.c")).read()
    survivors = []
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        os.makedirs(os.path.join(tmp, "paper_1006_0405_b200"))
        for f in ("__init__.py", "inputs.py", "dist.py"):
            shutil.copy(os.path.join(ROOT, "paper_1006_0405_b200", f), os.path.join(tmp, "paper_1006_0405_b200", f))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        for name, (old, new) in MUTANTS.items():
            assert src.count(old) >= 1, f"mutation site not found: {name}"
            open(os.path.join(tmp, "oracle", "ivm_oracle.c"), "w").write(src.replace(old, new, 1))
            so = os.path.join(tmp, "oracle", "liboracle.so")
            if os.path.exists(so):
                os.remove(so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                                *PINS], cwd=tmp, capture_output=True, text=True)
            killed = r.returncode != 0
            print(f"{'killed ' if killed else 'SURVIVED'}  {name}: {r.stdout.strip().splitlines()[-1]}")
            if not killed:
                survivors.append(name)
    print(f"{len(MUTANTS) - len(survivors)}/{len(MUTANTS)} mutants killed")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
