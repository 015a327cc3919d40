#!/usr/bin/env python3
"""Build an experiment variant of libivm.so with extra nvcc flags (A/B timing).

    python tools/build_variant.py NAME [-DFLAG ...]   ->  ab/libivm_NAME.so
"""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import paper_1006_0405_b200.build as b
    name, flags = sys.argv[1], sys.argv[2:]
    b.NVFLAGS = b.NVFLAGS + flags
    b.OUT = os.path.join(ROOT, "ab", f"libivm_{name}.so")
    b.OBJ = os.path.join(ROOT, "ab", f"obj_{name}")
    b.build(force=True)
    shutil.rmtree(b.OBJ, ignore_errors=True)
    print(b.OUT)
