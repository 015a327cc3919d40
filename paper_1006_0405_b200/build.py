"""Build libivm.so (sm_100a SASS, static cudart) in-tree.

    python -m paper_1006_0405_b200.build          # incremental
    python -m paper_1006_0405_b200.build --force  # rebuild everything
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libivm.so")
OBJ = os.path.join(HERE, "_obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--ftz=false",
                  "--prec-div=true", "--prec-sqrt=true", "--fmad=true", "-Xptxas", "-v",
                  "-I", os.path.join(ROOT, "include")]
CXXFLAGS = ["-O2", "-fPIC", "-std=gnu++17", "-fext-numeric-literals", "-I", os.path.join(ROOT, "include"),
            "-I", os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include")]

CU = ["ivm_kernels.cu", "ivm_v3.cu", "ivm_v4.cu", "ivm_v5.cu", "ivm_long.cu", "ivm_naive.cu", "ivm_disc.cu", "ivm_api.cu"]
CPP = ["ivm_planner.cpp", "ivm_multi.cpp"]
# every header under csrc/ is a dependency of every translation unit
HDR = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HDR] + [os.path.join(ROOT, "include", "ivm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    jobs = []
    for f in CU:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(obj, src):
            cmd = [NVCC, *NVFLAGS, "-c", src, "-o", obj]
            jobs.append((f, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                                  text=True)))
        objs.append(obj)
    failed = None
    for f, obj, pr in jobs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            failed = f
            continue
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(err)
        if verbose:
            sys.stderr.write(err)
    if failed:
        raise RuntimeError(f"nvcc failed on {failed}")
    for f in CPP:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        if force or _stale(obj, src):
            subprocess.check_call(["g++", *CXXFLAGS, "-c", src, "-o", obj])
        objs.append(obj)
    if force or not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", OUT, *objs,
               "-Xlinker", "-Bstatic", "-lquadmath", "-Xlinker", "-Bdynamic", "-lrt", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            # fall back to a dynamic libquadmath
            cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", OUT, *objs, "-lquadmath", "-ldl"]
            subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
