"""Build libbiluk.so in-tree for sm_100a (nvcc, static cudart).

    python -m paper_1703_01325_b200.build
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/plan.cpp", "csrc/psweep_plan.cpp", "csrc/abi.cu", "csrc/kernels.cu", "csrc/psweep.cu", "csrc/krylov.cu",
           "csrc/stages.cu", "csrc/gsweep.cu"]
HEADERS = ["csrc/biluk_internal.h", "csrc/device_util.cuh", "csrc/kernels.cuh", "../include/biluk.h"]
OUT = os.path.join(HERE, "_lib", "libbiluk.so")


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(os.path.join(HERE, f)) <= t for f in SOURCES + HEADERS + ["build.py"])


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC,-O3,-pthread", "-diag-suppress", "128", "-shared", "-o", OUT + ".tmp"]
    cmd += [os.path.join(HERE, s) for s in SOURCES] + ["-cudart", "static", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
