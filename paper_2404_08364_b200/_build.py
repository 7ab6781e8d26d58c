"""In-tree build of libflowwalk.so (nvcc, sm_100a only)."""

import os
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/fw_api.cu", "csrc/fw_walk.cu", "csrc/fw_trials.cu", "csrc/fw_ingest.cu"]
HEADERS = ["csrc/fw_common.cuh", "csrc/fw_walk.cuh", "../include/flowwalk.h"]
OUT = os.path.join(_HERE, "libflowwalk.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the reference's numba step_pass emits no FMAs; keep fp64 products and
    # sums separately rounded
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(os.path.join(_HERE, s)) > t for s in SOURCES + HEADERS)


def build(force=False, verbose=False, out=None, extra=()):
    out = out or OUT
    if not force and out == OUT and not needs_build():
        return OUT
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", out, *[os.path.join(_HERE, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=_HERE)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
