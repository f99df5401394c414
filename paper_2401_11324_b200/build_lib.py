"""Compile libbang.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels with the repository snapshot to the GPU box).

Each translation unit (the C-ABI + stand-alone kernels, and one per search
kernel family) is compiled in parallel, then linked with a static cudart."""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SRC = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
DEPS = SRC + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + \
    [os.path.join(os.path.dirname(HERE), "include", "bang.h")]
OUT = os.path.join(HERE, "libbang.so")
OBJ_DIR = os.path.join(CSRC, "build")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]
LINK_FLAGS = ["-shared", "-cudart", "static",   # no dependency on torch's cudart version
              "-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def _compile(src: str):
    obj = os.path.join(OBJ_DIR, os.path.basename(src)[:-3] + ".o")
    cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj, src]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return obj, cmd, res


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(OBJ_DIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=max(1, min(len(SRC), os.cpu_count() or 1))) as ex:
        results = list(ex.map(_compile, SRC))
    log = os.path.join(CSRC, "ptxas.log")
    with open(log, "w") as f:
        for _, cmd, res in results:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    failed = [r for r in results if r[2].returncode != 0]
    if failed:
        for _, _, res in failed:
            sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed; see {log}")
    cmd = [nvcc(), *LINK_FLAGS, "-o", OUT, *[r[0] for r in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc link failed ({res.returncode})")
    if verbose:
        for _, _, r in results:
            sys.stderr.write(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
