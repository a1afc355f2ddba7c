"""Compile libgpujoin.so in-tree for sm_100a (nvcc, -lineinfo).

Used by __graft_entry__.build() and `python -m paper_1809_09930_b200._build`.
The shared library is git-ignored but travels to the GPU box with gpurun.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgpujoin.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["gj_capi.cu", "gj_index.cu", "gj_join.cu", "gj_join32.cu", "gj_join_umma.cu", "gj_join_ws.cu", "gj_radix.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "gpujoin.h"))
    return any(os.path.getmtime(d) > t for d in deps)


# timing experiments only: extra nvcc flags (e.g. -DGJ_UMMA_EXPERIMENT=1) for an
# A/B copy of the package built by tools/ab_prep.sh; never set for the product build
EXTRA = os.environ.get("GJ_NVCC_EXTRA", "").split()


def _compile(src: str, extra: list) -> tuple:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    r = subprocess.run([NVCC, *FLAGS, *EXTRA, *extra, "-c", "-o", obj, src], capture_output=True, text=True)
    return obj, r


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc per translation unit (in parallel), then one shared link."""
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    extra = ["-Xptxas", "-v"] if verbose else []
    with ThreadPoolExecutor(max_workers=len(srcs)) as pool:
        results = list(pool.map(lambda s: _compile(s, extra), srcs))
    for obj, r in results:
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        if verbose:
            sys.stderr.write(r.stderr)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp",
           *[obj for obj, _ in results]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
