"""Build the sm_100a CUDA library ``libmpsylv_b200.so`` in-tree with nvcc.

The library is the product: every hot step of the solver is a kernel in
``csrc/``; ``include/mpsylv_b200.h`` is its C ABI.  Built in place so the
``.so`` travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmpsylv_b200.so")
SOURCES = [os.path.join(HERE, "csrc", "solver.cu")]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "177",
]


def _deps():
    d = os.path.join(HERE, "csrc")
    files = [os.path.join(d, f) for f in os.listdir(d)]
    files.append(os.path.join(ROOT, "include", "mpsylv_b200.h"))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("MSY_EXTRA_NVCC_FLAGS", "").split()  # developer A/B switches
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        print("[build]", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
