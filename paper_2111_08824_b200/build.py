"""Build recipe of the CUDA library ``csrc/liblj_b200.so`` (sm_100a only).

``python -m paper_2111_08824_b200.build`` or ``__graft_entry__.build()``.
nvcc cross-compiles here without a GPU; the .so is built in-tree so it
travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(CSRC, "liblj_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                   "--expt-relaxed-constexpr", "-I", INCLUDE]
SOURCES = ["lj_core.cu", "lj_grmi.cu", "lj_spline.cu", "lj_hash_staged.cu", "lj_spline_fit.cu", "lj_lsj.cu", "lj_multi.cu", "lj_spline_fit.cpp"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(INCLUDE, "lj_b200.h")]
    if not force and not _stale(LIB, deps + [__file__]):
        return LIB
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(CSRC, "build", src + ".o")
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        if force or _stale(obj, [path] + [os.path.join(CSRC, h) for h in HEADERS] +
                           [os.path.join(INCLUDE, "lj_b200.h"), __file__]):
            cmd = [NVCC] + CU_FLAGS + ["-c", path, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [CXX, "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
                       "-I", INCLUDE, "-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
