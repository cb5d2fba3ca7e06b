"""Build libcoral_s1.so in-tree for sm_100a (nvcc, no JIT cache): the shared library
travels with the repo snapshot to the GPU box."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "coral_s1.cu")
OUT = os.path.join(HERE, "_lib", "libcoral_s1.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in sorted(os.listdir(os.path.join(HERE, "csrc")))
        if f.endswith((".cu", ".cuh", ".h"))] + \
       [os.path.join(os.path.dirname(HERE), "include", "coral_s1.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              # the reference (Python/numba) never contracts a*b+c: keep fp64 bit-exact
              "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(d) > t for d in DEPS)


MAT_SRC = os.path.join(HERE, "csrc", "materialize.c")


def build_materialize(force: bool = False, verbose: bool = False) -> str:
    """CPython extension that turns device frontier items into template objects."""
    import sysconfig
    out = os.path.join(HERE, "_lib", "_materialize" + sysconfig.get_config_var("EXT_SUFFIX"))
    hdr = os.path.join(os.path.dirname(HERE), "include", "coral_s1.h")
    if not force and os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out)
                                                 for d in (MAT_SRC, hdr)):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-std=c11", "-I" + sysconfig.get_paths()["include"],
           "-o", out + ".tmp", MAT_SRC]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    build_materialize(force, verbose)
    if not force and not stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT + ".tmp", SRC]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
