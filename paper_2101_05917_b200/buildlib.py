"""In-tree build of libdiffpd_b200.so (sm_100a) — nvcc + g++, no JIT cache.

    python -m paper_2101_05917_b200.buildlib
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libdiffpd_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if p and os.path.exists(p):
            return p
    raise RuntimeError("nvcc not found")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cpp", ".h", ".cuh"))] + [
        os.path.join(os.path.dirname(HERE), "include", "diffpd_b200.h")]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    inc = ["-I", os.path.join(os.path.dirname(HERE), "include")]
    log = []
    setup_o = os.path.join(BUILD, "setup.o")
    log.append(_run(["g++", "-O3", "-std=c++17", "-fopenmp", "-fPIC", "-march=x86-64-v3",
                     "-c", os.path.join(CSRC, "setup.cpp"), "-o", setup_o] + inc))
    capi_o = os.path.join(BUILD, "capi.o")
    extra = [f"-DK1_MIN_BLOCKS={int(os.environ['PD_K1_MIN_BLOCKS'])}"] if os.environ.get("PD_K1_MIN_BLOCKS") else []
    log.append(_run([nvcc] + ARCH + extra + ["-O3", "-std=c++17", "-lineinfo", "-Xptxas", "-v",
                                     "-Xcompiler", "-fPIC", "-c", os.path.join(CSRC, "capi.cu"),
                                     "-o", capi_o] + inc))
    tmp = LIB + ".tmp"
    log.append(_run([nvcc] + ARCH + ["-shared", "-o", tmp, capi_o, setup_o, "-lgomp"]))
    os.replace(tmp, LIB)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
