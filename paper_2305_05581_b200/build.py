"""In-tree build of the sm_100a C-ABI library ``lib/libsdmrg_b200.so``.

One nvcc invocation over ``csrc/*.cu`` (``-gencode arch=compute_100a,
code=sm_100a -lineinfo``); the shared object lands inside the package so it
travels to the GPU box with the repo snapshot.  Rebuilds only when a source
or the public header is newer than the library.
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libsdmrg_b200.so")
HEADER = os.path.join(ROOT, "include", "sdmrg_b200.h")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-fopenmp",
         "-Xptxas", "-v", "--expt-relaxed-constexpr", "-lgomp"]


def nvcc():
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: cannot build the sm_100a library")
    return path


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh", ".h")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in sources() + [HEADER, __file__])


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    cu = [p for p in sources() if p.endswith(".cu")]
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + ARCH + FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", tmp] + cu
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + proc.stderr[-8000:])
    if verbose:
        sys.stderr.write(proc.stderr)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
        fh.write(" ".join(cmd) + "\n" + proc.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
