"""Build libpdssm.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

The library is several translation units (csrc/*.cu) compiled in parallel into
objects under paper_2605_19150_b200/build/ and linked into one shared object.
The ptxas resource logs (registers, spills, shared memory) go to build/ptxas_<unit>.txt
(git-ignored); commit a copy under profiles/ when it is evidence for a change.
"""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libpdssm.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def units():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(ROOT, "include", "pdssm.h")]
    return any(os.path.getmtime(s) > t for s in deps)


def _nvcc():
    return os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _compile(src, extra, bdir=BUILD):
    name = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(bdir, name + ".o")
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(bdir, f"ptxas_{name}.txt"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {name}:\n" + r.stderr[-8000:])
    os.replace(obj + ".tmp", obj)
    return obj


def build(force=False, verbose=False, extra=(), out=None):
    """Compile every csrc/*.cu unit (in parallel) and link libpdssm.so (or `out`: a tuning
    variant built with extra -D defines into its own object directory)."""
    lib = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    bdir = BUILD if out is None else os.path.join(BUILD, "variant_" + os.path.splitext(os.path.basename(out))[0])
    os.makedirs(bdir, exist_ok=True)
    srcs = units()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, list(extra), bdir), srcs))
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", lib + ".tmp",
           *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stderr[-8000:])
    os.replace(lib + ".tmp", lib)
    if verbose:
        for s in srcs:
            n = os.path.splitext(os.path.basename(s))[0]
            print(open(os.path.join(BUILD, f"ptxas_{n}.txt")).read())
    return lib


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":   # --variant NAME -DX=1 ...
        os.makedirs(os.path.join(PKG, "variants"), exist_ok=True)
        print(build(out=os.path.join(PKG, "variants", sys.argv[2] + ".so"), extra=sys.argv[3:]))
    else:
        build(force=True, verbose=False)
        print(LIB)
