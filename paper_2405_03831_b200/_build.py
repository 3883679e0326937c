"""In-tree build of the native libraries (invoked by ``__graft_entry__.build()``).

* ``libcosched_b200.so``: ``nvcc -gencode arch=compute_100a,code=sm_100a`` of
  ``csrc/sweep.cu``, static cudart, so the .so only needs the driver.
* ``libcosched_train.so``: ``nvcc`` (same flags) of ``csrc/train.cu``, the
  device-side trainer (include/cosched_train.h).
* ``libcosched_match.so``: ``g++`` of ``csrc/matching.cpp`` (host only).

Outputs sit next to the package sources (git-ignored, shipped to the GPU box
with the tree).  Rebuilds only when a source or header is newer.
"""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
CSRC = os.path.join(HERE, "csrc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
                     "-cudart", "static", f"-I{INCLUDE}"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra", f"-I{INCLUDE}"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose: bool) -> None:
    if verbose:
        print("+", " ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


def build_sweep(force: bool = False, verbose: bool = True) -> str:
    out = os.path.join(HERE, "libcosched_b200.so")
    src = os.path.join(CSRC, "sweep.cu")
    deps = [src, os.path.join(INCLUDE, "cosched_b200.h")] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    if force or _stale(out, deps):
        _run([_nvcc(), *NVCC_FLAGS, src, "-o", out], verbose)
    return out


def build_matcher(force: bool = False, verbose: bool = True) -> str:
    out = os.path.join(HERE, "libcosched_match.so")
    src = os.path.join(CSRC, "matching.cpp")
    deps = [src, os.path.join(INCLUDE, "cosched_match.h")]
    if force or _stale(out, deps):
        _run([os.environ.get("CXX", "g++"), *CXX_FLAGS, src, "-o", out], verbose)
    return out


def build_train(force: bool = False, verbose: bool = True) -> str:
    out = os.path.join(HERE, "libcosched_train.so")
    src = os.path.join(CSRC, "train.cu")
    deps = [src, os.path.join(INCLUDE, "cosched_train.h")]
    if force or _stale(out, deps):
        _run([_nvcc(), *NVCC_FLAGS, src, "-o", out], verbose)
    return out


def build_all(force: bool = False, verbose: bool = True) -> list:
    return [build_sweep(force, verbose), build_train(force, verbose), build_matcher(force, verbose)]


if __name__ == "__main__":
    import sys
    for path in build_all(force="--force" in sys.argv):
        print(path)
