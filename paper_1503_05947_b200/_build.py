"""In-tree build of the native library (sm_100a) and of the test oracle.

The product library ``paper_1503_05947_b200/librbd_b200.so`` is compiled with
nvcc for ``-gencode arch=compute_100a,code=sm_100a`` only (no multi-arch
dispatch). The oracle (``oracle/build/liborc.so``) is test infrastructure and
is built by ``oracle/Makefile``.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "librbd_b200.so")
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "build", "liborc.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-O3",
]


def _extra_flags():
    """Experiment knobs (e.g. RBD_NVCC_DEFS="-DRBD_P1_LOADS=20"); empty by default."""
    return os.environ.get("RBD_NVCC_DEFS", "").split()


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return (_sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(INCLUDE, "*.h")) + glob.glob(os.path.join(INCLUDE, "rbd", "*.hpp")))


def _stale(target, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit of csrc/ in parallel (one nvcc per unit),
    then link the shared library; the result replaces LIB atomically."""
    if not force and not _stale(LIB, _deps()):
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    with tempfile.TemporaryDirectory(prefix="rbd_build_") as tmp:
        def compile_one(src):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [_nvcc(), *NVCC_FLAGS, *_extra_flags(), "-Xcompiler", "-fPIC", "-c", "-I", INCLUDE, "-I", CSRC,
                   src, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-4000:]}")
            return obj
        srcs = _sources()
        with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
            objs = list(ex.map(compile_one, srcs))
        cmd = [_nvcc(), *NVCC_FLAGS, "-shared", *objs, "-o", LIB + ".tmp", "-ldl"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True, cwd=ROOT)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_oracle(force: bool = False) -> str:
    if not force and not _stale(ORACLE_LIB, glob.glob(os.path.join(ORACLE_DIR, "*.cpp"))
                                + glob.glob(os.path.join(ORACLE_DIR, "*.h"))
                                + [os.path.join(ORACLE_DIR, "Makefile")]):
        return ORACLE_LIB
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
    return ORACLE_LIB


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_library(force=force, verbose=verbose)
    build_oracle(force=force)


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv, verbose=True)
    print("built", LIB, ORACLE_LIB)
