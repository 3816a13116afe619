"""Build libeca_b200.so in-tree with nvcc for sm_100a (no torch JIT, no cache dir).

    python -m paper_2210_14771_b200.build          # incremental
    python -m paper_2210_14771_b200.build --force

The library is a plain C-ABI shared object (include/eca_b200.h) loaded with
ctypes; it links only the CUDA runtime.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libeca_b200.so"
OBJ = ROOT / "build" / "obj"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v", "-I", str(ROOT / "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def headers():
    return sorted(list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h")))


def needs_build(force: bool) -> bool:
    if force or not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources() + headers() + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not needs_build(force):
        return LIB
    OBJ.mkdir(parents=True, exist_ok=True)
    objs = []
    log = []
    for src in sources():
        obj = OBJ / (src.stem + ".o")
        # ECA_NVCC_DEFINES="-DX=1 ...": tuning experiments only
        extra = os.environ.get("ECA_NVCC_DEFINES", "").split()
        cmd = [nvcc(), *ARCH, *NVFLAGS, *extra, "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cpp":
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC",
                   "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src.name}")
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    # static cudart: the library must not bind to whichever libcudart.so.12
    # the host process (torch) loaded first
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    (ROOT / "build" / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
