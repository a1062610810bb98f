"""Build libevconv.so in-tree (sm_100a only; nvcc cross-compiles without a GPU).

    python -m paper_2303_04670_b200._build        # or: python paper_2303_04670_b200/_build.py

The library is a plain C-ABI shared object (include/evconv.h) with the CUDA
runtime linked statically, loaded by ``paper_2303_04670_b200._lib`` through
ctypes.  Object files are cached next to the sources and rebuilt when a
source or header is newer.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libevconv.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", str(INCLUDE)]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), *INCLUDE.glob("*.h")]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(verbose: bool = False, jobs: int = 8) -> Path:
    srcs = sorted(CSRC.glob("*.cu"))
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    procs = []
    objs = []
    for src in srcs:
        obj = objdir / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, src):
            cmd = [NVCC, *ARCH, *FLAGS, "-dc" if False else "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
            if len(procs) >= jobs:
                _drain(procs)
    _drain(procs)
    if not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        out = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        if out.returncode:
            raise RuntimeError(f"link failed:\n{out.stdout}")
    return LIB


def _drain(procs):
    errs = []
    for src, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode:
            errs.append(f"--- {src.name}\n{text}")
        elif text.strip():
            print(f"--- {src.name}\n{text}", file=sys.stderr)
    procs.clear()
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
