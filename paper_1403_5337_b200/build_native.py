"""Compile the sm_100a CUDA library in-tree: paper_1403_5337_b200/libhodlr_b200.so.

nvcc cross-compiles on a host without a GPU.  The shared library links the
CUDA runtime statically, so loading it needs no libcuda (only calling into the
device does).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = Path(os.environ["HK_LIB_OUT"]) if os.environ.get("HK_LIB_OUT") else PKG / "libhodlr_b200.so"
# experiment knob: extra nvcc flags (e.g. "-DHK_ACA_LB1") for variant builds written to HK_LIB_OUT
EXTRA = os.environ.get("HK_NVCC_EXTRA", "").split()
SOURCES = ["aca.cu", "lu.cu", "gj.cu", "gemm.cu", "solve.cu", "krylov.cu", "select.cu", "api.cpp",
           "graph.cpp", "validate.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh"))
    deps.append(INCLUDE / "hodlr_b200.h")
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    objdir = PKG / "build" / (LIB.stem if os.environ.get("HK_LIB_OUT") else "")
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = objdir / (src + ".o")
        cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-fvisibility=hidden", *EXTRA, "-I", str(INCLUDE), "-c", str(CSRC / src),
               "-o", str(obj)]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(str(obj))
    failed = False
    for cmd, pr in procs:
        out, _ = pr.communicate()
        if verbose or pr.returncode:
            sys.stderr.write(out.decode(errors="replace"))
        if pr.returncode:
            failed = True
            sys.stderr.write("FAILED: " + " ".join(cmd) + "\n")
    if failed:
        raise RuntimeError("nvcc build of libhodlr_b200.so failed")
    tmp = LIB.with_suffix(".so.tmp")
    link = [_nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-cudart", "static"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libhodlr_b200.so failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
