"""Build libaccord.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2412_11554_b200.build [--verbose]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libaccord.so")
SOURCES = ["api.cpp", "kernels.cu", "gemm_simt.cu", "gemm_tc.cu", "postproc.cu", "spmm_tma.cu",
           "quant_i8.cu"]
HEADERS = ["accord_internal.h", "tc_ptx.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "-cudart", "shared",
    "--expt-relaxed-constexpr",
]


def nvcc_path() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return p


def _newest_input_mtime() -> float:
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "accord.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files if os.path.exists(f))


def up_to_date() -> bool:
    return os.path.exists(OUT) and os.path.getmtime(OUT) >= _newest_input_mtime()


def build(verbose: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """defines/out: diagnostic variants (e.g. an A-B build next to the product
    library); the product is the default build to OUT."""
    global OUT
    if out is not None:
        prev, OUT = OUT, out
        try:
            return build(verbose, True, defines)
        finally:
            OUT = prev
    if not force and up_to_date():
        return OUT
    objdir = os.path.join(HERE, "build" if not defines else "build_variant")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s + ".o")
        cmd = [nvcc_path(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], *inc, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}")
        objs.append(obj)
    tmp = OUT + ".tmp"
    cmd = [nvcc_path(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           "-cudart", "shared", *objs, "-o", tmp, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("link failed")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force=True)
    print(OUT)
