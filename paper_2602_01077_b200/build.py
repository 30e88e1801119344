"""Builds the in-tree sm_100a shared library lib/libpisa_b200.so with nvcc.

Compiles each kernel translation unit with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (plain ``-arch=sm_100a``
also emits compute_100 PTX, which ptxas rejects for tcgen05) and links them with
the static CUDA runtime into one C-ABI library. Rebuilds only when a source is
newer than the library.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libpisa_b200.so")
SOURCES = ["k1_block_stats.cu", "k1c_block_norms.cu", "k2_select.cu", "k2p_pairing.cu", "k2q_overlap.cu", "k3_fused_attn.cu", "selftest_mma.cu",
           "generate.cu", "pisa_b200.cu"]
HEADERS = ["sm100.cuh", "kernels.h", os.path.join("..", "..", "include", "pisa_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS + [os.path.basename(__file__)]:
        p = os.path.join(CSRC, f) if f != os.path.basename(__file__) else os.path.abspath(__file__)
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    lib = LIB if not trace else os.path.join(LIBDIR, "libpisa_b200_trace.so")
    if not force and not trace and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj_trace" if trace else "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    logs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *(["-DPISA_TRACE=1"] if trace else []), "-I", CSRC,
               "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(f"== {src}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write("".join(logs))
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    with open(os.path.join(LIBDIR, "ptxas_trace.log" if trace else "ptxas.log"), "w") as f:
        f.write("".join(logs))
    if verbose:
        sys.stdout.write("".join(logs))
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv)
