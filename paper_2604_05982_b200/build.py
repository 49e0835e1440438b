"""Build libgtap.so (the C-ABI library) for sm_100a, in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, one object per
.cu (parallel), linked into paper_2604_05982_b200/libgtap.so. No torch
extension machinery: the library exports plain C symbols (include/gtap.h).
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libgtap.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]
SOURCES = ["runtime.cu", "table_fib.cu", "table_mergesort.cu", "table_spmv.cu", "table_bfs.cu", "table_nqueens.cu",
           "table_cilksort.cu", "table_tree.cu", "ubench.cu"]


def _digest(lib: str, extra) -> str:
    h = hashlib.sha256()
    for d in (CSRC, INCLUDE):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cuh", ".h")):
                with open(os.path.join(d, f), "rb") as fh:
                    h.update(f.encode() + fh.read())
    h.update(" ".join(ARCH + FLAGS + list(extra)).encode() + lib.encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, defines=(), out=None) -> str:
    """Compile every .cu in SOURCES and link libgtap.so (out/defines: diagnostic variants only)."""
    lib, bdir = LIB, BUILD
    if defines or out:
        tag = "_".join(d.lower().replace("=", "") for d in defines)
        lib = out or LIB.replace(".so", "_" + tag + ".so")
        bdir = BUILD + "_" + tag
    os.makedirs(bdir, exist_ok=True)
    stamp = os.path.join(bdir, "stamp")
    extra = (["-Xptxas", "-v"] if ptxas_v else []) + [f"-D{d}" for d in defines]
    dig = _digest(lib, [f"-D{d}" for d in defines])
    if not force and os.path.exists(lib) and os.path.exists(stamp) and open(stamp).read() == dig:
        return lib

    def compile_one(src):
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    if verbose or ptxas_v:
        for _, err in results:
            sys.stderr.write(err)
    tmp = lib + f".{os.getpid()}.tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *[o for o, _ in results], "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    with open(stamp, "w") as f:
        f.write(dig)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv, defines=defs))
