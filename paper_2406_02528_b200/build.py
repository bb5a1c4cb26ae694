"""Build libtern.so in-tree with nvcc for sm_100a.

Usage: python -m paper_2406_02528_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libtern.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["api.cu", "k_pack.cu", "k_quant.cu", "k_gemv.cu", "k_gemm.cu", "k_scan.cu", "k_selftest.cu", "k_shard.cu", "k_fcgscan.cu", "k_fin.cu", "k_fxp.cu", "k_gemm_sab.cu", "k_bwd.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}"]
HEADERS = ["common.cuh", "epilogue.cuh", "internal.h"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _compile(src: str, verbose: bool, obj_dir: str = OBJ, extra=()) -> str:
    obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
    dep = max([_mtime(os.path.join(CSRC, src))] + [_mtime(os.path.join(CSRC, h)) for h in HEADERS]
              + [_mtime(os.path.join(ROOT, "include", "tern.h"))])
    if _mtime(obj) >= dep:
        return obj
    cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".ptxas.log", "w") as f:
        f.write(r.stderr)
    if verbose:
        print(f"compiled {src}", file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace: the debug variant libtern_trace.so with the device timeline marks
    of every kernel compiled in (-DTERN_TRACE; tools/timeline.py)."""
    obj_dir = OBJ + "_trace" if trace else OBJ
    lib = LIB.replace("libtern.so", "libtern_trace.so") if trace else LIB
    extra = ("-DTERN_TRACE",) if trace else ()
    os.makedirs(obj_dir, exist_ok=True)
    if force:
        for s in SOURCES:
            o = os.path.join(obj_dir, s.replace(".cu", ".o"))
            if os.path.exists(o):
                os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, obj_dir, extra), SOURCES))
    if force or _mtime(lib) < max(_mtime(o) for o in objs):
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
               "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
