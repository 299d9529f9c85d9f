"""In-tree build of the CUDA library ``libwarmgp_b200.so`` for sm_100a.

Every translation unit is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked
into one shared object next to this file (it travels to the GPU box with the
repo snapshot).  Only CUDA 12.9 toolkit libraries are linked (cuBLAS for the
AP block GEMM, cuSOLVER for the AP block Cholesky); the driver API entry
point for TMA descriptors is resolved at run time.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libwarmgp_b200.so")
BUILD = os.path.join(HERE, "_build")
SOURCES = ["hv_simt.cu", "hv_tc.cu", "hv_f64.cu", "hv_i8.cu", "grad_rff.cu", "grad_tc.cu", "solver_kernels.cu", "exact.cu", "predict.cu", "runtime.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                   "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
                   "-Xptxas", "-warn-spills"] + os.environ.get("WGP_NVCC_DEFS", "").split()  # dev A/B variants


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    headers.append(os.path.join(ROOT, "include", "warmgp_b200.h"))
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc(), *flags(), "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(OUT, objs):
        run([nvcc(), *ARCH, "-shared", "-o", OUT, *objs, "-lcublas", "-lcusolver"])
    return OUT


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
