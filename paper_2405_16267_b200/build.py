"""Build libbicadmm.so in-tree: hand-written CUDA for sm_100a (nvcc, no JIT).

    python -m paper_2405_16267_b200.build        # or __graft_entry__.build()

Every translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (plain ``-arch=sm_100a``
would also emit compute_100 PTX, which cannot hold tcgen05/sm_100a-only code).
NCCL is not linked: the library dlopens libnccl.so.2 (torch's) on first
multi-rank use, using the nccl.h of the same pip package for its types.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libbicadmm.so")
SOURCES = ["k_gemv.cu", "k_gemv_c.cu", "k_gemv_dmma.cu", "k_prox.cu", "k_factor.cu", "k_gram_tc.cu", "k_outer.cu", "k_vec.cu", "k_fused4.cu", "k_fused4_r1.cu", "k_fused4_r2.cu", "k_fused4_r4.cu", "k_symv.cu", "comm.cu", "capi.cu", "ops.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _nccl_include() -> list:
    try:
        import nvidia.nccl  # noqa: F401
        for base in nvidia.nccl.__path__:
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return ["-I" + inc]
    except Exception:
        pass
    return []


def _flags() -> list:
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "--extended-lambda", "-Xcompiler", "-fPIC",
                   "-I" + os.path.join(ROOT, "include")] + _nccl_include()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + \
           [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    flags = _flags()

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
