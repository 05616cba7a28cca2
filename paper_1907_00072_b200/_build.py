"""Build libpgmres.so in-tree with nvcc for sm_100a (no torch JIT cache, so the
built library travels to the GPU box with the repo snapshot)."""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libpgmres.so")
# the same sources with the device-side invariant checks (PG_CHECKS=1)
LIB_CHECKED = os.path.join(HERE, "libpgmres_checked.so")
BUILD = os.path.join(ROOT, "build", "pgmres")

SOURCES = ["abi.cu", "spmv.cu", "ortho.cu", "host.cu", "ilu.cu", "step.cu", "chain.cu", "blasorder.cu", "march.cu", "planes.cu", "dist.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
    "-Xptxas", "-v",
    "-I", INCLUDE,
]


def _nccl_include():
    """nccl.h for the types of csrc/dist.cu (libnccl itself is dlopen'ed at
    run time): torch's wheel copy, else the system header."""
    try:
        import nvidia.nccl as nn
        for base in list(getattr(nn, "__path__", [])):
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except ImportError:
        pass
    return "/usr/include"


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libpgmres.so")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """nvcc the sources into libpgmres.so (checked: libpgmres_checked.so with
    -DPG_CHECKS=1, objects under build/pgmres_checked)."""
    headers = [os.path.join(INCLUDE, "pgmres.h"), os.path.join(CSRC, "internal.cuh"),
               os.path.join(CSRC, "pipeline.cuh"), os.path.join(CSRC, "sell.cuh")]
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    lib = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib, srcs + headers + [__file__]):
        return lib
    build_dir = BUILD + ("_checked" if checked else "")
    os.makedirs(build_dir, exist_ok=True)
    nvcc = _nvcc()
    extra = ["-DPG_CHECKS=1"] if checked else []

    def compile_one(src):
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", _nccl_include(), "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(res.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = lib + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    if verbose:
        for o in objs:
            print(open(o + ".ptxas.txt").read())
    return lib


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
