"""Build the native CUDA libraries in-tree (sm_100a): liboem.so (product) and
libdatagen_cuda.so (device input generator). nvcc cross-compiles here without a GPU.
(__graft_entry__.build() additionally builds the host generator and the test oracle.)"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
# developer hook (instrumented builds, e.g. -DSP_PROFILE); rebuild with force=True after changing it
NVFLAGS += os.environ.get("OEM_NVCC_EXTRA", "").split()

OEM_SRCS = ["api.cu", "gram.cu", "drule.cu", "path.cu", "logistic.cu", "cv.cu", "logit_ub.cu", "moments.cu", "stream.cu", "sparse.cu"]
OEM_HDRS = ["common.cuh", "internal.h"]
LIBOEM = os.path.join(PKG, "liboem.so")
DG_CUDA = os.path.join(ROOT, "datagen", "libdatagen_cuda.so")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[-1]}")
    return r.stderr


def build_liboem(force=False, verbose=False):
    csrc = os.path.join(PKG, "csrc")
    hdrs = [os.path.join(csrc, h) for h in OEM_HDRS] + [os.path.join(ROOT, "include", "oem.h")]
    objs = []
    jobs = []
    for s in OEM_SRCS:
        src = os.path.join(csrc, s)
        obj = os.path.join(csrc, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            extra = ["-Xptxas", "-v"] if verbose else []
            jobs.append([NVCC] + NVFLAGS + extra + ["-c", src, "-o", obj])
    with ThreadPoolExecutor(max_workers=4) as ex:
        for err in ex.map(_run, jobs):
            if verbose and err:
                sys.stderr.write(err)
    if force or jobs or _stale(LIBOEM, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIBOEM] + objs + ["-lnccl"])
    return LIBOEM


def build_datagen_cuda(force=False):
    src = os.path.join(ROOT, "datagen", "datagen_cuda.cu")
    hdr = os.path.join(ROOT, "include", "oem_datagen.h")
    if force or _stale(DG_CUDA, [src, hdr]):
        _run([NVCC] + NVFLAGS + ["--fmad=false", "-shared", "-o", DG_CUDA, src])
    return DG_CUDA


def build_native(force=False, verbose=False):
    build_datagen_cuda(force)
    build_liboem(force, verbose)


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built:", LIBOEM, DG_CUDA)
