"""Build the in-tree CUDA library ``paper_2209_08001_b200/lib/libnks.so`` for sm_100a.

    python -m paper_2209_08001_b200.build [--verbose] [--ptxas]

nvcc cross-compiles here without a GPU; the .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
BUILDDIR = os.path.join(PKG, "build")
LIB = os.path.join(LIBDIR, "libnks.so")
# experiments only: NKS_BUILD_TAG=x NKS_BUILD_DEFS="-DFOO=1" builds lib/libnks_x.so (load it with NKS_LIB)
TAG = os.environ.get("NKS_BUILD_TAG", "")
if TAG:
    LIB = os.path.join(LIBDIR, f"libnks_{TAG}.so")
    BUILDDIR = os.path.join(BUILDDIR, TAG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fvisibility=hidden"]


def _nccl():
    """NCCL of the PyTorch wheel (the library torch.distributed loads, so one NCCL lives in the process)."""
    import nvidia.nccl
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu*")) + glob.glob(os.path.join(PKG, "..", "include", "*.h")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(BUILDDIR, exist_ok=True)
    deps = _deps()
    if not force and not _stale(LIB, deps):
        return LIB
    extra = (["-Xptxas", "-v"] if ptxas else []) + os.environ.get("NKS_BUILD_DEFS", "").split()

    def compile_one(src):
        obj = os.path.join(BUILDDIR, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", _nccl()[0], "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose or ptxas:
            sys.stderr.write(r.stdout + r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    nccl_lib = _nccl()[1]
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcufft", "-lcudart", "-L", nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + nccl_lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, ptxas="--ptxas" in sys.argv))
