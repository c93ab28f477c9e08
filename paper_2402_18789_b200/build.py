"""In-tree build of libcoserve_cuda.so (sm_100a) and the host C++ pieces.

    python -m paper_2402_18789_b200.build [--force]

Compiles every csrc/*.cu and csrc/*.cpp with nvcc (-gencode arch=compute_100a,code=sm_100a
-lineinfo) into paper_2402_18789_b200/libcoserve_cuda.so.  Objects go to build/ (ignored);
the .so is git-ignored but travels to the GPU box with gpurun snapshots.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libcoserve_cuda.so")
# --trace: the same sources with -DCS_TRACE (in-kernel event timelines, scripts/trace_bwd.py)
OBJ_TRACE = os.path.join(ROOT, "build", "obj_trace")
LIB_TRACE = os.path.join(PKG, "libcoserve_cuda_trace.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "--expt-relaxed-constexpr"]


def _deps(src: str):
    heads = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "**", "*.h*"), recursive=True)
    return [src] + heads


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool, trace: bool = False):
    obj = os.path.join(OBJ_TRACE if trace else OBJ, os.path.basename(src) + ".o")
    if not force and not _stale(obj, _deps(src)):
        return obj, None
    flags = COMMON + (["-DCS_TRACE"] if trace else [])
    cmd = [NVCC] + ARCH + flags + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + flags + ["-x", "cu"] + ARCH + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"{' '.join(cmd)}\n{r.stdout}\n{r.stderr}"
    return obj, None


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    obj_dir, lib = (OBJ_TRACE, LIB_TRACE) if trace else (OBJ, LIB)
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, trace), srcs))
    errs = [e for _, e in results if e]
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n\n".join(errs))
    objs = [o for o, _ in results]
    if force or _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + [
            "-lcudart", "-L/usr/lib/x86_64-linux-gnu", "-l:libnccl.so.2"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv)
