"""Build libfem.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build().

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC, one object per
.cu (compiled in parallel), linked into paper_2602_12365_b200/libfem.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libfem.so")
BUILD = os.path.join(HERE, "build_obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dirs():
    """The NCCL torch loads (nvidia-nccl wheel), so one libnccl is in the process."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (list(spec.submodule_search_locations) if spec else []):
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                   "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"),
                   "-Xptxas", "-warn-spills", "-I" + _nccl_dirs()[0]] + \
        os.environ.get("FEM_NVCC_FLAGS", "").split()


def _needs_build(srcs, deps):
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in srcs + deps)


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "fem.h")]
    if not force and not _needs_build(srcs, deps):
        return SO
    os.makedirs(BUILD, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC] + _flags() + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = SO + ".tmp"
    inc, lib = _nccl_dirs()
    nccl = (["-L" + lib, "-Xlinker", "-l:libnccl.so.2"] if os.path.exists(os.path.join(lib, "libnccl.so.2")) else ["-lnccl"])
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + nccl + ["-lcudart_static",
                                                                    "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, SO)
    return SO


PEAK_SO = os.path.join(HERE, "libfem_peak.so")


def build_peak(force: bool = False) -> str:
    """Bench-only FP64 throughput microbenchmark (bench_tools/peak.cu)."""
    src = os.path.join(HERE, "bench_tools", "peak.cu")
    if force or not os.path.exists(PEAK_SO) or os.path.getmtime(PEAK_SO) < os.path.getmtime(src):
        cmd = [NVCC] + ARCH + ["-O3", "-Xcompiler", "-fPIC", "-shared", "-o", PEAK_SO, src]
        subprocess.check_call(cmd)
    return PEAK_SO


if __name__ == "__main__":
    build_peak(force="--force" in sys.argv)
    print(build(force="--force" in sys.argv, verbose=True))
