"""Build libpdnn.so (sm_100a) in-tree with nvcc.

    python -m paper_2008_08636_b200.build [--force] [--verbose]

Every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17`` (CUB from
the CUDA 12.9 toolkit; cudart linked statically) and linked into
``paper_2008_08636_b200/libpdnn.so``.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libpdnn.so")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "pdnn.h")]


LIB_DBG = os.path.join(HERE, "libpdnn_dbg.so")


def build(force: bool = False, verbose: bool = False, debug_knobs: bool = False, variant: str = "",
          defines=()) -> str:
    """Build libpdnn.so; with debug_knobs, libpdnn_dbg.so (-DPDNN_DEBUG_KNOBS:
    grid / poll / trace knobs read from the environment; probes under tools/
    load it explicitly, the product path never does)."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    # variant: a debug build with extra -D defines (compile-time experiments, tools/ only)
    BUILD = os.path.join(HERE, "build_dbg" + variant if debug_knobs else "build")
    LIB = LIB_DBG.replace(".so", variant + ".so") if debug_knobs else os.path.join(HERE, "libpdnn.so")
    flags = FLAGS + (["-DPDNN_DEBUG_KNOBS"] + ["-D" + d for d in defines] if debug_knobs else [])
    os.makedirs(BUILD, exist_ok=True)
    newest_dep = max(os.path.getmtime(p) for p in _deps())
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), newest_dep):
            extra = ["-Xptxas", "-v"] if verbose else []
            jobs.append([NVCC, *ARCH, *flags, *extra, "-c", s, "-o", o])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            res = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for c, r in zip(jobs, res):
            if r.returncode != 0 or verbose:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError("nvcc failed: " + " ".join(c))
    if jobs or force or not os.path.exists(LIB):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, debug_knobs="--debug-knobs" in sys.argv))
