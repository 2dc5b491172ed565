"""Build libpnx.so (sm_100a) in-tree with nvcc.

``python -m paper_2604_15645_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpnx.so")
SOURCES = ["pnx_capi.cu", "pnx_dp.cu", "launch_simt.cu", "launch_tc.cu", "launch_small.cu"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newest_source_mtime() -> float:
    ts = [os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)]
    ts.append(os.path.getmtime(os.path.join(ROOT, "include", "pnx.h")))
    return max(ts)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_source_mtime():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    objs, procs = [], []
    for src in SOURCES:  # translation units compile in parallel
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [nvcc, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd)))
        objs.append(obj)
    for src, p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {src}")
    tmp = LIB + ".tmp"
    # NCCL (the data-parallel group's all-reduce): link the libnccl.so.2 that torch
    # bundles (nvidia-nccl wheel, newer than the image's /usr/lib 2.27) when it is
    # there, with an rpath to it: whichever of libpnx / torch loads first, the one
    # libnccl.so.2 in the process satisfies both (libtorch_cuda needs 2.28 symbols)
    nccl = []
    try:
        import nvidia.nccl as _n  # noqa: F401  (namespace package)
        d = os.path.join(list(_n.__path__)[0], "lib")
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            nccl = ["-L" + d, "-Xlinker", "-rpath=" + d]
    except Exception:
        pass
    subprocess.run([nvcc, *GENCODE, "-shared", "-o", tmp, *objs, "-lcudart", *nccl, "-l:libnccl.so.2"], check=True)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
