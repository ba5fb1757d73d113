"""Build librgc.so (the C-ABI CUDA library) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librgc.so")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")


def _nccl_path() -> str:
    try:
        import nvidia.nccl  # type: ignore
        cands = []
        for p in getattr(nvidia.nccl, "__path__", []):
            cands += glob.glob(os.path.join(p, "lib", "libnccl.so.2"))
        if cands:
            return cands[0]
    except Exception:
        pass
    return ""


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "rgc.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


# per-translation-unit ptxas flags (experiments: RGC_PTXAS_COMPACT="-Xptxas -O1" builds K3 at
# ptxas -O1).  An earlier K3 design was only bit-exact at -O1 (ordered output misplaced from the
# second call on at -O3); the current K3 is bit-exact at -O3 on the whole parity suite and the
# 2/4-GPU runs, and ~2 us faster, so the default is -O3 again.
PTXAS = {"rgc_compact.cu": os.environ.get("RGC_PTXAS_COMPACT", "").split()}
UNITS = ["rgc_kernels.cu", "rgc_compact.cu", "rgc_select.cu", "rgc_p2p.cu", "rgc_decomp.cu", "rgc_asq.cu", "rgc_api.cu"]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    common = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-Xcompiler", "-fPIC", f"-DRGC_NCCL_PATH=\"{_nccl_path()}\"",
              "-I", INCLUDE]
    if verbose:
        common.append("-Xptxas=-v")
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for u in UNITS:
        o = os.path.join(objdir, u.replace(".cu", ".o"))
        cmd = common + PTXAS.get(u, []) + ["-c", os.path.join(CSRC, u), "-o", o]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-cudart", "static", "-o", tmp] + objs + ["-ldl", "-lpthread", "-lrt"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
