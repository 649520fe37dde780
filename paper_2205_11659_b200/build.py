"""Build libtreebbox.so (sm_100a) in-tree with nvcc.

    python -m paper_2205_11659_b200.build [--force]

The shared library exports the C ABI of include/treebbox.h.  Compiled with
-gencode arch=compute_100a,code=sm_100a -lineinfo, no fast-math (box min/max
must stay exact, DESIGN R12).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libtreebbox.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def _nccl_flags():
    """Link the NCCL that torch bundles (same library at run time)."""
    try:
        import nvidia.nccl  # type: ignore
        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    except Exception:
        return None
    inc = os.path.join(base, "include")
    lib = os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        return None
    so = sorted(glob.glob(os.path.join(lib, "libnccl.so*")))
    if not so:
        return None
    return ["-I" + inc, "-DTB_WITH_NCCL=1", "-L" + lib, "-l:" + os.path.basename(so[0]),
            "-Xlinker", "-rpath," + lib]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(INCLUDE, "*.h")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nccl = _nccl_flags() or []
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *FLAGS, "-I" + INCLUDE, "-shared", "-o", tmp, *sources(), *nccl]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libtreebbox.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
