"""Build libdpg.so in-tree with nvcc for sm_100a (no torch involved).

    python paper_cs_0308004_b200/build.py [--force]

Run it by path (or load it with :func:`load_builder`): importing the package
itself loads libdpg.so and fails loudly when it is missing or stale.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdpg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def nccl_flags() -> list[str]:
    """The NCCL headers and library of the nvidia-nccl wheel (comm.cu loads the
    library at run time); without them the multi-GPU C entries report
    DPG_ERR_NCCL."""
    try:
        import nvidia.nccl as m
        base = list(m.__path__)[0]
    except Exception:
        base = None
    if base and os.path.exists(os.path.join(base, "include", "nccl.h")):
        lib = os.path.join(base, "lib", "libnccl.so.2")
        return ["-I", os.path.join(base, "include"), f'-DDPG_NCCL_LIB="{lib}"']
    return ["-DDPG_NO_NCCL"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "dpg.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, *nccl_flags(), "-I", os.path.join(ROOT, "include"), *sources(),
           "-ldl", "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libdpg.so")
    with open(os.path.join(PKG, "ptxas_report.txt"), "w") as f:
        f.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
