"""How librelay.so is built (one place: the package, __graft_entry__.build()
and the tuning tools all use it).  Imports nothing from the package, so it
can run before the library exists."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "librelay.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in
           ("margin_kernels.cu", "scan_kernels.cu", "sample_kernels.cu", "relay_api.cu",
            "relay_comm.cu")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in ("relay_device.cuh", "relay_internal.h", "switch.cuh", "draw.cuh",
                                                    "p2p.cuh")] + \
          [os.path.join(REPO, "include", "relay.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]
LIBS = ["-ldl"]   # NCCL is dlopen'ed at run time (relay_comm.cu)


def nvcc() -> str:
    n = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return n if os.path.exists(n) else "nvcc"


def build_lib(out: str = LIB_PATH, defines=(), force: bool = False, verbose: bool = False) -> str:
    """Compile the sources for sm_100a into ``out`` (skipped when up to date
    and no ``defines`` are given)."""
    newest = max(os.path.getmtime(p) for p in SOURCES + HEADERS)
    if not force and not defines and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    tmp = out + ".tmp"
    cmd = [nvcc()] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-o", tmp] + SOURCES + LIBS
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out
