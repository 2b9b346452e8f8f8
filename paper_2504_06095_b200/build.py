"""Build the in-tree C-ABI library libntp_b200.so for sm_100a with nvcc.

    python -m paper_2504_06095_b200.build

The library is a plain shared object (extern "C" entry points, include/ntp_b200.h)
linked against a static CUDA runtime; Python binds it with ctypes.  It is built
in-tree so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libntp_b200.so")

SOURCES = ["ntp_planner.cpp", "ntp_sync.cu", "ntp_linear.cu", "ntp_multi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "ntp_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile (if stale or forced).  Concurrent callers -- e.g. the ranks of a
    torchrun job -- serialize on a file lock and each writes its own temporary,
    so the in-tree .so is replaced atomically exactly once."""
    import fcntl
    if not force and not _stale():
        return LIB
    with open(LIB + ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not _stale():  # another process built it meanwhile
            return LIB
        tmp = f"{LIB}.{os.getpid()}.tmp"
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
               "-Xcompiler", "-fPIC,-O3,-Wall", "-cudart", "static",
               "-I", os.path.join(ROOT, "include"), "-Xptxas", "-v" if verbose else "-O3",
               "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libntp_b200.so")
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
