"""Build the host (g++) copy of the device small-LA / sFFT-DT solver sources for CPU tests.

Test infrastructure: the same csrc/*.cuh code the CUDA kernels run, compiled for the
host with contraction disabled, so its numerics can be checked against numpy and the
oracle without a GPU.
"""

import ctypes
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def host_lib():
    global _lib
    if _lib is None:
        out = os.path.join(tempfile.gettempdir(), f"afft_host_{os.getuid()}.so")
        src = os.path.join(HERE, "smallla_host.cpp")
        deps = [src] + [os.path.join(HERE, "..", "..", "paper_2011_05749_b200", "csrc", f)
                        for f in ("smallla.cuh", "oneshot_core.cuh")]
        if not os.path.exists(out) or os.path.getmtime(out) < max(map(os.path.getmtime, deps)):
            subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                            "-o", out, src], check=True)
        lib = ctypes.CDLL(out)
        P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        lib.t_solve_bucket.argtypes = [P, I, I, P, I, I, L, L, L, P, P]
        lib.t_locate.argtypes = [P, I, I, I, L, L, L, P]
        _lib = lib
    return _lib
