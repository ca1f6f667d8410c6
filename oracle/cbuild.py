"""Build the plain-C oracle (oracle/c/*.c) into oracle/_build/liboracle.so.
Test infrastructure only (CPU baseline + large oracle checks)."""

from __future__ import annotations

import ctypes
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_build", "liboracle.so")


def build() -> str:
    srcs = sorted(glob.glob(os.path.join(HERE, "c", "*.c")))
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(s) for s in srcs):
        return OUT
    cmd = ["gcc", "-O3", "-mavx2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
           "-o", OUT] + srcs + ["-lm"]
    subprocess.run(cmd, check=True)
    return OUT


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I64, F32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_float
        L.oracle_eprop_accumulate_batch.argtypes = [P, P, I64, I64, P, P, P, I64, I64, P, P, P,
                                                    F32, F32, F32]
        L.oracle_eprop_accumulate_batch.restype = None
        L.oracle_lsig_fma.argtypes = [P, P, I64, I64, I64, P]
        L.oracle_lsig_fma.restype = None
        L.oracle_threads.argtypes = []
        L.oracle_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def eprop_accumulate_c(targets, row_length, pre_trace, psi, lsig, eps, ebar, grad, beta, rho,
                       alpha):
    import numpy as np
    for a, dt in ((targets, np.int32), (row_length, np.int32), (pre_trace, np.float32),
                  (psi, np.float32), (lsig, np.float32), (eps, np.float32), (ebar, np.float32),
                  (grad, np.float64)):
        assert a.dtype == dt and a.flags.c_contiguous
    P, S = targets.shape
    B, H = psi.shape
    lib().oracle_eprop_accumulate_batch(targets.ctypes.data, row_length.ctypes.data, P, S,
                                        pre_trace.ctypes.data, psi.ctypes.data, lsig.ctypes.data,
                                        B, H, eps.ctypes.data, ebar.ctypes.data, grad.ctypes.data,
                                        float(beta), float(rho), float(alpha))


def lsig_fma_c(d, w):
    """[B, H] float32 learning signal f32(sum_c d[:, c] * w[c]) with one fma
    per class, classes ascending (the device's order)."""
    import numpy as np
    d = np.ascontiguousarray(d, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    B, C = d.shape
    H = w.shape[1]
    out = np.empty((B, H), np.float32)
    lib().oracle_lsig_fma(d.ctypes.data, w.ctypes.data, B, C, H, out.ctypes.data)
    return out


def threads() -> int:
    """OpenMP threads the C oracle uses (the CPU baseline's core count)."""
    return int(lib().oracle_threads())
