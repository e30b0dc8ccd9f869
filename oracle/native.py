"""ctypes wrapper of ``oracle/liboracle.so`` (the C restatement) — TEST ONLY.

Built by ``build()`` (recipe: oracle/Makefile, or ``python -m oracle.native``).
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
SRC = HERE / "stc_oracle.c"
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11"]

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["gcc", *CFLAGS, "-o", str(LIB), str(SRC), "-lm"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        I = ctypes.c_int64
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_spmm_csr_f64.argtypes = [I, I, P, P, P, P, I, P, ctypes.c_int, P]
        L.orc_sddmm_csr_f64.argtypes = [I, P, P, P, P, P, I, I, P]
        L.orc_segsoftmax_f64.argtypes = [I, P, P, P]
        L.orc_mttkrp_f64.argtypes = [I, P, P, P, P, P, P, I, ctypes.c_int, P]
        _lib = L
    return _lib


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def spmm_csr(rowptr, colidx, vals, B, addend=None, relu=False, rows=None):
    """C (rows r0..r1 of) = act(A @ B + addend), float64, reference order."""
    rowptr, colidx, vals, B = _i64(rowptr), _i64(colidx), _f64(vals), _f64(B)
    m = len(rowptr) - 1
    r0, r1 = (0, m) if rows is None else rows
    k = B.shape[1]
    C = np.empty((r1 - r0, k), dtype=np.float64)
    D = None if addend is None else _f64(addend)
    lib().orc_spmm_csr_f64(r0, r1, _p(rowptr), _p(colidx), _p(vals), _p(B), k, _p(D), int(relu), _p(C))
    return C


def sddmm_csr(rowptr, colidx, maskvals, Q, K, tile=64):
    rowptr, colidx, Q, K = _i64(rowptr), _i64(colidx), _f64(Q), _f64(K)
    mv = None if maskvals is None else _f64(maskvals)
    S = np.empty(len(colidx), dtype=np.float64)
    lib().orc_sddmm_csr_f64(len(rowptr) - 1, _p(rowptr), _p(colidx), _p(mv), _p(Q), _p(K), Q.shape[1],
                            0 if tile is None else tile, _p(S))
    return S


def segment_softmax(rowptr, S):
    rowptr, S = _i64(rowptr), _f64(S)
    P = np.empty_like(S)
    lib().orc_segsoftmax_f64(len(rowptr) - 1, _p(rowptr), _p(S), _p(P))
    return P


def mttkrp(seg_ptr, j, k, vals, B, C, b_first=True):
    seg_ptr, j, k, vals, B, C = _i64(seg_ptr), _i64(j), _i64(k), _f64(vals), _f64(B), _f64(C)
    n_seg = len(seg_ptr) - 1
    R = B.shape[1]
    M = np.empty((n_seg, R), dtype=np.float64)
    lib().orc_mttkrp_f64(n_seg, _p(seg_ptr), _p(j), _p(k), _p(vals), _p(B), _p(C), R, int(b_first), _p(M))
    return M


if __name__ == "__main__":
    print(build(force=True))
