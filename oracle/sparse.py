"""O2 wrapper: trace definition with CSR operators, column by column, plain C + OpenMP.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  See sparse_o2.c for the
definition followed (Eq. 1, Eq. 5, Eq. 9).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sparse_o2.c")
_LIB = os.path.join(_HERE, "liboracle_o2.so")
_lib = None

TAU_REL = 1e-14  # DESIGN.md R6


def build(force: bool = False) -> str:
    """Compile sparse_o2.c into oracle/liboracle_o2.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.o2_unfold.restype = P
        lib.o2_unfold.argtypes = [ctypes.c_int, P, P, P, ctypes.c_int, P, P, P, P,
                                  ctypes.c_double, ctypes.c_int, ctypes.c_int]
        lib.o2_nnz.restype = ctypes.c_int64
        lib.o2_nnz.argtypes = [P]
        lib.o2_gap.argtypes = [P, P]
        lib.o2_fetch.argtypes = [P, P, P, P, P]
        lib.o2_free.argtypes = [P]
        lib.o2_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().o2_max_threads())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def frob(csr) -> float:
    return float(np.sqrt(np.sum(np.abs(csr.val) ** 2)))


def tau_q0(problem) -> float:
    """tau = 1e-14 (||H0||_F + sum_p gamma_p ||L_p||_F^2)  (R6)."""
    s = frob(problem.H0) + sum(g * frob(L) ** 2 for L, g in zip(problem.Ls, problem.gammas))
    return TAU_REL * s


def tau_q1(problem) -> float:
    return TAU_REL * frob(problem.H1)


def unfold_csr(H, Ls=(), gammas=(), tau: float = 0.0, with_k: bool = True, nthreads: int = 0):
    """Q (CSR with |q| > tau) and K for H, {L_p, gamma_p} given as workloads.ZCSR.

    Returns dict(row_ptr, col, val, K, gap={max_dropped, min_kept, max_imag}, seconds).
    """
    lib = _load()
    n = H.n
    keep = []  # keep numpy buffers alive during the call

    def arrs(A):
        rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.col, dtype=np.int32)
        v = np.ascontiguousarray(A.val, dtype=np.complex128)
        keep.extend([rp, ci, v])
        return rp, ci, v

    hrp, hci, hv = arrs(H)
    P = len(Ls)
    lrp = (ctypes.c_void_p * max(P, 1))()
    lci = (ctypes.c_void_p * max(P, 1))()
    lv = (ctypes.c_void_p * max(P, 1))()
    for p, L in enumerate(Ls):
        rp, ci, v = arrs(L)
        lrp[p], lci[p], lv[p] = rp.ctypes.data, ci.ctypes.data, v.ctypes.data
    g = np.ascontiguousarray(np.asarray(gammas, dtype=np.float64).reshape(-1) if P else np.zeros(1))
    t0 = time.perf_counter()
    res = lib.o2_unfold(n, _ptr(hrp), _ptr(hci), _ptr(hv), P,
                        ctypes.cast(lrp, ctypes.c_void_p), ctypes.cast(lci, ctypes.c_void_p),
                        ctypes.cast(lv, ctypes.c_void_p), _ptr(g), float(tau), int(with_k), int(nthreads))
    seconds = time.perf_counter() - t0
    try:
        nnz = int(lib.o2_nnz(res))
        m = n * n - 1
        row_ptr = np.empty(m + 1, dtype=np.int64)
        col = np.empty(max(nnz, 1), dtype=np.int32)
        val = np.empty(max(nnz, 1), dtype=np.float64)
        K = np.empty(m, dtype=np.float64)
        lib.o2_fetch(res, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(K))
        gap = np.empty(3, dtype=np.float64)
        lib.o2_gap(res, _ptr(gap))
    finally:
        lib.o2_free(res)
    return {
        "row_ptr": row_ptr, "col": col[:nnz], "val": val[:nnz], "K": K if with_k else None,
        "gap": {"max_dropped": float(gap[0]), "min_kept": float(gap[1]), "max_imag": float(gap[2])},
        "seconds": seconds,
    }


def unfold_problem(problem, nthreads: int = 0):
    """Q0 (+K) and, if the problem has a drive, Q1, each thresholded per DESIGN.md R6."""
    out = {"Q0": unfold_csr(problem.H0, problem.Ls, problem.gammas, tau_q0(problem), True, nthreads)}
    if problem.H1 is not None:
        out["Q1"] = unfold_csr(problem.H1, (), (), tau_q1(problem), False, nthreads)
    return out


def assert_gap(res, tau: float, factor: float = 1e3):
    """R6: the largest dropped |q| must be < tau/factor and the smallest kept > tau*factor."""
    gap = res["gap"]
    assert gap["max_dropped"] < tau / factor, f"dropped {gap['max_dropped']} vs tau {tau}"
    assert gap["min_kept"] > tau * factor, f"kept {gap['min_kept']} vs tau {tau}"
