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
        lib.o2_fetch_abs.argtypes = [P, P]
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
        absv = np.empty(max(nnz, 1), dtype=np.float64)
        lib.o2_fetch_abs(res, _ptr(absv))
        gap = np.empty(4, dtype=np.float64)
        lib.o2_gap(res, _ptr(gap))
    finally:
        lib.o2_free(res)
    return {
        "row_ptr": row_ptr, "col": col[:nnz], "val": val[:nnz], "K": K if with_k else None,
        "absum": absv[:nnz],
        "gap": {"max_dropped": float(gap[0]), "min_kept": float(gap[1]), "max_imag": float(gap[2]),
                "min_margin": float(gap[3])},
        "seconds": seconds,
    }


def unfold_problem(problem, nthreads: int = 0):
    """Q0 (+K) and, if the problem has a drive, Q1, each thresholded per DESIGN.md R6."""
    out = {"Q0": unfold_csr(problem.H0, problem.Ls, problem.gammas, tau_q0(problem), True, nthreads)}
    if problem.H1 is not None:
        out["Q1"] = unfold_csr(problem.H1, (), (), tau_q1(problem), False, nthreads)
    return out


def assert_gap(res, tau: float, factor: float = 1e3):
    """R6: the largest dropped |q| must be < tau/factor and the smallest kept
    > tau*factor (factor 1e3 as adopted; configs where this fails are FLAGGED in DESIGN.md R6
    and checked with assert_margin instead)."""
    gap = res["gap"]
    assert gap["max_dropped"] < tau / factor, f"dropped {gap['max_dropped']} vs tau {tau}"
    assert gap["min_kept"] > tau * factor, f"kept {gap['min_kept']} vs tau {tau}"


MARGIN_MIN = 50.0  # DESIGN.md R6: entries near tau lie >= 50 per-entry roundoff bounds away from it


def assert_margin(res, min_margin: float = MARGIN_MIN):
    """R6, the quantity that protects the pattern: for every entry with |q| <= 1e6 tau (kept or
    dropped), ||q| - tau| >= min_margin * 1e-16 * sum|terms| (sum|terms| = the absolute sum of
    the products that make up the entry, accumulated by O2), i.e. no ordering of the
    floating-point sum can move the entry across tau."""
    m = res["gap"]["min_margin"]
    assert m >= min_margin, f"roundoff margin {m} < {min_margin}"


# Configs on which the adopted R6 gap rule (kept > 1e3 tau) fails, with the measured
# min_kept / tau (R6 "flagged configs"); they are checked with assert_margin.
R6_FLAGGED = {"c3_banded_N512_P4": 543.45, "ring_N256_drive": 138.68, "sparse_N300_s21_P2": 520.36}


def assert_r6(res, tau: float, name: str = ""):
    """The stored-pattern checks of DESIGN.md R6 on an oracle result: the roundoff margin always;
    the 1e3 gap rule unless `name` is a flagged config, whose measured gap is asserted instead
    (within 1 % of the recorded value, so a change is noticed)."""
    assert_margin(res)
    if name in R6_FLAGGED:
        ratio = res["gap"]["min_kept"] / tau
        assert abs(ratio / R6_FLAGGED[name] - 1.0) < 1e-2, f"{name}: min_kept/tau {ratio} changed"
        assert res["gap"]["max_dropped"] < tau / 1e3
    else:
        assert_gap(res, tau)


def assert_entries_close(val_got, res, name: str = "Q"):
    """R7: normwise max |q_gpu - q_oracle| <= 1e-12 max |Q_oracle|, and per entry
    |q_gpu - q_oracle| <= 1e-12 |q_oracle| wherever the entry is well conditioned, cond =
    sum|terms| / |q| <= 100 (sum|terms| from O2).  Returns (normwise error, fraction of entries
    with cond <= 100, their worst relative error)."""
    val_got = np.asarray(val_got)
    ref = res["val"]
    if ref.size == 0:
        return 0.0, 1.0, 0.0
    scale = float(np.abs(ref).max())
    err = np.abs(val_got - ref)
    assert err.max() <= 1e-12 * scale, f"{name}: max err {err.max()} vs 1e-12 * {scale}"
    cond = res["absum"] / np.abs(ref)
    good = cond <= 100.0
    rel = err[good] / np.abs(ref[good])
    worst = float(rel.max()) if rel.size else 0.0
    assert worst <= 1e-12, f"{name}: per-entry rel err {worst} on an entry with cond <= 100"
    return float(err.max() / scale), float(good.mean()), worst


def assert_k_close(k_got, k_ref, what: str = "K", tau: float = 0.0):
    """R7 for K: max |K_gpu - K_oracle| <= 1e-12 max |K_oracle|.  Where K is numerically zero
    (max |K_oracle| <= tau, the R6 threshold of the problem: e.g. Hermitian or diagonal L_p, for
    which K == 0 exactly and the oracle holds only roundoff), max |K_gpu| <= tau; with tau = 0
    that is an exact-zero check."""
    k_got = np.asarray(k_got)
    k_ref = np.asarray(k_ref)
    scale = float(np.abs(k_ref).max()) if k_ref.size else 0.0
    if scale <= tau:
        got = float(np.abs(k_got).max()) if k_got.size else 0.0
        assert got <= tau, f"{what}: K is numerically zero (max |K_oracle| {scale} <= tau {tau}) but GPU has {got}"
        return 0.0
    err = float(np.abs(k_got - k_ref).max())
    assert err <= 1e-12 * scale, f"{what}: max err {err} vs 1e-12 * {scale}"
    return err / scale
