"""O1: dense textbook evaluation of the unfold (oracle; N <= ~64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    Q_sm = Tr(F_s L(F_m)),  K_s = Tr(F_s L(I/N))
    L(X) = -i[H, X] + sum_p gamma_p (L_p X L_p^+ - 1/2 {L_p^+ L_p, X})   (Eq. 1)

D_p is written in the paper as 1/2([L, X L^+] + [L X, L^+]); expanding
the two commutators gives L X L^+ - 1/2 (L^+ L X + X L^+ L), which is the form
used here (pinned against the commutator form in tests).

Q(t) = Q0 + eps(t) Q1 with Q0 from (H0, {L_p, gamma_p}) and Q1 from (H1, no
dissipators): the unfold is linear in H (Eq. 6; R10).
"""
from __future__ import annotations

import numpy as np

from .basis import generators


def lindbladian(H, Ls, gammas, X):
    """L(X) for one N x N matrix X (Eq. 1 with D_p in anticommutator form)."""
    out = -1j * (H @ X - X @ H)
    for L, g in zip(Ls, gammas):
        LdL = L.conj().T @ L
        out = out + g * (L @ X @ L.conj().T - 0.5 * (LdL @ X + X @ LdL))
    return out


def lindbladian_commutator_form(H, Ls, gammas, X):
    """L(X) with D_p = 1/2([L, X L^+] + [L X, L^+]) exactly as printed in P:52."""
    out = -1j * (H @ X - X @ H)
    for L, g in zip(Ls, gammas):
        Ld = L.conj().T
        A = X @ Ld
        B = L @ X
        out = out + g * 0.5 * ((L @ A - A @ L) + (B @ Ld - Ld @ B))
    return out


def _lindbladian_batched(H, Ls, gammas, X):
    """L(X_m) for a stack X[m] (same arithmetic as lindbladian())."""
    out = -1j * (H[None] @ X - X @ H[None])
    for L, g in zip(Ls, gammas):
        Ld = L.conj().T
        LdL = Ld @ L
        out = out + g * (L[None] @ X @ Ld[None] - 0.5 * (LdL[None] @ X + X @ LdL[None]))
    return out


def unfold_dense(H, Ls=(), gammas=(), chunk: int = 1024):
    """Dense (Q, K): Q_sm = Tr(F_s L(F_m)), K_s = Tr(F_s L(I/N)).

    H, Ls: dense complex N x N.  Returns real float64 Q (M x M) and K (M,).
    The imaginary parts are asserted to be roundoff (F_s and L(F_m) Hermitian).
    """
    H = np.asarray(H, dtype=np.complex128)
    n = H.shape[0]
    F = generators(n)
    M = F.shape[0]
    Fflat = F.reshape(M, n * n)  # row s: vec(F_s)
    Q = np.empty((M, M), dtype=np.float64)
    maxim = 0.0
    for m0 in range(0, M, chunk):
        LF = _lindbladian_batched(H, Ls, gammas, F[m0:m0 + chunk])  # L(F_m)
        # Tr(F_s L(F_m)) = sum_ij (F_s)_ij (L(F_m))_ji
        LFt = LF.transpose(0, 2, 1).reshape(LF.shape[0], n * n)
        block = Fflat @ LFt.T  # [s, m]
        maxim = max(maxim, float(np.abs(block.imag).max()))
        Q[:, m0:m0 + chunk] = block.real
    LI = lindbladian(H, Ls, gammas, np.eye(n, dtype=np.complex128) / n)
    Kc = np.einsum("sij,ji->s", F, LI)
    scale = max(1.0, float(np.abs(Q).max()))
    assert maxim <= 1e-11 * scale, f"Q imaginary residue {maxim}"
    assert float(np.abs(Kc.imag).max()) <= 1e-11 * scale
    return Q, Kc.real.copy()


def tau_scale(H0, Ls=(), gammas=()):
    """S = ||H0||_F + sum_p gamma_p ||L_p||_F^2 (R6); max|Q0| <= 2 S."""
    s = float(np.linalg.norm(H0))
    for L, g in zip(Ls, gammas):
        s += float(g) * float(np.linalg.norm(L)) ** 2
    return s


TAU_REL = 1e-14


def to_csr(Q: np.ndarray, tau: float):
    """Dense -> CSR keeping |q| > tau (R6).  Returns (row_ptr, col, val, gap)."""
    keep = np.abs(Q) > tau
    rows, cols = np.nonzero(keep)  # row-major => ascending cols within each row
    row_ptr = np.zeros(Q.shape[0] + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    dropped = np.abs(Q[~keep])
    gap = {
        "max_dropped": float(dropped.max()) if dropped.size else 0.0,
        "min_kept": float(np.abs(Q[keep]).min()) if keep.any() else np.inf,
    }
    return row_ptr, cols.astype(np.int32), Q[rows, cols].copy(), gap
