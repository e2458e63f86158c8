"""O3: the unfold of a GKSL generator given by a dense rate matrix A (oracle; F3 / F4).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md Eq. 7 writes the dissipator with a positive semidefinite M x M
rate matrix A = {a_jk} over the basis F_1..F_M:

    L_D(X) = 1/2 sum_jk a_jk ( [F_j, X F_k^+] + [F_j X, F_k^+] )

and P:568-570 asks for this summation with a dense, randomly generated A at N = 100
over > 10^3 realisations.  Expanding the two commutators with
F_k^+ = F_k (the basis is Hermitian, P:135-144 with reading R4):

    L_D(X) = sum_jk a_jk ( F_j X F_k - 1/2 {F_k F_j, X} )

which is the form evaluated here (pinned to the printed commutator form in tests).
With L(X) = -i[H, X] + L_D(X) (Eq. 1), the unfold is the plain definition

    Q_sm = Tr(F_s L(F_m)),   K_s = Tr(F_s L(I/N))

computed with dense matrices (no structure constants).  Cost O(M^2 N^3): N <= ~12.
"""
from __future__ import annotations

import numpy as np

from .basis import generators


def _weights(A, F):
    """B_k = sum_j a_jk F_j (M, N, N) and C = sum_jk a_jk F_k F_j (N, N)."""
    B = np.einsum("jk,jab->kab", A, F)
    C = np.einsum("kab,kbc->ac", F, B)  # sum_k F_k B_k = sum_jk a_jk F_k F_j
    return B, C


def lindbladian_gks(H, A, X):
    """L(X) = -i[H, X] + sum_jk a_jk (F_j X F_k - 1/2 {F_k F_j, X}) for one N x N X."""
    H = np.asarray(H, dtype=np.complex128)
    n = H.shape[0]
    out = -1j * (H @ X - X @ H)
    if A is None:
        return out
    F = generators(n)
    B, C = _weights(np.asarray(A, dtype=np.complex128), F)
    out = out + np.einsum("kab,bc,kcd->ad", B, X, F)  # sum_k B_k X F_k
    return out - 0.5 * (C @ X + X @ C)


def lindbladian_gks_printed(H, A, X):
    """L(X) with L_D exactly as printed in P:183: 1/2 sum a_jk ([F_j, X F_k^+] + [F_j X, F_k^+])."""
    H = np.asarray(H, dtype=np.complex128)
    n = H.shape[0]
    F = generators(n)
    out = -1j * (H @ X - X @ H)
    M = F.shape[0]
    for j in range(M):
        for k in range(M):
            a = A[j, k]
            if a == 0:
                continue
            Fj, Fkd = F[j], F[k].conj().T
            XF = X @ Fkd
            FX = Fj @ X
            out = out + 0.5 * a * ((Fj @ XF - XF @ Fj) + (FX @ Fkd - Fkd @ FX))
    return out


def unfold_gks(H, A=None):
    """Dense (Q, K) of L = -i[H, .] + L_D[A]:  Q_sm = Tr(F_s L(F_m)), K_s = Tr(F_s L(I/N)).

    H: N x N Hermitian; A: M x M Hermitian (PSD for a physical generator) or None.
    Returns real float64 Q (M, M) and K (M,); the imaginary parts are asserted to be
    roundoff (L preserves Hermiticity for Hermitian A).
    """
    H = np.asarray(H, dtype=np.complex128)
    n = H.shape[0]
    F = generators(n)
    M = F.shape[0]
    # L(F_m) for all m at once
    LF = -1j * (np.einsum("ab,mbc->mac", H, F) - np.einsum("mab,bc->mac", F, H))
    LI = np.zeros((n, n), dtype=np.complex128)
    if A is not None:
        A = np.asarray(A, dtype=np.complex128)
        B, C = _weights(A, F)
        # sum_k B_k F_m F_k for every m
        BF = np.einsum("kab,mbc->mkac", B, F)
        LF = LF + np.einsum("mkac,kcd->mad", BF, F)
        LF = LF - 0.5 * (np.einsum("ab,mbc->mac", C, F) + np.einsum("mab,bc->mac", F, C))
        LI = (np.einsum("kab,kbc->ac", B, F) - C) / n  # L_D(I/N) = (sum_k B_k F_k - C)/N
    # Tr(F_s L(F_m)) = sum_ij (F_s)_ij (L(F_m))_ji
    Qc = np.einsum("sij,mji->sm", F, LF)
    Kc = np.einsum("sij,ji->s", F, LI)
    scale = max(1.0, float(np.abs(Qc).max()))
    assert float(np.abs(Qc.imag).max()) <= 1e-11 * scale, "Q imaginary residue"
    assert float(np.abs(Kc.imag).max()) <= 1e-11 * scale, "K imaginary residue"
    return Qc.real.copy(), Kc.real.copy()


def rate_matrix_from_dissipators(Ls, gammas):
    """A = sum_p gamma_p l_p l_p^+ with l_{p,j} = Tr(F_j L_p) (Eq. 8 and the spectral form
    A = sum_p l_p l_p^+ of P:187-189; the L_p must be traceless, reading R3)."""
    Ls = [np.asarray(L, dtype=np.complex128) for L in Ls]
    n = Ls[0].shape[0]
    F = generators(n)
    M = F.shape[0]
    A = np.zeros((M, M), dtype=np.complex128)
    for L, g in zip(Ls, gammas):
        assert abs(np.trace(L)) < 1e-12 * max(1.0, np.abs(L).max()), "traceless L_p only (R3)"
        l = np.einsum("jab,ba->j", F, L)  # Tr(F_j L)
        A += g * np.outer(l, l.conj())
    return A
