"""SU(N) generator basis, projections and brute-force structure constants (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Basis (§II), 0-based indices a < b in [0, N), l in [1, N-1]:
    S_ab = (E_ab + E_ba)/sqrt(2)
    J_ab = -i (E_ab - E_ba)/sqrt(2)
    D^l  = (sum_{c<l} E_cc - l E_ll)/sqrt(l(l+1))
The stray factor i printed in D^l is dropped (R4): with it
D^l would be anti-Hermitian and Tr(F_i F_k) = delta_ik would fail.

Canonical order (R5): all S_ab in lexicographic (a, b)
order, then all J_ab in the same order, then D^1..D^{N-1}:
    idx(S_ab) = p(a,b),  idx(J_ab) = NP + p(a,b),  idx(D^l) = 2 NP + l - 1,
    p(a,b) = a(2N-a-1)/2 + (b-a-1),  NP = N(N-1)/2.
"""
from __future__ import annotations

import functools

import numpy as np

SQRT2 = np.sqrt(2.0)


def num_pairs(n: int) -> int:
    return n * (n - 1) // 2


def pair_index(n: int, a: int, b: int) -> int:
    """p(a,b) for 0 <= a < b < n (lexicographic rank of the pair)."""
    assert 0 <= a < b < n
    return a * (2 * n - a - 1) // 2 + (b - a - 1)


def gen_index(n: int, kind: str, a: int, b: int = -1) -> int:
    """Linear index of S_ab ('S'), J_ab ('J') or D^a ('D', a = l in [1, n-1])."""
    npairs = num_pairs(n)
    if kind == "S":
        return pair_index(n, a, b)
    if kind == "J":
        return npairs + pair_index(n, a, b)
    if kind == "D":
        assert 1 <= a <= n - 1
        return 2 * npairs + a - 1
    raise ValueError(kind)


@functools.lru_cache(maxsize=None)
def labels(n: int):
    """List of (kind, a, b) for s = 0..M-1 (for D: ('D', l, -1))."""
    out = []
    for kind in ("S", "J"):
        for a in range(n):
            for b in range(a + 1, n):
                out.append((kind, a, b))
    for l in range(1, n):
        out.append(("D", l, -1))
    return out


def generator(n: int, kind: str, a: int, b: int = -1) -> np.ndarray:
    """Dense N x N matrix of one generator (P:136-140 with the R4 reading)."""
    F = np.zeros((n, n), dtype=np.complex128)
    if kind == "S":
        F[a, b] = F[b, a] = 1.0 / SQRT2
    elif kind == "J":
        F[a, b] = -1j / SQRT2
        F[b, a] = 1j / SQRT2
    elif kind == "D":
        l = a
        F[np.arange(l), np.arange(l)] = 1.0
        F[l, l] = -float(l)
        F /= np.sqrt(l * (l + 1.0))
    else:
        raise ValueError(kind)
    return F


@functools.lru_cache(maxsize=8)
def generators(n: int) -> np.ndarray:
    """All M generators as a dense (M, N, N) complex128 array, canonical order."""
    return np.stack([generator(n, *lab) for lab in labels(n)])


def project_literal(A: np.ndarray) -> np.ndarray:
    """c_s = Tr(F_s A) for all s, by the literal dense trace (Eq. 5 inverse)."""
    n = A.shape[0]
    F = generators(n)
    return np.einsum("sij,ji->s", F, A)


def project(A: np.ndarray) -> np.ndarray:
    """c_s = Tr(F_s A) for all s, evaluating the trace only on F_s's support.

    Tr(S_ab A) = (A_ba + A_ab)/sqrt2 ; Tr(J_ab A) = (-i A_ba + i A_ab)/sqrt2 ;
    Tr(D^l A) = (sum_{c<l} A_cc - l A_ll)/sqrt(l(l+1)).   (Pinned to
    project_literal in tests.)  Returns complex; real for Hermitian A.
    """
    n = A.shape[0]
    iu, ju = np.triu_indices(n, 1)  # lexicographic (a, b) order == p(a,b)
    up, lo = A[iu, ju], A[ju, iu]
    cS = (lo + up) / SQRT2
    cJ = (-1j * lo + 1j * up) / SQRT2
    d = np.diag(A)
    l = np.arange(1, n)
    prefix = np.cumsum(d)[:-1]  # sum_{c<l} A_cc for l = 1..n-1
    cD = (prefix - l * d[1:]) / np.sqrt(l * (l + 1.0))
    return np.concatenate([cS, cJ, cD])


def reconstruct(v: np.ndarray, n: int) -> np.ndarray:
    """rho = I/N + sum_j v_j F_j (Eq. 5)."""
    F = generators(n)
    return np.eye(n, dtype=np.complex128) / n + np.einsum("s,sij->ij", v, F)


def reconstruct_fast(v: np.ndarray, n: int) -> np.ndarray:
    """Same as reconstruct() without forming all generators (for large N)."""
    npairs = num_pairs(n)
    iu, ju = np.triu_indices(n, 1)
    vS, vJ, vD = v[:npairs], v[npairs:2 * npairs], v[2 * npairs:]
    rho = np.zeros((n, n), dtype=np.complex128)
    rho[iu, ju] = (vS - 1j * vJ) / SQRT2
    rho[ju, iu] = (vS + 1j * vJ) / SQRT2
    l = np.arange(1, n)
    w = vD / np.sqrt(l * (l + 1.0))  # coefficient of (sum_{c<l} E_cc - l E_ll)
    # diag_c = 1/N + sum_{l > c} w_l - c w_c (the -l E_ll term for l = c >= 1)
    suffix = np.concatenate([np.cumsum(w[::-1])[::-1], [0.0]])  # suffix[c] = sum_{l>=c+1} w_l
    diag = np.full(n, 1.0 / n) + suffix
    diag[1:] -= l * w
    rho[np.arange(n), np.arange(n)] = diag
    return rho


def structure_constants(n: int):
    """Brute-force f_mns, d_mns over all triples (Eq. 4).

    f_mns = -i Tr(F_s [F_m, F_n]),  d_mns = Tr(F_s {F_m, F_n}).  Dense (M,M,M).
    """
    F = generators(n)
    prod = np.einsum("mij,njk->mnik", F, F)  # F_m F_n
    comm = prod - prod.transpose(1, 0, 2, 3)
    anti = prod + prod.transpose(1, 0, 2, 3)
    f = -1j * np.einsum("sij,mnji->mns", F, comm)
    d = np.einsum("sij,mnji->mns", F, anti)
    assert np.abs(f.imag).max() < 1e-12 and np.abs(d.imag).max() < 1e-12
    return f.real.copy(), d.real.copy()
