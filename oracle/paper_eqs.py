"""The paper's component formulas in generator space, from brute-force f and d (oracle pin).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Used only to pin O1
(oracle.dense) to the equations as printed, at N <= 6.

  h_m   = Tr(F_m H)                                   expansion after Eq. 5
  l_p,j = Tr(F_j L_p)                                 Eq. 8, P:188-192 (L_p = c_p I + sum_j l_p,j F_j)
  q_sn  = sum_m f_mns h_m                             Eq. 6
  r_sm  = -1/4 sum_p gamma_p sum_jkl l_j conj(l_k) (z_jlm f_kls + conj(z_klm) f_jls),
          z = f + i d                                 Eq. 10, reading R1
  k_s   = (i/N) sum_p gamma_p sum_jk l_j conj(l_k) f_jks
                                                      Eq. 11, reading R2
  h_eff = -sum_p gamma_p Im(conj(c_p) l_p)            reading R3 (trace of L_p)

R1: Eq. 10 as printed has prefactor -1/2 and never defines z.  With
    z = f + i d (the Alicki-Lendi convention named in BASELINE.json north_star)
    the prefactor that reproduces Tr(F_s L_D(F_m)) is -1/4.  The test
    tests/test_oracle_paper_eqs.py shows both that this reading matches O1 and
    that the printed -1/2 does not.
R2: Eq. 11 as printed omits gamma_p, which Eq. 10 carries; k_s must scale with
    the channel rate (L_D(I/N) = sum_p gamma_p/N [L_p, L_p^+]).
R3: Eq. 8 expands L_p over F_1..F_M only; a dissipator with a trace
    (configs[0], configs[3]) contributes the unitary term -i[H_eff, rho] with
    H_eff = sum_p gamma_p (i/2)(conj(c_p) L_p0 - c_p L_p0^+), c_p = Tr(L_p)/N.
"""
from __future__ import annotations

import numpy as np

from .basis import generators, project_literal


def coefficients(A):
    """(trace part c, generator coefficients Tr(F_j A)) of an N x N matrix."""
    n = A.shape[0]
    return np.trace(A) / n, project_literal(A)


def q_from_h(h, f):
    """Eq. 6: q_sn = sum_m f_mns h_m."""
    return np.einsum("mns,m->sn", f, h)


def r_from_l(l, gamma, f, d, prefactor=-0.25):
    """Eq. 10 with z = f + i d: r_sm = pref * gamma * sum_jkl l_j l*_k (z_jlm f_kls + conj(z_klm) f_jls)."""
    z = f + 1j * d
    t1 = np.einsum("j,k,jlm,kls->sm", l, l.conj(), z, f)
    t2 = np.einsum("j,k,klm,jls->sm", l, l.conj(), z.conj(), f)
    r = prefactor * gamma * (t1 + t2)
    return r


def k_from_l(l, gamma, f, n):
    """Eq. 11 with gamma_p (R2): k_s = (i/N) gamma sum_jk l_j l*_k f_jks."""
    return (1j / n) * gamma * np.einsum("j,k,jks->s", l, l.conj(), f)


def unfold_paper(H, Ls, gammas, f, d, r_prefactor=-0.25, fold_trace=True):
    """Q = Q_H(h + h_eff) + R, K from the paper's Eqs. 6, 10, 11 (dense, small N)."""
    n = H.shape[0]
    _, h = coefficients(H)
    assert np.abs(h.imag).max() < 1e-12
    h = h.real.copy()
    R = np.zeros((n * n - 1, n * n - 1), dtype=np.complex128)
    K = np.zeros(n * n - 1, dtype=np.complex128)
    for L, g in zip(Ls, gammas):
        c, l = coefficients(L)
        if fold_trace:
            h = h - g * np.imag(np.conj(c) * l)
        R += r_from_l(l, g, f, d, r_prefactor)
        K += k_from_l(l, g, f, n)
    Q = q_from_h(h, f) + R
    return Q, K


def generators_count(n):
    return generators(n).shape[0]
