"""Pins for oracle O3 (oracle.gks): the unfold of a generator given by a rate matrix A
(Eq. 7).

O3 is pinned to: the printed commutator form of Eq. 7; the N = 2 Bloch
equations (golden) through A = gamma l l^+; O1 (oracle.dense, itself pinned to the
paper's component equations) for A = sum_p gamma_p l_p l_p^+ (the spectral form,
P:187-189); the depolarising closed form A = gamma I (Fierz identity, derived below);
trace and Hermiticity preservation.
"""
import json
import os

import numpy as np
import pytest

from oracle import basis, dense, gks

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(n, rng):
    return rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))


def _herm(n, rng):
    X = _rand(n, rng)
    return (X + X.conj().T) / 2


def _wishart(m, rng, rank=None):
    G = rng.standard_normal((m, rank or m)) + 1j * rng.standard_normal((m, rank or m))
    return G @ G.conj().T / m


@pytest.mark.parametrize("n", [2, 3])
def test_expanded_equals_printed_commutator_form(n):
    rng = np.random.default_rng(40 + n)
    M = n * n - 1
    H, A, X = _herm(n, rng), _wishart(M, rng), _rand(n, rng)
    a = gks.lindbladian_gks(H, A, X)
    b = gks.lindbladian_gks_printed(H, A, X)
    assert np.abs(a - b).max() < 1e-12 * np.abs(a).max()


def test_bloch_n2_through_rate_matrix():
    gold = json.load(open(os.path.join(GOLDEN, "bloch_n2.json")))
    g = gold["gamma"]
    E01 = np.array([[0, 1], [0, 0]], dtype=complex)
    zero = np.zeros((2, 2), complex)
    for name, L in (("amplitude_damping_E01", E01), ("amplitude_damping_E10", E01.T.copy())):
        A = gks.rate_matrix_from_dissipators([L], [g])
        Q, K = gks.unfold_gks(zero, A)
        assert np.abs(Q - np.array(gold["cases"][name]["Q"])).max() < 1e-15, name
        assert np.abs(K - np.array(gold["cases"][name]["K"])).max() < 1e-15, name


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_spectral_form_equals_o1(n):
    rng = np.random.default_rng(50 + n)
    H = _herm(n, rng)
    Ls = []
    for _ in range(3):
        L = _rand(n, rng)
        Ls.append(L - np.trace(L) / n * np.eye(n))  # traceless (R3)
    gs = [0.3, 1.1, 0.05]
    A = gks.rate_matrix_from_dissipators(Ls, gs)
    Q, K = gks.unfold_gks(H, A)
    Qo, Ko = dense.unfold_dense(H, Ls, gs)
    sc = np.abs(Qo).max()
    assert np.abs(Q - Qo).max() < 1e-13 * sc
    assert np.abs(K - Ko).max() < 1e-13 * sc


@pytest.mark.parametrize("n", [2, 3, 6])
def test_depolarising_closed_form(n):
    """A = gamma I_M.  Fierz: sum_j F_j X F_j = Tr(X) I - X/N and sum_j F_j^2 = (M/N) I, so
    L_D(X) = gamma (Tr(X) I - N X): Q_D = -gamma N I_M, L_D(I/N) = 0 -> K = 0."""
    rng = np.random.default_rng(60 + n)
    H = _herm(n, rng)
    M = n * n - 1
    g = 0.37
    Q, K = gks.unfold_gks(H, g * np.eye(M))
    QH, KH = dense.unfold_dense(H)
    assert np.abs(Q - (QH - g * n * np.eye(M))).max() < 1e-13 * max(1.0, np.abs(Q).max())
    assert np.abs(K).max() < 1e-14


@pytest.mark.parametrize("n", [3, 4])
def test_trace_and_hermiticity_preservation(n):
    rng = np.random.default_rng(70 + n)
    M = n * n - 1
    H, A = _herm(n, rng), _wishart(M, rng)
    X = _herm(n, rng)
    LX = gks.lindbladian_gks(H, A, X)
    assert abs(np.trace(LX)) < 1e-12 * np.abs(LX).max()
    assert np.abs(LX - LX.conj().T).max() < 1e-12 * np.abs(LX).max()
    # Q, K reproduce L on a random density matrix: Q v + K = proj(L(rho))  (Eq. 9)
    Q, K = gks.unfold_gks(H, A)
    B = _rand(n, rng)
    rho = B @ B.conj().T
    rho /= np.trace(rho)
    v = basis.project(rho).real
    lhs = Q @ v + K
    rhs = basis.project(gks.lindbladian_gks(H, A, rho)).real
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(rhs).max()


def test_hamiltonian_only_is_skew():
    rng = np.random.default_rng(80)
    H = _herm(4, rng)
    Q, K = gks.unfold_gks(H, None)
    assert np.abs(Q + Q.T).max() < 1e-14 * np.abs(Q).max()
    assert np.abs(K).max() == 0.0
