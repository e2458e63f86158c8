"""Input generators: the dimer operators against an independent two-mode Fock construction."""
import numpy as np
import pytest

from workloads import ZCSR, config, dimer_dissipator, dimer_drive, dimer_hamiltonian


def _two_mode(n):
    """b1, b2 on the (n x n)-dim two-mode space with occupations 0..n-1 each, and the
    projector onto the (n-1)-boson sector ordered by a = n1 (Eq. 12)."""
    b = np.diag(np.sqrt(np.arange(1, n)), 1)  # single-mode annihilation
    I = np.eye(n)
    b1, b2 = np.kron(b, I), np.kron(I, b)
    # basis state |n1, n2> has index n1 * n + n2 ; sector n1 + n2 = n-1, ordered by n1
    idx = [a * n + (n - 1 - a) for a in range(n)]
    return b1, b2, idx


@pytest.mark.parametrize("n", [2, 3, 6, 9])
def test_dimer_operators(n):
    b1, b2, idx = _two_mode(n)
    d = lambda A: A.conj().T  # noqa: E731
    n1, n2 = d(b1) @ b1, d(b2) @ b2
    J, U = 1.0, 2.0
    H = -J * (d(b1) @ b2 + d(b2) @ b1) + (U / (2 * n)) * (n1 @ (n1 - np.eye(n * n)) + n2 @ (n2 - np.eye(n * n)))
    L = (d(b1) + d(b2)) @ (b1 - b2)
    sec = np.ix_(idx, idx)
    assert np.abs(dimer_hamiltonian(n).to_dense() - H[sec]).max() < 1e-12
    assert np.abs(dimer_dissipator(n).to_dense() - L[sec]).max() < 1e-12
    assert np.abs(dimer_drive(n).to_dense() - (n2 - n1)[sec]).max() < 1e-12


def test_configs_shapes():
    for i, (n, P, drive) in enumerate([(4, 1, False), (64, 1, False), (256, 1, True), (512, 4, False), (1000, 1, True)]):
        p = config(i)
        assert p.n == n and len(p.Ls) == P and (p.H1 is not None) == drive
        H = p.H0
        assert H.row_ptr[-1] == H.nnz and (np.diff(H.row_ptr) >= 0).all()
        if n <= 512:
            Hd = H.to_dense()
            assert np.abs(Hd - Hd.conj().T).max() == 0.0


def test_zcsr_roundtrip():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((7, 7)) * (rng.random((7, 7)) < 0.3)
    z = ZCSR.from_dense(A + 0j)
    assert np.array_equal(z.to_dense(), A + 0j)
    assert all((np.diff(z.col[z.row_ptr[r]:z.row_ptr[r + 1]]) > 0).all() for r in range(7))


def test_gks_ensemble_recipe():
    """F3 inputs (F3 'ensemble reading'): H Hermitian (GUE), A = G G^+ Hermitian
    positive semidefinite with Tr A = N; seeded, so two draws with one seed agree."""
    import numpy as np

    from workloads import gks_ensemble

    n, B = 4, 3
    H, A = gks_ensemble(n, B, seed=9)
    H2, A2 = gks_ensemble(n, B, seed=9)
    assert np.array_equal(H, H2) and np.array_equal(A, A2)
    for b in range(B):
        assert np.abs(H[b] - H[b].conj().T).max() == 0.0
        assert np.abs(A[b] - A[b].conj().T).max() < 1e-12 * np.abs(A[b]).max()
        assert abs(np.trace(A[b]).real - n) < 1e-12
        assert np.linalg.eigvalsh(A[b]).min() > -1e-12


def test_rank_p_coefficients_band():
    """band > 0: only S_ab / J_ab with b - a <= band (and all D^l) carry a coefficient, so
    L = sum_j l_j F_j is banded (checked through the oracle's basis)."""
    import numpy as np

    from oracle import basis
    from workloads import rank_p_coefficients

    n = 9
    l, g = rank_p_coefficients(n, 2, seed=1, band=2)
    F = basis.generators(n)
    for p in range(2):
        L = np.einsum("j,jab->ab", l[p], F)
        r, c = np.nonzero(np.abs(L) > 0)
        assert np.abs(r - c).max() <= 2
    assert np.all((g >= 0.05) & (g <= 0.5))
