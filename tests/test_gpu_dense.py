"""GPU parity of the dense rate-matrix unfold sun_unfold_dense (Eq. 7
P:181-185) against the oracles.

Small N: element by element against O3 (oracle.gks, the trace definition with dense A).
Larger N (ragged against the 32-lane scans, several warps' worth of D^l): the spectral form
A = sum_p gamma_p l_p l_p^+ against O2 (oracle.sparse) on the operators L_p = sum_j l_pj F_j,
and the depolarising closed form A = gamma I (Q = Q_H - gamma N I, K = 0).
Tolerance (R7 reading): normwise, max |Q_gpu - Q_oracle| <= 1e-12 max |Q_oracle|.
"""
import numpy as np
import pytest
import torch

from oracle import basis, gks, sparse
from workloads import ZCSR, gks_ensemble, rank_p_coefficients

pytestmark = pytest.mark.gpu


def _sun():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1812_11626_b200 as sun

    return sun


def _dev(x):
    return torch.tensor(x, dtype=torch.complex128, device="cuda")


def _operator(l, n):
    """L = sum_j l_j F_j for complex coefficients (oracle.basis.reconstruct_fast, real parts)."""
    e = np.eye(n) / n
    return (basis.reconstruct_fast(l.real, n) - e) + 1j * (basis.reconstruct_fast(l.imag, n) - e)


def _csr_dense(r, m):
    Q = np.zeros((m, m))
    rp, c, v = r["row_ptr"], r["col"], r["val"]
    for s in range(m):
        Q[s, c[rp[s]:rp[s + 1]]] = v[rp[s]:rp[s + 1]]
    return Q


@pytest.mark.parametrize("n,batch", [(2, 3), (3, 2), (4, 2), (5, 1), (7, 2)])
def test_dense_vs_o3(n, batch):
    sun = _sun()
    H, A = gks_ensemble(n, batch, seed=100 + n)
    Q, K = sun.unfold_dense(_dev(H), _dev(A))
    torch.cuda.synchronize()
    Q, K = Q.cpu().numpy(), K.cpu().numpy()
    for b in range(batch):
        Qo, Ko = gks.unfold_gks(H[b], A[b])
        sc = np.abs(Qo).max()
        assert np.abs(Q[b] - Qo).max() <= 1e-12 * sc, (n, b)
        assert np.abs(K[b] - Ko).max() <= 1e-12 * sc, (n, b)


@pytest.mark.parametrize("n", [2, 6])
def test_dense_hamiltonian_only(n):
    sun = _sun()
    H, _ = gks_ensemble(n, 1, seed=7)
    Q, K = sun.unfold_dense(_dev(H[0]), None)
    Qo, Ko = gks.unfold_gks(H[0], None)
    assert np.abs(Q.cpu().numpy() - Qo).max() <= 1e-12 * np.abs(Qo).max()
    assert np.abs(K.cpu().numpy()).max() == 0.0


def test_dense_chunking_is_bitwise_stable():
    sun = _sun()
    n, batch = 5, 4
    H, A = gks_ensemble(n, batch, seed=3)
    Hd, Ad = _dev(H), _dev(A)
    Q1, K1 = sun.unfold_dense(Hd, Ad, chunk=1)
    Q4, K4 = sun.unfold_dense(Hd, Ad, chunk=4)
    assert torch.equal(Q1, Q4) and torch.equal(K1, K4)
    # one realisation alone gives the same bits as inside the batch
    Qs, Ks = sun.unfold_dense(Hd[2], Ad[2])
    assert torch.equal(Qs, Q4[2]) and torch.equal(Ks, K4[2])


@pytest.mark.parametrize("n,P", [(17, 3), (32, 2), (33, 2), (40, 3)])
def test_dense_spectral_form_vs_o2(n, P):
    """A = sum_p gamma_p l_p l_p^+ (rank P, dense in the F basis) against O2 on L_p = sum_j l_pj F_j."""
    sun = _sun()
    m = n * n - 1
    l, g = rank_p_coefficients(n, P, seed=n)
    A = np.zeros((m, m), dtype=np.complex128)
    for p in range(P):
        A += g[p] * np.outer(l[p], l[p].conj())
    rng = np.random.default_rng(500 + n)
    X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    H = (X + X.conj().T) / 2
    Q, K = sun.unfold_dense(_dev(H), _dev(A))
    Q, K = Q.cpu().numpy(), K.cpu().numpy()
    # oracle side: the operators L_p = sum_j l_pj F_j (traceless), through O2's trace definition
    Ls = [ZCSR.from_dense(_operator(l[p], n)) for p in range(P)]
    r = sparse.unfold_csr(ZCSR.from_dense(H), Ls, list(g), tau=0.0)
    Qo = _csr_dense(r, m)
    sc = np.abs(Qo).max()
    assert np.abs(Q - Qo).max() <= 1e-12 * sc
    assert np.abs(K - r["K"]).max() <= 1e-12 * sc


def test_dense_banded_spectral_form_vs_o2_full_size():
    """N = 100 (the F3 size): A = sum_p gamma_p l_p l_p^+ with l_p supported on a band
    of generators (so L_p = sum_j l_pj F_j is banded and O2 is fast) against O2."""
    sun = _sun()
    n, P = 100, 2
    m = n * n - 1
    l, g = rank_p_coefficients(n, P, seed=7, band=2)
    Ad = torch.zeros((m, m), dtype=torch.complex128, device="cuda")
    for p in range(P):
        lp = _dev(l[p])
        Ad += g[p] * torch.outer(lp, lp.conj())
    rng = np.random.default_rng(900)
    X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    H = (X + X.conj().T) / 2
    Q, K = sun.unfold_dense(_dev(H), Ad)
    Q, K = Q.cpu().numpy(), K.cpu().numpy()
    Ls = [ZCSR.from_dense(_operator(l[p], n)) for p in range(P)]
    r = sparse.unfold_csr(ZCSR.from_dense(H), Ls, list(g), tau=0.0)
    Qo = _csr_dense(r, m)
    sc = np.abs(Qo).max()
    assert np.abs(Q - Qo).max() <= 1e-12 * sc
    assert np.abs(K - r["K"]).max() <= 1e-12 * sc


@pytest.mark.parametrize("n", [16, 32, 40, 64, 100])
def test_dense_depolarising_closed_form(n):
    """A = gamma I: L_D(X) = gamma (Tr(X) I - N X) (Fierz), so Q = Q_H - gamma N I and K = 0."""
    sun = _sun()
    m = n * n - 1
    gam = 0.25
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    H = (X + X.conj().T) / 2
    A = torch.eye(m, dtype=torch.complex128, device="cuda") * gam
    Q, K = sun.unfold_dense(_dev(H), A)
    r = sparse.unfold_csr(ZCSR.from_dense(H), [], [], tau=0.0)
    Qo = _csr_dense(r, m) - gam * n * np.eye(m)
    Q = Q.cpu().numpy()
    assert np.abs(Q - Qo).max() <= 1e-12 * np.abs(Qo).max()
    assert np.abs(K.cpu().numpy()).max() <= 1e-12 * np.abs(Qo).max()


def test_dense_errors():
    sun = _sun()
    H = torch.zeros((1, 3, 3), dtype=torch.complex128, device="cuda")
    with pytest.raises(sun.SunError):
        sun.unfold_dense(H, None, work=torch.empty(4, dtype=torch.complex128, device="cuda"))
    assert sun.dense_work_bytes(1) == 0 and sun.dense_work_bytes(2000) == 0
    assert sun.dense_work_bytes(3, 2) == 2 * sun.dense_work_bytes(3, 1)
    # batch 0 is a no-op
    Q, K = sun.unfold_dense(torch.zeros((0, 3, 3), dtype=torch.complex128, device="cuda"), None)
    assert Q.numel() == 0 and K.numel() == 0
