"""Pins for the unfold oracles O1 (oracle.dense) and O2 (oracle.sparse).

O1 is pinned to: the N=2 Bloch equations (golden), the paper's own component
formulas Eq. 6 / Eq. 10 (R1) / Eq. 11 (R2) with brute-force f, d, trace
preservation, the rho-level apply check and special cases.  O2 is pinned to O1
(bit-exact pattern, values) and to the apply check at the BASELINE sizes.
"""
import json
import os

import numpy as np
import scipy.sparse as sp
import pytest

from oracle import basis, dense, paper_eqs, sparse
from workloads import (ZCSR, banded_random_problem, config, dense_random_problem, dimer_problem)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(n, rng):
    return rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))


def test_bloch_n2_closed_forms():
    gold = json.load(open(os.path.join(GOLDEN, "bloch_n2.json")))
    w, g = gold["omega"], gold["gamma"]
    sz = np.diag([1.0, -1.0]).astype(complex)
    E01 = np.array([[0, 1], [0, 0]], dtype=complex)
    zero = np.zeros((2, 2), complex)
    cases = {
        "hamiltonian": (w / 2 * sz, [], []),
        "amplitude_damping_E01": (zero, [E01], [g]),
        "amplitude_damping_E10": (zero, [E01.T.copy()], [g]),
        "dephasing": (zero, [sz], [g]),
    }
    for name, (H, Ls, gs) in cases.items():
        Q, K = dense.unfold_dense(H, Ls, gs)
        assert np.abs(Q - np.array(gold["cases"][name]["Q"])).max() < 1e-15, name
        assert np.abs(K - np.array(gold["cases"][name]["K"])).max() < 1e-15, name
        r = sparse.unfold_csr(ZCSR.from_dense(H), [ZCSR.from_dense(L) for L in Ls], gs, tau=1e-15)
        Qs = np.zeros((3, 3))
        for s in range(3):
            lo, hi = r["row_ptr"][s], r["row_ptr"][s + 1]
            Qs[s, r["col"][lo:hi]] = r["val"][lo:hi]
        assert np.abs(Qs - np.array(gold["cases"][name]["Q"])).max() < 1e-15, name
        assert np.abs(r["K"] - np.array(gold["cases"][name]["K"])).max() < 1e-15, name


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_o1_equals_paper_equations(n):
    rng = np.random.default_rng(10 + n)
    A = _rand(n, rng)
    H = (A + A.conj().T) / 2
    Ls = [_rand(n, rng), _rand(n, rng)]  # with traces: exercises reading R3
    gs = [0.7, 0.2]
    f, d = basis.structure_constants(n)
    Q, K = dense.unfold_dense(H, Ls, gs)
    Qp, Kp = paper_eqs.unfold_paper(H, Ls, gs, f, d)
    scale = np.abs(Q).max()
    assert np.abs(Qp.imag).max() < 1e-13 * scale and np.abs(Kp.imag).max() < 1e-13 * scale
    assert np.abs(Q - Qp.real).max() < 1e-13 * scale
    assert np.abs(K - Kp.real).max() < 1e-13 * scale
    # the readings matter: printed -1/2 (R1), Eq. 11 without gamma (R2), no trace fold-in (R3)
    Qh, _ = paper_eqs.unfold_paper(H, Ls, gs, f, d, r_prefactor=-0.5)
    assert np.abs(Q - Qh.real).max() > 1e-3 * scale
    Qn, _ = paper_eqs.unfold_paper(H, Ls, gs, f, d, fold_trace=False)
    assert np.abs(Q - Qn.real).max() > 1e-3 * scale
    Kg = sum(paper_eqs.k_from_l(basis.project_literal(L), 1.0, f, n) for L in Ls)
    assert np.abs(K - Kg.real).max() > 1e-3 * np.abs(K).max()


@pytest.mark.parametrize("n", [2, 3, 6])
def test_o1_hamiltonian_part_skew_and_specials(n):
    rng = np.random.default_rng(n)
    A = _rand(n, rng)
    H = (A + A.conj().T) / 2
    Q, K = dense.unfold_dense(H)
    assert np.abs(Q + Q.T).max() < 1e-13 * np.abs(Q).max()  # Q^T = -Q
    assert np.abs(K).max() == 0.0
    # gamma = 0 -> no dissipative part; Hermitian L -> K = 0; additivity over channels
    L1, L2 = _rand(n, rng), _rand(n, rng)
    Q0, _ = dense.unfold_dense(H, [L1], [0.0])
    assert np.abs(Q0 - Q).max() < 1e-14
    Lh = L1 + L1.conj().T
    _, Kh = dense.unfold_dense(H, [Lh], [0.3])
    assert np.abs(Kh).max() < 1e-13
    Qa, Ka = dense.unfold_dense(H, [L1, L2], [0.3, 0.4])
    Q1_, K1_ = dense.unfold_dense(H, [L1], [0.3])
    Q2_, K2_ = dense.unfold_dense(0 * H, [L2], [0.4])
    assert np.abs(Qa - (Q1_ + Q2_)).max() < 1e-12 * np.abs(Qa).max()
    assert np.abs(Ka - (K1_ + K2_)).max() < 1e-12 * np.abs(Ka).max()


@pytest.mark.parametrize("n", [2, 3, 5])
def test_lindbladian_forms_and_trace_preservation(n):
    rng = np.random.default_rng(n + 100)
    A = _rand(n, rng)
    H = (A + A.conj().T) / 2
    Ls = [_rand(n, rng)]
    X = _rand(n, rng)
    a = dense.lindbladian(H, Ls, [0.4], X)
    b = dense.lindbladian_commutator_form(H, Ls, [0.4], X)
    assert np.abs(a - b).max() < 1e-13
    assert abs(np.trace(a)) < 1e-13  # Tr L(X) = 0
    # => the identity component of L(F_m) vanishes: sum over a Q column of Tr(I L(F_m)) = 0
    F = basis.generators(n)
    for m in range(F.shape[0]):
        assert abs(np.trace(dense.lindbladian(H, Ls, [0.4], F[m]))) < 1e-13


def _random_density(n, rng):
    B = _rand(n, rng)
    rho = B @ B.conj().T
    return rho / np.trace(rho)


def _apply_csr(r, v):
    rp, ci, val = r["row_ptr"], r["col"], r["val"]
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    out = np.zeros(len(rp) - 1)
    np.add.at(out, rows, val * v[ci])
    return out


@pytest.mark.parametrize("n", [2, 4, 7])
def test_apply_check_dense(n):
    """dv/dt = Q v + K equals the coefficients of L(rho) (Eq. 9)."""
    rng = np.random.default_rng(n + 7)
    A = _rand(n, rng)
    H = (A + A.conj().T) / 2
    Ls = [_rand(n, rng)]
    Q, K = dense.unfold_dense(H, Ls, [0.6])
    for _ in range(3):
        rho = _random_density(n, rng)
        v = basis.project(rho).real
        lhs = Q @ v + K
        rhs = basis.project(dense.lindbladian(H, Ls, [0.6], rho))
        assert np.abs(rhs.imag).max() < 1e-13
        assert np.abs(lhs - rhs.real).max() < 1e-12 * max(1, np.abs(rhs).max())


CASES = [
    dense_random_problem(2, seed=1),
    dense_random_problem(3, seed=2, P=2),
    dense_random_problem(6, seed=3),
    dimer_problem(2, True), dimer_problem(3, True), dimer_problem(7, True), dimer_problem(16, True),
    banded_random_problem(9, seed=4, wH=2, wL=1, P=2, drive_w=1),
    banded_random_problem(20, seed=5),
    config(0),
]


@pytest.mark.parametrize("prob", CASES, ids=lambda p: p.name)
def test_o2_equals_o1(prob):
    H = prob.H0.to_dense()
    Ls = [L.to_dense() for L in prob.Ls]
    Q, K = dense.unfold_dense(H, Ls, prob.gammas)
    tau = sparse.tau_q0(prob)
    rp, ci, val, gap = dense.to_csr(Q, tau)
    r = sparse.unfold_csr(prob.H0, prob.Ls, prob.gammas, tau)
    assert np.array_equal(rp, r["row_ptr"]) and np.array_equal(ci, r["col"])
    assert np.abs(val - r["val"]).max() <= 1e-13 * np.abs(val).max()
    sparse.assert_k_close(r["K"], K, prob.name + ":K", tau)
    assert np.abs(K - r["K"]).max() <= 1e-13 * np.abs(K).max() or np.abs(K).max() <= tau
    sparse.assert_r6(r, tau, prob.name)
    if prob.H1 is not None:
        Q1, _ = dense.unfold_dense(prob.H1.to_dense())
        t1 = sparse.tau_q1(prob)
        rp1, ci1, v1, _ = dense.to_csr(Q1, t1)
        r1 = sparse.unfold_csr(prob.H1, (), (), t1, with_k=False)
        assert np.array_equal(rp1, r1["row_ptr"]) and np.array_equal(ci1, r1["col"])
        assert np.abs(v1 - r1["val"]).max() <= 1e-13 * np.abs(v1).max()


def test_o2_c1_matches_o1():
    prob = config(1)
    H = prob.H0.to_dense()
    Q, K = dense.unfold_dense(H, [L.to_dense() for L in prob.Ls], prob.gammas)
    tau = sparse.tau_q0(prob)
    rp, ci, val, _ = dense.to_csr(Q, tau)
    r = sparse.unfold_csr(prob.H0, prob.Ls, prob.gammas, tau)
    assert np.array_equal(rp, r["row_ptr"]) and np.array_equal(ci, r["col"])
    assert np.abs(val - r["val"]).max() <= 1e-12 * np.abs(val).max()
    sparse.assert_k_close(r["K"], K, prob.name + ":K", tau)


def _dense_lindblad_coeffs(prob, rho, eps):
    n = prob.n
    H = prob.H0.to_dense()
    if prob.H1 is not None:
        H = H + eps * prob.H1.to_dense()
    out = -1j * (H @ rho - rho @ H)
    for L, g in zip(prob.Ls, prob.gammas):
        Ld = L.to_dense()
        LdL = Ld.conj().T @ Ld
        out += g * (Ld @ rho @ Ld.conj().T - 0.5 * (LdL @ rho + rho @ LdL))
    return basis.project(out).real


@pytest.mark.parametrize("idx", [2, 3])
def test_o2_apply_check_baseline_configs(idx):
    """Q(t) v + K = proj L(t)(rho) at BASELINE configs[2], configs[3] (global invariant)."""
    prob = config(idx)
    r = sparse.unfold_problem(prob)
    sparse.assert_r6(r["Q0"], sparse.tau_q0(prob), prob.name)
    rng = np.random.default_rng(idx)
    rho = _random_density(prob.n, rng)
    v = basis.project(rho).real
    eps = 1.0 + 1.5 * np.sin(0.37)
    lhs = _apply_csr(r["Q0"], v) + r["Q0"]["K"]
    if "Q1" in r:
        lhs = lhs + eps * _apply_csr(r["Q1"], v)
    rhs = _dense_lindblad_coeffs(prob, rho, eps)
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(rhs).max()


def test_o2_nnz_regression_dimer_banded():
    """Closed-form nnz fits measured by SURVEY.md Appendix B (regression pin, not a paper value)."""
    for n in (6, 16, 34):  # the survey fit holds for even N (all BASELINE dimers)
        r = sparse.unfold_problem(dimer_problem(n, True))
        assert len(r["Q0"]["col"]) == (37 * n * n - 103 * n + 70) // 2
        assert len(r["Q1"]["col"]) == n * (n - 1)
    for n in (16, 32):
        p = banded_random_problem(n, seed=3)
        r = sparse.unfold_csr(p.H0, p.Ls, p.gammas, sparse.tau_q0(p))
        assert len(r["col"]) == int(70.5 * n * n - 322.5 * n + 379)


def _labels_of(n, m):
    """(kind, a, b) of generator index m (R5)."""
    np_ = n * (n - 1) // 2
    if m < 2 * np_:
        p = m if m < np_ else m - np_
        a = 0
        while p >= n - 1 - a:
            p -= n - 1 - a
            a += 1
        return ("S" if m < np_ else "J"), a, a + 1 + p
    return "D", m - 2 * np_ + 1, -1


@pytest.mark.parametrize("idx,nrand,nd", [(2, 200, 255), (3, 60, 30), (4, 24, 8)])
def test_o2_columns_match_o1_samples(idx, nrand, nd):
    """O2 against the textbook definition O1 (Q_sm = Tr(F_s L(F_m)), dense
    matrices) on sampled columns at the BASELINE sizes c2-c4 where O1 cannot run
    whole: random S/J columns plus D columns (all at c2).  Pattern of each column bit-exact under
    R6, values within 1e-12 max|Q| (R7)."""
    prob = config(idx)
    n, m = prob.n, prob.m
    r = sparse.unfold_problem(prob)["Q0"]
    tau = sparse.tau_q0(prob)
    Qc = sp.csr_matrix((r["val"], r["col"], r["row_ptr"]), shape=(m, m)).tocsc()
    scale = np.abs(r["val"]).max()
    H = prob.H0.to_dense()
    Ls = [L.to_dense() for L in prob.Ls]
    rng = np.random.default_rng(100 + idx)
    cols = list(rng.choice(n * (n - 1), size=nrand, replace=False))
    dcols = n * (n - 1) + np.linspace(0, n - 2, nd).round().astype(int)
    for mcol in cols + list(dcols):
        kind, a, b = _labels_of(n, int(mcol))
        F = basis.generator(n, kind, a, b)
        col = basis.project(dense.lindbladian(H, Ls, prob.gammas, F))
        assert np.abs(col.imag).max() <= 1e-12 * scale
        col = col.real
        keep = np.nonzero(np.abs(col) > tau)[0]
        lo, hi = Qc.indptr[mcol], Qc.indptr[mcol + 1]
        assert np.array_equal(Qc.indices[lo:hi], keep), (idx, mcol, kind, a, b)
        assert np.abs(Qc.data[lo:hi] - col[keep]).max(initial=0.0) <= 1e-12 * scale
        assert np.abs(np.delete(col, keep)).max(initial=0.0) < tau
