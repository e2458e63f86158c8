"""GPU parity of the propagation rows against oracle.propagate.

F1: sun_rk4 (fixed-step RK4 of dv/dt = (Q0 + eps(t) Q1) v + K) vs RK4 on rho (Eq. 1) projected
(small N), and vs RK4 on v with the oracle's O2 matrices (BASELINE sizes).  F2: sun_expand_state
vs Tr(F_s rho); sun_state_diag vs diag(rho).  Tolerance: normwise 1e-12 of max|v| (RK4 adds
O(steps) roundings of size 1e-16 |Q| |v| h)."""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import basis, propagate, sparse
from workloads import ZCSR, banded_random_problem, config, dimer_problem

pytestmark = pytest.mark.gpu


def _sun():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1812_11626_b200 as sun

    return sun


def _dense_random_rho(n, seed):
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    rho = B @ B.conj().T
    return rho / np.trace(rho)


@pytest.mark.parametrize("n", [2, 6, 33, 100])
def test_state_reconstruct(n):
    """rho(T) (Step 3.2): sun_state_reconstruct(v) against oracle basis.reconstruct(v) and
    against the density matrix v was projected from (Eq. 5 is an isometry for Tr rho = 1)."""
    sun = _sun()
    rho = _dense_random_rho(n, 40 + n)
    v = basis.project(rho).real
    got = sun.state_reconstruct(torch.tensor(v, device="cuda"), n).cpu().numpy()
    ref = basis.reconstruct_fast(v, n)
    assert np.abs(got - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max())
    assert np.abs(got - rho).max() <= 1e-13 * max(1.0, np.abs(rho).max())


def test_expand_state_and_populations():
    sun = _sun()
    for n, seed in ((2, 0), (6, 1), (33, 2)):
        rho = _dense_random_rho(n, seed)
        v = sun.expand_state(ZCSR.from_dense(rho)).cpu().numpy()
        ref = basis.project(rho).real
        assert np.abs(v - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max())
        d = sun.state_diag(torch.tensor(ref, device="cuda"), n).cpu().numpy()
        assert np.abs(d - np.diag(rho).real).max() <= 1e-14
    # the paper's initial state |0><0| at N = 1000
    n = 1000
    rho0 = ZCSR.from_triplets(n, [0], [0], [1.0])
    v = sun.expand_state(rho0)
    d = sun.state_diag(v, n).cpu().numpy()
    assert abs(d[0] - 1.0) < 1e-13 and np.abs(d[1:]).max() < 1e-13


def _csr_np(q, m):
    return sp.csr_matrix((q["val"], q["col"], q["row_ptr"]), shape=(m, m))


@pytest.mark.parametrize("n", [3, 8])
def test_rk4_matches_rk4_on_rho(n):
    sun = _sun()
    prob = dimer_problem(n, True)
    Q0, Q1, K = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    rho0 = np.zeros((n, n), complex)
    rho0[0, 0] = 1.0
    v = sun.expand_state(ZCSR.from_dense(rho0))
    h, steps, t0 = 0.05, 20, 0.3
    sun.rk4(Q0, Q1, K, v, h, steps, t0=t0, eps0=1.0, eps1=1.5, omega=1.0)
    rho = propagate.rk4_rho(prob.H0.to_dense(), prob.H1.to_dense(), [L.to_dense() for L in prob.Ls], prob.gammas,
                            rho0, t0, h, steps, eps0=1.0, eps1=1.5, omega=1.0)
    ref = basis.project(rho).real
    assert np.abs(v.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("idx", [2, 4])
def test_rk4_matches_oracle_sparse_rk4_at_baseline_sizes(idx):
    sun = _sun()
    prob = config(idx)
    Q0, Q1, K = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    ref = sparse.unfold_problem(prob)
    m = prob.m
    rho0 = ZCSR.from_triplets(prob.n, [0], [0], [1.0])
    v0 = sun.expand_state(rho0)
    v = v0.clone()
    # BASELINE's dissipator has no gamma/(N-1) prefactor (reading R9): |lambda|max ~ gamma N^2,
    # so RK4 needs h |lambda| < 2.8; h = 1e-5 is stable at N <= 1000
    h, steps = 1e-5, 3
    sun.rk4(Q0, Q1, K, v, h, steps, eps0=1.0, eps1=1.5, omega=1.0)
    # (1) the integrator alone: RK4 on v with the GPU's own Q0, Q1, K on the CPU
    gq = lambda q: {"row_ptr": q.row_ptr.cpu().numpy(), "col": q.col.cpu().numpy(), "val": q.val.cpu().numpy()}  # noqa
    vown = propagate.rk4_v(_csr_np(gq(Q0), m), _csr_np(gq(Q1), m), K.cpu().numpy(), v0.cpu().numpy(), 0.0, h, steps,
                           eps0=1.0, eps1=1.5, omega=1.0)
    assert np.abs(v.cpu().numpy() - vown).max() <= 1e-13 * np.abs(vown).max()
    # (2) end to end against the oracle's matrices: the unfold's normwise tolerance (1e-12 max|Q|
    # per entry, R7) propagated through the steps: |dv| <= steps h (1 + eps) L dQ |v|
    Qo0, Qo1 = _csr_np(ref["Q0"], m), _csr_np(ref["Q1"], m)
    vref = propagate.rk4_v(Qo0, Qo1, ref["Q0"]["K"], v0.cpu().numpy(), 0.0, h, steps, eps0=1.0, eps1=1.5, omega=1.0)
    rowlen = np.diff(ref["Q0"]["row_ptr"]).max()
    bound = steps * h * 3.5 * rowlen * 1e-12 * np.abs(ref["Q0"]["val"]).max() * np.abs(vref).max() * 2
    assert np.abs(v.cpu().numpy() - vref).max() <= bound + 1e-13 * np.abs(vref).max()
    # populations stay a probability distribution
    d = sun.state_diag(v, prob.n).cpu().numpy()
    assert abs(d.sum() - 1.0) < 1e-12


def test_rk4_zero_steps_and_errors():
    sun = _sun()
    prob = dimer_problem(5, False)
    Q0, Q1, K = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    v = torch.arange(24, dtype=torch.float64, device="cuda")
    w = v.clone()
    sun.rk4(Q0, None, K, v, 0.1, 0)
    assert torch.equal(v, w)
    assert sun.lib().sun_rk4(None, None, None, 0.0, 0.0, 0.0, 0.0, 0.1, 1, None, None, None) == 1  # SUN_ERR_ARG
    assert sun.lib().sun_state_diag(None, 5, None, None) == 1


@pytest.mark.parametrize("idx", [0, 2, 3])
def test_unfold_split_sums_to_q0(idx):
    """F4: Q_H (Eq. 6) + R (Eq. 10) == Q0 as matrices; K identical; R = 0 without dissipators."""
    sun = _sun()
    prob = config(idx)
    QH, R, Q1, K = sun.unfold_split(prob.H0, prob.H1, prob.Ls, prob.gammas)
    Q0, Q1b, K0 = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    m = prob.m
    tocsr = lambda q: sp.csr_matrix((q.val.cpu().numpy(), q.col.cpu().numpy(), q.row_ptr.cpu().numpy()), shape=(m, m))  # noqa
    diff = (tocsr(QH) + tocsr(R) - tocsr(Q0)).toarray() if m < 5000 else None
    scale = np.abs(Q0.val.cpu().numpy()).max()
    if diff is not None:
        assert np.abs(diff).max() <= 1e-12 * scale
    else:
        d = tocsr(QH) + tocsr(R) - tocsr(Q0)
        assert (np.abs(d.data).max() if d.nnz else 0.0) <= 1e-12 * scale
    sparse.assert_k_close(K.cpu().numpy(), K0.cpu().numpy(), "split:K", sparse.tau_q0(prob))
    # Q_H is skew-symmetric
    A = tocsr(QH)
    assert abs(A + A.T).max() <= 1e-12 * max(1.0, abs(A).max())


@pytest.mark.parametrize("n,drive", [(3, True), (16, True), (33, False), (130, True)])
def test_rk4_matrix_free_matches_csr_rk4(n, drive):
    """sun_rk4_plan (Q regenerated per stage) against sun_rk4 on the assembled CSR (pinned above
    to the oracle) and, at n = 3, against RK4 on rho itself (Eq. 1)."""
    sun = _sun()
    prob = dimer_problem(n, drive)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    Q0, Q1, K = plan.run()
    assert plan.info()["mode_q0"] == 0
    v0 = sun.expand_state(ZCSR.from_triplets(n, [0], [0], [1.0]))
    h, steps, t0 = (0.05 if n <= 16 else 1e-3), 12, 0.3
    kw = dict(t0=t0, eps0=1.0, eps1=1.5, omega=1.0) if drive else dict(t0=t0)
    va = v0.clone()
    sun.rk4(Q0, Q1, K, va, h, steps, **kw)
    vb = v0.clone()
    plan.rk4(vb, h, steps, **kw)
    torch.cuda.synchronize()
    a, b = va.cpu().numpy(), vb.cpu().numpy()
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()
    if n == 3:
        rho0 = np.zeros((n, n), complex)
        rho0[0, 0] = 1.0
        rho = propagate.rk4_rho(prob.H0.to_dense(), prob.H1.to_dense(), [L.to_dense() for L in prob.Ls], prob.gammas,
                                rho0, t0, h, steps, eps0=1.0, eps1=1.5, omega=1.0)
        ref = basis.project(rho).real
        assert np.abs(b - ref).max() <= 1e-12 * np.abs(ref).max()
    plan.close()


def test_rk4_matrix_free_full_size_and_errors():
    sun = _sun()
    prob = config(4)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    Q0, Q1, K = plan.run()
    v0 = sun.expand_state(ZCSR.from_triplets(prob.n, [0], [0], [1.0]))
    va, vb = v0.clone(), v0.clone()
    sun.rk4(Q0, Q1, K, va, 1e-5, 3, eps0=1.0, eps1=1.5, omega=1.0)
    plan.rk4(vb, 1e-5, 3, eps0=1.0, eps1=1.5, omega=1.0)
    a, b = va.cpu().numpy(), vb.cpu().numpy()
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()
    plan.close()
    # not counted yet -> state error; a mode-2 plan (c3 widths) -> unsupported
    p2 = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    with pytest.raises(sun.SunError):
        p2.rk4(v0.clone(), 1e-5, 1)
    p2.close()
    # a mode-1 plan (runtime widths) -> unsupported
    p1 = banded_random_problem(70, seed=9, wH=15, wL=7, P=1)
    pm = sun.Plan(p1.H0, p1.H1, p1.Ls, p1.gammas)
    pm.run()
    with pytest.raises(sun.SunError, match="unsupported"):
        pm.rk4(sun.expand_state(ZCSR.from_triplets(p1.n, [0], [0], [1.0])), 1e-5, 1)
    pm.close()


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("which", ["small_P1", "small_P4", "c3"])
def test_rk4_matrix_free_wide(which, mode, monkeypatch):
    """Plans of widths (4, 2), thread-per-pair (mode 0, default) or warp-per-pair (mode 2,
    SUNFOLD_MODE2=1) count/fill: the matrix-free RK4 against the CSR RK4."""
    monkeypatch.setenv("SUNFOLD_MODE2", "1" if mode == 2 else "0")
    sun = _sun()
    prob = {"small_P1": lambda: banded_random_problem(50, seed=11, wH=4, wL=2, P=1),
            "small_P4": lambda: banded_random_problem(64, seed=6),
            "c3": lambda: config(3)}[which]()
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    Q0, Q1, K = plan.run()
    assert plan.info()["mode_q0"] == mode
    v0 = sun.expand_state(ZCSR.from_triplets(prob.n, [0], [0], [1.0]))
    va, vb = v0.clone(), v0.clone()
    h, steps = 1e-4, 5
    sun.rk4(Q0, None, K, va, h, steps)
    plan.rk4(vb, h, steps)
    a, b = va.cpu().numpy(), vb.cpu().numpy()
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()
    plan.close()


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_apply_matrix_free_matches_csr_apply(idx):
    """sun_apply_plan (Q regenerated) against sun_apply on the assembled CSR."""
    sun = _sun()
    prob = config(idx)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    Q0, Q1, K = plan.run()
    v = torch.linspace(-1.0, 1.0, prob.m, dtype=torch.float64, device="cuda")
    a = sun.apply(Q0, Q1, 1.3, K, v).cpu().numpy()
    b = plan.apply(v, 1.3).cpu().numpy()
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()
    plan.close()


def _oracle_mats(prob):
    ref = sparse.unfold_problem(prob)
    m = prob.m
    Q0 = _csr_np(ref["Q0"], m)
    Q1 = _csr_np(ref["Q1"], m) if "Q1" in ref else None
    return ref, Q0, Q1, ref["Q0"]["K"]


@pytest.mark.parametrize("idx", [2, 3, 4])
def test_matrix_free_apply_and_rk4_against_oracle(idx):
    """The matrix-free apply (sun_apply_plan) and RK4 (sun_rk4_plan) directly against the oracle:
    y = (Q0 + eps Q1) v + K and RK4 on v with O2's matrices (oracle.propagate.rk4_v), at c2-c4.
    Bound: R7's entrywise tolerance 1e-12 max|Q| carried through the row sums (apply) and the
    steps (RK4)."""
    sun = _sun()
    prob = config(idx)
    ref, Qo0, Qo1, Ko = _oracle_mats(prob)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    plan.run()
    rng = np.random.default_rng(7 + idx)
    rho = _dense_random_rho(prob.n, 90 + idx) if prob.n <= 512 else None
    v = basis.project(rho).real if rho is not None else rng.standard_normal(prob.m) / prob.n
    eps = 1.0 + 1.5 * np.sin(0.7)
    y = plan.apply(torch.tensor(v, device="cuda"), eps).cpu().numpy()
    yref = Qo0 @ v + Ko + (eps * (Qo1 @ v) if Qo1 is not None else 0.0)
    rowlen = np.diff(ref["Q0"]["row_ptr"]).max()
    qmax = np.abs(ref["Q0"]["val"]).max()
    bound = 1e-12 * qmax * np.abs(v).max() * rowlen * (1 + abs(eps)) + 1e-12 * np.abs(Ko).max()
    assert np.abs(y - yref).max() <= bound + 1e-13 * np.abs(yref).max()
    v0 = sun.expand_state(ZCSR.from_triplets(prob.n, [0], [0], [1.0]))
    h, steps = 1e-5, 3
    kw = dict(eps0=1.0, eps1=1.5, omega=1.0) if Qo1 is not None else {}
    vg = v0.clone()
    plan.rk4(vg, h, steps, **kw)
    vref = propagate.rk4_v(Qo0, Qo1, Ko, v0.cpu().numpy(), 0.0, h, steps, **kw)
    b2 = steps * h * 3.5 * rowlen * 1e-12 * qmax * np.abs(vref).max() * 2
    assert np.abs(vg.cpu().numpy() - vref).max() <= b2 + 1e-13 * np.abs(vref).max()
    plan.close()


@pytest.mark.parametrize("idx", [0, 2, 3])
def test_unfold_split_against_oracle(idx):
    """F4: Q_H (Eq. 6) and R (Eq. 10) of unfold_split, each against O2 directly: O2 on
    (H0, no dissipators) and on (0, {L_p, gamma_p}); K against O2's K."""
    sun = _sun()
    prob = config(idx)
    QH, R, Q1, K = sun.unfold_split(prob.H0, prob.H1, prob.Ls, prob.gammas)
    n = prob.n
    zero = ZCSR.from_dense(np.zeros((n, n), complex))
    tauH = sparse.TAU_REL * sparse.frob(prob.H0)
    tauR = sparse.TAU_REL * sum(g * sparse.frob(L) ** 2 for L, g in zip(prob.Ls, prob.gammas))
    rH = sparse.unfold_csr(prob.H0, (), (), tauH, with_k=False)
    rR = sparse.unfold_csr(zero, prob.Ls, prob.gammas, tauR)
    for got, want, nm in ((QH, rH, "QH"), (R, rR, "R")):
        assert np.array_equal(got.row_ptr.cpu().numpy(), want["row_ptr"]), nm
        assert np.array_equal(got.col.cpu().numpy(), want["col"]), nm
        sparse.assert_entries_close(got.val.cpu().numpy(), want, nm)
    sparse.assert_k_close(K.cpu().numpy(), rR["K"], "split:K", tauR)
