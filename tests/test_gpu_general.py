"""GPU parity of the general-pattern mode (mode 3, sunfold_general.cu) against the oracle O2.

Operators of any pattern ("any complex N x N matrix could be chosen as an
operator L_p"; the paper's dense case, Table II): a periodic ring (entry (0, N-1)),
random sparse H and L_p with 4 nonzeros per row at random columns, dense L_p, and a jump into
a superposition (one dense column).  Same bar as tests/test_gpu_parity.py: bit-exact pattern,
normwise 1e-12 values (R7), K within 1e-12 max|K|, the oracle's pattern robust (R6).  The mode is
also forced on banded inputs (SUN_PLAN_GENERAL) and run with a 16-candidate merge buffer
(SUN_PLAN_SMALLCAP: key-range chunks, histogram refinement and the single-key reduction).
"""
import numpy as np
import pytest
import torch

from oracle import sparse
from workloads import (ZCSR, Problem, banded_random_problem, column_jump_problem, config, dense_dissipator_problem,
                       dense_random_problem, dimer_problem, random_sparse_problem, ring_dimer_problem)

pytestmark = pytest.mark.gpu

_REF = {}


def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1812_11626_b200 as sun

    return sun


def _np(t):
    return t.detach().cpu().numpy()


def _ref(prob):
    if prob.name not in _REF:
        _REF[prob.name] = sparse.unfold_problem(prob)
    return _REF[prob.name]


def _compare_csr(got, ref, name):
    """Bit-exact pattern; values per R7 (normwise 1e-12, and 1e-12 per entry where cond <= 100)."""
    rp, col, val = _np(got.row_ptr), _np(got.col), _np(got.val)
    assert np.array_equal(rp, ref["row_ptr"]), f"{name}: row_ptr differs"
    assert np.array_equal(col, ref["col"]), f"{name}: col differs"
    return sparse.assert_entries_close(val, ref, name)[0]


def _check(sun, prob, mode_expected=3, determinism=True, **plan_kw):
    ref = _ref(prob)
    tau0 = sparse.tau_q0(prob)
    sparse.assert_r6(ref["Q0"], tau0, prob.name)
    if prob.H1 is not None:
        sparse.assert_r6(ref["Q1"], sparse.tau_q1(prob), prob.name + ":Q1")
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas, **plan_kw)
    info = plan.info()
    assert info["mode_q0"] == mode_expected, info
    Q0, Q1, K = plan.run()
    torch.cuda.synchronize()
    assert abs(info["tau_q0"] - tau0) <= 1e-12 * tau0 or info["tau_q0"] == 0.0
    _compare_csr(Q0, ref["Q0"], prob.name + ":Q0")
    sparse.assert_k_close(_np(K), ref["Q0"]["K"], prob.name + ":K", tau0)
    if prob.H1 is not None:
        _compare_csr(Q1, ref["Q1"], prob.name + ":Q1")
    else:
        assert Q1 is None
    if determinism:
        A = plan.run()
        B = plan.run_two_pass()
        torch.cuda.synchronize()
        for X in (A, B):
            assert torch.equal(Q0.row_ptr, X[0].row_ptr) and torch.equal(Q0.col, X[0].col)
            assert torch.equal(Q0.val, X[0].val) and torch.equal(K, X[2])
            if Q1 is not None:
                assert torch.equal(Q1.val, X[1].val) and torch.equal(Q1.col, X[1].col)
    plan.close()
    return Q0, Q1, K


GENERAL = [
    ring_dimer_problem(256, drive=True),          # (i) periodic ring, entry (0, N-1)
    random_sparse_problem(300, seed=21, P=2),     # (ii) 4 nonzeros per row at random columns
    dense_dissipator_problem(24, seed=0),         # (iii) dense L_p (the paper's dense case)
    dense_dissipator_problem(48, seed=0),
    dense_dissipator_problem(17, seed=2, P=2),
    random_sparse_problem(40, seed=5, P=2, drive=True),  # non-diagonal sparse drive
    random_sparse_problem(77, seed=6, per_row=3, P=1),   # odd sizes, ragged rows
    column_jump_problem(20, seed=0),
    ring_dimer_problem(33, drive=False),
]


@pytest.mark.parametrize("prob", GENERAL, ids=lambda p: p.name)
def test_general_patterns(prob):
    """Operators beyond every band limit take mode 3 automatically and match the oracle."""
    sun = _gpu()
    _check(sun, prob)


FORCED = [
    config(0), config(1), config(2),
    dense_random_problem(2, seed=1), dense_random_problem(3, seed=2, P=2), dense_random_problem(8, seed=5, P=3),
    dimer_problem(2, True), dimer_problem(3, True), dimer_problem(16, True), dimer_problem(33, True),
    banded_random_problem(9, seed=4, wH=2, wL=1, P=2, drive_w=1),
    banded_random_problem(20, seed=5),
    banded_random_problem(70, seed=9, wH=15, wL=7, P=1),
]


@pytest.mark.parametrize("prob", FORCED, ids=lambda p: p.name)
def test_general_mode_forced_on_banded_inputs(prob):
    """SUN_PLAN_GENERAL: the general mode on inputs the band kernels also take; oracle parity,
    and the same CSR pattern as the banded plan (values within 1e-12 normwise)."""
    sun = _gpu()
    Q0, Q1, K = _check(sun, prob, general=True)
    B = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    assert torch.equal(Q0.row_ptr, B[0].row_ptr) and torch.equal(Q0.col, B[0].col)


SMALLCAP = [
    dense_dissipator_problem(24, seed=0),
    dense_dissipator_problem(9, seed=3, P=3),
    column_jump_problem(20, seed=0),
    random_sparse_problem(40, seed=5, P=2, drive=True),
    ring_dimer_problem(33, drive=True),
    config(0),
]


@pytest.mark.parametrize("prob", SMALLCAP, ids=lambda p: p.name)
def test_general_mode_small_buffer(prob):
    """SUN_PLAN_SMALLCAP (16-candidate buffer): every row goes through key-range chunks planned
    from histograms (with refinement), keys with more than 16 terms through the single-key
    reduction; oracle parity and determinism still hold."""
    sun = _gpu()
    _check(sun, prob, small_cap=True)


def test_general_edge_cases():
    """P = 0, gamma = 0, zero Hamiltonian, H only with a wide pattern, N = 2."""
    sun = _gpu()
    n = 20  # dense: half-bandwidth 19 > 15
    rng = np.random.default_rng(7)
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    Hd = ZCSR.from_dense(A + A.conj().T)                    # dense H, no dissipator
    _check(sun, Problem("denseH_P0", n, Hd, None, [], []))
    L = ZCSR.from_dense(rng.standard_normal((n, n)) + 0j)
    _check(sun, Problem("denseL_g0", n, Hd, None, [L], [0.0]))  # gamma = 0
    Z = ZCSR.from_dense(np.zeros((n, n), complex))
    _check(sun, Problem("pure_diss_dense", n, Z, None, [L], [0.7]))
    Q0, Q1, K = sun.Plan(Z, None, [], [], general=True).run()
    assert Q0.nnz == 0 and int(Q0.row_ptr[-1]) == 0 and torch.count_nonzero(K) == 0
    two = dense_random_problem(2, seed=4, P=2)
    _check(sun, two, general=True)


def test_general_capacity_and_errors():
    """sun_run into a short output reports SUN_ERR_CAPACITY and refills exactly; a non-Hermitian
    wide H is rejected; the matrix-free RK4 is reported unsupported on a general plan."""
    sun = _gpu()
    prob = random_sparse_problem(40, seed=5, P=2, drive=True)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    A = plan.run()
    small = plan._alloc(A[0].nnz - 5, A[1].nnz)
    C = plan.run(out=small)
    torch.cuda.synchronize()
    assert torch.equal(A[0].col, C[0].col) and torch.equal(A[0].val, C[0].val)
    v = torch.zeros(prob.m, dtype=torch.float64, device="cuda")
    with pytest.raises(sun.SunError, match="unsupported"):
        plan.rk4(v, 1e-3, 1)
    plan.close()
    rng = np.random.default_rng(3)
    B = rng.standard_normal((30, 30)) + 1j * rng.standard_normal((30, 30))
    with pytest.raises(sun.SunError, match="Hermitian"):
        sun.unfold(ZCSR.from_dense(B), None, [], [])


def test_general_workspace_guard():
    """No device write lands beyond the workspace the library is given (mode 3)."""
    sun = _gpu()
    prob = dense_dissipator_problem(17, seed=2, P=2)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas, guard_bytes=1 << 16)
    plan.run()
    plan.run_two_pass()
    torch.cuda.synchronize()
    assert plan.workspace_guard_intact()
    plan.close()


STASH = [
    random_sparse_problem(300, seed=21, P=2),
    ring_dimer_problem(256, drive=True),
    dense_dissipator_problem(24, seed=0),
    random_sparse_problem(40, seed=5, P=2, drive=True),
    column_jump_problem(20, seed=0),
]


@pytest.mark.parametrize("prob", STASH, ids=lambda p: p.name)
def test_general_stash_bit_identical(prob):
    """Light-row stash (sun_plan_set_stash): the count pass writes each light
    pair's assembled rows, the fill copies them.  Output bit-identical to the plan without a
    stash (the fill assembling every row itself); both equal the oracle (test_general_patterns
    runs with the stash, the default)."""
    sun = _gpu()
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    assert plan.stash is not None and plan.info()["mode_q0"] == 3
    A = plan.run()
    A2 = plan.run_two_pass()
    assert not plan.set_stash(False) and plan.stash is None
    B = plan.run()
    torch.cuda.synchronize()
    for X in (A2, B):
        for i in (0, 1):
            if A[i] is None:
                assert X[i] is None
                continue
            assert torch.equal(A[i].row_ptr, X[i].row_ptr) and torch.equal(A[i].col, X[i].col)
            assert torch.equal(A[i].val, X[i].val)
        assert torch.equal(A[2], X[2])
    ref = _ref(prob)
    _compare_csr(A[0], ref["Q0"], prob.name + ":Q0")
    plan.close()


def test_general_stash_abi():
    """sun_plan_stash_bytes is 0 for banded plans and set_stash rejects them; changing the stash
    requires a new count pass before the next fill (SUN_ERR_STATE)."""
    import ctypes

    sun = _gpu()
    L = sun.lib()
    prob = config(2)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    assert int(L.sun_plan_stash_bytes(plan._plan)) == 0 and plan.stash is None
    buf = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    assert L.sun_plan_set_stash(plan._plan, ctypes.c_void_p(buf.data_ptr()), ctypes.c_size_t(1 << 20)) != 0
    plan.close()
    prob = random_sparse_problem(40, seed=5, P=2, drive=True)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    nb = int(L.sun_plan_stash_bytes(plan._plan))
    assert nb > 0 and plan.stash is not None and plan.stash.numel() == nb
    assert L.sun_plan_set_stash(plan._plan, ctypes.c_void_p(plan.stash.data_ptr()), ctypes.c_size_t(nb - 1)) != 0
    nnz = plan.count()
    plan.set_stash(True)
    with pytest.raises(Exception):
        plan.fill(*nnz)
    plan.close()
