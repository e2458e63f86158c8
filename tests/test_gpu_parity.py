"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle O2.

Bar (BASELINE.json north_star; R6/R7):
  * CSR pattern (row_ptr, col) bit-exact;
  * values: max |q_gpu - q_oracle| <= 1e-12 max |q_oracle| per matrix (normwise, R7),
    and per-entry relative error <= 1e-12 wherever the entry has cond = sum|terms|/|q| <= 100;
  * K: max |K_gpu - K_oracle| <= 1e-12 max |K_oracle| (exact zeros where K == 0);
  * the oracle's pattern is robust (R6): gap kept > 1e3 tau > 1e6 dropped (flagged configs
    excepted, R6) and every entry near tau >= 50 roundoff bounds away from it;
  * bitwise determinism across runs; Q1 of a diagonal drive exactly skew-symmetric.
"""
import numpy as np
import pytest
import torch

from oracle import basis, sparse
from workloads import (ZCSR, banded_random_problem, config, dense_random_problem, dimer_problem)

pytestmark = pytest.mark.gpu


def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1812_11626_b200 as sun

    return sun


def _np(t):
    return t.detach().cpu().numpy()


def _compare_csr(got, ref, name):
    """Bit-exact pattern; values per R7 (normwise 1e-12, and 1e-12 per entry where cond <= 100)."""
    rp, col, val = _np(got.row_ptr), _np(got.col), _np(got.val)
    assert np.array_equal(rp, ref["row_ptr"]), f"{name}: row_ptr differs"
    assert np.array_equal(col, ref["col"]), f"{name}: col differs"
    return sparse.assert_entries_close(val, ref, name)[0]


def _run(sun, prob):
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    Q0, Q1, K = plan.run()
    torch.cuda.synchronize()
    info = plan.info()
    return plan, Q0, Q1, K, info


def _check_problem(sun, prob, determinism=True):
    ref = sparse.unfold_problem(prob)
    tau0 = sparse.tau_q0(prob)
    sparse.assert_r6(ref["Q0"], tau0, prob.name)
    if prob.H1 is not None:
        sparse.assert_r6(ref["Q1"], sparse.tau_q1(prob), prob.name + ":Q1")
    plan, Q0, Q1, K, info = _run(sun, prob)
    assert abs(info["tau_q0"] - tau0) <= 1e-12 * tau0
    _compare_csr(Q0, ref["Q0"], prob.name + ":Q0")
    sparse.assert_k_close(_np(K), ref["Q0"]["K"], prob.name + ":K", tau0)
    if prob.H1 is not None:
        _compare_csr(Q1, ref["Q1"], prob.name + ":Q1")
    else:
        assert Q1 is None
    if determinism:
        Q0b, Q1b, Kb = plan.run()
        torch.cuda.synchronize()
        assert torch.equal(Q0.row_ptr, Q0b.row_ptr) and torch.equal(Q0.col, Q0b.col)
        assert torch.equal(Q0.val, Q0b.val) and torch.equal(K, Kb)
        if Q1 is not None:
            assert torch.equal(Q1.val, Q1b.val)
    plan.close()
    return Q0, Q1, K, info


SMALL = [
    dense_random_problem(2, seed=1),
    dense_random_problem(3, seed=2, P=2),
    dense_random_problem(4, seed=0),
    dense_random_problem(6, seed=3),
    dense_random_problem(8, seed=5, P=3),
    dimer_problem(2, True), dimer_problem(3, True), dimer_problem(5, True), dimer_problem(16, True),
    dimer_problem(33, True), dimer_problem(130, True),
    banded_random_problem(9, seed=4, wH=2, wL=1, P=2, drive_w=1),
    banded_random_problem(20, seed=5),
    banded_random_problem(64, seed=6),
    banded_random_problem(97, seed=7, wH=1, wL=3, P=2),
    banded_random_problem(150, seed=8, wH=5, wL=0, P=1, drive_w=2),
    banded_random_problem(70, seed=9, wH=15, wL=7, P=1),
    banded_random_problem(50, seed=11, wH=4, wL=2, P=1),   # widths (4, 2), one dissipator
    banded_random_problem(45, seed=12, wH=3, wL=0, P=1),   # mode 0 widths (3, 0)
    banded_random_problem(77, seed=13, wH=1, wL=1, P=2),   # mode 0 widths (2, 1), runtime P
    dimer_problem(1300, True),                               # fill with a barrier per far tile (N >= 1200)
]


@pytest.mark.parametrize("prob", SMALL, ids=lambda p: p.name)
def test_parity_small(prob):
    sun = _gpu()
    _check_problem(sun, prob)


@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4])
def test_parity_baseline_configs(idx):
    """Full element-by-element parity at every BASELINE.json config (c4 = N=1000, the bench case)."""
    sun = _gpu()
    prob = config(idx)
    Q0, Q1, K, info = _check_problem(sun, prob, determinism=(idx == 4))
    if Q1 is not None and idx in (2, 4):
        # diagonal drive: Q1 exactly skew-symmetric, one entry per S/J row
        rp, col, val = _np(Q1.row_ptr), _np(Q1.col), _np(Q1.val)
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
        d = {(int(r), int(c)): v for r, c, v in zip(rows, col, val)}
        for (r, c), v in d.items():
            assert d[(c, r)] == -v


WIDE = [banded_random_problem(50, seed=11, wH=4, wL=2, P=1), banded_random_problem(64, seed=6),
        banded_random_problem(300, seed=21, wH=4, wL=2, P=3, drive_w=1)]


@pytest.mark.parametrize("which", ["w50_P1", "w64_P4", "w300_P3_drive", "c3"])
def test_wide_band_modes(which, monkeypatch):
    """Widths (4, 2) (c3's): the thread-per-pair staged path (mode 0, the default) and the
    warp-per-pair path (mode 2, SUNFOLD_MODE2=1) both match the oracle, and agree bit for bit."""
    sun = _gpu()
    prob = config(3) if which == "c3" else WIDE[["w50_P1", "w64_P4", "w300_P3_drive"].index(which)]
    outs = []
    for m2 in ("0", "1"):
        monkeypatch.setenv("SUNFOLD_MODE2", m2)
        if which != "c3" or m2 == "1":  # c3 in the default mode: test_parity_baseline_configs
            Q0, Q1, K, info = _check_problem(sun, prob, determinism=False)
        else:
            plan, Q0, Q1, K, info = _run(sun, prob)
            plan.close()
        assert info["mode_q0"] == (2 if m2 == "1" else 0), info
        outs.append((Q0, Q1, K))
    (a0, a1, ak), (b0, b1, bk) = outs
    for x, y in ((a0, b0),) + (((a1, b1),) if a1 is not None else ()):
        assert torch.equal(x.row_ptr, y.row_ptr) and torch.equal(x.col, y.col) and torch.equal(x.val, y.val)
    assert torch.equal(ak, bk)


@pytest.mark.parametrize("idx", [2, 3])
def test_scan_near_fused_switch(idx, monkeypatch):
    """SUNFOLD_SCAN_NEAR=1 (A/B switch, off by default: measured slower): sun_run writes the near
    rows from the scan's launch (k_scan_near0, near warps wait on per-chunk flags of the chained
    scan).  Its outputs equal the two-pass path's bit for bit, direct and graph-replayed."""
    sun = _gpu()
    monkeypatch.setenv("SUNFOLD_SCAN_NEAR", "1")
    prob = config(idx)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    for _ in range(3):
        Q0, Q1, K = plan.run()
    R0, R1, RK = plan.run_two_pass()
    torch.cuda.synchronize()
    assert Q0.nnz == R0.nnz and torch.equal(Q0.row_ptr, R0.row_ptr)
    assert torch.equal(Q0.col, R0.col) and torch.equal(Q0.val, R0.val) and torch.equal(K, RK)
    if Q1 is not None:
        assert Q1.nnz == R1.nnz and torch.equal(Q1.col, R1.col) and torch.equal(Q1.val, R1.val)
    plan.close()


def test_nnz_readback_pooled_slots():
    """sun_run returns nnz as soon as the fill has stored this sequence's header (mapped
    slot, sequence number last).  Plans created one after another reuse pooled slots that hold
    other plans' sequence numbers; every run must still report its own problem's nnz, equal to
    the two-pass (count -> synchronous readback -> fill) result, with identical outputs."""
    sun = _gpu()
    probs = [config(1), config(2), dimer_problem(40, True), config(1), config(2), config(3)]
    for prob in probs:
        plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
        for _ in range(3):  # first call direct, then graph capture and replay
            Q0, Q1, K = plan.run()
        R0, R1, RK = plan.run_two_pass()
        torch.cuda.synchronize()
        assert Q0.nnz == R0.nnz and torch.equal(Q0.col, R0.col) and torch.equal(Q0.val, R0.val)
        assert torch.equal(K, RK)
        if Q1 is not None:
            assert Q1.nnz == R1.nnz and torch.equal(Q1.val, R1.val)
        plan.close()


def test_phase_timing():
    """sun_plan_set_timing / sun_plan_phase_ms: event records around the count and fill passes
    inside the (captured) sequence; outputs unchanged, phase times positive, state errors."""
    sun = _gpu()
    prob = config(2)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    ref = plan.run()
    with pytest.raises(sun.SunError):
        plan.phase_ms()  # timing off
    plan.set_timing(True)
    with pytest.raises(sun.SunError):
        plan.phase_ms()  # no timed sequence yet
    for _ in range(3):  # direct, then captured with event-record nodes, then replayed
        out = plan.run()
        c, f = plan.phase_ms()
        assert c > 0 and f > 0
    torch.cuda.synchronize()
    assert torch.equal(out[0].val, ref[0].val) and torch.equal(out[1].val, ref[1].val) and torch.equal(out[2], ref[2])
    plan.count()
    c, f = plan.phase_ms()
    assert c > 0 and f == -1.0
    plan.set_timing(False)
    plan.close()


def test_apply_matches_lindbladian_c4():
    """Q(t) v + K from the GPU (sun_apply) equals proj L(t)(rho) for a random density matrix."""
    sun = _gpu()
    prob = config(4)
    Q0, Q1, K = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    rng = np.random.default_rng(4)
    n = prob.n
    B = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    rho = B @ B.conj().T
    rho /= np.trace(rho)
    v = basis.project(rho).real
    eps = 1.0 + 1.5 * np.sin(0.3)
    y = sun.apply(Q0, Q1, eps, K, torch.tensor(v, device="cuda"))
    H = prob.H0.to_dense() + eps * prob.H1.to_dense()
    L = prob.Ls[0].to_dense()
    g = prob.gammas[0]
    LdL = L.conj().T @ L
    Lr = -1j * (H @ rho - rho @ H) + g * (L @ rho @ L.conj().T - 0.5 * (LdL @ rho + rho @ LdL))
    ref = basis.project(Lr).real
    assert np.abs(_np(y) - ref).max() <= 1e-12 * np.abs(ref).max()


def test_apply_against_oracle_spmv_c3():
    sun = _gpu()
    prob = config(3)
    ref = sparse.unfold_problem(prob)["Q0"]
    Q0, Q1, K = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    v = np.random.default_rng(3).standard_normal(prob.m)
    y = _np(sun.apply(Q0, None, 0.0, K, torch.tensor(v, device="cuda")))
    rows = np.repeat(np.arange(prob.m), np.diff(ref["row_ptr"]))
    yr = np.zeros(prob.m)
    np.add.at(yr, rows, ref["val"] * v[ref["col"]])
    yr += ref["K"]
    assert np.abs(y - yr).max() <= 1e-12 * np.abs(yr).max()


def _csr_from_lengths(lens, m, seed):
    """A random square CSR (m rows) with the given row lengths: ascending distinct columns per row."""
    rng = np.random.default_rng(seed)
    rp = np.zeros(m + 1, dtype=np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.empty(rp[-1], dtype=np.int32)
    for r in range(m):
        col[rp[r]:rp[r + 1]] = np.sort(rng.choice(m, size=int(lens[r]), replace=False))
    return rp, col, rng.standard_normal(rp[-1])


@pytest.mark.parametrize("shape", ["short", "one_long_among_short", "all_long", "wide_multi_tile", "empty_rows",
                                   "single_row", "no_entries"])
def test_apply_row_shapes(shape):
    """sun_apply (a7, Eq. 9) on synthetic CSR matrices that reach every summation path of
    the streamed kernel (thread per row, a long segment summed by its warp, G lanes per intersecting
    row, rows spanning several tiles, rows per CTA below 256, ragged last block), against the plain
    definition y_r = sum_k Q0[r,k] x_k + eps sum_k Q1[r,k] x_k + K_r in fp64."""
    sun = _gpu()
    rng = np.random.default_rng(5)
    m = {"single_row": 1, "all_long": 300, "wide_multi_tile": 2600}.get(shape, 1301)
    if shape == "short":
        l0 = rng.integers(0, 30, m)
    elif shape == "one_long_among_short":
        l0 = rng.integers(5, 25, m)
        l0[[3, 700, 1300]] = [1200, 900, 1301]
    elif shape == "all_long":
        l0 = rng.integers(150, 300, m)
    elif shape == "wide_multi_tile":
        l0 = rng.integers(2200, 2600, m)  # every row longer than a 2048-entry tile, 8 rows per CTA
    elif shape == "empty_rows":
        l0 = np.where(rng.random(m) < 0.7, 0, rng.integers(1, 400, m))
    elif shape == "single_row":
        l0 = np.array([1])
    else:
        l0 = np.zeros(m, dtype=np.int64)
    l1 = np.minimum(rng.integers(0, 4, m), m)
    A0, A1 = _csr_from_lengths(l0, m, 1), _csr_from_lengths(l1, m, 2)
    x, Kv, eps = rng.standard_normal(m), rng.standard_normal(m), 0.7

    def dev(A):
        # entries at an offset inside a larger buffer when empty (a null data pointer is an error)
        rp, col, val = (torch.tensor(a, device="cuda") for a in A)
        if col.numel() == 0:
            col, val = torch.zeros(4, dtype=torch.int32, device="cuda")[:0], torch.zeros(4, dtype=torch.float64, device="cuda")[:0]
        return sun.CSR(rp, col, val)

    def ref(A):
        rp, col, val = A
        y = np.zeros(m)
        for r in range(m):
            y[r] = np.dot(val[rp[r]:rp[r + 1]], x[col[rp[r]:rp[r + 1]]])
        return y

    want = ref(A0) + eps * ref(A1) + Kv
    scale = np.abs(want).max() + 1.0
    xd = torch.tensor(x, device="cuda")
    for Q1, K, w in ((dev(A1), torch.tensor(Kv, device="cuda"), want), (None, None, ref(A0))):
        got = _np(sun.apply(dev(A0), Q1, eps, K, xd))
        assert np.abs(got - w).max() <= 1e-12 * scale, (shape, np.abs(got - w).max())
        again = _np(sun.apply(dev(A0), Q1, eps, K, xd))
        assert np.array_equal(got, again), "sun_apply is deterministic"


def test_edge_cases():
    sun = _gpu()
    n = 6
    # H only (P = 0), no drive
    p = dimer_problem(n, False)
    p.Ls, p.gammas = [], []
    _check_problem(sun, p)
    # gamma = 0 -> same as H only
    q = dimer_problem(n, False)
    q.gammas = [0.0]
    Q0a, _, Ka, _ = _check_problem(sun, q)
    assert torch.count_nonzero(Ka) == 0
    # zero Hamiltonian and no dissipator: empty Q0
    z = ZCSR.from_dense(np.zeros((n, n), complex))
    Q0, Q1, K = sun.unfold(z, None, [], [])
    assert Q0.nnz == 0 and int(Q0.row_ptr[-1]) == 0 and torch.count_nonzero(K) == 0
    # pure dissipation (H = 0) with a traceful L
    rng = np.random.default_rng(1)
    L = rng.standard_normal((5, 5)) + 1j * rng.standard_normal((5, 5))
    from workloads import Problem
    pd = Problem("pure_diss", 5, ZCSR.from_dense(np.zeros((5, 5), complex)), None, [ZCSR.from_dense(L)], [0.4])
    _check_problem(sun, pd)


def test_error_codes():
    sun = _gpu()
    rng = np.random.default_rng(0)
    A = rng.standard_normal((5, 5)) + 1j * rng.standard_normal((5, 5))
    with pytest.raises(sun.SunError, match="Hermitian"):
        sun.unfold(ZCSR.from_dense(A), None, [], [])  # not Hermitian
    H = ZCSR.from_dense(A + A.conj().T)
    with pytest.raises(sun.SunError, match="rate"):
        sun.Plan(H, None, [ZCSR.from_dense(A)], [-0.1])
    big = banded_random_problem(60, seed=1, wH=16, wL=0, P=0)  # beyond the band kernels: general mode
    assert sun.Plan(big.H0, None, [], []).info()["mode_q0"] == 3
    p = dimer_problem(8, True)
    plan = sun.Plan(p.H0, p.H1, p.Ls, p.gammas)
    plan.count()
    nnz0, nnz1 = plan.nnz()
    with pytest.raises(sun.SunError, match="capacity"):
        plan.fill(nnz0 - 1, nnz1)
    other = dimer_problem(9, False)
    with pytest.raises(sun.SunError, match="dimension"):
        sun.Plan(p.H0, None, other.Ls, other.gammas)
    plan.close()


def test_run_single_pass_matches_two_pass_and_capacity_fallback():
    """sun_run (no host round trip) == sun_count/sun_plan_nnz/sun_unfold, byte for byte; an
    undersized output is reported (SUN_ERR_CAPACITY) and refilled exactly."""
    sun = _gpu()
    prob = config(2)
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    b0, b1 = plan.nnz_bound()
    A = plan.run()  # first call: capacity = structural bound
    B = plan.run_two_pass()
    torch.cuda.synchronize()
    assert A[0].nnz <= b0 and A[1].nnz <= b1
    for x, y in ((A[0], B[0]), (A[1], B[1])):
        assert torch.equal(x.row_ptr, y.row_ptr) and torch.equal(x.col, y.col) and torch.equal(x.val, y.val)
    assert torch.equal(A[2], B[2])
    small = plan._alloc(A[0].nnz - 7, A[1].nnz)
    C = plan.run(out=small)
    torch.cuda.synchronize()
    assert torch.equal(C[0].col, B[0].col) and torch.equal(C[0].val, B[0].val)
    plan.close()


def test_plan_rerun_uses_current_operator_values():
    """A plan re-runs the whole path on the operators' current values (bench.py's step): the
    device values of H0 and L are changed in place between run() calls (same pattern, new
    values, also a different tau), and each result equals the oracle for those values."""
    sun = _gpu()
    from workloads import Problem

    prob = dimer_problem(40, True)
    H0 = sun.DeviceZCSR.from_host(prob.H0)
    H1 = sun.DeviceZCSR.from_host(prob.H1)
    Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
    plan = sun.Plan(H0, H1, Ls, prob.gammas)
    for scale_h, scale_l in ((1.0, 1.0), (1.7, 0.6), (0.3, 2.5)):
        if (scale_h, scale_l) != (1.0, 1.0):
            H0.val.mul_(scale_h)
            Ls[0].val.mul_(scale_l)
        Q0, Q1, K = plan.run()
        torch.cuda.synchronize()
        h0 = ZCSR(prob.H0.n, prob.H0.row_ptr, prob.H0.col, H0.val.cpu().numpy())
        l0 = ZCSR(prob.Ls[0].n, prob.Ls[0].row_ptr, prob.Ls[0].col, Ls[0].val.cpu().numpy())
        cur = Problem("rerun", prob.n, h0, prob.H1, [l0], prob.gammas)
        ref = sparse.unfold_problem(cur)
        _compare_csr(Q0, ref["Q0"], "rerun:Q0")
        _compare_csr(Q1, ref["Q1"], "rerun:Q1")
        sparse.assert_k_close(_np(K), ref["Q0"]["K"], "rerun:K", sparse.tau_q0(cur))
    plan.close()


def test_wrapper_accepts_dense_and_sparse_torch_inputs():
    """The Python wrapper's operator marshalling: dense torch / numpy and torch
    sparse-CSR inputs give the same unfold as host CSR; outputs convert to torch sparse CSR."""
    sun = _gpu()
    prob = dimer_problem(20, True)
    ref = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    dense = [torch.tensor(x.to_dense(), device="cuda") for x in (prob.H0, prob.H1, prob.Ls[0])]
    got = sun.unfold(dense[0], dense[1].to_sparse_csr(), [prob.Ls[0].to_dense()], prob.gammas)
    torch.cuda.synchronize()
    for a, b in ((ref[0], got[0]), (ref[1], got[1])):
        assert torch.equal(a.row_ptr, b.row_ptr) and torch.equal(a.col, b.col) and torch.equal(a.val, b.val)
    assert torch.equal(ref[2], got[2])
    T = ref[0].to_torch()
    D = T.to_dense().cpu().numpy()
    rp, c, v = _np(ref[0].row_ptr), _np(ref[0].col), _np(ref[0].val)
    for s in (0, 5, ref[0].m - 1):
        assert np.array_equal(np.nonzero(D[s])[0], c[rp[s]:rp[s + 1]])
        assert np.array_equal(D[s, c[rp[s]:rp[s + 1]]], v[rp[s]:rp[s + 1]])


def test_side_stream_matches_default_stream():
    """Every call takes the caller's stream (C-ABI `void* stream`): a plan bound to a side stream
    gives the default stream's results bit for bit (unfold, run, apply, both RK4 paths)."""
    sun = _gpu()
    prob = dimer_problem(60, True)
    ref_plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    R = ref_plan.run()
    v = torch.linspace(-1, 1, prob.m, dtype=torch.float64, device="cuda")
    ya = sun.apply(R[0], R[1], 0.9, R[2], v)
    va = v.clone()
    sun.rk4(R[0], R[1], R[2], va, 1e-4, 3, eps0=1.0, eps1=0.5)
    vma = v.clone()
    ref_plan.rk4(vma, 1e-4, 3, eps0=1.0, eps1=0.5)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas, stream=s)
        S1 = plan.run()
        S2 = plan.run()
        yb = sun.apply(S2[0], S2[1], 0.9, S2[2], v, stream=s)
        vb = v.clone()
        sun.rk4(S2[0], S2[1], S2[2], vb, 1e-4, 3, eps0=1.0, eps1=0.5, stream=s)
        vmb = v.clone()
        plan.rk4(vmb, 1e-4, 3, eps0=1.0, eps1=0.5)
    s.synchronize()
    for A, B in ((R, S1), (R, S2)):
        assert torch.equal(A[0].row_ptr, B[0].row_ptr) and torch.equal(A[0].col, B[0].col)
        assert torch.equal(A[0].val, B[0].val) and torch.equal(A[1].val, B[1].val) and torch.equal(A[2], B[2])
    assert torch.equal(ya, yb) and torch.equal(va, vb) and torch.equal(vma, vmb)
    plan.close()
    ref_plan.close()


def test_stream_argument_without_stream_context():
    """A call given `stream=s` while the caller's current stream stays the default one: the work
    is ordered after the current stream (inputs copied there just before) and the workspace,
    outputs and scratch belong to `s`, so memory freed by unfold()'s plan is not reused by the
    current stream while `s` still runs.  Results equal the default-stream ones."""
    sun = _gpu()
    prob = dimer_problem(60, True)
    R = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    v = torch.linspace(-1, 1, prob.m, dtype=torch.float64, device="cuda")
    ya = sun.apply(R[0], R[1], 0.9, R[2], v)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    outs = []
    for k in range(3):
        H0 = sun.DeviceZCSR.from_host(prob.H0)  # made on the current stream
        H1 = sun.DeviceZCSR.from_host(prob.H1)
        Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
        S = sun.unfold(H0, H1, Ls, prob.gammas, stream=s)
        junk = torch.full((1 << 22,), float(k), dtype=torch.float64, device="cuda")  # reuse pressure
        y = sun.apply(S[0], S[1], 0.9, S[2], v, stream=s)
        outs.append((S, y))
        del junk
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas, stream=s)
    P1 = plan.run()
    s.synchronize()
    for S, y in outs + [(P1, ya)]:
        assert torch.equal(R[0].row_ptr, S[0].row_ptr) and torch.equal(R[0].col, S[0].col)
        assert torch.equal(R[0].val, S[0].val) and torch.equal(R[1].val, S[1].val) and torch.equal(R[2], S[2])
        assert torch.equal(ya, y)
    plan.close()
