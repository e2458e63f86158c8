"""Out-of-bounds write checks (compute-sanitizer is not available on the GPU pool): every
device entry point writes into buffers followed by guard regions filled with a sentinel, and
the guards must be intact afterwards.  Covers the unfold in modes 0/1/2 (single pass, two
pass, graphs on and off), apply, both RK4 paths, the state maps, the dense unfold and the
structure constants."""
import numpy as np
import pytest
import torch

from workloads import ZCSR, banded_random_problem, config, dimer_problem, gks_ensemble

pytestmark = pytest.mark.gpu
G = 4096  # guard elements


def _sun():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1812_11626_b200 as sun

    return sun


class Guarded:
    def __init__(self, n, dtype, fill):
        self.full = torch.full((n + G,), fill, dtype=dtype, device="cuda")
        self.fill = fill
        self.n = n

    @property
    def t(self):
        return self.full[: self.n]

    def intact(self):
        tail = self.full[self.n:]
        return bool((tail == self.fill).all().item())


def _guarded_csr(sun, m, nnz):
    rp, col, val = Guarded(m + 1, torch.int64, -7), Guarded(nnz, torch.int32, -7), Guarded(nnz, torch.float64, 7.5e300)
    return (rp, col, val), sun.CSR(rp.t, col.t, val.t)


@pytest.mark.parametrize("prob", [config(0), config(1), config(2), config(3), dimer_problem(1300, True),
                                  banded_random_problem(70, seed=9, wH=15, wL=7, P=1),
                                  banded_random_problem(50, seed=11, wH=4, wL=2, P=1)],
                         ids=lambda p: p.name)
def test_unfold_writes_stay_in_bounds(prob):
    sun = _sun()
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas, guard_bytes=1 << 16)
    ref = plan.run()
    n0, n1 = ref[0].nnz, (ref[1].nnz if ref[1] is not None else 0)
    m = prob.m
    for graphs in (True, False):
        plan.set_graphs(graphs)
        g0, Q0 = _guarded_csr(sun, m, n0)
        g1, Q1 = _guarded_csr(sun, m, n1) if ref[1] is not None else ((), None)
        gk = Guarded(m, torch.float64, 7.5e300)
        out = plan.run(out=(Q0, Q1, gk.t))
        torch.cuda.synchronize()
        assert all(g.intact() for g in (*g0, *g1, gk)), "output guard overwritten (run)"
        assert torch.equal(out[0].col, ref[0].col) and torch.equal(out[0].val, ref[0].val)
        # undersized capacity: nothing written beyond it either
        if n0 > 8:
            g0s, Q0s = _guarded_csr(sun, m, n0 - 8)
            gks = Guarded(m, torch.float64, 7.5e300)
            plan._caps = None
            try:
                plan.run(out=(Q0s, Q1, gks.t))
            except sun.SunError:
                pass
            torch.cuda.synchronize()
            assert all(g.intact() for g in (*g0s, gks)), "output guard overwritten (small capacity)"
        # two-pass API into guarded buffers
        plan.count()
        a, b = plan.nnz()
        g0, Q0 = _guarded_csr(sun, m, a)
        g1, Q1 = _guarded_csr(sun, m, b) if ref[1] is not None else ((), None)
        gk = Guarded(m, torch.float64, 7.5e300)
        plan.fill(a, b, out=(Q0, Q1, gk.t))
        torch.cuda.synchronize()
        assert all(g.intact() for g in (*g0, *g1, gk)), "output guard overwritten (two pass)"
    assert plan.workspace_guard_intact(), "workspace guard overwritten"
    # apply and the CSR RK4 with guarded vectors / scratch
    v = Guarded(m, torch.float64, 0.25)
    v.t.copy_(torch.linspace(-1, 1, m, dtype=torch.float64, device="cuda"))
    y = Guarded(m, torch.float64, 7.5e300)
    sun.apply(ref[0], ref[1], 0.7, ref[2], v.t, out=y.t)
    nb = int(sun.lib().sun_rk4_work_bytes(m))
    w = Guarded((nb + 7) // 8, torch.float64, 7.5e300)
    sun.rk4(ref[0], ref[1], ref[2], v.t, 1e-6, 2, eps0=1.0, eps1=0.5, work=w.t)
    torch.cuda.synchronize()
    assert v.intact() and y.intact() and w.intact()
    if plan.info()["mode_q0"] == 0 and (prob.H1 is None or plan.info()["w_h1"] == 0):
        nbm = int(sun.lib().sun_rk4_plan_work_bytes(plan._plan))
        wm = Guarded((nbm + 7) // 8, torch.float64, 7.5e300)
        plan.rk4(v.t, 1e-6, 2, eps0=1.0, eps1=0.5, work=wm.t)
        torch.cuda.synchronize()
        assert v.intact() and wm.intact() and plan.workspace_guard_intact()
    plan.close()


def test_state_maps_dense_and_structure_constants_stay_in_bounds():
    sun = _sun()
    n = 33
    m = n * n - 1
    v = Guarded(m, torch.float64, 0.5)
    v.t.copy_(torch.linspace(-0.01, 0.01, m, dtype=torch.float64, device="cuda"))
    d = Guarded(n, torch.float64, 7.5e300)
    assert sun.lib().sun_state_diag(v.t.data_ptr(), n, d.t.data_ptr(), None) == 0
    rho = Guarded(2 * n * n, torch.float64, 7.5e300)
    assert sun.lib().sun_state_reconstruct(v.t.data_ptr(), n, rho.t.data_ptr(), None) == 0
    vout = Guarded(m, torch.float64, 7.5e300)
    rho_csr = sun.DeviceZCSR.from_host(ZCSR.from_dense(np.eye(n) / n))
    s = sun._zcsr_struct(rho_csr)
    import ctypes

    assert sun.lib().sun_expand_state(ctypes.addressof(s), vout.t.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert v.intact() and d.intact() and rho.intact() and vout.intact()
    # dense unfold
    nd, B = 6, 3
    md = nd * nd - 1
    H, A = gks_ensemble(nd, B, seed=5)
    Hd = torch.tensor(H, dtype=torch.complex128, device="cuda")
    Ad = torch.tensor(A, dtype=torch.complex128, device="cuda")
    Q = Guarded(B * md * md, torch.float64, 7.5e300)
    K = Guarded(B * md, torch.float64, 7.5e300)
    nb = sun.dense_work_bytes(nd, 2)
    W = Guarded((nb + 15) // 16, torch.complex128, 0.0)
    W.fill = 0.0
    sun.unfold_dense(Hd, Ad, Q.t.view(B, md, md), K.t.view(B, md), work=W.t)
    torch.cuda.synchronize()
    assert Q.intact() and K.intact() and W.intact()
    # structure constants
    cnt = sun.structure_constants(nd, "d", count_only=True)
    idx = Guarded(3 * cnt, torch.int32, -9)
    val = Guarded(cnt, torch.float64, 7.5e300)
    wb = int(sun.lib().sun_sc_work_bytes(nd))
    ws = Guarded((wb + 7) // 8, torch.int64, -9)
    out = ctypes.c_int64()
    assert sun.lib().sun_structure_constants(nd, 1, idx.t.data_ptr(), val.t.data_ptr(), cnt, ctypes.addressof(out),
                                             ws.t.data_ptr(), wb, None) == 0
    assert out.value == cnt and idx.intact() and val.intact() and ws.intact()
