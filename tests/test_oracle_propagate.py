"""Pins for oracle.propagate (F1/F2 rows): RK4 on rho against exp(L T), order 4, invariants,
and RK4 on v (O1's Q, K) == proj(RK4 on rho)."""
import numpy as np
import scipy.linalg

from oracle import basis, dense, propagate


def _rand(n, rng):
    return rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))


def _problem(n, seed):
    rng = np.random.default_rng(seed)
    A = _rand(n, rng)
    H = (A + A.conj().T) / 2
    Ls = [_rand(n, rng) * 0.5]
    B = _rand(n, rng)
    rho0 = B @ B.conj().T
    rho0 /= np.trace(rho0)
    return H, Ls, [0.7], rho0


def test_rk4_rho_converges_with_order_4_to_expm():
    n = 3
    H, Ls, gs, rho0 = _problem(n, 1)
    T = 0.5
    E = propagate.liouvillian_matrix(H, Ls, gs)
    exact = (scipy.linalg.expm(E * T) @ rho0.reshape(-1, order="F")).reshape(n, n, order="F")
    errs = []
    for steps in (10, 20, 40):
        rho = propagate.rk4_rho(H, None, Ls, gs, rho0, 0.0, T / steps, steps)
        errs.append(np.abs(rho - exact).max())
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 13.0 < r1 < 19.0 and 13.0 < r2 < 19.0, errs  # 2^4 = 16
    assert errs[-1] < 1e-8


def test_rk4_rho_preserves_trace_and_hermiticity():
    H, Ls, gs, rho0 = _problem(4, 2)
    H1 = np.diag(np.arange(4.0)).astype(complex)
    rho = propagate.rk4_rho(H, H1, Ls, gs, rho0, 0.0, 0.01, 50, eps0=1.0, eps1=1.5, omega=1.0)
    assert abs(np.trace(rho) - 1.0) < 1e-13
    assert np.abs(rho - rho.conj().T).max() < 1e-13


def test_rk4_v_with_o1_equals_projected_rk4_rho_driven():
    n = 4
    H, Ls, gs, rho0 = _problem(n, 3)
    H1 = np.diag([1.0, -0.5, 0.25, 2.0]).astype(complex)
    Q0, K = dense.unfold_dense(H, Ls, gs)
    Q1, _ = dense.unfold_dense(H1)
    v0 = basis.project(rho0).real
    h, steps = 0.02, 40
    v = propagate.rk4_v(Q0, Q1, K, v0, 0.1, h, steps, eps0=1.0, eps1=1.5, omega=1.0)
    rho = propagate.rk4_rho(H, H1, Ls, gs, rho0, 0.1, h, steps, eps0=1.0, eps1=1.5, omega=1.0)
    assert np.abs(v - basis.project(rho).real).max() < 1e-13


def test_state_maps_are_inverse():
    n = 5
    rng = np.random.default_rng(4)
    B = _rand(n, rng)
    rho = B @ B.conj().T
    rho /= np.trace(rho)
    v = basis.project(rho).real
    assert np.abs(basis.reconstruct_fast(v, n) - rho).max() < 1e-14
    assert np.abs(np.diag(basis.reconstruct_fast(v, n)).real - np.diag(rho).real).max() < 1e-14
