"""Oracle for the propagation rows: RK4 on the density operator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA path.

F1 (PAPER.md Step 3.1): the paper integrates dv/dt = [Q(t) + R] v + K (Eq. 9,
P:194-198) with the fixed-step fourth-order Runge-Kutta method.  The oracle integrates the
GKSL equation itself, drho/dt = L(t) rho (Eq. 1) with H(t) = H0 + eps(t) H1 and
eps(t) = eps0 + eps1 sin(omega t) (Eq. 12 drive; reading R10), with the same
classic RK4 step:
    k1 = L(t) rho, k2 = L(t + h/2)(rho + h/2 k1), k3 = L(t + h/2)(rho + h/2 k2),
    k4 = L(t + h)(rho + h k3),  rho <- rho + h/6 (k1 + 2 k2 + 2 k3 + k4).
Since rho -> v (Eq. 5) is affine and maps L(t) onto (Q0 + eps Q1) v + K exactly, RK4 on v
reproduces proj(RK4 on rho) up to rounding.  Pins (tests/test_oracle_propagate.py): order-4
convergence to exp(L T) rho(0) (scipy.linalg.expm of the vectorised Liouvillian) for a static
problem, trace and Hermiticity preservation, and agreement with RK4 on v with O1's Q and K.

F2 (Step 2.6 P:456-457, Eq. 5; observable P:259-261): v(0) = Tr(F_s rho(0)) is
oracle.basis.project; the populations are diag(reconstruct(v)).
"""
from __future__ import annotations

import numpy as np

from .dense import lindbladian


def eps_of(t: float, eps0: float, eps1: float, omega: float) -> float:
    """eps(t) = eps0 + eps1 sin(omega t) (reading R10)."""
    return eps0 + eps1 * np.sin(omega * t)


def rk4_rho(H0, H1, Ls, gammas, rho0, t0: float, h: float, nsteps: int, eps0=0.0, eps1=0.0, omega=1.0):
    """Classic RK4 of drho/dt = L(t) rho (Eq. 1) with H(t) = H0 + eps(t) H1 (H1 may be None)."""
    rho = np.array(rho0, dtype=np.complex128)

    def L(t, X):
        H = H0 if H1 is None else H0 + eps_of(t, eps0, eps1, omega) * H1
        return lindbladian(H, Ls, gammas, X)

    for i in range(nsteps):
        t = t0 + i * h
        k1 = L(t, rho)
        k2 = L(t + h / 2, rho + h / 2 * k1)
        k3 = L(t + h / 2, rho + h / 2 * k2)
        k4 = L(t + h, rho + h * k3)
        rho = rho + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    return rho


def rk4_v(Q0, Q1, K, v0, t0: float, h: float, nsteps: int, eps0=0.0, eps1=0.0, omega=1.0):
    """Classic RK4 of dv/dt = (Q0 + eps(t) Q1) v + K (Eq. 9) with given (dense or scipy) Q."""
    v = np.array(v0, dtype=np.float64)

    def f(t, x):
        y = Q0 @ x + K
        if Q1 is not None:
            y = y + eps_of(t, eps0, eps1, omega) * (Q1 @ x)
        return y

    for i in range(nsteps):
        t = t0 + i * h
        k1 = f(t, v)
        k2 = f(t + h / 2, v + h / 2 * k1)
        k3 = f(t + h / 2, v + h / 2 * k2)
        k4 = f(t + h, v + h * k3)
        v = v + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    return v


def liouvillian_matrix(H, Ls, gammas):
    """The N^2 x N^2 matrix of X -> L(X) on column-stacked vec(X) (for expm pins)."""
    n = H.shape[0]
    E = np.zeros((n * n, n * n), dtype=np.complex128)
    for k in range(n * n):
        X = np.zeros(n * n, dtype=np.complex128)
        X[k] = 1.0
        E[:, k] = lindbladian(H, Ls, gammas, X.reshape(n, n, order="F")).reshape(-1, order="F")
    return E
