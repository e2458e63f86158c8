"""Seeded synthetic inputs for the SU(N) unfold (shared by the oracle, the tests and bench.py).

This module holds NO arithmetic of the method (no basis, no structure constants,
no Lindbladian).  It only builds the N x N input operators H0, H1, {L_p} and the
rates {gamma_p} for the five BASELINE.json configurations, as complex128 CSR
arrays in host memory.  Both sides of every parity test (the CUDA path through
the C-ABI and the CPU oracle) consume exactly these arrays.

Recipes (DESIGN.md "Input recipe" restates them):

* c0  N=4, P=1.  rng = numpy.random.default_rng(0).  A = g(N,N) + i g(N,N)
      (real block drawn first, then imaginary block), H = (A + A^H)/2 (dense,
      has a trace).  Then L1 = g(N,N) + i g(N,N) (dense, has a trace).
      gamma_1 = 1.0.  No drive.                      BASELINE.json configs[0]
* c1  Bose-Hubbard dimer, N=64 states (N-1 bosons), Fock index a = n1,
      n2 = N-1-a:  H = -J(b1^+ b2 + b2^+ b1) + (U/2N) sum_j n_j(n_j-1), J=1, U=2;
      L = (b1^+ + b2^+)(b1 - b2), gamma = 0.1.  No drive.  configs[1]
      (Eq. 12-13, with BASELINE's normalisation.)
* c2  c1 at N=256 plus H1 = n2 - n1 = diag(N-1-2a); eps(t) = 1 + 1.5 sin t.
* c3  N=512 random banded.  rng = default_rng(3).  H: for each diagonal offset
      k = 1..3 (in that order) draw re = g(N-k), im = g(N-k) and set
      H[a, a+k] = re + i im, H[a+k, a] = conj; then the real diagonal g(N).
      Then for p = 1..4: for k = -2..2 (in that order) draw re = g(N-|k|),
      im = g(N-|k|) and set L_p[a, a+k] (a ranging over valid rows ascending).
      Finally gamma = uniform(0.05, 0.5, size=4).            configs[3]
* c4  c2's dimer and drive at N=1000 with c1's dissipator.   configs[4]

CSR layout (the C-ABI's sun_zcsr): row_ptr int64[N+1], col int32[nnz] ascending
within each row, val complex128[nnz] (== interleaved re,im float64[2 nnz]).
Exact zeros are not stored.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np


@dataclasses.dataclass
class ZCSR:
    """N x N complex operator in CSR form (host numpy arrays)."""

    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col: np.ndarray  # int32 [nnz]
    val: np.ndarray  # complex128 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n), dtype=np.complex128)
        for r in range(self.n):
            lo, hi = int(self.row_ptr[r]), int(self.row_ptr[r + 1])
            out[r, self.col[lo:hi]] = self.val[lo:hi]
        return out

    @staticmethod
    def from_dense(a: np.ndarray) -> "ZCSR":
        a = np.asarray(a, dtype=np.complex128)
        n = a.shape[0]
        assert a.shape == (n, n)
        rows, cols = np.nonzero(a)
        order = np.lexsort((cols, rows))
        rows, cols = rows[order], cols[order]
        row_ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        row_ptr = np.cumsum(row_ptr).astype(np.int64)
        return ZCSR(n, row_ptr, cols.astype(np.int32), a[rows, cols].copy())

    @staticmethod
    def from_triplets(n: int, rows, cols, vals) -> "ZCSR":
        """Build from (row, col, value) triplets; duplicates are not allowed, zeros dropped."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.complex128)
        keep = vals != 0
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        if rows.size > 1:
            dup = (rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])
            assert not dup.any(), "duplicate (row, col) in triplets"
        row_ptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(row_ptr, rows + 1, 1)
        row_ptr = np.cumsum(row_ptr).astype(np.int64)
        return ZCSR(n, row_ptr, cols.astype(np.int32), vals)


@dataclasses.dataclass
class Problem:
    """One unfold problem: H(t) = H0 + eps(t) H1 and dissipators {(L_p, gamma_p)}."""

    name: str
    n: int
    H0: ZCSR
    H1: Optional[ZCSR]
    Ls: List[ZCSR]
    gammas: List[float]
    eps: Optional[dict] = None  # drive eps(t) = eps0 + eps1 sin(omega t) (R10)

    @property
    def m(self) -> int:
        return self.n * self.n - 1


# ----------------------------------------------------------------------------
# Bose-Hubbard dimer (Eq. 12; Eq. 13, P:242-245;
# normalisation and sign per BASELINE.json configs[1], R8/R9/R11)
# ----------------------------------------------------------------------------

def dimer_hamiltonian(n: int, J: float = 1.0, U: float = 2.0) -> ZCSR:
    """H = -J(b1^+ b2 + b2^+ b1) + (U/2N) sum_j n_j(n_j - 1) in the Fock basis a = n1."""
    a = np.arange(n, dtype=np.float64)
    n1, n2 = a, (n - 1) - a
    diag = (U / (2.0 * n)) * (n1 * (n1 - 1.0) + n2 * (n2 - 1.0))
    off = -J * np.sqrt((a[:-1] + 1.0) * (n - 1.0 - a[:-1]))  # H[a+1,a] = H[a,a+1]
    rows = np.concatenate([np.arange(n), np.arange(n - 1), np.arange(1, n)])
    cols = np.concatenate([np.arange(n), np.arange(1, n), np.arange(n - 1)])
    vals = np.concatenate([diag, off, off]).astype(np.complex128)
    return ZCSR.from_triplets(n, rows, cols, vals)


def dimer_drive(n: int) -> ZCSR:
    """H1 = n2 - n1 = diag(N-1-2a) (the operator multiplying eps(t) in Eq. 12)."""
    a = np.arange(n)
    return ZCSR.from_triplets(n, a, a, ((n - 1) - 2 * a).astype(np.complex128))


def dimer_dissipator(n: int) -> ZCSR:
    """L = (b1^+ + b2^+)(b1 - b2) = n1 - n2 - b1^+ b2 + b2^+ b1 (no prefactor, R9)."""
    a = np.arange(n, dtype=np.float64)
    diag = 2.0 * a - (n - 1.0)
    s = np.sqrt((a[:-1] + 1.0) * (n - 1.0 - a[:-1]))
    rows = np.concatenate([np.arange(n), np.arange(1, n), np.arange(n - 1)])
    cols = np.concatenate([np.arange(n), np.arange(n - 1), np.arange(1, n)])
    # L[a+1, a] = -s_a ; L[a, a+1] = +s_a
    vals = np.concatenate([diag, -s, s]).astype(np.complex128)
    return ZCSR.from_triplets(n, rows, cols, vals)


def dimer_problem(n: int, drive: bool, gamma: float = 0.1, name: str = "", U: float = 2.0) -> Problem:
    return Problem(
        name=name or f"dimer_N{n}",
        n=n,
        H0=dimer_hamiltonian(n, U=U),
        H1=dimer_drive(n) if drive else None,
        Ls=[dimer_dissipator(n)],
        gammas=[gamma],
        eps={"eps0": 1.0, "eps1": 1.5, "omega": 1.0} if drive else None,
    )


# ----------------------------------------------------------------------------
# Random inputs
# ----------------------------------------------------------------------------

def dense_random_problem(n: int = 4, seed: int = 0, gamma: float = 1.0, P: int = 1) -> Problem:
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    H = (A + A.conj().T) / 2.0
    Ls = []
    for _ in range(P):
        Ls.append(ZCSR.from_dense(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))))
    return Problem(f"dense_N{n}_s{seed}", n, ZCSR.from_dense(H), None, Ls, [gamma] * P)


def _band_hermitian(rng, n: int, w: int) -> np.ndarray:
    H = np.zeros((n, n), dtype=np.complex128)
    for k in range(1, w + 1):
        if n - k <= 0:
            continue
        re = rng.standard_normal(n - k)
        im = rng.standard_normal(n - k)
        idx = np.arange(n - k)
        H[idx, idx + k] = re + 1j * im
        H[idx + k, idx] = re - 1j * im
    H[np.arange(n), np.arange(n)] = rng.standard_normal(n)
    return H


def _band_general(rng, n: int, w: int) -> np.ndarray:
    L = np.zeros((n, n), dtype=np.complex128)
    for k in range(-w, w + 1):
        m = n - abs(k)
        if m <= 0:
            continue
        re = rng.standard_normal(m)
        im = rng.standard_normal(m)
        rows = np.arange(m) if k >= 0 else np.arange(-k, n)
        L[rows, rows + k] = re + 1j * im
    return L


def banded_random_problem(n: int = 512, seed: int = 3, wH: int = 3, wL: int = 2, P: int = 4,
                          drive_w: Optional[int] = None) -> Problem:
    rng = np.random.default_rng(seed)
    H = _band_hermitian(rng, n, wH)
    Ls = [_band_general(rng, n, wL) for _ in range(P)]
    gammas = rng.uniform(0.05, 0.5, size=P).tolist()
    H1 = None
    if drive_w is not None:
        H1 = ZCSR.from_dense(_band_hermitian(rng, n, drive_w))
    return Problem(f"banded_N{n}_s{seed}", n, ZCSR.from_dense(H), H1,
                   [ZCSR.from_dense(L) for L in Ls], gammas)


def ring_dimer_problem(n: int, drive: bool = True, gamma: float = 0.1, J: float = 1.0) -> Problem:
    """General-pattern case (i): the dimer of R8/R9/R11 closed into a ring -- H gains the hopping
    -J (E_{0,N-1} + E_{N-1,0}) and L the antisymmetric pair +E_{0,N-1} - E_{N-1,0} (entry (0, N-1):
    half-bandwidth N-1, beyond every banded mode).  Deterministic."""
    base = dimer_problem(n, drive, gamma=gamma)
    H = base.H0.to_dense()
    H[0, n - 1] += -J
    H[n - 1, 0] += -J
    L = base.Ls[0].to_dense()
    L[0, n - 1] += 1.0
    L[n - 1, 0] -= 1.0
    return Problem(f"ring_N{n}" + ("_drive" if drive else ""), n, ZCSR.from_dense(H), base.H1, [ZCSR.from_dense(L)],
                   [gamma])


def random_sparse_problem(n: int = 300, seed: int = 21, per_row: int = 4, P: int = 2, drive: bool = False) -> Problem:
    """General-pattern case (ii): H and every L_p with `per_row` nonzeros per row at uniformly
    random columns (no band).  rng = default_rng(seed).  H: for each row a, `per_row // 2` columns
    drawn without replacement (excluding a), entries g + i g (real then imaginary draw per row)
    mirrored conjugate (so rows hold about per_row entries), then a real diagonal g(N).  Then for
    p = 1..P: for each row, `per_row` distinct columns and entries g + i g.  gamma ~ U[0.05, 0.5].
    drive: H1 = the same recipe's real symmetric pattern with entries g (one more draw)."""
    rng = np.random.default_rng(seed)
    H = np.zeros((n, n), dtype=np.complex128)
    k = max(per_row // 2, 1)
    for a in range(n):
        cols = rng.choice(np.delete(np.arange(n), a), size=k, replace=False)
        re, im = rng.standard_normal(k), rng.standard_normal(k)
        H[a, cols] += re + 1j * im
        H[cols, a] += re - 1j * im
    H[np.arange(n), np.arange(n)] += rng.standard_normal(n)
    Ls = []
    for _ in range(P):
        L = np.zeros((n, n), dtype=np.complex128)
        for a in range(n):
            cols = rng.choice(n, size=per_row, replace=False)
            L[a, cols] = rng.standard_normal(per_row) + 1j * rng.standard_normal(per_row)
        Ls.append(ZCSR.from_dense(L))
    gammas = list(rng.uniform(0.05, 0.5, size=P))
    H1 = None
    if drive:
        D = np.zeros((n, n), dtype=np.complex128)
        for a in range(n):
            cols = rng.choice(np.delete(np.arange(n), a), size=k, replace=False)
            v = rng.standard_normal(k)
            D[a, cols] += v
            D[cols, a] += v
        H1 = ZCSR.from_dense(D)
    return Problem(f"sparse_N{n}_s{seed}_P{P}", n, ZCSR.from_dense(H), H1, Ls, gammas)


def dense_dissipator_problem(n: int, seed: int = 0, P: int = 1, gamma: float = 0.5) -> Problem:
    """General-pattern case (iii), the paper's dense-L case (Table II): the
    dimer Hamiltonian with P dense random dissipators L_p = g + i g (traceful).  rng = default_rng(seed)."""
    rng = np.random.default_rng(seed)
    Ls = [ZCSR.from_dense(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) for _ in range(P)]
    return Problem(f"denseL_N{n}_s{seed}_P{P}", n, dimer_hamiltonian(n), None, Ls, [gamma] * P)


def column_jump_problem(n: int, seed: int = 0) -> Problem:
    """A jump into a superposition, L = |psi><0| (one dense column), plus the dimer H: many
    candidate terms share one output key (the single-key path of the general mode)."""
    rng = np.random.default_rng(seed)
    psi = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    L = np.zeros((n, n), dtype=np.complex128)
    L[:, 0] = psi
    return Problem(f"coljump_N{n}_s{seed}", n, dimer_hamiltonian(n), None, [ZCSR.from_dense(L)], [0.3])


def config(idx: int) -> Problem:
    """The five BASELINE.json configurations (index = position in configs[])."""
    if idx == 0:
        return dense_random_problem(4, seed=0, gamma=1.0)
    if idx == 1:
        return dimer_problem(64, drive=False, name="c1_dimer_N64")
    if idx == 2:
        return dimer_problem(256, drive=True, name="c2_dimer_N256_drive")
    if idx == 3:
        p = banded_random_problem(512, seed=3)
        p.name = "c3_banded_N512_P4"
        return p
    if idx == 4:
        return dimer_problem(1000, drive=True, name="c4_dimer_N1000_drive")
    raise ValueError(idx)


def u_scan_problem(idx: int, rank: int, world: int, dU: float = 0.25) -> Problem:
    """Rank `rank`'s share of a U scan (the bifurcation-diagram axis, PAPER.md P:259-261,
    Fig. 2): the dimer of configs[idx] (1, 2 or 4) at U = 2 + rank * dU.  Every
    rank's problem has the same pattern sizes; ranks share nothing (multi-GPU = independent
    unfolds, no data-path collective).  Other configs are not U-parametrised and are
    replicated."""
    if world <= 1 or idx not in (1, 2, 4):
        return config(idx)
    n = {1: 64, 2: 256, 4: 1000}[idx]
    U = 2.0 + rank * dU
    return dimer_problem(n, drive=idx != 1, name=f"{CONFIG_NAMES[idx]}_U{U:g}", U=U)


CONFIG_NAMES = {
    0: "c0_dense_N4_P1",
    1: "c1_dimer_N64",
    2: "c2_dimer_N256_drive",
    3: "c3_banded_N512_P4",
    4: "c4_dimer_N1000_drive",
}


# ---- F3: ensembles of random dense generators ------------------------------
# The ensemble of ref. [Karol] is not in the container; the reading used here (F3):
# H from the GUE (H = (X + X^+)/2, X complex Ginibre), rate matrix A = G G^+ with G a complex
# Ginibre M x r matrix (a Wishart GKS matrix, positive semidefinite), normalised to Tr A = N.
def gks_ensemble(n: int, batch: int, seed: int = 0, rank: int = 0):
    """(H (batch, N, N) complex128, A (batch, M, M) complex128) host arrays, seeded."""
    rng = np.random.default_rng(seed)
    m = n * n - 1
    r = rank or m
    H = np.empty((batch, n, n), dtype=np.complex128)
    A = np.empty((batch, m, m), dtype=np.complex128)
    for b in range(batch):
        X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        H[b] = (X + X.conj().T) / 2
        G = rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r))
        Ab = G @ G.conj().T
        A[b] = Ab * (n / np.trace(Ab).real)
    return H, A


def gks_ensemble_torch(n: int, batch: int, seed: int = 0, device="cuda"):
    """The same recipe drawn on the device with torch (large N: the Wishart product is an
    M x M x M complex GEMM); not bitwise equal to gks_ensemble."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    m = n * n - 1
    H = torch.empty((batch, n, n), dtype=torch.complex128, device=device)
    A = torch.empty((batch, m, m), dtype=torch.complex128, device=device)
    for b in range(batch):
        X = torch.randn((n, n), dtype=torch.complex128, device=device, generator=gen) * np.sqrt(2.0)
        H[b] = (X + X.conj().T) / 2
        G = torch.randn((m, m), dtype=torch.complex128, device=device, generator=gen) * np.sqrt(2.0)
        torch.matmul(G, G.conj().T, out=A[b])
        A[b] *= n / torch.diagonal(A[b]).real.sum()
        del G
    return H, A


def rank_p_coefficients(n: int, P: int, seed: int = 0, band: int = 0):
    """Random complex coefficient vectors l_p (P, M) and rates gamma_p (P,) for A = sum_p
    gamma_p l_p l_p^+ (the spectral form).  band > 0: only the S_ab / J_ab with
    b - a <= band (and every D^l) get a coefficient (generator order R5), so that
    L_p = sum_j l_pj F_j is banded."""
    rng = np.random.default_rng(seed)
    m = n * n - 1
    l = rng.standard_normal((P, m)) + 1j * rng.standard_normal((P, m))
    if band > 0:
        npairs = n * (n - 1) // 2
        keep = np.ones(m, dtype=bool)
        q = 0
        for a in range(n):
            for b in range(a + 1, n):
                if b - a > band:
                    keep[q] = keep[npairs + q] = False
                q += 1
        l[:, ~keep] = 0.0
    g = rng.uniform(0.05, 0.5, size=P)
    return l, g
