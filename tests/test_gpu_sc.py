"""GPU parity of the structure-constant generator sun_structure_constants (
PAPER.md Step 2.2 P:328-355, Eqs. 2-4).

Pinned to: brute-force f, d over all triples (oracle.basis.structure_constants) at N = 2..6,
element by element; the paper's counts NZ_F, NZ_D (tests/golden/nz_counts.json and the
closed forms) up to N = 200; and the hot path itself: Q_H[s, n] = sum_m h_m f_mns (Eq. 6,
P:171-174) from the generated f equals the unfold's Q for a Hamiltonian-only generator.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import basis
from workloads import ZCSR

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _sun():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1812_11626_b200 as sun

    return sun


def _dense(idx, val, m):
    T = np.zeros((m, m, m))
    i = idx.cpu().numpy()
    np.add.at(T, (i[:, 0], i[:, 1], i[:, 2]), val.cpu().numpy())
    return T


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_structure_constants_vs_brute_force(n):
    sun = _sun()
    m = n * n - 1
    f_ref, d_ref = basis.structure_constants(n)
    gold = json.load(open(os.path.join(GOLDEN, "nz_counts.json")))["counts"][str(n)]
    for which, ref, count in (("f", f_ref, gold[0]), ("d", d_ref, gold[1])):
        idx, val = sun.structure_constants(n, which)
        assert idx.shape[0] == count, (which, idx.shape[0], count)
        keys = idx.cpu().numpy()
        assert len({tuple(k) for k in keys}) == count  # every ordered triple once
        T = _dense(idx, val, m)
        assert np.abs(T - ref).max() < 1e-14, which


@pytest.mark.parametrize("n", [10, 37, 64, 200])
def test_structure_constant_counts(n):
    sun = _sun()
    nz_f = 5 * n**3 - 9 * n**2 - 2 * n + 6
    nz_d = 6 * n**3 - n * (21 * n + 7) // 2 + 1
    assert sun.structure_constants(n, "f", count_only=True) == nz_f
    assert sun.structure_constants(n, "d", count_only=True) == nz_d


def test_eq6_contraction_matches_unfold():
    """Q_H[s, n] = sum_m h_m f_mns with the generated f equals the unfold of -i[H, .]."""
    sun = _sun()
    n = 7
    m = n * n - 1
    rng = np.random.default_rng(77)
    X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    H = (X + X.conj().T) / 2
    h = basis.project(H).real  # h_m = Tr(F_m H)
    idx, val = sun.structure_constants(n, "f")
    i = idx.cpu().numpy()
    v = val.cpu().numpy()
    Q = np.zeros((m, m))
    np.add.at(Q, (i[:, 2], i[:, 1]), h[i[:, 0]] * v)  # Q[s, n] += h_m f_mns
    Q0, _, K = sun.unfold(ZCSR.from_dense(H), None, [], [])
    G = np.zeros((m, m))
    rp, c, w = Q0.row_ptr.cpu().numpy(), Q0.col.cpu().numpy(), Q0.val.cpu().numpy()
    for s in range(m):
        G[s, c[rp[s]:rp[s + 1]]] = w[rp[s]:rp[s + 1]]
    assert np.abs(G - Q).max() <= 1e-12 * np.abs(Q).max()
