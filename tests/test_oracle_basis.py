"""Pins for oracle.basis: generators, projection (Eq. 5), f/d (Eq. 4)."""
import json
import os

import numpy as np
import pytest

from oracle import basis

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 16, 32])
def test_orthonormal_hermitian_traceless(n):
    F = basis.generators(n)
    M = n * n - 1
    assert F.shape == (M, n, n)
    flat = F.reshape(M, n * n)
    gram = flat @ flat.T.conj()  # Tr(F_i F_k^+) = Tr(F_i F_k) for Hermitian F
    assert np.abs(gram - np.eye(M)).max() < 1e-12
    assert np.abs(F - F.conj().transpose(0, 2, 1)).max() == 0.0
    assert np.abs(np.trace(F, axis1=1, axis2=2)).max() < 1e-12
    nnz = (np.abs(F) > 0).sum(axis=(1, 2))
    npairs = n * (n - 1) // 2
    assert (nnz[: 2 * npairs] == 2).all()
    assert (nnz[2 * npairs:] == np.arange(2, n + 1)).all()  # D^l has l+1 entries


@pytest.mark.parametrize("n", [2, 3, 7, 64])
def test_index_map_bijection(n):
    labs = basis.labels(n)
    seen = set()
    for s, (kind, a, b) in enumerate(labs):
        assert basis.gen_index(n, kind, a, b) == s
        seen.add(s)
    assert len(seen) == n * n - 1
    # lexicographic pair order
    ps = [basis.pair_index(n, a, b) for a in range(n) for b in range(a + 1, n)]
    assert ps == list(range(n * (n - 1) // 2))


def test_generator_examples():
    # SPEC.md S:55-57 examples restated: N=2 D^1 = diag(1,-1)/sqrt2 ; N=3 D^2 = diag(1,1,-2)/sqrt6
    assert np.allclose(basis.generator(2, "D", 1), np.diag([1, -1]) / np.sqrt(2))
    assert np.allclose(basis.generator(3, "D", 2), np.diag([1, 1, -2]) / np.sqrt(6))
    sx = np.array([[0, 1], [1, 0]])
    sy = np.array([[0, -1j], [1j, 0]])
    assert np.allclose(basis.generator(2, "S", 0, 1), sx / np.sqrt(2))
    assert np.allclose(basis.generator(2, "J", 0, 1), sy / np.sqrt(2))


@pytest.mark.parametrize("n", [2, 3, 6, 11])
def test_projection_and_reconstruction(n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    c_lit = basis.project_literal(A)
    assert np.abs(basis.project(A) - c_lit).max() < 1e-13
    # completeness: A = Tr(A)/N I + sum_s Tr(F_s A) F_s
    F = basis.generators(n)
    rec = np.trace(A) / n * np.eye(n) + np.einsum("s,sij->ij", c_lit, F)
    assert np.abs(rec - A).max() < 1e-12
    v = rng.standard_normal(n * n - 1)
    assert np.abs(basis.reconstruct(v, n) - basis.reconstruct_fast(v, n)).max() < 1e-14
    rho = basis.reconstruct(v, n)
    assert abs(np.trace(rho) - 1) < 1e-14
    assert np.abs(basis.project(rho).real - v).max() < 1e-13


def test_nz_counts_match_paper():
    gold = json.load(open(os.path.join(GOLDEN, "nz_counts.json")))
    for n_str, (nzf, nzd) in gold["counts"].items():
        n = int(n_str)
        f, d = basis.structure_constants(n)
        assert int((np.abs(f) > 1e-12).sum()) == nzf
        assert int((np.abs(d) > 1e-12).sum()) == nzd


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_f_antisymmetric_d_symmetric_and_algebra(n):
    f, d = basis.structure_constants(n)
    for perm, sign in [((1, 0, 2), -1), ((0, 2, 1), -1), ((2, 1, 0), -1), ((1, 2, 0), 1), ((2, 0, 1), 1)]:
        assert np.abs(f - sign * f.transpose(perm)).max() < 1e-13
        assert np.abs(d - d.transpose(perm)).max() < 1e-13
    # Eqs. 2-3 as matrix identities
    F = basis.generators(n)
    M = F.shape[0]
    rng = np.random.default_rng(0)
    for _ in range(20):
        i, k = rng.integers(0, M, 2)
        comm = F[i] @ F[k] - F[k] @ F[i]
        anti = F[i] @ F[k] + F[k] @ F[i]
        assert np.abs(comm - 1j * np.einsum("l,lab->ab", f[i, k], F)).max() < 1e-13
        assert np.abs(anti - (2.0 / n) * (i == k) * np.eye(n) - np.einsum("l,lab->ab", d[i, k], F)).max() < 1e-13


def test_su3_gellmann_values():
    gold = json.load(open(os.path.join(GOLDEN, "su3_gellmann.json")))
    f, d = basis.structure_constants(3)
    idx = [basis.gen_index(3, k, a, b) for k, a, b in gold["gellmann_to_ours"]]
    import itertools

    def expected(table, antisym):
        out = np.zeros((8, 8, 8))
        for a, b, c, expr in table:
            val = float(eval(expr, {"sqrt": np.sqrt}))
            for perm in itertools.permutations(range(3)):
                tri = [(a, b, c)[p] - 1 for p in perm]
                sign = 1.0
                if antisym:
                    sign = np.linalg.det(np.eye(3)[list(perm)])
                out[tri[0], tri[1], tri[2]] = sign * val
        return out

    fg = expected(gold["f"], True)
    dg = expected(gold["d"], False)
    ours_f = f[np.ix_(idx, idx, idx)]
    ours_d = d[np.ix_(idx, idx, idx)]
    assert np.abs(ours_f - np.sqrt(2) * fg).max() < 1e-13
    assert np.abs(ours_d - np.sqrt(2) * dg).max() < 1e-13
