"""GPU parity of the small float64 kernels: generalized eigensolve and CholQR."""

import numpy as np
import pytest
import scipy.linalg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spb():
    import paper_1708_07481_b200 as spb

    return spb


def _spd_pair(m, seed, cond_b=10.0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, m))
    a = a + a.T
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    ev = np.geomspace(1.0, cond_b, m)
    b = (q * ev) @ q.T
    return a, b


@pytest.mark.parametrize("m", [1, 2, 3, 7, 21, 47, 48, 63, 100, 147, 164, 165, 170, 256, 257, 324, 401, 528])
def test_sygv_matches_lapack(spb, m):
    from paper_1708_07481_b200.lobpcg import _solve_small

    a, b = _spd_pair(m, m)
    nev = max(1, m // 3)
    th, c = _solve_small(a, b, nev)
    want = scipy.linalg.eigh(a, b, eigvals_only=True)[:nev]
    scale = max(1.0, np.abs(want).max())
    assert np.allclose(th, want, rtol=0, atol=1e-11 * scale)
    # B-orthonormal columns and residual
    assert np.allclose(c.T @ b @ c, np.eye(nev), atol=1e-10)
    res = a @ c - b @ c * th[None, :]
    assert np.abs(res).max() < 1e-9 * scale


def test_sygv_identity_b_and_clusters(spb):
    from paper_1708_07481_b200.lobpcg import _solve_small

    # repeated eigenvalues (K4-like) and exact zero
    q, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((12, 12)))
    ev = np.array([0.0, 4.0, 4.0, 4.0, 5.0, 5.0 + 1e-12, 7, 8, 9, 10, 11, 12.0])
    a = (q * ev) @ q.T
    th, c = _solve_small(a, None, 7)
    assert np.allclose(th, ev[:7], atol=1e-11)
    assert np.allclose(c.T @ c, np.eye(7), atol=1e-10)
    assert np.abs(a @ c - c * th).max() < 1e-10


def test_sygv_conditioning_errors(spb):
    from paper_1708_07481_b200.lobpcg import _solve_small

    a, _ = _spd_pair(10, 1)
    b = np.eye(10)
    b[3, 3] = 1e-9  # cond 1e9 > 1/sqrt(eps)
    with pytest.raises(spb.ConditioningError):
        _solve_small(a, b, 3)
    b[3, 3] = -1.0
    with pytest.raises(spb.ConditioningError):
        _solve_small(a, b, 3)
    a[0, 0] = np.nan
    with pytest.raises(spb.ConditioningError):
        _solve_small(a, np.eye(10), 3)
    # near the threshold the exact path decides: cond 5e7 passes, 8e7 fails
    a, _ = _spd_pair(10, 2)
    b = np.diag(np.r_[np.ones(9), 1.0 / 5e7])
    _solve_small(a, b, 3)
    b = np.diag(np.r_[np.ones(9), 1.0 / 8e7])
    with pytest.raises(spb.ConditioningError):
        _solve_small(a, b, 3)


def test_orthonormalize_and_rank_repair(spb):
    rng = np.random.default_rng(1234)
    x = rng.standard_normal((40, 6))
    spb.orthonormalize(x)
    assert np.allclose(x.T @ x, np.eye(6), atol=1e-12)
    x = rng.standard_normal((40, 5))
    x[:, 3] = x[:, 0]
    x[:, 4] = 0.0
    spb.orthonormalize(x, rng)
    assert np.allclose(x.T @ x, np.eye(5), atol=1e-10)
    with pytest.raises(spb.DomainError):
        spb.orthonormalize(np.zeros((6, 2)))
    with pytest.raises(spb.DomainError):
        spb.orthonormalize(rng.standard_normal((3, 5)))


def test_rayleigh_ritz_full_basis(spb):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((30, 30))
    a = a + a.T
    op = spb.DenseOperator(a)
    basis = rng.standard_normal((30, 30))
    spb.orthonormalize(basis, rng)
    vals, coeff = spb.rayleigh_ritz(op, basis)
    assert np.allclose(vals, np.linalg.eigvalsh(a), atol=1e-8)
    ritz = basis @ coeff
    assert np.allclose(ritz.T @ (a @ ritz), np.diag(vals), atol=1e-7)


@pytest.mark.parametrize("w", [49, 108, 176, 256])
def test_orthonormalize_wide_blocks(spb, w):
    # CholQR widths of C2..C4 (l = 49, 108, 176) and beyond: single-CTA LDL'
    # and cluster Cholesky paths
    rng = np.random.default_rng(w)
    x = rng.standard_normal((4 * w + 100, w)) * np.geomspace(1.0, 1e3, w)[None, :]
    spb.orthonormalize(x)
    assert np.allclose(x.T @ x, np.eye(w), atol=1e-11)


def test_sygv_not_pd_cluster(spb):
    from paper_1708_07481_b200.lobpcg import _solve_small

    a, b = _spd_pair(300, 5)
    b[150, 150] = -50.0  # indefinite B in the cluster Cholesky range
    with pytest.raises(spb.ConditioningError):
        _solve_small(a, b, 10)
