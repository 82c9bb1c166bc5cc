"""float32 storage: the Rayleigh-Ritz re-solve on an orthonormalised P when G_B is
ill-conditioned (lobpcg.cu orth_p) keeps long solves on the spectrum."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spb():
    import paper_1708_07481_b200 as spb

    return spb


def test_long_float32_solve_stays_on_spectrum(spb):
    from paper_1708_07481_b200.dcsbm import DcsbmSpec, generate_dcsbm

    spec = DcsbmSpec(n=900, blocks=4, arcs=18000, alpha=30.0, ratio=30.0, seed=2)
    e, truth = generate_dcsbm(spec)
    g = spb.from_edges(e, spec.n)
    hist = []
    x0 = np.random.default_rng(0).standard_normal((spec.n, 6))
    st = spb.lobpcg_solve(spb.LaplacianOperator(g), x0, spb.SolverConfig(block_size=6, tol=1e-6, max_iter=300, seed=0),
                          n_converge=5, callback=lambda it, th, nr: hist.append(th[0]), precision="float32")
    ref = spb.lobpcg_solve(spb.LaplacianOperator(g), x0, spb.SolverConfig(block_size=6, tol=1e-6, max_iter=300, seed=0),
                           n_converge=5, precision="float64")
    # the Laplacian is PSD: no Ritz value may fall below -(float32 floor)
    assert min(hist) > -1e-4
    assert st.iterations < 150 and ref.iterations < 150
    np.testing.assert_allclose(st.eigenvalues[:5], ref.eigenvalues[:5], atol=1e-4 * ref.eigenvalues[-1])
    assert st.solve_stats["orth_p"] >= 1
