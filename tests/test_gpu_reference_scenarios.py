"""The reference test suite's solver / spectral / streaming scenarios
(pkg/tests/test_lobpcg.py, test_spectral.py, test_streaming.py), restated for
the device path: the same inputs and the same asserted properties, run through
this package's public API on the GPU (float64 storage where the reference
asserts float64 tolerances, both storages where the property is
precision-independent)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spb():
    import paper_1708_07481_b200 as spb

    return spb


def _dense_laplacian(edges, n):
    a = np.zeros((n, n))
    for e in edges:
        u, v = int(e[0]), int(e[1])
        w = float(e[2]) if len(e) > 2 else 1.0
        if u != v:
            a[u, v] += w
            a[v, u] += w
    return np.diag(a.sum(1)) - a


def _op(spb, edges, n):
    e = np.array([(a, b) for a, b, *_ in edges], dtype=np.int64).reshape(-1, 2)
    w = np.array([x[2] if len(x) > 2 else 1.0 for x in edges], dtype=np.float64)
    g = spb.from_edges(e, n, weights=w if any(len(x) > 2 for x in edges) else None)
    return spb.LaplacianOperator(g)


def _random_graph(rng, n, m):
    e = rng.integers(0, n, size=(m, 2))
    return e, _dense_laplacian(e, n)


def _angle(u, v):
    qu, _ = np.linalg.qr(u)
    qv, _ = np.linalg.qr(v)
    s = np.linalg.svd(qu.T @ qv, compute_uv=False)
    return float(np.arccos(np.clip(s.min(), -1.0, 1.0)))


# ---- lobpcg_solve ---------------------------------------------------------------

def test_path_and_complete_graph_spectra(spb):
    op = _op(spb, [(0, 1), (1, 2)], 3)
    st = spb.lobpcg_solve(op, spb.random_init(3, 3, 0), spb.SolverConfig.high_accuracy(3, seed=0),
                          precision="float64")
    assert np.allclose(st.eigenvalues, [0.0, 1.0, 3.0], atol=1e-10) and st.converged.all()
    edges = [(i, j) for i in range(4) for j in range(i + 1, 4)]
    st = spb.lobpcg_solve(_op(spb, edges, 4), spb.random_init(4, 4, 1),
                          spb.SolverConfig.high_accuracy(4, seed=1), precision="float64")
    assert np.allclose(st.eigenvalues, [0.0, 4.0, 4.0, 4.0], atol=1e-9)


def test_two_triangles_component_indicators(spb):
    edges = [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]
    st = spb.lobpcg_solve(_op(spb, edges, 6), spb.random_init(6, 3, 0),
                          spb.SolverConfig.high_accuracy(3, seed=0), precision="float64")
    assert np.allclose(st.eigenvalues, [0.0, 0.0, 3.0], atol=1e-8)
    ind = np.zeros((6, 2))
    ind[:3, 0] = 1.0
    ind[3:, 1] = 1.0
    assert _angle(st.vectors[:, :2], ind) < 1e-6


@pytest.mark.parametrize("precision", ["float32", "float64"])
def test_ritz_partial_traces_monotone(spb, precision):
    rng = np.random.default_rng(23)
    e, _ = _random_graph(rng, 250, 1200)
    op = spb.LaplacianOperator(spb.from_edges(e, 250))
    hist = []
    spb.lobpcg_solve(op, spb.random_init(250, 6, 3),
                     spb.SolverConfig(block_size=6, tol=1e-12, max_iter=25, seed=3),
                     callback=lambda it, vals, norms: hist.append(np.array(vals)),
                     precision=precision)
    traces = np.cumsum(np.array(hist), axis=1)
    slack = (1e-8 if precision == "float64" else 1e-5) * op.scale_hint
    assert np.all(np.diff(traces, axis=0) <= slack)


def test_eigenvalue_range_and_dense_oracle(spb):
    rng = np.random.default_rng(29)
    e, dense = _random_graph(rng, 100, 400)
    op = spb.LaplacianOperator(spb.from_edges(e, 100))
    st = spb.lobpcg_solve(op, spb.random_init(100, 5, 0), spb.SolverConfig.high_accuracy(5),
                          precision="float64")
    assert np.all(st.eigenvalues >= -1e-9) and np.all(st.eigenvalues <= 2 * op.scale_hint + 1e-9)
    want = np.linalg.eigvalsh(dense)[:5]
    assert np.allclose(st.eigenvalues, want, atol=1e-8 * max(1.0, want.max()))


def test_callback_sequence_and_unconverged_state(spb):
    op = _op(spb, [(0, 1), (1, 2), (2, 3)], 4)
    seen = []
    st = spb.lobpcg_solve(op, spb.random_init(4, 2, 1), spb.SolverConfig.high_accuracy(2, seed=1),
                          callback=lambda it, vals, norms: seen.append(it), precision="float64")
    assert seen == list(range(len(seen)))
    assert len(seen) in (st.iterations, st.iterations + 1)
    rng = np.random.default_rng(3)
    e, _ = _random_graph(rng, 200, 900)
    op = spb.LaplacianOperator(spb.from_edges(e, 200))
    st = spb.lobpcg_solve(op, spb.random_init(200, 6, 0),
                          spb.SolverConfig(block_size=6, tol=1e-14, max_iter=3, seed=0))
    assert st.iterations == 3 and not st.converged.all()
    assert st.vectors.shape == (200, 6)


def test_n_converge_limits_the_gate(spb):
    rng = np.random.default_rng(13)
    e, dense = _random_graph(rng, 120, 500)
    op = spb.LaplacianOperator(spb.from_edges(e, 120))
    cfg = spb.SolverConfig(block_size=8, tol=1e-7, max_iter=300, seed=5)
    full = spb.lobpcg_solve(op, spb.random_init(120, 8, 5), cfg, precision="float64")
    part = spb.lobpcg_solve(op, spb.random_init(120, 8, 5), cfg, n_converge=3, precision="float64")
    assert part.iterations <= full.iterations
    ev = np.linalg.eigvalsh(dense)
    assert np.abs(part.eigenvalues[:3] - ev[:3]).max() < 1e-5 * max(1.0, ev[-1])


def test_full_block_exact_and_shape_errors(spb):
    edges = [(0, 1, 2.0), (1, 2, 1.0), (0, 2, 0.5)]
    st = spb.lobpcg_solve(_op(spb, edges, 3), spb.random_init(3, 3, 2),
                          spb.SolverConfig.high_accuracy(3, seed=2), precision="float64")
    assert np.allclose(st.eigenvalues, np.linalg.eigvalsh(_dense_laplacian(edges, 3)), atol=1e-9)
    op = _op(spb, [(0, 1)], 2)
    with pytest.raises(spb.ContractError):
        spb.lobpcg_solve(op, spb.random_init(2, 2, 0), spb.SolverConfig(block_size=1))
    with pytest.raises(spb.DomainError):
        spb.lobpcg_solve(op, np.ones((2, 3)), spb.SolverConfig(block_size=3))


def test_work_blocks_budget(spb):
    rng = np.random.default_rng(19)
    e, _ = _random_graph(rng, 60, 200)
    st = spb.lobpcg_solve(spb.LaplacianOperator(spb.from_edges(e, 60)), spb.random_init(60, 4, 0),
                          spb.SolverConfig(block_size=4))
    assert st.work_blocks == 6


# ---- partition_static -------------------------------------------------------------

def _cliques(sizes):
    edges, off = [], 0
    for s in sizes:
        edges += [(off + i, off + j) for i in range(s) for j in range(i + 1, s)]
        off += s
    return np.array(edges, dtype=np.int64), off


@pytest.mark.parametrize("c", [2, 3, 4])
def test_component_count_recovered(spb, c):
    e, n = _cliques([6] * c)
    part, st, gap = spb.partition_static(spb.from_edges(e, n),
                                         spb.SolverConfig.high_accuracy(c + 2, seed=0),
                                         precision="float64")
    assert gap.k == c and part.k == c
    # every clique is one block
    lab = part.labels.reshape(c, 6)
    assert all(len(set(r)) == 1 for r in lab) and len(set(lab[:, 0])) == c


def test_fix_k_overrides_gap_and_tiny_graph(spb):
    e, n = _cliques([6, 6])
    part, _, gap = spb.partition_static(spb.from_edges(e, n), spb.SolverConfig.high_accuracy(5, seed=0),
                                        k_expected=3, fix_k=True, precision="float64")
    assert gap.k == 2 and part.k <= 3
    with pytest.raises(spb.DomainError):
        spb.partition_static(spb.empty_graph(0), spb.SolverConfig(block_size=2))
    part, _, _ = spb.partition_static(spb.from_edges(np.array([[0, 1]]), 2),
                                      spb.SolverConfig(block_size=2, seed=0), precision="float64")
    assert part.labels.size == 2


def test_planted_model_recovery(spb):
    from paper_1708_07481_b200.dcsbm import DcsbmSpec, generate_dcsbm

    spec = DcsbmSpec(n=900, blocks=4, arcs=18000, alpha=30.0, ratio=30.0, seed=2)
    e, truth = generate_dcsbm(spec)
    part, _, gap = spb.partition_static(spb.from_edges(e, spec.n), spb.SolverConfig(block_size=6, tol=1e-6, max_iter=300, seed=0),
                                        k_expected=4, fix_k=True)
    assert spb.partition_match(spb.contingency(truth, part.labels)) > 0.95


# ---- streaming ------------------------------------------------------------------

def _two_cliques():
    e, _ = _cliques([6, 6])
    return e


def test_stream_stage_one_same_for_both_modes_and_fixed_point(spb):
    e = _two_cliques()
    cfg = spb.SolverConfig(block_size=4, tol=1e-8, max_iter=200, seed=3)
    perm = np.random.default_rng(0).permutation(len(e))
    stages = [spb.StreamStage(index=i + 1, mode="emerging", edge_delta=e[c], n_after=12)
              for i, c in enumerate(np.array_split(perm, 2))]
    w = spb.partition_stream(spb.empty_graph(12), stages, cfg, init_mode="warm", precision="float64")
    r = spb.partition_stream(spb.empty_graph(12), stages, cfg, init_mode="random", precision="float64")
    assert np.array_equal(w[0].partition.labels, r[0].partition.labels)
    assert np.array_equal(w[0].eigenstate.eigenvalues, r[0].eigenstate.eigenvalues)
    assert w[0].init_mode == "random" and w[1].init_mode == "warm"
    truth = np.array([0] * 6 + [1] * 6)
    for res in (w, r):
        assert spb.partition_match(spb.contingency(truth, res[-1].partition.labels)) == 1.0
    fixed = [spb.StreamStage(index=1, mode="emerging", edge_delta=e, n_after=12),
             spb.StreamStage(index=2, mode="emerging", edge_delta=np.empty((0, 2), np.int64), n_after=12)]
    res = spb.partition_stream(spb.empty_graph(12), fixed, cfg, init_mode="warm", k_expected=2,
                               precision="float64")
    assert res[1].iterations <= 2
    assert np.array_equal(res[0].partition.labels, res[1].partition.labels)


def test_resolve_from_warm_converges_fast(spb):
    op = spb.LaplacianOperator(spb.from_edges(_two_cliques(), 12))
    cfg = spb.SolverConfig(block_size=3, tol=1e-4, max_iter=100)
    st = spb.lobpcg_solve(op, spb.random_init(12, 3, seed=2), cfg, precision="float64")
    again = spb.lobpcg_solve(op, spb.warm_start(st, 12), cfg, precision="float64")
    assert again.iterations <= 2
