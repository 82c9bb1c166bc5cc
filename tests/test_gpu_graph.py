"""GPU parity of (a) CSR build + degrees and (b) Laplacian SpMM against the oracle."""

import numpy as np
import pytest

import oracle
from tests.golden.cases import small_graph_cases
from tests.helpers import config_input, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spb():
    import paper_1708_07481_b200 as spb

    return spb


@pytest.mark.parametrize("name", sorted(small_graph_cases()))
def test_small_graphs_bit_exact(spb, golden_graph, name):
    edges, n, w = small_graph_cases()[name]
    g = spb.from_edges(edges, n, weights=w)
    gold = golden_graph
    assert np.array_equal(g.row_offsets, gold[f"{name}/a_indptr"])
    assert np.array_equal(g.col_indices, gold[f"{name}/a_indices"])
    assert np.array_equal(g.weights, gold[f"{name}/a_data"])
    s = spb.symmetrize(g)
    assert np.array_equal(s.row_offsets, gold[f"{name}/w_indptr"])
    assert np.array_equal(s.col_indices, gold[f"{name}/w_indices"])
    assert np.array_equal(s.weights, gold[f"{name}/w_data"])
    assert np.array_equal(spb.degrees(g), gold[f"{name}/deg"])
    x = np.random.default_rng(11).standard_normal((n, 3))
    y = spb.laplacian_apply(g, spb.degrees(g), x)
    assert np.allclose(y, gold[f"{name}/y"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_config_graphs_bit_exact(spb, golden_graph, cfg):
    spec, edges, _ = config_input(cfg)
    gold = golden_graph
    g = spb.from_edges(edges, spec.n)
    assert sha(g.row_offsets, g.col_indices, g.weights) == str(gold[f"{cfg}/a_sha"])
    s = spb.symmetrize(g)
    assert sha(s.row_offsets, s.col_indices, s.weights) == str(gold[f"{cfg}/w_sha"])
    assert sha(spb.degrees(g)) == str(gold[f"{cfg}/deg_sha"])
    x = np.random.default_rng(5).standard_normal((spec.n, 8))
    y = spb.laplacian_apply(g, spb.degrees(g), x)
    assert np.allclose(np.linalg.norm(y, axis=0), gold[f"{cfg}/y_colnorm"], rtol=1e-12)
    assert np.allclose(y[:64], gold[f"{cfg}/y_head"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("ncols", [1, 3, 8, 21, 49, 108, 176])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_spmm_widths_vs_oracle(spb, ncols, dtype):
    import torch

    spec, edges, _ = config_input("c1")
    g = spb.from_edges(edges, spec.n)
    op = spb.LaplacianOperator(g)
    ip, ix, dv = oracle.directed_csr(edges, spec.n)
    ref_op = oracle.LaplacianRef(ip, ix, dv, spec.n)
    x = np.random.default_rng(ncols).standard_normal((spec.n, ncols))
    want = ref_op.apply(x)
    ld = ((ncols + 7) // 8) * 8
    tdt = torch.float32 if dtype == "float32" else torch.float64
    xt = torch.zeros(spec.n, ld, dtype=tdt, device="cuda")
    xt[:, :ncols] = torch.from_numpy(x).to(xt)
    yt = torch.full_like(xt, 7.0)
    from paper_1708_07481_b200.graph import _spmm

    _spmm(g, op.device_degrees(dtype), xt[:, :ncols], yt[:, :ncols], dtype)
    got = yt[:, :ncols].double().cpu().numpy()
    tol = 1e-5 if dtype == "float32" else 1e-12
    assert np.allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())
    # padding columns untouched
    assert torch.all(yt[:, ncols:] == 7.0)
    assert op.scale_hint == float(oracle.directed_degrees(ip, ix, dv, spec.n).max())


def test_domain_errors(spb):
    with pytest.raises(spb.DomainError):
        spb.from_edges([(0, 5)], 3)
    with pytest.raises(spb.DomainError):
        spb.from_edges([(0, 1, -1.0)], 2)


def test_apply_delta_matches_bulk(spb):
    first = [(0, 1, 1.0), (2, 0, 2.0)]
    second = [(1, 3, 1.0), (0, 1, 1.0)]
    g = spb.apply_delta(spb.from_edges(first, 3), second, 4)
    h = spb.from_edges(first + second, 4)
    assert np.array_equal(g.row_offsets, h.row_offsets)
    assert np.array_equal(g.col_indices, h.col_indices)
    assert np.allclose(g.weights, h.weights)
    assert spb.degrees(g).tolist() == [4.0, 3.0, 2.0, 1.0]


def test_load_edge_list_native_matches_from_edges(spb, tmp_path):
    spec, edges, _ = config_input("c1", seed=0)
    rng = np.random.default_rng(5)
    # integer-valued weights: duplicate sums are exact in any order (the reference's
    # order of summing duplicates is scipy's unstable per-row sort)
    w = rng.integers(1, 5, len(edges)).astype(np.float64)
    path = tmp_path / "c1.tsv"
    with open(path, "w") as fh:
        fh.write("# DC-SBM c1\n")
        for (a, b), x in zip(edges, w):
            fh.write(f"{a + 1}\t{b + 1}\t{float(x)!r}\n")
    g = spb.load_edge_list(path, base=1, num_vertices=spec.n)
    dref = oracle.directed_csr(edges, spec.n, w)
    assert np.array_equal(g.row_offsets, dref[0]) and np.array_equal(g.col_indices, dref[1])
    assert np.array_equal(g.weights, dref[2])
    ref = oracle.symmetrize_csr(*dref, spec.n)
    sym = spb.symmetrize(g)
    assert np.array_equal(sym.row_offsets, ref[0]) and np.array_equal(sym.col_indices, ref[1])
    assert np.array_equal(sym.weights, ref[2])
    # errors keep the reference's types and line numbers
    bad = tmp_path / "bad.tsv"
    bad.write_text("1 2\n2 3\n3 x\n")
    with pytest.raises(spb.ParseError, match="line 3"):
        spb.load_edge_list(bad)


def test_symmetrize_twice_doubles_weights(spb):
    """reference test_graph.py:193-198: W(W) = 2W (AS_SYMMETRIC graphs)."""
    g = spb.from_edges([(0, 1, 2.0), (1, 2, 1.0), (2, 0, 0.5)], 3)
    once = spb.symmetrize(g)
    twice = spb.symmetrize(once)
    assert np.array_equal(twice.col_indices, once.col_indices)
    assert np.allclose(twice.weights, 2.0 * once.weights)
    assert np.array_equal(spb.degrees(twice), 2.0 * spb.degrees(once))


def test_symmetrize_modes(spb):
    """reference test_graph.py:182-191, :201-210."""
    g = spb.symmetrize(spb.from_edges([(0, 1, 1.0)], 2))
    assert g.to_dense().tolist() == [[0.0, 1.0], [1.0, 0.0]]
    d = spb.symmetrize(spb.from_edges([(0, 1, 2.0), (1, 0, 3.0)], 2)).to_dense()
    assert d[0, 1] == 5.0 and d[1, 0] == 5.0
    g = spb.symmetrize(spb.from_edges([(0, 1, 2.0), (1, 0, 3.0), (1, 2, 4.0)], 3), mode="logical")
    assert set(g.weights.tolist()) == {1.0}
    with pytest.raises(spb.DomainError):
        spb.symmetrize(spb.from_edges([(0, 1)], 2), mode="other")


@pytest.mark.parametrize("hub", [900, 3000])
def test_hub_rows_both_build_paths(spb, hub):
    """Rows up to 1024 entries take the bucket build (shared-memory row sort); a hub
    row beyond that sends the whole build down the radix-sort path. Both bit-exact
    against the oracle, with duplicate, antiparallel and weighted arcs."""
    rng = np.random.default_rng(hub)
    n = hub + 50
    leaves = rng.integers(1, n, size=hub)
    edges = np.concatenate([np.stack([np.zeros(hub, np.int64), leaves], 1),
                            np.stack([leaves[: hub // 3], np.zeros(hub // 3, np.int64)], 1),
                            rng.integers(0, n, size=(4 * n, 2))])
    w = rng.integers(1, 4, size=len(edges)).astype(np.float64) * 0.5
    g = spb.from_edges(np.column_stack([edges, w]), n)
    ip, ix, dv = oracle.directed_csr(np.column_stack([edges, w]), n)
    assert np.array_equal(g.row_offsets, ip) and np.array_equal(g.col_indices, ix)
    assert np.array_equal(g.weights, dv)
    wp, wx, wv = oracle.symmetrize_csr(ip, ix, dv, n)
    s = spb.symmetrize(g)
    assert np.array_equal(s.row_offsets, wp) and np.array_equal(s.col_indices, wx)
    assert np.array_equal(s.weights, wv)
    assert np.array_equal(spb.degrees(g), oracle.directed_degrees(ip, ix, dv, n))


@pytest.mark.parametrize("rows,cols", [(300_001, 7), (2_100_000, 3)])
def test_staged_h2d_copies_and_narrows_bit_exactly(rows, cols):
    """spb_h2d_staged (csrc/h2d.cu), the multi-threaded pinned-ring upload behind
    from_edges / lobpcg_solve for large numpy inputs: a ragged element count (last chunk
    partial, chunks spread over the threads) arrives bit-identical, and float64 ->
    float32 narrowing equals numpy's astype."""
    import torch

    from paper_1708_07481_b200 import _h2d

    rng = np.random.default_rng(rows)
    x = rng.standard_normal((rows, cols)) * 10.0 ** rng.integers(-30, 30, size=(rows, 1))
    assert x.nbytes >= _h2d._SMALL
    dev = torch.device("cuda", 0)
    assert torch.equal(_h2d.to_device(x, dev).cpu(), torch.from_numpy(x))
    assert torch.equal(_h2d.to_device(x, dev, np.float32).cpu(), torch.from_numpy(x.astype(np.float32)))
    e = rng.integers(-2**62, 2**62, size=(rows, cols))
    assert torch.equal(_h2d.to_device(e, dev).cpu(), torch.from_numpy(e))
