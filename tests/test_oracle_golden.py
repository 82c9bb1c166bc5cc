"""Pin the CPU oracle (oracle/) against fixtures produced by the real reference.

The fixtures come from tests/golden/make_golden.py, which imported
/root/reference/pkg/src/specpart in the build container.
"""

import numpy as np
import pytest

import oracle
from oracle.lobpcg_ref import SolverCfg, lobpcg_ref, random_init
from tests.golden.cases import qrcp_cases, small_graph_cases
from tests.helpers import config_input, sha, solve_cases


@pytest.mark.parametrize("name", sorted(small_graph_cases()))
def test_small_graph_build_bit_exact(golden_graph, name):
    edges, n, w = small_graph_cases()[name]
    ip, ix, dv = oracle.directed_csr(edges, n, w)
    g = golden_graph
    assert np.array_equal(ip, g[f"{name}/a_indptr"])
    assert np.array_equal(ix, g[f"{name}/a_indices"])
    assert np.array_equal(dv, g[f"{name}/a_data"])
    wp, wx, wv = oracle.symmetrize_csr(ip, ix, dv, n)
    assert np.array_equal(wp, g[f"{name}/w_indptr"])
    assert np.array_equal(wx, g[f"{name}/w_indices"])
    assert np.array_equal(wv, g[f"{name}/w_data"])
    d = oracle.directed_degrees(ip, ix, dv, n)
    assert np.array_equal(d, g[f"{name}/deg"])
    x = np.random.default_rng(11).standard_normal((n, 3))
    y = oracle.laplacian_apply(ip, ix, dv, n, d, x)
    assert np.allclose(y, g[f"{name}/y"], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_config_graph_build_bit_exact(golden_graph, cfg):
    spec, edges, _ = config_input(cfg)
    g = golden_graph
    assert sha(edges) == str(g[f"{cfg}/edges_sha"]), "DC-SBM generator drifted"
    ip, ix, dv = oracle.directed_csr(edges, spec.n)
    assert sha(ip, ix, dv) == str(g[f"{cfg}/a_sha"])
    wp, wx, wv = oracle.symmetrize_csr(ip, ix, dv, spec.n)
    assert sha(wp, wx, wv) == str(g[f"{cfg}/w_sha"])
    d = oracle.directed_degrees(ip, ix, dv, spec.n)
    assert sha(d) == str(g[f"{cfg}/deg_sha"])
    x = np.random.default_rng(5).standard_normal((spec.n, 8))
    y = oracle.laplacian_apply(ip, ix, dv, spec.n, d, x)
    assert np.allclose(np.linalg.norm(y, axis=0), g[f"{cfg}/y_colnorm"], rtol=1e-12)
    assert np.allclose(y[:64], g[f"{cfg}/y_head"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", sorted(solve_cases()))
def test_small_solves_match_reference(golden_solve, name):
    edges, n, l, kw, xseed = solve_cases()[name]
    ip, ix, dv = oracle.directed_csr(edges, n)
    op = oracle.LaplacianRef(ip, ix, dv, n)
    ht, hr = [], []
    st = lobpcg_ref(op, random_init(n, l, xseed), SolverCfg(block_size=l, **kw),
                    callback=lambda it, t, r: (ht.append(t), hr.append(r)))
    g = golden_solve
    scale = max(1.0, op.scale_hint)
    assert st.iterations == int(g[f"{name}/iterations"])
    assert np.allclose(st.eigenvalues, g[f"{name}/theta"], rtol=1e-9, atol=1e-9 * scale)
    ref_h = g[f"{name}/hist_theta"]
    assert len(ht) == len(ref_h)
    assert np.allclose(np.array(ht), ref_h, rtol=1e-8, atol=1e-8 * scale)
    a, b = np.array(hr), g[f"{name}/hist_norms"]
    # early history tight; in long high-accuracy solves nearly-degenerate tail
    # columns drift chaotically once residuals fall below ~1e-6*scale, so the
    # history is compared as |log10 ratio| <= 0.05 above that level (measured:
    # oracle vs reference differ by 3% at callback 92 of the 224-callback rand150)
    assert np.allclose(a[:30], b[:30], rtol=1e-6, atol=1e-10 * scale)
    big = b > 1e-6 * scale
    assert np.all(np.abs(np.log10(a[big] / b[big])) <= 0.05)


@pytest.mark.parametrize("name", sorted(qrcp_cases()))
def test_qrcp_matches_reference(golden_qrcp, name):
    x = qrcp_cases()[name]
    piv = oracle.spectral_ref.qrcp_pivots_ref(x)
    assert np.array_equal(piv, golden_qrcp[f"{name}/pivots"])
    labels, _ = oracle.qrcp_assign_ref(x)
    assert np.array_equal(labels, golden_qrcp[f"{name}/labels"])


@pytest.mark.parametrize("key", ["c1_s0", "c1_s1", "c1_s0_10x", "c2_s0"])
def test_partition_static_matches_reference(golden_partition, key):
    cfg, s = key.split("_")[0], int(key.split("_")[1][1:])
    spec, edges, truth = config_input(cfg, seed=s)
    g = golden_partition
    assert sha(edges) == str(g[f"{key}/edges_sha"])
    k = spec.blocks
    l = oracle.block_size_for(k)
    x0 = np.random.default_rng(s).standard_normal((spec.n, l))
    ht, hr = [], []
    labels, st, gap = oracle.partition_static_ref(
        edges, spec.n, SolverCfg(block_size=l, tol=float(g[f"{key}/tol"]),
                                 max_iter=int(g[f"{key}/max_iter"]), seed=s),
        k_expected=k, x0=x0, callback=lambda it, t, r: (ht.append(t), hr.append(r)))
    assert st.iterations == int(g[f"{key}/iterations"])
    assert np.allclose(st.eigenvalues, g[f"{key}/theta"], rtol=1e-8, atol=1e-8)
    assert np.allclose(np.array(hr), g[f"{key}/hist_norms"], rtol=1e-6)
    assert np.array_equal(labels, g[f"{key}/labels"].astype(np.int64))
    pm = oracle.partition_match(truth, labels)
    assert abs(pm - g[f"{key}/pm_pr_pp"][0]) < 1e-12


def _stream_stages(mode):
    from paper_1708_07481_b200.dcsbm import DcsbmSpec, emerging_slices, generate_dcsbm, snowball_slices

    spec = DcsbmSpec(n=1500, blocks=6, arcs=30_000, alpha=3.0, ratio=8.0, seed=11)
    edges, _ = generate_dcsbm(spec)
    if mode == "emerging":
        return spec, [(d, spec.n) for d in emerging_slices(edges, 5, seed=11)]
    return spec, snowball_slices(edges, spec.n, 5, seed=11)[1]


@pytest.mark.parametrize("key", ["emerging_warm", "emerging_random", "snowball_warm", "snowball_random"])
def test_stream_matches_reference(key):
    from tests.conftest import load_golden

    g = load_golden("stream")
    mode, init = key.split("_")
    spec, stages = _stream_stages(mode)
    res = oracle.partition_stream_ref(stages, SolverCfg(block_size=8, tol=1e-4, max_iter=200, seed=11),
                                      init_mode=init, k_expected=spec.blocks, fix_k=True)
    assert [r["iterations"] for r in res] == g[f"{key}/iterations"].tolist()
    for i, r in enumerate(res):
        assert np.allclose(r["theta"], g[f"{key}/theta{i}"], rtol=1e-7, atol=1e-7)
        assert oracle.partition_match(g[f"{key}/labels{i}"].astype(np.int64), r["labels"]) >= 0.999
