"""GPU k-means mode (parity unpinned: the reference has no k-means). Checked
against a float64 numpy Lloyd iteration from the same seeds, and for recovery
on well-separated spectral embeddings."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lloyd(x, seeds, iters=100):
    mu = x[seeds].copy()
    lab = np.full(len(x), -1)
    for _ in range(iters):
        d = (mu ** 2).sum(1)[None, :] - 2 * x @ mu.T
        new = np.argmin(d, axis=1)
        if np.array_equal(new, lab):
            break
        lab = new
        for c in range(len(mu)):
            if np.any(lab == c):
                mu[c] = x[lab == c].mean(0)
    return lab


def test_kmeans_matches_numpy_lloyd():
    import paper_1708_07481_b200 as spb

    rng = np.random.default_rng(0)
    centers = rng.standard_normal((6, 5)) * 4
    x = np.concatenate([c + rng.standard_normal((300, 5)) for c in centers])
    seeds = np.array([0, 300, 600, 900, 1200, 1500])
    part, info = spb.assign_clusters_kmeans(x, 6, seeds=seeds, return_info=True)
    want = _lloyd(x, seeds)
    from oracle import partition_match

    assert partition_match(want, part.labels) == 1.0
    assert info["iterations"] >= 1


def test_kmeans_on_partition_embedding():
    import paper_1708_07481_b200 as spb
    from tests.helpers import config_input

    spec, edges, truth = config_input("c1", seed=0)
    g = spb.from_edges(edges, spec.n)
    l = spb.block_size_for(spec.blocks)
    cfg = spb.SolverConfig(block_size=l, tol=1e-12, max_iter=50, seed=0)
    part, st, _ = spb.partition_static(g, cfg, k_expected=spec.blocks, fix_k=True, precision="float64")
    km = spb.assign_clusters_kmeans(st.device_vectors[:, : spec.blocks], spec.blocks)
    km2, _, _ = spb.partition_static(g, cfg, k_expected=spec.blocks, fix_k=True,
                                     precision="float64", assign="kmeans")
    from oracle import partition_match

    assert partition_match(km.labels, km2.labels) == 1.0
    # Lloyd refinement from the QRCP seeds does not lose the planted structure
    q, m = partition_match(truth, part.labels), partition_match(truth, km.labels)
    print(f"qrcp {q:.4f} kmeans {m:.4f}")
    assert q > 0.7 and m > q - 0.05


def test_kmeans_float32_and_normalize():
    import paper_1708_07481_b200 as spb
    import torch

    rng = np.random.default_rng(1)
    centers = rng.standard_normal((4, 3)) * 5
    x = np.concatenate([c + rng.standard_normal((200, 3)) for c in centers])
    seeds = np.array([5, 205, 405, 605])
    p32 = spb.assign_clusters_kmeans(torch.tensor(x, dtype=torch.float32, device="cuda"), 4, seeds=seeds)
    want = _lloyd(x, seeds)
    from oracle import partition_match

    assert partition_match(want, p32.labels) > 0.995
    xn = x / np.linalg.norm(x, axis=1, keepdims=True)
    pn = spb.assign_clusters_kmeans(x, 4, seeds=seeds, normalize_rows=True)
    assert partition_match(_lloyd(xn, seeds), pn.labels) > 0.995


@pytest.mark.parametrize("k", [44, 98, 160])
def test_kmeans_tensor_core_distance_gemm(k):
    """float32 embeddings take the tcgen05 distance GEMM with the fused argmin epilogue
    (k <= 128: one epilogue warp per row; 128 < k <= 192, C4's k = 160: two column
    halves combined through shared memory). Against a float64 numpy Lloyd from the same
    seeds; clusters are well separated, so near-ties are rare."""
    import torch

    import paper_1708_07481_b200 as spb
    from oracle import partition_match

    rng = np.random.default_rng(k)
    n_per = 300
    centers = rng.standard_normal((k, k)) * 3.0
    x = np.concatenate([c + rng.standard_normal((n_per, k)) for c in centers])
    perm = rng.permutation(len(x))
    x = x[perm]
    inv = np.argsort(perm)
    seeds = np.sort(inv[np.arange(k) * n_per])  # one row of each cluster
    xt = torch.tensor(x, dtype=torch.float32, device="cuda")
    part, info = spb.assign_clusters_kmeans(xt, k, seeds=seeds, return_info=True)
    want = _lloyd(x.astype(np.float32).astype(np.float64), seeds)
    agree = partition_match(want, part.labels)
    print(f"\nk={k}: tensor-core k-means agreement {agree:.5f}, {info['iterations']} Lloyd steps")
    assert agree > 0.999


def test_kmeans_contract_errors():
    import paper_1708_07481_b200 as spb

    with pytest.raises(spb.ContractError):
        spb.assign_clusters_kmeans(np.zeros((3, 2)), 4)
    with pytest.raises(spb.ContractError):
        spb.assign_clusters_kmeans(np.zeros((10, 2)), 3)  # k > width with default seeds


def test_contingency_device_matches_host():
    import torch

    import paper_1708_07481_b200 as spb
    from paper_1708_07481_b200.metrics import contingency_device

    rng = np.random.default_rng(3)
    for n, kt, kf in [(1000, 5, 7), (200_000, 44, 44), (50_000, 160, 300)]:
        t = rng.integers(0, kt, n)
        f = rng.integers(0, kf, n)
        t[0], f[0] = kt - 1, kf - 1
        dev = contingency_device(torch.tensor(t, device="cuda"), torch.tensor(f, device="cuda"))
        host = spb.contingency(t, f)
        assert np.array_equal(dev.counts, host.counts) and dev.n == host.n
        assert spb.partition_match(dev) == spb.partition_match(host)
