"""Host-side logic that needs no GPU: gap detection, block sizes, Partition,
label I/O, metrics, solver config, and the DC-SBM / stream input generators."""

import numpy as np
import pytest

import paper_1708_07481_b200 as spb
from paper_1708_07481_b200.dcsbm import CONFIGS, DcsbmSpec, emerging_slices, generate_dcsbm, snowball_slices


class TestDetectGap:
    def test_clear_gap(self):
        r = spb.detect_gap([0.0, 0.01, 0.02, 5.0, 5.1])
        assert r.k == 3 and r.reliable

    def test_unreliable_falls_back_to_argmax(self):
        r = spb.detect_gap([0.0, 1.0, 2.0, 3.5, 4.0])
        assert not r.reliable and r.k == 3

    def test_validation(self):
        with pytest.raises(spb.DomainError):
            spb.detect_gap([0.0, 1.0], k_min=2)
        with pytest.raises(spb.DomainError):
            spb.detect_gap([0.0, 2.0, 1.0])
        with pytest.raises(spb.DomainError):
            spb.detect_gap([0.0, 1.0, 2.0], alpha=1.0)

    def test_matches_oracle_on_random_spectra(self):
        import oracle

        rng = np.random.default_rng(0)
        for _ in range(200):
            lam = np.sort(rng.random(int(rng.integers(3, 30))) * rng.choice([1.0, 100.0]))
            r = spb.detect_gap(lam)
            k, rel, conf = oracle.detect_gap_ref(lam)
            assert (r.k, r.reliable) == (k, rel)
            assert r.confidence == pytest.approx(conf)


@pytest.mark.parametrize("k,l", [(1, 3), (2, 4), (8, 10), (19, 21), (20, 22), (32, 36), (44, 49), (98, 108), (160, 176)])
def test_block_size_for(k, l):
    assert spb.block_size_for(k) == l


def test_partition_from_labels_and_io(tmp_path):
    p = spb.Partition.from_labels([5, 3, 3, 9])
    assert p.labels.tolist() == [1, 0, 0, 2] and p.k == 3
    path = tmp_path / "l.tsv"
    spb.write_labels(p, path)
    assert np.array_equal(spb.read_labels(path).labels, p.labels)
    with pytest.raises(spb.ContractError):
        spb.Partition(np.array([0, 2]), 2)


def test_metrics_match_oracle():
    import oracle

    rng = np.random.default_rng(3)
    for _ in range(20):
        t = rng.integers(0, 5, 200)
        f = rng.integers(0, 7, 200)
        table = spb.contingency(t, f)
        assert spb.partition_match(table) == pytest.approx(oracle.partition_match(t, f))
        assert spb.pairwise_recall(table) == pytest.approx(oracle.pairwise_recall(t, f))
        assert spb.pairwise_precision(table) == pytest.approx(oracle.pairwise_precision(t, f))


def test_solver_config_semantics():
    cfg = spb.SolverConfig(block_size=5)
    assert cfg.tol == 1e-4 and cfg.max_iter == 20 and cfg.lock_tol == pytest.approx(1e-5)
    assert spb.SolverConfig.high_accuracy(block_size=5).tol == 1e-10
    with pytest.raises(spb.DomainError):
        spb.SolverConfig(block_size=0)


def test_random_init_is_numpy_pcg64():
    a = spb.random_init(50, 4, seed=9)
    assert np.array_equal(a, np.random.default_rng(9).standard_normal((50, 4)))


class TestGenerators:
    def test_dcsbm_shapes_and_mix(self):
        spec = CONFIGS["c1"]
        e, z = generate_dcsbm(spec)
        assert e.shape == (spec.arcs, 2) and z.shape == (spec.n,)
        within = (z[e[:, 0]] == z[e[:, 1]]).mean()
        assert abs(within - spec.ratio / (spec.ratio + 1)) < 0.02
        deg = np.bincount(e.ravel(), minlength=spec.n)
        assert abs(deg.mean() - 2 * spec.arcs / spec.n) < 1e-9

    def test_seeded(self):
        a = generate_dcsbm(DcsbmSpec(n=300, blocks=4, arcs=2000, seed=4))
        b = generate_dcsbm(DcsbmSpec(n=300, blocks=4, arcs=2000, seed=4))
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])

    def test_emerging_and_snowball(self):
        e, _ = generate_dcsbm(DcsbmSpec(n=400, blocks=4, arcs=3000, seed=1))
        sl = emerging_slices(e, 10, seed=1)
        assert sum(len(s) for s in sl) == len(e)
        relabel, stages = snowball_slices(e, 400, 10, seed=1)
        assert sorted(relabel.tolist()) == list(range(400))
        assert sum(len(s[0]) for s in stages) == len(e)
        prev = 0
        for delta, n_after in stages:
            assert n_after >= prev
            if len(delta):
                assert delta.max() < n_after
            prev = n_after


class TestPrecisionAndState:
    def test_default_precision_promotes_below_f32_floor(self, monkeypatch):
        from paper_1708_07481_b200.lobpcg import default_precision

        monkeypatch.delenv("SPB_PRECISION", raising=False)
        assert default_precision() == "float32"
        assert default_precision(1e-4) == "float32"
        with pytest.warns(UserWarning, match="float32 residual floor"):
            assert default_precision(spb.SolverConfig.high_accuracy(4).tol) == "float64"
        monkeypatch.setenv("SPB_PRECISION", "float32")
        assert default_precision(1e-12) == "float32"  # explicit choice wins

    def test_eigenstate_save_load_roundtrip(self, tmp_path):
        """EigenState.save/load as .npz (lobpcg.py:108-129)."""
        rng = np.random.default_rng(0)
        st = spb.EigenState(np.array([0.0, 1.5, 2.0]), rng.standard_normal((7, 3)),
                            np.array([1e-3, 2e-3, 3e-3]), 11, np.array([True, False, True]),
                            work_blocks=6)
        path = tmp_path / "state.npz"
        st.save(path)
        back = spb.EigenState.load(path)
        assert np.array_equal(back.eigenvalues, st.eigenvalues)
        assert np.array_equal(back.vectors, st.vectors)
        assert np.array_equal(back.residual_norms, st.residual_norms)
        assert back.iterations == 11 and back.work_blocks == 6
        assert np.array_equal(back.converged, st.converged)
        assert back.block_size == 3
