"""GPU: the row-sharded driver path (gather buffer, remapped local CSR, all-reduce
hooks) on one rank reproduces the unsharded solve exactly."""

import numpy as np
import pytest

from tests.helpers import config_input

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["float32", "float64"])
def test_single_rank_sharded_equals_unsharded(precision):
    import paper_1708_07481_b200 as spb
    from paper_1708_07481_b200.sharded import RowShardedLaplacian, partition_static_sharded

    spec, edges, truth = config_input("c1", seed=0)
    k = spec.blocks
    l = spb.block_size_for(k)
    x0 = np.random.default_rng(0).standard_normal((spec.n, l))
    g = spb.from_edges(edges, spec.n)
    cfg = spb.SolverConfig(block_size=l, tol=1e-12, max_iter=20, seed=0)
    a, sa, _ = spb.partition_static(g, cfg, k_expected=k, fix_k=True, x0=x0, precision=precision)
    op = RowShardedLaplacian(g)
    assert op.nranks == 1 and op.n_local == spec.n
    b, sb, _ = partition_static_sharded(g, cfg, k_expected=k, fix_k=True, x0=x0,
                                        precision=precision, op=op)
    assert sa.iterations == sb.iterations
    assert np.array_equal(sa.eigenvalues, sb.eigenvalues)
    assert np.array_equal(a.labels, b.labels)
