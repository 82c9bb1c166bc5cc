"""GPU: the tcgen05 3xTF32 Gram (mode 1) and the CUDA-core float64 Gram (mode 0)
against an exact float64 product of the same float32 inputs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gram(u, v, mode, dtype="float32"):
    import torch

    from paper_1708_07481_b200 import _native as N

    tdt = torch.float32 if dtype == "float32" else torch.float64
    code = N.F32 if dtype == "float32" else N.F64
    n, p = u.shape
    q = v.shape[1]
    ldu = ((p + 7) // 8) * 8 + 8  # padded row stride, like the solver's blocks
    ldv = ((q + 7) // 8) * 8
    ut = torch.zeros((n, ldu), dtype=tdt, device="cuda")
    vt = torch.zeros((n, ldv), dtype=tdt, device="cuda")
    ut[:, :p] = torch.from_numpy(u).to(ut)
    vt[:, :q] = torch.from_numpy(v).to(vt)
    out = torch.full((p, q), np.nan, dtype=torch.float64, device="cuda")
    L = N.lib()
    wsb = L.spb_gram_workspace(p, q, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(L.spb_gram(code, mode, N.ptr(ut), ldu, p, N.ptr(vt), ldv, q, n, N.ptr(out), q,
                       N.ptr(ws), wsb, N.stream()))
    return out.cpu().numpy()


@pytest.mark.parametrize("n,p,q", [(1000, 21, 63), (5003, 49, 147), (50000, 147, 294),
                                   (20000, 176, 352), (7000, 324, 324), (300, 8, 8), (77, 3, 5)])
def test_tensor_core_gram_accuracy(n, p, q):
    rng = np.random.default_rng(n + p + q)
    u = rng.standard_normal((n, p)).astype(np.float32)
    v = rng.standard_normal((n, q)).astype(np.float32)
    exact = u.astype(np.float64).T @ v.astype(np.float64)
    scale = np.abs(u.astype(np.float64)).T @ np.abs(v.astype(np.float64))
    g1 = _gram(u, v, 1)
    assert np.all(np.isfinite(g1))
    err = np.abs(g1 - exact) / scale
    assert err.max() < 2e-6, err.max()
    g0 = _gram(u, v, 0)
    assert np.abs(g0 - exact).max() <= 1e-12 * scale.max()


def test_fp64_mode_gram():
    rng = np.random.default_rng(2)
    u = rng.standard_normal((999, 13))
    v = rng.standard_normal((999, 7))
    g = _gram(u, v, 0, dtype="float64")
    assert np.allclose(g, u.T @ v, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("n,p,q", [(1000, 21, 63), (5003, 49, 147), (50000, 147, 294),
                                   (40000, 176, 352), (70000, 324, 324), (300, 8, 8), (77, 3, 5),
                                   (33000, 130, 90)])
def test_ozaki_int8_gram_accuracy(n, p, q):
    """spb_gram mode 2: int8 tcgen05 with five signed 7-bit digits per value and exact
    int32 sums (error O(2^-35) of the column maxima per product)."""
    rng = np.random.default_rng(n + 7 * p + q)
    u = rng.standard_normal((n, p)).astype(np.float32)
    v = rng.standard_normal((n, q)).astype(np.float32)
    v[:, 0] = 0.0  # an all-zero column

    def rel_err(u, v):
        exact = u.astype(np.float64).T @ v.astype(np.float64)
        scale = np.abs(u.astype(np.float64)).T @ np.abs(v.astype(np.float64))
        g = _gram(u, v, 2)
        assert np.all(np.isfinite(g)) and np.all(g[:, 0] == 0.0)
        return (np.abs(g - exact) / np.maximum(scale, 1e-300)).max()

    assert rel_err(u, v) < 1e-10
    # one entry 1e3 x larger per column of U: the shared column scale costs
    # ~10 bits of the other entries' digits (the scheme's known dynamic-range cost)
    u[5, :] *= 1e3
    assert rel_err(u, v) < 1e-7


@pytest.mark.parametrize("n,blocks,arcs", [(60000, 20, 1_200_000), (40000, 98, 1_000_000)])
def test_ozaki_rr_grams_track_dmma_in_the_solver(n, blocks, arcs):
    """The solver's Rayleigh-Ritz Grams on the Ozaki int8 path (default for C3/C4-sized
    bases) follow the float64 DMMA path: same iteration count, Ritz values within 1e-6
    relative, residual histories within 0.01 in log10, labels agree. With 98 blocks
    (l = 108 > one Ozaki column tile) the Ozaki run also takes the fused projection +
    CholQR step ([X | R]'R from one packing, lobpcg.cu project_orth) and the split
    G_B / G_A launches with the side-stream Cholesky, against the two-step float64 path."""
    import os

    import paper_1708_07481_b200 as spb
    from paper_1708_07481_b200.dcsbm import DcsbmSpec, generate_dcsbm

    spec = DcsbmSpec(n=n, blocks=blocks, arcs=arcs, alpha=3.0, ratio=5.0, seed=4)
    e, truth = generate_dcsbm(spec)
    g = spb.from_edges(e, spec.n)
    l = spb.block_size_for(spec.blocks)
    x0 = np.random.default_rng(4).standard_normal((spec.n, l))
    out = {}
    old = os.environ.get("SPB_GRAM")
    try:
        for mode in ("dmma", "oz"):
            os.environ["SPB_GRAM"] = mode
            hist = []
            part, st, _ = spb.partition_static(
                g, spb.SolverConfig(block_size=l, tol=1e-12, max_iter=12, seed=4), k_expected=spec.blocks,
                fix_k=True, x0=x0, callback=lambda it, th, nr: hist.append(nr[:spec.blocks].max()))
            out[mode] = (part.labels, st, np.array(hist))
    finally:
        if old is None:
            os.environ.pop("SPB_GRAM", None)
        else:
            os.environ["SPB_GRAM"] = old
    (la, sa, ha), (lb, sb, hb) = out["dmma"], out["oz"]
    assert sa.iterations == sb.iterations
    rel = np.abs(sa.eigenvalues - sb.eigenvalues) / np.maximum(np.abs(sa.eigenvalues), 1e-6 * sa.eigenvalues.max())
    assert rel.max() < 1e-6, rel.max()
    assert np.abs(np.log10(ha) - np.log10(hb)).max() < 0.01
    assert spb.partition_match(spb.contingency(la, lb)) > 0.999


@pytest.mark.parametrize("n,p", [(60000, 176), (9000, 49), (40000, 324)])
def test_ozaki_self_gram_packs_once(n, p):
    """U'U through spb_gram mode 2 with the same device block for both operands (the
    solver's CholQR Gram at C4): one packed operand, same accuracy as two."""
    import torch

    from paper_1708_07481_b200 import _native as N

    rng = np.random.default_rng(n + p)
    u = (rng.standard_normal((n, p)) * rng.random(n)[:, None]).astype(np.float32)
    ld = ((p + 7) // 8) * 8
    ut = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
    ut[:, :p] = torch.from_numpy(u).cuda()
    out = torch.full((p, p), np.nan, dtype=torch.float64, device="cuda")
    L = N.lib()
    wsb = L.spb_gram_workspace(p, p, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(L.spb_gram(N.F32, 2, N.ptr(ut), ld, p, N.ptr(ut), ld, p, n, N.ptr(out), p,
                       N.ptr(ws), wsb, N.stream()))
    g = out.cpu().numpy()
    u64 = u.astype(np.float64)
    exact = u64.T @ u64
    scale = np.abs(u64).T @ np.abs(u64)
    assert np.all(np.isfinite(g))
    # rows scaled by U(0, 1): the digits are relative to each column's maximum
    assert (np.abs(g - exact) / scale).max() < 1e-9
    two = _gram(u, u, 2)  # separate operand copies: the two-operand path
    assert (np.abs(g - two) / scale).max() < 1e-9


def test_fused_projection_guard_with_preconditioner():
    """A preconditioned residual has a large component inside span(X): the fused
    projection + CholQR of the Ozaki path (lobpcg.cu project_orth) must hand such
    blocks to the two-step sequence (energy guard in projected_gram), so a Jacobi-
    preconditioned float32 solve with l = 108 follows the float64-product path."""
    import os

    import paper_1708_07481_b200 as spb
    from paper_1708_07481_b200.dcsbm import DcsbmSpec, generate_dcsbm

    spec = DcsbmSpec(n=30000, blocks=98, arcs=750_000, alpha=3.0, ratio=5.0, seed=6)
    e, _ = generate_dcsbm(spec)
    g = spb.from_edges(e, spec.n)
    d = np.maximum(spb.degrees(g), 1.0)
    l = spb.block_size_for(spec.blocks)
    x0 = np.random.default_rng(6).standard_normal((spec.n, l))
    cfg = spb.SolverConfig(block_size=l, tol=1e-12, max_iter=8, seed=6)
    out = {}
    old = os.environ.get("SPB_GRAM")
    try:
        for mode in ("dmma", "oz"):
            os.environ["SPB_GRAM"] = mode
            hist = []
            st = spb.lobpcg_solve(spb.LaplacianOperator(g), x0, cfg, precond=lambda r: r / d[:, None],
                                  precision="float32",
                                  callback=lambda it, th, nr: hist.append(nr[:spec.blocks].max()))
            out[mode] = (st, np.array(hist))
    finally:
        if old is None:
            os.environ.pop("SPB_GRAM", None)
        else:
            os.environ["SPB_GRAM"] = old
    (sa, ha), (sb, hb) = out["dmma"], out["oz"]
    assert sa.iterations == sb.iterations
    rel = np.abs(sa.eigenvalues - sb.eigenvalues) / np.maximum(np.abs(sa.eigenvalues), 1e-6 * sa.eigenvalues.max())
    assert rel.max() < 1e-5, rel.max()
    assert np.abs(np.log10(ha) - np.log10(hb)).max() < 0.01


def test_ozaki_path_with_soft_locked_columns():
    """Soft locking on the Ozaki path (l = 108): with a loose soft_lock_tol columns
    leave the active set, so R is narrower than X (na < l), P is compacted and the
    packed [X | R] view, the Rayleigh-Ritz operand width and the kept X planes all
    change from iteration to iteration. Same iteration count, Ritz values and
    residual history as the float64-product path."""
    import os

    import paper_1708_07481_b200 as spb
    from paper_1708_07481_b200.dcsbm import DcsbmSpec, generate_dcsbm

    spec = DcsbmSpec(n=30000, blocks=98, arcs=900_000, alpha=3.0, ratio=8.0, seed=9)
    e, _ = generate_dcsbm(spec)
    g = spb.from_edges(e, spec.n)
    l = spb.block_size_for(spec.blocks)
    x0 = np.random.default_rng(9).standard_normal((spec.n, l))
    # probe: the lock threshold is the median residual after 6 iterations, so about half
    # of the columns are locked from then on
    probe = []
    op = spb.LaplacianOperator(g)
    spb.lobpcg_solve(op, x0, spb.SolverConfig(block_size=l, tol=1e-12, max_iter=6, seed=9),
                     precision="float32", callback=lambda it, th, nr: probe.append((np.array(th), np.array(nr))))
    th6, nr6 = probe[-1]
    scale = max(abs(float(th6[-1])), op.scale_hint)
    lock = float(np.median(nr6)) / scale
    cfg = spb.SolverConfig(block_size=l, tol=1e-12, max_iter=14, seed=9, soft_lock_tol=lock)
    out = {}
    old = os.environ.get("SPB_GRAM")
    try:
        for mode in ("dmma", "oz"):
            os.environ["SPB_GRAM"] = mode
            hist = []
            st = spb.lobpcg_solve(spb.LaplacianOperator(g), x0, cfg, precision="float32",
                                  callback=lambda it, th, nr: hist.append(np.array(nr)))
            out[mode] = (st, np.array(hist))
    finally:
        if old is None:
            os.environ.pop("SPB_GRAM", None)
        else:
            os.environ["SPB_GRAM"] = old
    (sa, ha), (sb, hb) = out["dmma"], out["oz"]
    locked = int((ha[-1] < lock * scale).sum())
    print(f"\nsoft lock: {locked} of {l} columns below the lock threshold at the end, "
          f"iterations {sa.iterations} / {sb.iterations}")
    assert locked > 0, "the case must lock columns to exercise na < l"
    assert sa.iterations == sb.iterations
    rel = np.abs(sa.eigenvalues - sb.eigenvalues) / np.maximum(np.abs(sa.eigenvalues), 1e-6 * sa.eigenvalues.max())
    assert rel.max() < 1e-5, rel.max()
    big = ha > 1e-3 * ha.max()
    assert np.abs(np.log10(ha[big]) - np.log10(hb[big])).max() < 0.02
