"""Generate golden fixtures by running the REAL reference (``specpart``) here.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Outputs ``tests/golden/*.npz`` (committed). Inputs are regenerated at test time
from the seeds stored in each fixture (DC-SBM via paper_1708_07481_b200.dcsbm,
small random graphs via numpy), and each fixture stores a sha256 of the input
arcs so a generator drift is detected instead of silently changing the pin.
BLAS is pinned to one thread: the reference is only byte-stable that way
(SURVEY.md §8(c)).
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import specpart  # noqa: E402
from specpart import graph as rg  # noqa: E402
from specpart import lobpcg as rl  # noqa: E402
from specpart import spectral as rs  # noqa: E402
from specpart import metrics as rm  # noqa: E402

from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402
from tests.golden.cases import small_graph_cases, qrcp_cases  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def graph_fixture():
    out = {}
    for name, (edges, n, weights) in small_graph_cases().items():
        g = rg.from_edges(edges, n, weights=weights)
        s = rg.symmetrize(g)
        d = rg.degrees(g)
        x = np.random.default_rng(11).standard_normal((n, 3))
        y = rg.laplacian_apply(g, d, x)
        out[f"{name}/a_indptr"] = g.row_offsets
        out[f"{name}/a_indices"] = g.col_indices
        out[f"{name}/a_data"] = g.weights
        out[f"{name}/w_indptr"] = s.row_offsets
        out[f"{name}/w_indices"] = s.col_indices
        out[f"{name}/w_data"] = s.weights
        out[f"{name}/deg"] = d
        out[f"{name}/y"] = y
    for cfg in ("c1", "c2"):
        spec = CONFIGS[cfg]
        edges, truth = generate_dcsbm(spec)
        g = rg.from_edges(edges, spec.n)
        s = rg.symmetrize(g)
        d = rg.degrees(g)
        x = np.random.default_rng(5).standard_normal((spec.n, 8))
        y = rg.laplacian_apply(g, d, x)
        out[f"{cfg}/edges_sha"] = np.array(sha(edges))
        out[f"{cfg}/a_sha"] = np.array(sha(g.row_offsets, g.col_indices, g.weights))
        out[f"{cfg}/w_sha"] = np.array(sha(s.row_offsets, s.col_indices, s.weights))
        out[f"{cfg}/deg_sha"] = np.array(sha(d))
        out[f"{cfg}/nnz"] = np.array([g.nnz, s.nnz])
        out[f"{cfg}/y_colnorm"] = np.linalg.norm(y, axis=0)
        out[f"{cfg}/y_head"] = y[:64]
    np.savez_compressed(HERE / "graph.npz", **out)


def solve_fixture():
    """Small exact-spectrum and random-graph solves (test_lobpcg.py style)."""
    out = {}
    cases = {
        "path3": ([(0, 1), (1, 2)], 3, 3, rl.SolverConfig.high_accuracy(block_size=3, seed=0), 0),
        "k4": ([(i, j) for i in range(4) for j in range(i + 1, 4)], 4, 4,
               rl.SolverConfig.high_accuracy(block_size=4, seed=1), 1),
        "two_tri": ([(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)], 6, 3,
                    rl.SolverConfig.high_accuracy(block_size=3, seed=0), 0),
    }
    rng = np.random.default_rng(7)
    ends = rng.integers(0, 150, size=(600, 2))
    w = rng.random(600) * 2.0
    cases["rand150"] = (np.column_stack([ends, w[:, None]]), 150, 8,
                        rl.SolverConfig.high_accuracy(block_size=8, seed=1), 1)
    rng = np.random.default_rng(5)
    ends = rng.integers(0, 300, size=(1500, 2))
    w = rng.random(1500) * 2.0
    cases["rand300_20it"] = (np.column_stack([ends, w[:, None]]), 300, 8,
                             rl.SolverConfig(block_size=8, tol=1e-14, max_iter=20, seed=4), 4)
    for name, (edges, n, l, cfg, xseed) in cases.items():
        op = rg.LaplacianOperator(rg.from_edges(edges, n))
        hist_t, hist_r = [], []
        st = rl.lobpcg_solve(op, rl.random_init(n, l, xseed), cfg,
                             callback=lambda it, t, r: (hist_t.append(t), hist_r.append(r)))
        out[f"{name}/theta"] = st.eigenvalues
        out[f"{name}/norms"] = st.residual_norms
        out[f"{name}/iterations"] = np.array(st.iterations)
        out[f"{name}/hist_theta"] = np.array(hist_t)
        out[f"{name}/hist_norms"] = np.array(hist_r)
        out[f"{name}/vectors"] = st.vectors
    np.savez_compressed(HERE / "solve.npz", **out)


def partition_fixture(cfg_name, seeds, max_iter, ten_x=False):
    """partition_static on a DC-SBM config (SURVEY.md §8(d) reference mapping)."""
    spec0 = CONFIGS[cfg_name]
    out = {}
    for s in seeds:
        spec = spec0.__class__(**{**spec0.__dict__, "seed": s})
        edges, truth = generate_dcsbm(spec)
        g = rg.from_edges(edges, spec.n)
        k = spec.blocks
        l = rs.block_size_for(k)
        x0 = np.random.default_rng(s).standard_normal((spec.n, l))
        tol = 1e-12
        if ten_x:
            seen = {}
            op = rg.LaplacianOperator(g)
            rl.lobpcg_solve(op, x0, rl.SolverConfig(block_size=l, tol=1e-12, max_iter=1, seed=s),
                            n_converge=min(k + 1, l),
                            callback=lambda it, t, r: seen.setdefault(it, (t, r)))
            t0, r0 = seen[0]
            scale = max(abs(t0[l - 1]), op.scale_hint)
            tol = 0.1 * r0[: k + 1].max() / scale
        hist_t, hist_r = [], []
        orig = rl.lobpcg_solve

        def spy(op, x, c, precond=None, n_converge=None, callback=None):
            return orig(op, x, c, precond=precond, n_converge=n_converge,
                        callback=lambda it, t, r: (hist_t.append(t), hist_r.append(r)))

        rs.lobpcg_solve = spy
        try:
            part, st, gap = rs.partition_static(
                g, rl.SolverConfig(block_size=l, tol=tol, max_iter=max_iter, seed=s),
                k_expected=k, fix_k=True, x0=x0)
        finally:
            rs.lobpcg_solve = orig
        table = rm.contingency(truth, part)
        key = f"{cfg_name}_s{s}" + ("_10x" if ten_x else "")
        out[f"{key}/edges_sha"] = np.array(sha(edges))
        out[f"{key}/tol"] = np.array(tol)
        out[f"{key}/max_iter"] = np.array(max_iter)
        out[f"{key}/theta"] = st.eigenvalues
        out[f"{key}/norms"] = st.residual_norms
        out[f"{key}/iterations"] = np.array(st.iterations)
        out[f"{key}/hist_theta"] = np.array(hist_t)
        out[f"{key}/hist_norms"] = np.array(hist_r)
        out[f"{key}/labels"] = part.labels.astype(np.int16)
        out[f"{key}/gap"] = np.array([gap.k, int(gap.reliable)])
        out[f"{key}/pm_pr_pp"] = np.array([rm.partition_match(table), rm.pairwise_recall(table),
                                           rm.pairwise_precision(table)])
        print(key, "iters", st.iterations, "pm/pr/pp", out[f"{key}/pm_pr_pp"], flush=True)
    return out


def qrcp_fixture():
    out = {}
    for name, x in qrcp_cases().items():
        _, _, piv = __import__("scipy.linalg").linalg.qr(x.T, mode="economic", pivoting=True)
        out[f"{name}/pivots"] = piv[: x.shape[1]]
        import warnings

        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            out[f"{name}/labels"] = rs.assign_clusters_qrcp(x).labels
    np.savez_compressed(HERE / "qrcp.npz", **out)


def stream_fixture():
    """partition_stream of the reference on small DC-SBM streams (emerging, snowball)."""
    from specpart import streaming as rstr
    from paper_1708_07481_b200.dcsbm import DcsbmSpec, emerging_slices, snowball_slices

    out = {}
    spec = DcsbmSpec(n=1500, blocks=6, arcs=30_000, alpha=3.0, ratio=8.0, seed=11)
    edges, truth = generate_dcsbm(spec)
    k = spec.blocks
    streams = {
        "emerging": [(d, spec.n) for d in emerging_slices(edges, 5, seed=11)],
        "snowball": snowball_slices(edges, spec.n, 5, seed=11)[1],
    }
    for mode, st in streams.items():
        stages = [rstr.StreamStage(index=i + 1, mode=mode, edge_delta=d, n_after=n)
                  for i, (d, n) in enumerate(st)]
        for init in ("warm", "random"):
            cfg = rl.SolverConfig(block_size=8, tol=1e-4, max_iter=200, seed=11)
            res = rstr.partition_stream(rg.empty_graph(0), stages, cfg, init_mode=init,
                                        k_expected=k, fix_k=True)
            key = f"{mode}_{init}"
            out[f"{key}/iterations"] = np.array([r.iterations for r in res])
            for i, r in enumerate(res):
                out[f"{key}/theta{i}"] = r.eigenstate.eigenvalues
                out[f"{key}/labels{i}"] = r.partition.labels.astype(np.int16)
            print(key, [r.iterations for r in res], flush=True)
    np.savez_compressed(HERE / "stream.npz", **out)


def main():
    assert specpart.__version__ == "0.1.0"
    graph_fixture()
    solve_fixture()
    stream_fixture()
    qrcp_fixture()
    out = {}
    out.update(partition_fixture("c1", seeds=[0, 1], max_iter=20))
    out.update(partition_fixture("c1", seeds=[0], max_iter=30, ten_x=True))
    out.update(partition_fixture("c2", seeds=[0], max_iter=20))
    np.savez_compressed(HERE / "partition.npz", **out)


if __name__ == "__main__":
    main()
