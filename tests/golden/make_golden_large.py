"""Golden fixtures at the large configs (C3, C4, C5) from the REAL reference.

Run in the build container only (it imports ``specpart`` from /root/reference):

    python tests/golden/make_golden_large.py c3     # -> tests/golden/large_c3.npz
    python tests/golden/make_golden_large.py c4     # -> tests/golden/large_c4.npz
    python tests/golden/make_golden_large.py c5     # -> tests/golden/stream_c5.npz

BLAS is pinned to one thread (byte-stable reference). Inputs
are regenerated at test time from the seeds (``dcsbm.generate_dcsbm``) and
checked against the stored ``edges_sha``.

* C3 (seed 0): the SURVEY §8(d) "10x rule": ``tol = 0.1 * r0 / scale`` from an
  it=0 dry run, ``max_iter=30``; full ``partition_static(..., fix_k=True)``.
* C4 (seed 0): CSR/degree shas plus a ``max_iter=3`` pin (history, theta,
  labels after 3 expansions). ``c4full`` runs the full 10x-rule solve (about
  an hour of CPU here) into ``large_c4full.npz``.
* C5: the C2 graph streamed over 10 stages, emerging and BFS-snowball orders,
  warm and random starts, per-stage tolerance = the 10x rule of the final
  graph (``tol`` stored), ``max_iter=30``.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
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
from specpart import streaming as rstr  # noqa: E402

from paper_1708_07481_b200.dcsbm import (  # noqa: E402
    CONFIGS, emerging_slices, generate_dcsbm, snowball_slices)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def ten_x_tol(g, x0, l, k, seed):
    """T = 0.1 * max_{j<k+1} r_j(it=0) / scale(it=0)."""
    seen = {}
    op = rg.LaplacianOperator(g)
    rl.lobpcg_solve(op, x0, rl.SolverConfig(block_size=l, tol=1e-12, max_iter=1, seed=seed),
                    n_converge=min(k + 1, l),
                    callback=lambda it, t, r: seen.setdefault(it, (t, r)))
    t0, r0 = seen[0]
    scale = max(abs(t0[l - 1]), op.scale_hint)
    return 0.1 * r0[: k + 1].max() / scale


def graph_pins(out, key, edges, n):
    t = time.perf_counter()
    g = rg.from_edges(edges, n)
    s = rg.symmetrize(g)
    d = rg.degrees(g)
    out[f"{key}/edges_sha"] = np.array(sha(edges))
    out[f"{key}/a_sha"] = np.array(sha(g.row_offsets, g.col_indices, g.weights))
    out[f"{key}/w_sha"] = np.array(sha(s.row_offsets, s.col_indices, s.weights))
    out[f"{key}/deg_sha"] = np.array(sha(d))
    out[f"{key}/nnz"] = np.array([g.nnz, s.nnz])
    out[f"{key}/w_maxweight"] = np.array(s.weights.max())
    print(key, "graph", g.nnz, s.nnz, f"{time.perf_counter() - t:.1f}s", flush=True)
    return g


def run_partition(out, key, g, truth, spec, l, x0, tol, max_iter):
    k = spec.blocks
    hist_t, hist_r, stamps = [], [], []
    orig = rl.lobpcg_solve

    def spy(op, x, c, precond=None, n_converge=None, callback=None):
        def cb(it, t, r):
            stamps.append(time.perf_counter())
            hist_t.append(t)
            hist_r.append(r)
        return orig(op, x, c, precond=precond, n_converge=n_converge, callback=cb)

    rs.lobpcg_solve = spy
    t0 = time.perf_counter()
    try:
        part, st, gap = rs.partition_static(
            g, rl.SolverConfig(block_size=l, tol=tol, max_iter=max_iter, seed=spec.seed),
            k_expected=k, fix_k=True, x0=x0)
    finally:
        rs.lobpcg_solve = orig
    total = time.perf_counter() - t0
    table = rm.contingency(truth, part)
    out[f"{key}/tol"] = np.array(tol)
    out[f"{key}/max_iter"] = np.array(max_iter)
    out[f"{key}/theta"] = st.eigenvalues
    out[f"{key}/norms"] = st.residual_norms
    out[f"{key}/iterations"] = np.array(st.iterations)
    out[f"{key}/hist_theta"] = np.array(hist_t)
    out[f"{key}/hist_norms"] = np.array(hist_r)
    out[f"{key}/labels"] = part.labels.astype(np.uint8 if part.labels.max() < 256 else np.uint16)
    out[f"{key}/gap"] = np.array([gap.k, int(gap.reliable)])
    out[f"{key}/pm_pr_pp"] = np.array([rm.partition_match(table), rm.pairwise_recall(table),
                                       rm.pairwise_precision(table)])
    st_ = np.array(stamps)
    # reference timings here (8-core container, 1 BLAS thread): informational only
    out[f"{key}/ref_seconds"] = np.array([total, (st_[-1] - st_[0]) / max(1, len(st_) - 1)])
    print(key, "iters", st.iterations, "pm/pr/pp", out[f"{key}/pm_pr_pp"],
          f"total {total:.1f}s", flush=True)


def static_case(cfg_name, max_iter, ten_x, fname, seed=0):
    spec0 = CONFIGS[cfg_name]
    spec = spec0.__class__(**{**spec0.__dict__, "seed": seed})
    edges, truth = generate_dcsbm(spec)
    out = {}
    key = f"{cfg_name}_s{seed}"
    g = graph_pins(out, key, edges, spec.n)
    l = rs.block_size_for(spec.blocks)
    x0 = np.random.default_rng(seed).standard_normal((spec.n, l))
    tol = ten_x_tol(g, x0, l, spec.blocks, seed) if ten_x else 1e-12
    print(key, "tol", tol, flush=True)
    run_partition(out, key, g, truth, spec, l, x0, tol, max_iter)
    np.savez_compressed(HERE / fname, **out)


def stream_case(sens=False):
    spec = CONFIGS["c2"]
    edges, truth = generate_dcsbm(spec)
    k = spec.blocks
    l = rs.block_size_for(k)
    g_full = rg.from_edges(edges, spec.n)
    x0 = np.random.default_rng(spec.seed).standard_normal((spec.n, l))
    tol = ten_x_tol(g_full, x0, l, k, spec.seed)
    print("c5 tol", tol, flush=True)
    out = {"tol": np.array(tol), "max_iter": np.array(30), "stages": np.array(10),
           "edges_sha": np.array(sha(edges))}
    relabel, snow = snowball_slices(edges, spec.n, 10, seed=spec.seed)
    streams = {
        "emerging": ([(d, spec.n) for d in emerging_slices(edges, 10, seed=spec.seed)],
                     truth),
        "snowball": (snow, truth[np.argsort(relabel)]),
    }
    fname = "stream_c5_sens.npz" if sens else "stream_c5.npz"
    for mode, (st, tr) in streams.items():
        stages = [rstr.StreamStage(index=i + 1, mode=mode, edge_delta=d, n_after=n)
                  for i, (d, n) in enumerate(st)]
        for init in (("warm",) if sens else ("warm", "random")):
            cfg = rl.SolverConfig(block_size=l, tol=tol, max_iter=30, seed=spec.seed)
            hists = []
            orig = rstr.lobpcg_solve

            def spy(op, x, c, precond=None, n_converge=None, callback=None):
                h = []
                hists.append(h)
                return orig(op, x, c, precond=precond, n_converge=n_converge,
                            callback=lambda it, t, r: h.append(r[: k + 1].max()))

            rstr.lobpcg_solve = spy
            try:
                res = rstr.partition_stream(rg.empty_graph(0), stages, cfg, init_mode=init,
                                            k_expected=k, fix_k=True)
            finally:
                rstr.lobpcg_solve = orig
            key = f"{mode}_{init}"
            out[f"{key}/iterations"] = np.array([r.iterations for r in res])
            out[f"{key}/seconds"] = np.array([r.wall_time for r in res])
            pms = []
            for i, r in enumerate(res):
                out[f"{key}/theta{i}"] = r.eigenstate.eigenvalues
                out[f"{key}/hist{i}"] = np.array(hists[i])
                n_i = len(r.partition.labels)
                table = rm.contingency(tr[:n_i], r.partition)
                pms.append([rm.partition_match(table), rm.pairwise_recall(table),
                            rm.pairwise_precision(table)])
            out[f"{key}/pm_pr_pp"] = np.array(pms)
            out[f"{key}/labels_last"] = res[-1].partition.labels.astype(np.uint8)
            print(key, [r.iterations for r in res],
                  [round(r.wall_time, 1) for r in res], flush=True)
            np.savez_compressed(HERE / fname, **out)


def main():
    assert specpart.__version__ == "0.1.0"
    what = sys.argv[1]
    if what == "c3":
        static_case("c3", 30, True, "large_c3.npz")
    elif what == "c4":
        static_case("c4", 3, False, "large_c4.npz")
    elif what == "c4full":
        static_case("c4", 30, True, "large_c4full.npz")
    elif what == "c5":
        stream_case()
    elif what == "c5sens":
        # the reference's own round-off sensitivity: the warm streams again with
        # OPENBLAS_NUM_THREADS=8 (a different BLAS summation order)
        assert os.environ.get("OPENBLAS_NUM_THREADS") == "8"
        stream_case(sens=True)
    else:
        raise SystemExit(f"unknown case {what}")


if __name__ == "__main__":
    main()
