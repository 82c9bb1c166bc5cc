"""Streaming partition — restatement of ``specpart/streaming.py`` (TEST INFRASTRUCTURE ONLY).

warm_start (streaming.py:83-103), partition_stream (:126-192): per stage the
cumulative directed graph is rebuilt (graph.py:281-297), the solve is warm- or
random-started with per-stage seeds from SeedSequence(cfg.seed), then gap
detection and QRCP assignment.
"""

from __future__ import annotations

import numpy as np

from .graph_ref import LaplacianRef, coerce_edges, directed_csr
from .lobpcg_ref import SolverCfg, lobpcg_ref, random_init
from .spectral_ref import block_size_for, detect_gap_ref, qrcp_assign_ref


def warm_start_ref(prev_vectors, n_new, fill="zero", seed=0):
    n_old, l = prev_vectors.shape
    out = np.empty((n_new, l))
    out[:n_old] = prev_vectors
    if n_new > n_old:
        out[n_old:] = 0.0 if fill == "zero" else np.random.default_rng(seed).standard_normal((n_new - n_old, l))
    return out


def partition_stream_ref(stages, cfg: SolverCfg, init_mode="warm", k_expected=None, fix_k=False,
                         fill="zero", alpha=3.0, k_min=2):
    """stages: list of (delta_edges (m,2), n_after). Returns per-stage dicts."""
    l = block_size_for(k_expected) if k_expected is not None else cfg.block_size
    run = SolverCfg(block_size=l, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed,
                    soft_lock_tol=cfg.soft_lock_tol, deflate_ones=cfg.deflate_ones)
    nc = min(k_expected + 1, l) if k_expected is not None else None
    seeds = np.random.SeedSequence(cfg.seed).generate_state(len(stages))
    arcs = np.empty((0, 2), dtype=np.int64)
    prev = None
    out = []
    for (delta, n_after), seed in zip(stages, seeds):
        arcs = np.concatenate([arcs, np.asarray(delta, dtype=np.int64).reshape(-1, 2)])
        ip, ix, dv = directed_csr(arcs, n_after)
        op = LaplacianRef(ip, ix, dv, n_after)
        if init_mode == "warm" and prev is not None:
            x0 = warm_start_ref(prev, n_after, fill, int(seed))
        else:
            x0 = random_init(n_after, l, int(seed))
        st = lobpcg_ref(op, x0, run, n_converge=nc)
        k, rel, _ = detect_gap_ref(st.eigenvalues, k_min=min(k_min, l - 1), alpha=alpha)
        k_used = k_expected if (fix_k and k_expected is not None) else k
        labels, _ = qrcp_assign_ref(st.vectors[:, :k_used])
        out.append({"iterations": st.iterations, "theta": st.eigenvalues, "labels": labels})
        prev = st.vectors
    return out
