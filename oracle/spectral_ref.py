"""Gap detection, QRCP assignment, static pipeline — restatement (TEST INFRASTRUCTURE ONLY).

Follows ``specpart/spectral.py`` of the reference:
* ``detect_gap``            spectral.py:89-131
* ``assign_clusters_qrcp``  spectral.py:134-170 (dgeqp3 pivots of X', sorted seeds,
                            cond <= 1e12, Psi = X X[J]^-1, argmax |Psi|, zero rows -> 0,
                            label compaction as Partition.from_labels spectral.py:63-70)
* ``block_size_for``        spectral.py:173-177
* ``partition_static``      spectral.py:180-218
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

from .graph_ref import LaplacianRef, directed_csr
from .lobpcg_ref import SolverCfg, lobpcg_ref, random_init

GAP_FLOOR = 1e-12


def block_size_for(k):
    return k + max(2, math.ceil(0.1 * k))


def detect_gap_ref(lam, k_min=2, alpha=3.0):
    """Returns (k, reliable, confidence) (spectral.py:89-131)."""
    lam = np.asarray(lam, dtype=np.float64)
    inc = np.maximum(np.diff(lam), 0.0)
    floor = GAP_FLOOR * abs(float(lam[-1]))
    k = None
    for cand in range(max(k_min, 2), lam.size):
        if inc[cand - 1] > alpha * max(float(inc[: cand - 1].max()), floor):
            k = cand
            break
    reliable = k is not None
    if k is None:
        k = int(np.argmax(inc)) + 1
    if k >= 2:
        den = max(float(inc[: k - 1].max()), floor)
        conf = float(inc[k - 1] / den) if den > 0 else 0.0
    else:
        conf = 0.0
    return k, reliable, conf


def qrcp_pivots_ref(x):
    """First k column pivots of dgeqp3 on X' (spectral.py:153)."""
    _, _, piv = scipy.linalg.qr(x.T, mode="economic", pivoting=True)
    return piv[: x.shape[1]]


def qrcp_assign_ref(x):
    """Compacted labels (spectral.py:134-170); raises ValueError on a singular seed block."""
    x = np.asarray(x, dtype=np.float64)
    k = x.shape[1]
    seeds = np.sort(qrcp_pivots_ref(x))
    s = x[seeds, :]
    if np.linalg.cond(s) > 1e12:
        raise ValueError("seed rows numerically singular")
    psi = np.linalg.solve(s.T, x.T).T
    raw = np.argmax(np.abs(psi), axis=1)
    raw[~np.any(x, axis=1)] = 0
    _, compact = np.unique(raw, return_inverse=True)
    return compact.astype(np.int64), seeds


def partition_static_ref(edges, n, cfg: SolverCfg, k_expected, fix_k=True, x0=None,
                         alpha=3.0, k_min=2, callback=None):
    """Edge list -> (labels, state, (k, reliable)) (spectral.py:180-218)."""
    indptr, indices, data = directed_csr(edges, n)
    l = min(block_size_for(k_expected), n)
    run = SolverCfg(block_size=l, tol=cfg.tol, max_iter=cfg.max_iter, seed=cfg.seed,
                    soft_lock_tol=cfg.soft_lock_tol, deflate_ones=cfg.deflate_ones)
    start = random_init(n, l, cfg.seed) if x0 is None else x0
    op = LaplacianRef(indptr, indices, data, n)
    state = lobpcg_ref(op, start, run, n_converge=min(k_expected + 1, l), callback=callback)
    gap = detect_gap_ref(state.eigenvalues, k_min=min(k_min, l - 1), alpha=alpha)
    k_used = k_expected if fix_k else gap[0]
    labels, _ = qrcp_assign_ref(state.vectors[:, :k_used])
    return labels, state, gap
