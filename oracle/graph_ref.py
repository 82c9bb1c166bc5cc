"""Graph build and Laplacian apply — numpy restatement (TEST INFRASTRUCTURE ONLY).

Follows ``specpart/graph.py`` of the reference:
* ``_coerce_edges``      graph.py:106-132
* ``from_edges``         graph.py:135-145 (self-loops dropped, duplicates summed,
                         columns sorted)
* ``symmetrize``         graph.py:220-236 (W = A + A'; scipy's csr binop keeps
                         only non-zero sums)
* ``degrees``            graph.py:239-250 (bincount over rows + bincount over cols)
* ``laplacian_apply``    graph.py:253-278 (Y = d*X - A X - A' X)
* ``LaplacianOperator``  graph.py:300-317 (n, scale_hint = max d, apply)

The construction is a stable lexsort + segmented ``np.add.reduceat`` instead
of scipy's coo->csr, so it is an independent route to the same arrays.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


class OracleDomainError(ValueError):
    pass


class OracleContractError(ValueError):
    pass


def coerce_edges(edges, weights=None):
    """(m,2|3) edges -> int64 src, int64 dst, float64 w (graph.py:106-132)."""
    if isinstance(edges, np.ndarray) and edges.ndim == 2:
        arr = edges
    else:
        arr = np.asarray(list(edges), dtype=np.float64)
        if arr.size == 0:
            arr = arr.reshape(0, 2)
    if arr.ndim != 2 or arr.shape[1] not in (2, 3):
        raise OracleContractError("edges must be (m, 2) or (m, 3)")
    src = arr[:, 0].astype(np.int64)
    dst = arr[:, 1].astype(np.int64)
    if weights is not None:
        w = np.asarray(weights, dtype=np.float64)
        if w.shape != (src.size,):
            raise OracleContractError("weights length does not match edges")
    elif arr.shape[1] == 3:
        w = arr[:, 2].astype(np.float64)
    else:
        w = np.ones(src.size)
    if np.any(w < 0):
        raise OracleDomainError("negative edge weight")
    return src, dst, w


def _segment_csr(rows, cols, vals, n, drop_zero=False):
    """Sort (row, col) stably, sum equal keys in input order, emit CSR."""
    order = np.lexsort((cols, rows))
    r, c, v = rows[order], cols[order], vals[order]
    if r.size:
        new = np.empty(r.size, dtype=bool)
        new[0] = True
        new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        heads = np.flatnonzero(new)
        v = np.add.reduceat(v, heads)
        r, c = r[heads], c[heads]
    if drop_zero:
        keep = v != 0
        r, c, v = r[keep], c[keep], v[keep]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=indptr[1:])
    return indptr, c.astype(np.int64), v.astype(np.float64)


def directed_csr(edges, n, weights=None):
    """``from_edges``: directed A with duplicates summed (graph.py:135-145)."""
    src, dst, w = coerce_edges(edges, weights)
    if src.size and (min(src.min(), dst.min()) < 0 or max(src.max(), dst.max()) >= n):
        raise OracleDomainError("edge endpoint out of range")
    keep = src != dst
    return _segment_csr(src[keep], dst[keep], w[keep], n)


def symmetrize_csr(indptr, indices, data, n):
    """W = A + A' from a canonical directed CSR (graph.py:220-236)."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    allr = np.concatenate([rows, indices])
    allc = np.concatenate([indices, rows])
    allv = np.concatenate([data, data])
    return _segment_csr(allr, allc, allv, n, drop_zero=True)


def directed_degrees(indptr, indices, data, n, symmetric=False):
    """``degrees``: bincount(rows, w) [+ bincount(cols, w)] (graph.py:239-250)."""
    rows = np.repeat(np.arange(n), np.diff(indptr))
    d = np.bincount(rows, weights=data, minlength=n)
    if not symmetric:
        d = d + np.bincount(indices, weights=data, minlength=n)
    return d


def laplacian_apply(indptr, indices, data, n, d, x, symmetric=False):
    """Y = d*X - A X (- A' X) (graph.py:253-278)."""
    a = sp.csr_matrix((data, indices, indptr), shape=(n, n))
    y = d[:, None] * x
    y -= a @ x
    if not symmetric:
        y -= a.T @ x
    return y


class LaplacianRef:
    """Operator protocol n / scale_hint / apply (graph.py:300-317)."""

    def __init__(self, indptr, indices, data, n, symmetric=False):
        self.n = int(n)
        self._a = sp.csr_matrix((data, indices, indptr), shape=(n, n))
        self._sym = bool(symmetric)
        self.degrees = directed_degrees(indptr, indices, data, n, symmetric)
        self.scale_hint = float(self.degrees.max()) if self.n else 1.0

    def apply(self, x, out=None):
        y = self.degrees[:, None] * x if x.ndim == 2 else self.degrees * x
        y = y - self._a @ x
        if not self._sym:  # transpose product formed per call, as graph.py:277
            y = y - self._a.T @ x
        if out is not None:
            out[...] = y
            return out
        return y
