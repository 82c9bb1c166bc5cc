"""Partition quality scores — restatement of ``specpart/metrics.py`` (TEST INFRASTRUCTURE ONLY).

contingency (metrics.py:65-75), PM via an exact assignment (metrics.py:78-93),
PR / PP from integer pair counts (metrics.py:96-122).
"""

from __future__ import annotations

import numpy as np
from scipy.optimize import linear_sum_assignment


def _compact(lab):
    _, c = np.unique(np.asarray(lab), return_inverse=True)
    return c.astype(np.int64)


def contingency_counts(truth, found):
    t, f = _compact(truth), _compact(found)
    kt, kf = int(t.max()) + 1, int(f.max()) + 1
    return np.bincount(t * kf + f, minlength=kt * kf).reshape(kt, kf)


def _c2(v):
    v = v.astype(np.int64)
    return int((v * (v - 1) // 2).sum())


def partition_match(truth, found):
    c = contingency_counts(truth, found)
    side = max(c.shape)
    pad = np.zeros((side, side), dtype=np.int64)
    pad[: c.shape[0], : c.shape[1]] = c
    r, k = linear_sum_assignment(pad, maximize=True)
    return int(pad[r, k].sum()) / int(c.sum())


def pairwise_recall(truth, found):
    c = contingency_counts(truth, found)
    return _c2(c.ravel()) / _c2(c.sum(axis=1))


def pairwise_precision(truth, found):
    c = contingency_counts(truth, found)
    return _c2(c.ravel()) / _c2(c.sum(axis=0))
