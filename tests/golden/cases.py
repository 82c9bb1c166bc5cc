"""Deterministic small inputs shared by make_golden.py and the tests."""

from __future__ import annotations

import numpy as np


def small_graph_cases():
    """name -> (edges, n, weights-or-None); includes duplicates, self-loops, zeros."""
    rng = np.random.default_rng(2024)
    cases = {
        "path3": (np.array([[0, 1], [1, 2]]), 3, None),
        "one_weighted": (np.array([[0.0, 1.0, 2.0]]), 2, None),
        "dups_loops": (np.array([[0, 1, 1.0], [0, 1, 2.5], [1, 1, 9.0]]), 2, None),
        "antiparallel": (np.array([[0, 1, 2.0], [1, 0, 3.0], [1, 2, 4.0]]), 3, None),
        "zero_weight": (np.array([[0, 1, 0.0], [1, 2, 1.0], [2, 1, 0.0]]), 3, None),
        "empty": (np.empty((0, 2), dtype=np.int64), 4, None),
        "isolated": (np.array([[0, 1], [1, 2], [2, 0]]), 6, None),
    }
    e = rng.integers(0, 40, size=(300, 2))
    cases["rand_w40"] = (e, 40, rng.uniform(0.0, 8.0, size=300))
    e = rng.integers(0, 200, size=(2000, 2))
    cases["rand_u200"] = (e, 200, None)
    e = rng.integers(0, 100, size=(800, 2))
    cases["rand_int100"] = (e, 100, rng.integers(0, 5, size=800).astype(np.float64))
    return cases


def _indicator(sizes):
    n = sum(sizes)
    x = np.zeros((n, len(sizes)))
    s = 0
    for j, c in enumerate(sizes):
        x[s : s + c, j] = 1.0 / np.sqrt(c)
        s += c
    return x


def qrcp_cases():
    rng = np.random.default_rng(77)
    q3, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    z = np.zeros((5, 2))
    z[0, 0] = 1.0
    z[1, 1] = 1.0
    g, _ = np.linalg.qr(rng.standard_normal((300, 7)))
    blocks = _indicator([40, 25, 60, 35, 40])
    noisy = blocks + 0.01 * rng.standard_normal(blocks.shape)
    noisy, _ = np.linalg.qr(noisy)
    return {
        "indicator": _indicator([4, 6]),
        "rotated": _indicator([5, 7, 3]) @ q3,
        "zero_rows": z,
        "single": np.full((4, 1), 0.5),
        "gauss300x7": g,
        "noisy_blocks": noisy,
    }
