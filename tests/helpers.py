"""Shared helpers for the test-suite (hashing, config inputs)."""

from __future__ import annotations

import hashlib

import numpy as np

from paper_1708_07481_b200.dcsbm import CONFIGS, DcsbmSpec, generate_dcsbm


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


# l = 108 > one Ozaki column tile at a size the one-GPU multi-rank tests can run: with
# SPB_GRAM=oz the solve takes the int8 Rayleigh-Ritz Grams and the fused projection +
# CholQR step (lobpcg.cu project_orth) that C3 / C4 take by default.
OZ108 = DcsbmSpec(n=40000, blocks=98, arcs=1_000_000, alpha=3.0, ratio=5.0, seed=4)


def config_input(name, seed=None):
    spec = OZ108 if name == "oz108" else CONFIGS[name]
    if seed is not None:
        spec = spec.__class__(**{**spec.__dict__, "seed": seed})
    edges, truth = generate_dcsbm(spec)
    return spec, edges, truth


def solve_cases():
    """Inputs of tests/golden/make_golden.py::solve_fixture (same seeds)."""
    cases = {
        "path3": ([(0, 1), (1, 2)], 3, 3, dict(tol=1e-10, max_iter=500, seed=0), 0),
        "k4": ([(i, j) for i in range(4) for j in range(i + 1, 4)], 4, 4,
               dict(tol=1e-10, max_iter=500, seed=1), 1),
        "two_tri": ([(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)], 6, 3,
                    dict(tol=1e-10, max_iter=500, seed=0), 0),
    }
    rng = np.random.default_rng(7)
    ends = rng.integers(0, 150, size=(600, 2))
    w = rng.random(600) * 2.0
    cases["rand150"] = (np.column_stack([ends, w[:, None]]), 150, 8,
                        dict(tol=1e-10, max_iter=500, seed=1), 1)
    rng = np.random.default_rng(5)
    ends = rng.integers(0, 300, size=(1500, 2))
    w = rng.random(1500) * 2.0
    cases["rand300_20it"] = (np.column_stack([ends, w[:, None]]), 300, 8,
                             dict(tol=1e-14, max_iter=20, seed=4), 4)
    return cases
