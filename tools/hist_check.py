"""Residual-history deviation of the rand300_20it golden case (debug helper)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1708_07481_b200 as spb  # noqa: E402
from tests.conftest import load_golden  # noqa: E402
from tests.helpers import solve_cases  # noqa: E402

gs = load_golden("solve")
edges, n, l, kw, xseed = solve_cases()["rand300_20it"]
op = spb.LaplacianOperator(spb.from_edges(edges, n))
for prec in ("float32", "float64"):
    hr = []
    spb.lobpcg_solve(op, spb.random_init(n, l, xseed), spb.SolverConfig(block_size=l, **kw),
                     callback=lambda it, t, r: hr.append(r), precision=prec)
    a, b = np.array(hr), gs["rand300_20it/hist_norms"]
    eps = 1e-16 if prec == "float64" else 6e-8
    floor = 1e3 * eps * op.scale_hint
    big = b > floor
    dev = np.abs(np.log10(a[big] / b[big]))
    i = np.argmax(dev)
    print(prec, "scale", op.scale_hint, "floor", floor, "max dev", dev.max(), "at ref", b[big][i], "ours", a[big][i])
