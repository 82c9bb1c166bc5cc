"""Per-phase cycle breakdown of the warp-per-column tridiagonalisation (SPB_TRI_TRACE).

    python tools/tri_trace_wc.py [--m 147]
Stamps (warp of the last column, lane 0): 0 step top -> 1 row k arrived ->
2 reflector + p_i pushed -> 3 p_k arrived -> 4 update + row k+1 pushed -> 5 K term.
"""
import argparse
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=147)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
tf = tempfile.mktemp(suffix=".trace")
os.environ["SPB_TRI_TRACE"] = tf
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_07481_b200.lobpcg import _solve_small  # noqa: E402

rng = np.random.default_rng(0)
x = rng.standard_normal((a.m, a.m))
ga = x + x.T
for _ in range(a.reps):
    _solve_small(ga, None)
lines = Path(tf).read_text().split("\n")
blocks, cur = [], None
for ln in lines:
    if ln.startswith("m "):
        print(ln)
        cur = []
        blocks.append(cur)
    elif ln.strip():
        cur.append([int(v) for v in ln.split()])
t = np.array(blocks[-1], dtype=np.float64)
t = t[:, [0, 1, 5, 6, 2, 3, 4]]
names = ["wait row k", "loads+fma+reduce", "sqrt/div", "p push", "wait p_k", "update+row push"]
d = np.diff(t, axis=1)
nxt = t[1:, 0] - t[:-1, 6]
tot = t[-1, 6] - t[0, 0]
print(f"m={a.m} steps={len(t)} total cycles {tot:.0f} ({tot / len(t):.0f}/step)")
for i in range(6):
    print(f"  {names[i]:14s} mean {d[:, i].mean():7.1f}  first {d[:8, i].mean():7.1f}  last {d[-8:, i].mean():7.1f}")
print(f"  {'loop':14s} mean {nxt.mean():7.1f}")
