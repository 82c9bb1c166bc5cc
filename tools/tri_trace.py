"""Per-phase cycle breakdown of the cluster tridiagonalisation (SPB_TRI_TRACE).

    python tools/tri_trace.py [--m 147]
Phases (CTA 0, thread 0): 0 top sync -> 1 matvec -> 2 sync -> 3 p/dot pushed
-> 4 exchange waited -> 5 own update -> 6 next reflector -> next step.
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
        cur = []
        blocks.append(cur)
    elif ln.strip():
        cur.append([int(v) for v in ln.split()])
t = np.array(blocks[-1], dtype=np.float64)
names = ["matvec", "sync2", "p+dot push", "exchange wait", "own update", "reflect(k+1)", "top sync"]
d = np.diff(t, axis=1)
nxt = t[1:, 0] - t[:-1, 6]
print(f"m={a.m} steps={len(t)} total cycles {t[-1, 6] - t[0, 0]:.0f} ({(t[-1, 6] - t[0, 0]) / len(t):.0f}/step)")
for i in range(6):
    print(f"  {names[i]:14s} mean {d[:, i].mean():7.1f}  first {d[:8, i].mean():7.1f}  last {d[-8:, i].mean():7.1f}")
print(f"  {names[6]:14s} mean {nxt.mean():7.1f}  first {nxt[:8].mean():7.1f}  last {nxt[-8:].mean():7.1f}")
if t.shape[1] > 7:
    ok = (t[:, 7] >= t[:, 2]) & (t[:, 7] <= t[:, 3])
    s1, s2 = t[ok, 7] - t[ok, 2], t[ok, 3] - t[ok, 7]
    print(f"  (p+dot push = group sum {s1.mean():.1f} + pushes/warp_sum/bar {s2.mean():.1f})")
