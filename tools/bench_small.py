"""Per-kernel device time of the projected eigensolve (spb_sygv) at given sizes.

    python tools/bench_small.py --m 147 [--gb] [--reps 10] [--nev 49]
"""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_07481_b200.lobpcg import _solve_small  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, nargs="+", default=[147])
ap.add_argument("--nev", type=int, default=0)
ap.add_argument("--gb", action="store_true", help="generalized problem (Cholesky of G_B)")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--lib", default="")
a = ap.parse_args()
if a.lib:
    from paper_1708_07481_b200 import _native as N
    N.LIB_PATH = Path(a.lib)
for m in a.m:
    rng = np.random.default_rng(0)
    x = rng.standard_normal((m, m))
    ga = x + x.T
    gb = None
    if a.gb:
        y = rng.standard_normal((4 * m, m))
        gb = y.T @ y / (4 * m)
    nev = a.nev or m // 3
    _solve_small(ga, gb, nev)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            _solve_small(ga, gb, nev)
        torch.cuda.synchronize()
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA and "spb" in ev.name:
            nm = ev.name.replace("void ", "").replace("spb::", "").replace("(anonymous namespace)::", "")
            nm = nm.split("(")[0]
            tot[nm] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
            cnt[nm] += 1
    print(f"m={m} nev={nev} gb={a.gb}: " + ", ".join(
        f"{k} {tot[k] / a.reps:.1f}us" for k in sorted(tot, key=lambda k: -tot[k])))
