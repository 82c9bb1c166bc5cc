"""A/B: whole-partition device time of a config with a given libspb200.so build.

    python tools/ab_step.py [--lib path/to/libspb200.so] [--config c3] [--steps 8]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
ap = argparse.ArgumentParser()
ap.add_argument("--lib", default="")
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=8)
a = ap.parse_args()
from paper_1708_07481_b200 import _native as N  # noqa: E402

if a.lib:
    N.LIB_PATH = Path(a.lib)
import bench  # noqa: E402
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402
from paper_1708_07481_b200.spectral import partition_device  # noqa: E402

spec = CONFIGS[a.config]
edges, _ = generate_dcsbm(spec)
k = spec.blocks
l = spb.block_size_for(k)
x0 = torch.from_numpy(np.random.default_rng(0).standard_normal((spec.n, l))).cuda()
src = torch.from_numpy(np.ascontiguousarray(edges[:, 0])).cuda()
dst = torch.from_numpy(np.ascontiguousarray(edges[:, 1])).cuda()
tol, mi = (bench.golden_tol(a.config) or 1e-12, 30) if a.config in ("c3", "c4") else (1e-12, 20)
cfg = spb.SolverConfig(block_size=l, tol=tol, max_iter=mi, seed=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts, its = [], []
for s in range(a.steps + 2):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g = spb.from_edges((src, dst), spec.n)
    _, _, st, _ = partition_device(g, cfg, k, fix_k=True, x0=x0, precision="float32")
    e1.record()
    torch.cuda.synchronize()
    if s >= 2:
        ts.append(e0.elapsed_time(e1))
        its.append(st.iterations)
print(f"{a.lib or 'tree'} {a.config}: median {np.median(ts):.2f} ms min {min(ts):.2f} iterations {set(its)}")
