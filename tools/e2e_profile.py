"""cProfile of the public-API end-to-end call (host arcs + x0 -> host labels).

    python tools/e2e_profile.py [--config c2]
"""
import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--precision", default="float32")
a = ap.parse_args()
spec = CONFIGS[a.config]
edges, _ = generate_dcsbm(spec)
k = spec.blocks
l = spb.block_size_for(k)
x0 = np.random.default_rng(0).standard_normal((spec.n, l))
edges_pinned = np.ascontiguousarray(edges)  # pageable, as bench.py's e2e
tol = 1e-12
if a.config in ("c3", "c4"):
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench

    tol = bench.golden_tol(a.config) or 1e-12
    a.iters = 30
cfg = spb.SolverConfig(block_size=l, tol=tol, max_iter=a.iters, seed=0)


def step():
    g = spb.from_edges(edges_pinned, spec.n)
    part, st, gap = spb.partition_static(g, cfg, k, fix_k=True, x0=x0, precision=a.precision)
    torch.cuda.synchronize()
    return part


step()
t0 = time.perf_counter()
step()
print(f"e2e wall {1e3 * (time.perf_counter() - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)

# per-phase wall times (synchronised): host arcs -> graph, x0 staging, solve, assignment
from paper_1708_07481_b200.graph import LaplacianOperator  # noqa: E402
from paper_1708_07481_b200.lobpcg import _x0_device  # noqa: E402

for rep in range(10):
    ts = []
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = spb.from_edges(edges_pinned, spec.n)
    torch.cuda.synchronize()
    ts.append(("from_edges", time.perf_counter() - t))
    t = time.perf_counter()
    xd = _x0_device(x0, spec.n, l)
    torch.cuda.synchronize()
    ts.append(("x0_stage", time.perf_counter() - t))
    t = time.perf_counter()
    xd = torch.from_numpy(x0).to("cuda")
    torch.cuda.synchronize()
    ts.append(("x0_pageable", time.perf_counter() - t))
    t = time.perf_counter()
    part, st, gap = spb.partition_static(g, cfg, k, fix_k=True, x0=x0, precision=a.precision)
    torch.cuda.synchronize()
    ts.append(("partition_static(host x0)", time.perf_counter() - t))
    print("  ".join(f"{nm} {1e3 * v:.1f} ms" for nm, v in ts))
