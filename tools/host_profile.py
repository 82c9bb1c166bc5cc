"""cProfile of the host side of one partition step (where the GPU waits on Python).

    python tools/host_profile.py [--config c3] [--iters 10]
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
from paper_1708_07481_b200.spectral import partition_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--tol", type=float, default=1e-12)
a = ap.parse_args()
spec = CONFIGS[a.config]
edges, _ = generate_dcsbm(spec)
k = spec.blocks
l = spb.block_size_for(k)
x0 = np.random.default_rng(0).standard_normal((spec.n, l))
dev = torch.device("cuda", 0)
src = torch.from_numpy(np.ascontiguousarray(edges[:, 0])).to(dev)
dst = torch.from_numpy(np.ascontiguousarray(edges[:, 1])).to(dev)
x0_d = torch.from_numpy(x0).to(dev)
cfg = spb.SolverConfig(block_size=l, tol=a.tol, max_iter=a.iters, seed=0)


def step():
    g = spb.from_edges((src, dst), spec.n)
    out = partition_device(g, cfg, k, fix_k=True, x0=x0_d)
    torch.cuda.synchronize()
    return out


step()
t0 = time.perf_counter()
step()
print(f"wall {1e3 * (time.perf_counter() - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# per-phase wall times (synchronised) over a few steps
from paper_1708_07481_b200.graph import LaplacianOperator  # noqa: E402

for rep in range(6):
    ts = []
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = spb.from_edges((src, dst), spec.n)
    torch.cuda.synchronize()
    ts.append(("from_edges", time.perf_counter() - t))
    t = time.perf_counter()
    op = LaplacianOperator(g)
    torch.cuda.synchronize()
    ts.append(("operator", time.perf_counter() - t))
    t = time.perf_counter()
    st = spb.lobpcg_solve(op, x0_d, cfg, n_converge=min(k + 1, l))
    torch.cuda.synchronize()
    ts.append(("solve", time.perf_counter() - t))
    print("  ".join(f"{nm} {1e3 * v:.1f} ms" for nm, v in ts), "iters", st.iterations)
