"""Per-kernel device time of one partition step (torch.profiler / CUPTI).

    python tools/profile_step.py [--config c2] [--precision float32]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402
from paper_1708_07481_b200.spectral import partition_device  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--precision", default="float32")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--tol", type=float, default=1e-12)
a = ap.parse_args()
spec = CONFIGS[a.config]
edges, truth = generate_dcsbm(spec)
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
    return partition_device(g, cfg, k, fix_k=True, x0=x0_d, precision=a.precision)


for _ in range(2):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
step()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
print(f"wall per step {wall*1e3:.1f} ms")
agg = {}
for ev in prof.events():
    if ev.device_type is not None and str(ev.device_type).endswith("CUDA"):
        name = ev.name.replace("(anonymous namespace)::", "").split("(")[0][-90:]
        d = agg.setdefault(name, [0, 0.0])
        d[0] += 1
        d[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"sum of kernel time {tot/1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{t/1e3:9.3f} ms  {c:5d}  {name}")
