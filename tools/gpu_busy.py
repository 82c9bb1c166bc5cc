"""Kernel-busy fraction of one partition step: sum of CUPTI kernel durations over the
CUDA-event time of the step (the rest is launch latency and host synchronisations).

    python tools/gpu_busy.py [c2|c3]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.spectral import partition_device  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
spec, edges, truth, k, l, x0, max_iter = bench.workload(cfg_name)
dev = torch.device("cuda", 0)
src = torch.from_numpy(np.ascontiguousarray(edges[:, 0])).to(dev)
dst = torch.from_numpy(np.ascontiguousarray(edges[:, 1])).to(dev)
x0_d = torch.from_numpy(x0).to(dev)
tol = bench.golden_tol(cfg_name) or 1e-12
cfg = spb.SolverConfig(block_size=l, tol=tol, max_iter=max_iter, seed=0)


def step():
    g = spb.from_edges((src, dst), spec.n)
    return partition_device(g, cfg, k, fix_k=True, x0=x0_d, precision="float32")


for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
busy = 0.0
n = 0
for ev in prof.events():
    if ev.device_type is not None and str(ev.device_type).endswith("CUDA"):
        t = getattr(ev, "device_time_total", None) or ev.cuda_time_total
        busy += t
        n += 1
ms = e0.elapsed_time(e1)
print(f"{cfg_name}: step {ms:.2f} ms (under the profiler), kernels {n}, busy {busy / 1e3:.2f} ms "
      f"({100 * busy / 1e3 / ms:.0f} %)")
