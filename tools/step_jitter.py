"""Per-step diagnostics of the C3 device step: CUDA-event ms, host wall ms, caching-
allocator growth (reserved bytes, cudaMalloc count) -- for hunting sporadic slow steps.

    python tools/step_jitter.py [steps] [gc: 0|1]
"""
import gc
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402
from paper_1708_07481_b200.spectral import partition_device  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
use_gc = len(sys.argv) > 2 and sys.argv[2] == "1"
spec = CONFIGS["c3"]
edges, _ = generate_dcsbm(spec)
k = spec.blocks
l = spb.block_size_for(k)
dev = torch.device("cuda", 0)
src = torch.from_numpy(np.ascontiguousarray(edges[:, 0])).to(dev)
dst = torch.from_numpy(np.ascontiguousarray(edges[:, 1])).to(dev)
x0 = torch.from_numpy(np.random.default_rng(0).standard_normal((spec.n, l))).to(dev)
cfg = spb.SolverConfig(block_size=l, tol=bench.golden_tol("c3"), max_iter=30, seed=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
if not use_gc:
    gc.collect()
    gc.disable()
keep = None
for i in range(steps):
    flush.zero_()
    torch.cuda.synchronize()
    s0 = torch.cuda.memory_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    g = spb.from_edges((src, dst), spec.n)
    t1 = time.perf_counter()
    keep = partition_device(g, cfg, k, fix_k=True, x0=x0, precision="float32")
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s1 = torch.cuda.memory_stats()
    print(f"step {i:2d}: {e0.elapsed_time(e1):8.2f} ms  host from_edges {1e3 * (t1 - t0):6.2f}  "
          f"partition {1e3 * (t2 - t1):7.2f}  reserved {s1['reserved_bytes.all.current'] / 2**30:6.2f} GiB  "
          f"cudaMalloc +{s1['num_device_alloc'] - s0['num_device_alloc']}  "
          f"cudaFree +{s1['num_device_free'] - s0['num_device_free']}  "
          f"alloc_retries +{s1['num_alloc_retries'] - s0['num_alloc_retries']}", flush=True)
