"""Time one k-means Lloyd assignment pass at C3/C4 shapes: the tcgen05 distance GEMM
with the fused argmin (float32) against the thread-per-row kernel (float64 input).

    python tools/bench_kmeans.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.spectral import _kmeans_device  # noqa: E402

for n, k in [(500_000, 98), (2_000_000, 160), (50_000, 44)]:
    rng = np.random.default_rng(0)
    x = torch.randn((n, k), device="cuda", dtype=torch.float32)
    seeds = torch.as_tensor(np.sort(rng.choice(n, k, replace=False)), dtype=torch.int32, device="cuda")
    for dt in (torch.float32, torch.float64):
        xx = x.to(dt)
        _kmeans_device(xx, k, seeds, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            _kmeans_device(xx, k, seeds, 1)  # one Lloyd step: init + assign (+ update)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = n * k * xx.element_size() / (ms * 1e-3) / 1e9
        print(f"n={n} k={k} {str(dt):14s}: {ms:.3f} ms per Lloyd step ({gbs:.0f} GB/s of X)")
