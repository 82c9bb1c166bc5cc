"""Time spb_block_update (modes 0 / 1) on solver shapes; GB/s of compulsory traffic.

    python tools/bench_update.py [--reps 20]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_07481_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--shapes", default="50000x147x49,50000x49x49,500000x324x108,500000x108x108,2000000x528x176")
a = ap.parse_args()
L = N.lib()
for sh in a.shapes.split(","):
    n, w, q = map(int, sh.split("x"))
    ld = ((w + 7) // 8) * 8
    ldo = ((q + 7) // 8) * 8
    x = torch.randn((n, ld), device="cuda")
    c = torch.randn((w, q), device="cuda", dtype=torch.float64)
    out = torch.empty((n, ldo), device="cuda")
    wsb = L.spb_block_update_workspace(w, q)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    line = f"{sh:>18s}"
    for mode in (0, 1):
        def run():
            N.check(L.spb_block_update(N.F32, mode, N.ptr(x), ld, w, N.ptr(c), q, q, 1.0, None, 0,
                                       N.ptr(out), ldo, n, N.ptr(ws), wsb, N.stream()))
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        gb = (4.0 * n * w + 4.0 * n * q) / 1e9
        line += f"   mode {mode}: {ms * 1e3:8.1f} us {gb / ms * 1e3:7.0f} GB/s"
    print(line, flush=True)
