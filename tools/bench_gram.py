"""Time spb_gram (C-ABI) on solver-shaped blocks; prints ms and TFLOP/s per shape.

    python tools/bench_gram.py [--mode 0] [--reps 10] [--dtype float32]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_07481_b200 import _native as N  # noqa: E402
import os  # noqa: E402

if os.environ.get("SPB_LIBV"):  # experiment builds (tools/build_variant.py)
    N.LIB_PATH = Path(os.environ["SPB_LIBV"])

ap = argparse.ArgumentParser()
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--dtype", default="float32")
ap.add_argument("--profile", action="store_true")
ap.add_argument("--shapes", default="500000x108x108,500000x324x324,50000x147x147,50000x49x49,2000000x176x176")
a = ap.parse_args()
tdt = torch.float32 if a.dtype == "float32" else torch.float64
code = N.F32 if a.dtype == "float32" else N.F64
L = N.lib()
for sh in a.shapes.split(","):
    n, p, q = map(int, sh.split("x"))
    ld = ((max(p, q) + 7) // 8) * 8
    u = torch.randn((n, ld), dtype=tdt, device="cuda")
    v = torch.randn((n, ld), dtype=tdt, device="cuda")
    out = torch.empty((p, q), dtype=torch.float64, device="cuda")
    wsb = L.spb_gram_workspace(p, q, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")

    def run():
        N.check(L.spb_gram(code, a.mode, N.ptr(u), ld, p, N.ptr(v), ld, q, n, N.ptr(out), q,
                           N.ptr(ws), wsb, N.stream()))

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
    ref = (u[:, :p].double().T @ v[:, :q].double())
    err = ((out - ref).abs().max() / (u[:, :p].abs().double().T @ v[:, :q].abs().double()).max()).item()
    print(f"{sh:>20s}  {ms:8.3f} ms  {2.0*n*p*q/ms/1e9:7.2f} TFLOP/s  relerr {err:.2e}", flush=True)
    if a.profile:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            run()
            torch.cuda.synchronize()
        for ev in prof.key_averages():
            if ev.device_time_total > 0:
                print(f"      {ev.key[:70]:70s} {ev.device_time_total:9.1f} us  x{ev.count}")
