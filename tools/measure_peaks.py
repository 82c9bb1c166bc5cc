#!/usr/bin/env python
"""Measure the tensor-pipe peaks the Gram rooflines are quoted against.

Same method as MEASURED_PEAKS.json's bf16 entry (torch.matmul 8192^3, best of 10,
CUDA events), for the pipes this repo's Grams use: FP64 (DMMA), TF32 (3xTF32
tcgen05 kind::tf32) and INT8 (Ozaki tcgen05 kind::i8, torch._int_mm). Writes
profiles/r02/peaks_tensor.json. Run on the B200 box:

    python tools/measure_peaks.py
"""

from __future__ import annotations

import json
import time
from pathlib import Path

import torch

OUT = Path(__file__).resolve().parent.parent / "profiles" / "r02" / "peaks_tensor.json"


def best_of(fn, flops, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return flops / (best * 1e-3) / 1e12, best


def main():
    torch.cuda.set_device(0)
    n = 8192
    res = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "torch matmul n=8192 (2 n^3 ops), best of 10 after 3 warm-up, CUDA events"}
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    res["fp64_tflops"], res["fp64_ms"] = best_of(lambda: a @ b, 2.0 * n**3)
    del a, b
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, dtype=torch.float32, device="cuda")
    b = torch.randn(n, n, dtype=torch.float32, device="cuda")
    res["tf32_tflops"], res["tf32_ms"] = best_of(lambda: a @ b, 2.0 * n**3)
    torch.backends.cuda.matmul.allow_tf32 = False
    res["fp32_simt_tflops"], res["fp32_simt_ms"] = best_of(lambda: a @ b, 2.0 * n**3)
    del a, b
    ai = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
    bi = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    try:
        res["int8_tops"], res["int8_ms"] = best_of(lambda: torch._int_mm(ai, bi), 2.0 * n**3)
    except RuntimeError as e:  # no int8 GEMM in this build
        res["int8_tops"], res["int8_error"] = None, str(e)[:200]
    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
