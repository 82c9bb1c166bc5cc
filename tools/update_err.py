"""Error of the block update kernels (modes 0 / 1) against float64, by K.

    python tools/update_err.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from tests.test_gpu_update import _run  # noqa: E402

for n, w, q in [(20000, 8, 64), (20000, 32, 64), (20000, 64, 64), (20000, 147, 64), (20000, 324, 64),
                (20000, 1024, 64)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    ld = ((w + 7) // 8) * 8
    a_full = torch.randn((n, ld), device="cuda", generator=g)
    a = a_full[:, :w]
    c = torch.randn((w, q), device="cuda", generator=g, dtype=torch.float64) / np.sqrt(w)
    c32 = c.float().double()
    want = a.double() @ c32
    mag = a.double().abs() @ c32.abs()
    line = f"K={w:5d}"
    for mode in (0, 1):
        got = _run(mode, a_full, c, 1.0, None, ((q + 7) // 8) * 8)
        e = (got.double() - want).abs() / mag
        line += f"   mode {mode}: max {e.max().item():.2e} mean {e.mean().item():.2e}"
    print(line, flush=True)
