"""Host staging of the C3 x0 block (float64 -> float32 while copying to pinned chunks):
thread-count sweep, and numpy's conversion rate per thread.

    python tools/stage_bench.py
"""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_07481_b200 import _h2d  # noqa: E402

x = np.random.default_rng(0).standard_normal((500_000, 108))
dev = torch.device("cuda", 0)
print("cpus", os.cpu_count())
dst = np.empty(x.shape, dtype=np.float32)
for _ in range(2):
    t = time.perf_counter()
    np.copyto(dst, x, casting="unsafe")
    dt = time.perf_counter() - t
print(f"numpy copyto f64->f32, 1 thread: {1e3 * dt:.1f} ms ({x.nbytes / dt / 1e9:.1f} GB/s read)")
for threads in (2, 4, 6, 8, 12, 16):
    _h2d._THREADS = threads
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        y = _h2d.to_device(x, dev, np.float32)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    ok = bool(torch.equal(y.cpu(), torch.from_numpy(x.astype(np.float32))))
    print(f"threads {threads:2d}: {1e3 * min(ts):6.2f} ms min, {1e3 * np.median(ts):6.2f} median, bit-identical {ok}")
e = np.random.default_rng(1).integers(0, 500_000, size=(10_000_000, 2))
for threads in (4, 8, 16):
    _h2d._THREADS = threads
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        y = _h2d.to_device(e, dev)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"arcs int64 {e.nbytes >> 20} MiB threads {threads:2d}: {1e3 * min(ts):6.2f} ms min, "
          f"{1e3 * np.median(ts):6.2f} median, identical {bool(torch.equal(y.cpu(), torch.from_numpy(e)))}")
