"""Small deterministic target for ncu: N partition steps of a config (no profiler inside).

    python tools/ncu_target.py [c2|c3|c4] [steps] [float32|float64]
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200 import _native as _N  # noqa: E402

if os.environ.get("SPB_LIBV"):  # experiment builds (tools/build_variant.py)
    _N.LIB_PATH = Path(os.environ["SPB_LIBV"])
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402
from paper_1708_07481_b200.spectral import partition_device  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
precision = sys.argv[3] if len(sys.argv) > 3 else "float32"  # explicit: no tol-based promotion
spec = CONFIGS[cfg_name]
edges, truth = generate_dcsbm(spec)
k = spec.blocks
l = spb.block_size_for(k)
x0 = np.random.default_rng(0).standard_normal((spec.n, l))
dev = torch.device("cuda", 0)
src = torch.from_numpy(np.ascontiguousarray(edges[:, 0])).to(dev)
dst = torch.from_numpy(np.ascontiguousarray(edges[:, 1])).to(dev)
x0_d = torch.from_numpy(x0).to(dev)
tol, max_iter = 1e-12, 20
if cfg_name in ("c3", "c4"):  # the 10x stop rule the reference produced (bench.golden_tol)
    import bench

    tol, max_iter = bench.golden_tol(cfg_name) or 1e-12, 30
cfg = spb.SolverConfig(block_size=l, tol=tol, max_iter=max_iter, seed=0)
for _ in range(steps):
    g = spb.from_edges((src, dst), spec.n)
    partition_device(g, cfg, k, fix_k=True, x0=x0_d, precision=precision)
torch.cuda.synchronize()
print("done")
