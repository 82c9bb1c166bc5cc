"""Time the solver's SpMM (R block, ld = 3 lp) in the locality order on a config's graph.

    python tools/bench_spmm_order.py [--lib variant.so] [--config c3] [--reps 20]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
ap = argparse.ArgumentParser()
ap.add_argument("--lib", default="")
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
from paper_1708_07481_b200 import _native as N  # noqa: E402

if a.lib:
    N.LIB_PATH = Path(a.lib)
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402

spec = CONFIGS[a.config]
edges, _ = generate_dcsbm(spec)
g = spb.from_edges(edges, spec.n)
n, l = spec.n, spb.block_size_for(spec.blocks)
lp = (l + 7) // 8 * 8
ld = 3 * lp
op = spb.LaplacianOperator(g, vertex_order=True)
h = op.native("float32", l)
x = torch.randn((n, ld), device="cuda")
y = torch.empty_like(x)
L = N.lib()


def run():
    N.check(L.spb_laplacian_spmm(N.F32, 0, n, h.row_ptr, h.col, h.val, h.deg, N.ptr(x[:, lp:]), ld, l,
                                 N.ptr(y[:, lp:]), ld, N.stream()))


for _ in range(3):
    run()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(a.reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{a.lib or 'tree'} {a.config}: {np.median(ts) * 1e3:.1f} us")
