"""Time the Laplacian SpMM (C-ABI) on a DC-SBM config's graph.

    python tools/bench_spmm.py [--config c2] [--reps 20]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200 import _native as N  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--cols", type=int, default=0)
ap.add_argument("--ld", type=int, default=0, help="row stride of X/Y (solver: 3 * padded l)")
a = ap.parse_args()
spec = CONFIGS[a.config]
edges, _ = generate_dcsbm(spec)
g = spb.from_edges(edges, spec.n)
l = a.cols or spb.block_size_for(spec.blocks)
ld = a.ld or ((l + 7) // 8) * 8
n = spec.n
row_ptr, col, _, nnz = g.device_csr()
vals = g._w_csr.values("float32")
deg = g.device_degrees().float().contiguous()
x = torch.randn((n, ld), device="cuda", dtype=torch.float32)
y = torch.empty_like(x)
L = N.lib()


def run():
    N.check(L.spb_laplacian_spmm(N.F32, 0, n, N.ptr(row_ptr), N.ptr(col), N.ptr(vals), N.ptr(deg),
                                 N.ptr(x), ld, l, N.ptr(y), ld, N.stream()))


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
ms = float(np.median(ts))
ref = deg[:, None] * x[:, :l] - torch.sparse_csr_tensor(row_ptr.long(), col[:nnz].long(), vals[:nnz],
                                                         size=(n, n)).matmul(x[:, :l])
err = ((y[:, :l] - ref).abs().max() / ref.abs().max()).item()
gath = 4.0 * int(nnz) * l
print(f"{a.config} n={n} nnz={int(nnz)} cols={l}: {ms * 1e3:.1f} us  gather {gath / ms / 1e6:.0f} GB/s  relerr {err:.1e}")
