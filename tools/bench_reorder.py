"""Experiment: SpMM time under vertex orderings (natural / planted truth / smoothed-LSH).

    python tools/bench_reorder.py [--config c3] [--steps 3] [--bits 16]

Timing tool only (torch builds the permuted CSR); the product ordering is in csrc.
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
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--bits", type=int, default=16)
a = ap.parse_args()
spec = CONFIGS[a.config]
edges, truth = generate_dcsbm(spec)
g = spb.from_edges(edges, spec.n)
n = spec.n
l = spb.block_size_for(spec.blocks)
lp = ((l + 7) // 8) * 8
ld = 3 * lp
rp, col, _, nnz = g.device_csr()
nnz = int(nnz)
rp = rp[: n + 1].long()
col = col[:nnz].long()
vals = g._w_csr.values("float32")[:nnz].contiguous()
deg = g.device_degrees().float().contiguous()
L = N.lib()
dev = torch.device("cuda")


def permuted(perm):
    """CSR of P W P^T with new row i = old row perm[i]; per-row entry order kept."""
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(n, device=dev)
    cnt = (rp[1:] - rp[:-1])[perm]
    nrp = torch.zeros(n + 1, dtype=torch.long, device=dev)
    nrp[1:] = torch.cumsum(cnt, 0)
    row_of = torch.repeat_interleave(torch.arange(n, device=dev), cnt)
    pos = torch.arange(nnz, device=dev) - nrp[row_of]
    src = rp[perm][row_of] + pos
    return (nrp.int().contiguous(), inv[col[src]].int().contiguous(), vals[src].contiguous(),
            deg[perm].contiguous())


flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def time_spmm(rpi, ci, cv, dg, tag):
    x = torch.randn((n, ld), device=dev, dtype=torch.float32)
    y = torch.empty_like(x)

    def run():
        N.check(L.spb_laplacian_spmm(N.F32, 0, n, N.ptr(rpi), N.ptr(ci), N.ptr(cv), N.ptr(dg),
                                     N.ptr(x), ld, l, N.ptr(y), ld, N.stream()))
    for _ in range(3):
        run()
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
    print(f"{tag:>28s}: {ms * 1e3:8.1f} us  gather {4.0 * nnz * l / ms / 1e6:6.0f} GB/s", flush=True)
    return ms


def locality(perm, tag):
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(n, device=dev)
    row_of = torch.repeat_interleave(torch.arange(n, device=dev), rp[1:] - rp[:-1])
    d = (inv[row_of] - inv[col]).abs().float()
    print(f"{tag:>28s}: median |i-j| {d.median().item():9.0f}  frac<8192 {(d < 8192).float().mean().item():.3f}")


ident = torch.arange(n, device=dev)
time_spmm(rp.int(), col.int(), vals, deg, "natural")
locality(ident, "natural")
tz = torch.as_tensor(truth, device=dev)
pt = torch.sort(tz * n + ident).indices
time_spmm(*permuted(pt), "planted truth (upper bound)")
locality(pt, "planted truth")

# the product ordering (csrc/reorder.cu) at several walk lengths, timed
from paper_1708_07481_b200 import graph as G  # noqa: E402

for steps in (2, 3, 4, 5, 6, 8):
    G.ORDER_STEPS = steps
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        o = G._VertexOrder(g._w_csr, n)
        rpo, co, vo = o.csr(g._w_csr, "float32")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    perm = o.perm.long()
    dg = o.gather(deg)
    tag = f"product steps={steps}"
    print(f"{tag:>28s}: order + permute {np.median(ts) * 1e3:8.1f} us", flush=True)
    locality(perm, tag)
    if truth is not None:
        tp = torch.as_tensor(truth, device=dev)[perm]
        print(f"{tag:>28s}: same block as next {(tp[1:] == tp[:-1]).float().mean().item():.3f}")
    time_spmm(rpo, co, vo, dg, tag)
