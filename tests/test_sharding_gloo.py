"""Host logic of the row-sharded solve, on CPU with torch.distributed/gloo (world 2).

The GPU path (paper_1708_07481_b200/sharded.py + csrc/lobpcg.cu) places the
collectives as follows: all-gather of the SpMM input block (gathered layout
rank * n_max + local row), float64 all-reduce of every Gram partial and of the
column sums, small problems solved redundantly. This test runs the same
decomposition in numpy on two gloo ranks and checks it reproduces the
single-process oracle, plus the row partition and the column remap.
"""

import os
import socket

import numpy as np
import pytest
import scipy.linalg
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1708_07481_b200.dcsbm import DcsbmSpec, generate_dcsbm
from paper_1708_07481_b200.sharded import partition_rows


def _graph():
    spec = DcsbmSpec(n=600, blocks=4, arcs=8000, alpha=3.0, ratio=6.0, seed=5)
    edges, _ = generate_dcsbm(spec)
    ip, ix, dv = oracle.directed_csr(edges, spec.n)
    wp, wx, wv = oracle.symmetrize_csr(ip, ix, dv, spec.n)
    deg = oracle.directed_degrees(ip, ix, dv, spec.n)
    return spec, edges, (ip, ix, dv), (wp, wx, wv), deg


def test_partition_rows_balanced():
    _, _, _, (wp, _, _), _ = _graph()
    for r in (1, 2, 3, 4, 8):
        b = partition_rows(wp, r)
        assert b[0] == 0 and b[-1] == len(wp) - 1 and np.all(np.diff(b) >= 1)
        cost = (wp[b[1:]] - wp[b[:-1]]) + np.diff(b)
        assert cost.max() <= cost.sum() / r * 1.1 + 250


def _shard_csr(wp, wx, wv, bounds, rank, n_max):
    """numpy restatement of spb_csr_shard."""
    r0, r1 = bounds[rank], bounds[rank + 1]
    rp = wp[r0:r1 + 1] - wp[r0]
    cols = wx[wp[r0]:wp[r1]]
    owner = np.searchsorted(bounds, cols, side="right") - 1
    return rp, owner * n_max + (cols - bounds[owner]), wv[wp[r0]:wp[r1]]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, edges, (ip, ix, dv), (wp, wx, wv), deg = _graph()
        n = spec.n
        bounds = partition_rows(wp, world)
        n_max = int(np.diff(bounds).max())
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        lrp, lcol, lval = _shard_csr(wp, wx, wv, bounds, rank, n_max)
        ldeg = deg[r0:r1]

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        def apply(x_local):  # all-gather + local rows of d*X - W X
            pad = np.zeros((n_max, x_local.shape[1]))
            pad[: r1 - r0] = x_local
            out = [torch.empty(n_max, x_local.shape[1], dtype=torch.float64) for _ in range(world)]
            dist.all_gather(out, torch.from_numpy(pad))
            xg = torch.cat(out).numpy()
            y = ldeg[:, None] * xg[rank * n_max + np.arange(r1 - r0)]
            for i in range(r1 - r0):
                s, e = lrp[i], lrp[i + 1]
                y[i] -= lval[s:e] @ xg[lcol[s:e]]
            return y

        def gram(a, b):
            return allreduce(a.T @ b)

        def cholqr(b):
            c = np.linalg.cholesky(0.5 * (gram(b, b) + gram(b, b).T))
            return b @ scipy.linalg.solve_triangular(c.T, np.eye(b.shape[1]), lower=False)

        l, iters = 6, 8
        x0 = np.random.default_rng(3).standard_normal((n, l))
        X = cholqr(x0[r0:r1].copy())
        LX = apply(X)
        th, C = scipy.linalg.eigh(0.5 * (gram(X, LX) + gram(X, LX).T), 0.5 * (gram(X, X) + gram(X, X).T))
        X, LX = X @ C, LX @ C
        P = LP = None
        hist = []
        for it in range(iters + 1):
            R = LX - X * th[None, :l]
            hist.append(np.sqrt(allreduce((R * R).sum(axis=0))))
            if it == iters:
                break
            R = R - X @ gram(X, R)
            R = cholqr(R)
            LR = apply(R)
            if P is not None:
                pn = np.sqrt(allreduce((P * P).sum(axis=0)))
                P, LP = P / pn, LP / pn
            B = np.concatenate([X, R] + ([P] if P is not None else []), axis=1)
            LB = np.concatenate([LX, LR] + ([LP] if LP is not None else []), axis=1)
            ga, gb = gram(B, LB), gram(B, B)
            th, C = scipy.linalg.eigh(0.5 * (ga + ga.T), 0.5 * (gb + gb.T))
            C = C[:, :l]
            P, LP = B[:, l:] @ C[l:], LB[:, l:] @ C[l:]
            X, LX = B @ C, LB @ C
        q.put((rank, np.array(th[:l]), np.array(hist)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_decomposition_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (t, h)) for r, t, h in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    assert res[0][0].tolist() == res[1][0].tolist(), "ranks must agree bitwise (replicated solves)"
    # single-process oracle on the same input (no soft locking is triggered at tol 1e-14)
    spec, edges, (ip, ix, dv), _, _ = _graph()
    op = oracle.LaplacianRef(ip, ix, dv, spec.n)
    hist = []
    st = oracle.lobpcg_ref(op, np.random.default_rng(3).standard_normal((spec.n, 6)),
                           oracle.SolverCfg(block_size=6, tol=1e-14, max_iter=8, seed=0),
                           callback=lambda it, t, r: hist.append(r))
    assert np.allclose(res[0][1], np.array(hist), rtol=1e-7, atol=1e-9)
