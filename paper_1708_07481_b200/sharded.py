"""Row-sharded multi-GPU solves: one process per GPU.

Each rank builds only its own contiguous row range of the symmetrised CSR W
directly from the whole arc list (``spb_csr_build_rows``: bit-identical rows,
columns remapped to the all-gathered layout, no whole-graph CSR anywhere); the
row ranges balance arc endpoints + rows and are computed identically on every
rank from the arc list, so the build needs no collective. The device LOBPCG
driver then runs with

* an all-gather of the operator's input block before every SpMM;
* float64 all-reduces of the Gram partials and column sums (norms, means);
* the small projected problems solved redundantly (identical on every rank).

Transport: NCCL over NVLink (``transport="nccl"``, the production path), or the
host transport (``transport="host"``): the same driver with every collective
staged through host memory and done by torch.distributed on a CPU (gloo) group.
The host transport exists so the multi-rank code path runs -- and is tested --
with several ranks on one GPU (no kernel ever waits on another rank).

The assignment all-gathers the first k eigenvector columns and runs the QRCP
kernel on every rank, so every rank returns the same labels.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _h2d
from . import _native as N
from .errors import ContractError, DomainError, SolverError, SpecpartError
from .graph import DTYPES, SparseGraph, _device, _device_arcs
from .lobpcg import EigenState, SolverConfig, _Bridge, default_precision, random_init
from .spectral import GapResult, Partition, block_size_for, detect_gap

__all__ = ["partition_rows", "arc_row_bounds", "RowShardedLaplacian", "lobpcg_solve_sharded",
           "partition_static_sharded", "partition_edges_sharded"]


def partition_rows(row_ptr: np.ndarray, nranks: int) -> np.ndarray:
    """Contiguous row ranges balanced by (nnz + rows); returns bounds[nranks + 1]."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = row_ptr.size - 1
    if nranks < 1:
        raise DomainError("nranks must be positive")
    cost = row_ptr + np.arange(n + 1)
    targets = cost[-1] * np.arange(1, nranks) / nranks
    inner = np.searchsorted(cost, targets, side="left")
    bounds = np.concatenate([[0], inner, [n]]).astype(np.int64)
    return np.maximum.accumulate(np.clip(bounds, 0, n))


def arc_row_bounds(src: torch.Tensor, dst: torch.Tensor, n: int, nranks: int) -> np.ndarray:
    """Row ranges balanced by (arc endpoints + rows), from the arc list alone.

    Every rank computes the same bounds (integer counts, no collective); an
    endpoint count is the number of W entries of the row before duplicate arcs
    merge, so the balance matches ``partition_rows`` on W up to duplicates.
    """
    if nranks < 1:
        raise DomainError("nranks must be positive")
    keep = src != dst
    cnt = torch.bincount(src[keep], minlength=n) + torch.bincount(dst[keep], minlength=n)
    cost = torch.zeros(n + 1, dtype=torch.int64, device=src.device)
    cost[1:] = torch.cumsum(cnt + 1, 0)
    targets = (cost[-1].double() * torch.arange(1, nranks, device=src.device, dtype=torch.float64)
               / nranks)
    inner = torch.searchsorted(cost.double(), targets, side="left")
    b = torch.cat([torch.zeros(1, dtype=torch.int64, device=src.device), inner,
                   torch.full((1,), n, dtype=torch.int64, device=src.device)]).cpu().numpy()
    return np.maximum.accumulate(np.clip(b, 0, n))


class _Comm:
    """Communicator for the sharded driver.

    ``transport="nccl"``: NCCL communicator from a unique id broadcast over
    torch.distributed. ``transport="host"``: collectives staged through host
    memory on a torch.distributed CPU group (gloo).
    """

    def __init__(self, group=None, transport: str = "nccl"):
        import torch.distributed as dist

        if transport not in ("nccl", "host"):
            raise DomainError(f"unknown transport {transport!r}")
        self.transport = transport
        self.group = group
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        L = N.lib()
        h = C.c_void_p()
        if transport == "host":
            self._cbs = self._host_callbacks(dist)
            N.check(L.spb_comm_init_host(self.nranks, self.rank, self._cbs[0], self._cbs[1], None,
                                         C.byref(h)))
        else:
            uid = (C.c_char * 128)()
            if self.nranks > 1:
                if self.rank == 0:
                    N.check(L.spb_comm_unique_id(uid, 128))
                obj = [bytes(uid) if self.rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                C.memmove(uid, obj[0], 128)
            N.check(L.spb_comm_init(self.nranks, self.rank, uid, C.byref(h)))
        self.handle = h

    def _host_callbacks(self, dist):
        group, nranks = self.group, self.nranks
        self.exc = None

        def allreduce(_u, buf, count):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(buf, (int(count),)))
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                return 0
            except BaseException as e:  # noqa: BLE001
                self.exc = e
                return 1

        def allgather(_u, send, recv, nbytes):
            try:
                nb = int(nbytes)
                snd = torch.frombuffer((C.c_char * nb).from_address(send), dtype=torch.uint8).clone()
                rcv = torch.frombuffer((C.c_char * (nb * nranks)).from_address(recv), dtype=torch.uint8)
                dist.all_gather(list(rcv.chunk(nranks)), snd, group=group)
                return 0
            except BaseException as e:  # noqa: BLE001
                self.exc = e
                return 1

        return N.ALLREDUCE_CB(allreduce), N.ALLGATHER_CB(allgather)

    def allreduce_max(self, value: float) -> float:
        if self.nranks == 1:
            return float(value)
        import torch.distributed as dist

        dev = "cpu" if self.transport == "host" else _device()
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def all_gather_rows(self, pad: torch.Tensor) -> torch.Tensor:
        import torch.distributed as dist

        if self.transport == "host":
            src = pad.cpu()
            out = torch.empty((self.nranks * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype)
            dist.all_gather(list(out.chunk(self.nranks)), src, group=self.group)
            return out.to(pad.device)
        out = torch.empty((self.nranks * pad.shape[0],) + tuple(pad.shape[1:]), dtype=pad.dtype,
                          device=pad.device)
        dist.all_gather_into_tensor(out, pad, group=self.group)
        return out

    def __del__(self):
        try:
            N.lib().spb_comm_destroy(self.handle)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class RowShardedLaplacian:
    """This rank's rows of L = D - W, in the gathered-column layout.

    Built from the graph's arc list (``g`` may be a lazily built SparseGraph:
    its whole-graph CSR is never formed here).
    """

    def __init__(self, g: SparseGraph, group=None, comm: _Comm | None = None,
                 transport: str = "nccl"):
        self.graph = g
        self.comm = comm or _Comm(group, transport)
        self.nranks, self.rank = self.comm.nranks, self.comm.rank
        self.n = g.n_vertices
        if self.n < self.nranks:
            raise ContractError("a rank received no rows; use fewer ranks")
        src, dst, w, m = g._src, g._dst, g._w, g._m
        self.bounds = arc_row_bounds(src, dst, self.n, self.nranks)
        self.row_begin = int(self.bounds[self.rank])
        self.row_end = int(self.bounds[self.rank + 1])
        self.n_local = self.row_end - self.row_begin
        self.n_max = int(np.diff(self.bounds).max())
        if self.n_local < 1:
            raise ContractError("a rank received no rows; use fewer ranks")
        dev = _device()
        L = N.lib()
        b = torch.from_numpy(self.bounds.astype(np.int32)).to(dev)
        cap = max(1, 2 * m)
        wsb = L.spb_csr_build_workspace(m, self.n, N.CSR_SYMMETRIZED)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        self.row_ptr = torch.empty(self.n_local + 1, dtype=torch.int32, device=dev)
        col = torch.empty(cap, dtype=torch.int32, device=dev)
        val = torch.empty(cap, dtype=torch.float64, device=dev)
        self.deg64 = torch.empty(self.n_local, dtype=torch.float64, device=dev)
        nnz = C.c_int64(0)
        N.check(L.spb_csr_build_rows(N.ptr(src), N.ptr(dst), N.ptr(w), m, self.n, self.row_begin,
                                     self.row_end, N.ptr(b), self.nranks, self.n_max, N.ptr(ws), wsb,
                                     N.ptr(self.row_ptr), N.ptr(col), N.ptr(val), N.ptr(self.deg64),
                                     C.byref(nnz), N.stream()))
        del ws
        self.nnz_local = int(nnz.value)
        self.col = col[: max(self.nnz_local, 1)].clone()
        self.val64 = val[: max(self.nnz_local, 1)].clone()
        mx = C.c_double(0.0)
        N.check(L.spb_max_f64(N.ptr(self.deg64), self.n_local, C.byref(mx), N.stream()))
        self.scale_hint = self.comm.allreduce_max(float(mx.value))  # global max degree
        self._cast = {}

    def _typed(self, dtype):
        if dtype == "float64":
            return self.val64, self.deg64
        if dtype not in self._cast:
            v = self.val64.to(torch.float32)
            d = self.deg64.to(torch.float32)
            self._cast[dtype] = (v, d)
        return self._cast[dtype]

    def native(self, dtype: str):
        v, d = self._typed(dtype)
        op = N.Operator()
        op.kind = N.OP_LAPLACIAN
        op.n = self.n_local
        op.row_ptr = N.ptr(self.row_ptr)
        op.col = N.ptr(self.col)
        op.val = N.ptr(v)
        op.deg = N.ptr(d)
        op.dense = None
        op.scale_hint = self.scale_hint
        sh = N.Shard(comm=self.comm.handle if self.nranks > 1 else None, nranks=self.nranks,
                     rank=self.rank, n_global=self.n, row_begin=self.row_begin, n_max=self.n_max)
        op._keep = (v, d)
        return op, sh


def lobpcg_solve_sharded(op: RowShardedLaplacian, x0, config: SolverConfig, n_converge=None,
                         callback=None, *, precision: str | None = None) -> EigenState:
    """lobpcg_solve on this rank's rows; x0 is the global (n, l) block (host)."""
    precision = precision or default_precision(config.tol)
    if not isinstance(x0, torch.Tensor):
        x0 = np.asarray(x0, dtype=np.float64)
    if x0.ndim != 2 or x0.shape[0] != op.n:
        raise ContractError(f"x0 must be ({op.n}, block_size)")
    l = x0.shape[1]
    if l != config.block_size:
        raise ContractError(f"x0 has {l} columns but config.block_size is {config.block_size}")
    nc = l if n_converge is None else int(n_converge)
    code, tdt = DTYPES[precision]
    L = N.lib()
    native, sh = op.native(precision)
    dev = _device()
    if isinstance(x0, torch.Tensor):
        x0_d = x0[op.row_begin:op.row_end].to(device=dev, dtype=torch.float64).contiguous()
    else:
        x0_d = _h2d.to_device(np.ascontiguousarray(x0[op.row_begin:op.row_end]), dev)
    wsb = L.spb_lobpcg_workspace_sharded(code, op.n_local, l, op.nranks, op.n_max)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    cfg = N.SolverConfigC(block_size=l, max_iter=config.max_iter, tol=config.tol,
                          lock_tol=config.lock_tol, n_converge=nc, deflate_ones=int(config.deflate_ones),
                          has_precond=0, reserved=1 if os.environ.get("SPB_PROFILE_SPMM") == "1" else 0)
    bridge = _Bridge(callback, np.random.default_rng(config.seed), None, l)
    theta, norms, conv, stats = (C.c_double * l)(), (C.c_double * l)(), (C.c_uint8 * l)(), (C.c_int64 * 16)()
    status = L.spb_lobpcg_solve_sharded(C.byref(native), C.byref(sh), code, N.ptr(x0_d), C.byref(cfg),
                                        bridge.it, bridge.refill, None, N.ptr(ws), wsb, theta, norms,
                                        conv, stats, N.stream())
    if bridge.exc is not None:
        raise bridge.exc
    if getattr(op.comm, "exc", None) is not None:
        raise op.comm.exc
    state = None
    if status in (N.OK, N.E_SOLVER):
        xp, ldx = C.c_void_p(), C.c_int64()
        N.check(L.spb_lobpcg_result_block(code, op.n_local, l, N.ptr(ws), C.byref(xp), C.byref(ldx)))
        vec = torch.empty((op.n_local, l), dtype=tdt, device=dev)
        N.check(L.spb_copy_block(code, xp.value, ldx.value, code, N.ptr(vec), l, op.n_local, l, N.stream()))
        state = EigenState(np.array(theta[:]), vec, np.array(norms[:]), int(stats[0]),
                           np.array(conv[:], dtype=bool), work_blocks=6)
        state.solve_stats = dict(zip(("iterations", "spmm_calls", "rr_calls", "drop_p",
                                      "rebuild", "orth_p"), [int(x) for x in stats[:6]]))
        state.solve_stats.update(spmm_us=int(stats[7]), spmm_bytes=int(stats[8]),
                                 spmm_cols=int(stats[9]),
                                 gram_us=int(stats[12]), gram_calls=int(stats[13]),
                                 gram_mflop=int(stats[14]))
        state.row_range = (op.row_begin, op.row_end)
    if status == N.OK:
        return state
    msg = (L.spb_last_error() or b"").decode(errors="replace")
    if status in (N.E_SOLVER, N.E_SOLVER_NOSTATE):
        raise SolverError(msg, state=state)
    N.check(status)
    raise SpecpartError(msg)


def _gather_rows(op: RowShardedLaplacian, local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather variable-length row blocks (padded to n_max) into the global block."""
    if op.nranks == 1:
        return local
    pad = torch.zeros((op.n_max, local.shape[1]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = op.comm.all_gather_rows(pad)
    parts = [out[r * op.n_max: r * op.n_max + int(op.bounds[r + 1] - op.bounds[r])] for r in range(op.nranks)]
    return torch.cat(parts).contiguous()


def assign_clusters_qrcp_sharded(op: RowShardedLaplacian, emb: torch.Tensor, k: int):
    """assign_clusters_qrcp (spectral.py:134-170) on the row-sharded embedding
    (this rank's rows): k global argmax pivot steps over the communicator
    (spb_assign_qrcp_sharded), labels of the local rows.

    Returns (local labels int32 device tensor, pivots (global rows, device), info)."""
    if emb.dtype not in (torch.float32, torch.float64):
        raise ContractError("embedding must be float32 or float64")
    emb = emb if emb.stride(1) == 1 else emb.contiguous()
    code = N.F32 if emb.dtype == torch.float32 else N.F64
    L = N.lib()
    _, sh = op.native("float64")
    nl = emb.shape[0]
    if nl != op.n_local:
        raise ContractError("embedding rows do not match this rank's rows")
    wsb = L.spb_assign_workspace_sharded(nl, k, op.nranks)
    ws = torch.empty(wsb, dtype=torch.uint8, device=emb.device)
    labels = torch.empty(max(nl, 1), dtype=torch.int32, device=emb.device)
    pivots = torch.empty(k, dtype=torch.int32, device=emb.device)
    info = (C.c_double * 4)()
    status = L.spb_assign_qrcp_sharded(code, N.ptr(emb), emb.stride(0), nl, k, C.byref(sh),
                                       N.ptr(ws), wsb, N.ptr(labels), N.ptr(pivots), info, N.stream())
    if getattr(op.comm, "exc", None) is not None:
        raise op.comm.exc
    N.check(status)
    return labels[:nl], pivots, list(info)


def partition_static_sharded(g: SparseGraph, cfg: SolverConfig, k_expected: int | None = None, *,
                             alpha: float = 3.0, k_min: int = 2, fix_k: bool = False, x0=None,
                             precision: str | None = None, group=None, op: RowShardedLaplacian | None = None,
                             callback=None):
    """partition_static with the rows of the operator split across the ranks of ``group``."""
    n = g.n_vertices
    if n < 1:
        raise DomainError("cannot partition an empty graph")
    l = block_size_for(k_expected) if k_expected is not None else cfg.block_size
    l = min(l, n)
    cfg_run = cfg.replace(block_size=l)
    start = random_init(n, l, cfg.seed) if x0 is None else x0
    nc = min(k_expected + 1, l) if k_expected is not None else None
    op = op or RowShardedLaplacian(g, group)
    state = lobpcg_solve_sharded(op, start, cfg_run, n_converge=nc, precision=precision,
                                 callback=callback)
    gap = (detect_gap(state.eigenvalues, k_min=min(k_min, l - 1), alpha=alpha) if l >= 2
           else GapResult(k=1, increments=np.empty(0), confidence=0.0, reliable=False))
    k_used = k_expected if (fix_k and k_expected is not None) else gap.k
    # distributed QRCP: global argmax pivot steps, local labels, then one gather of labels
    local, _, info = assign_clusters_qrcp_sharded(op, state.device_vectors[:, :k_used], k_used)
    labels = _gather_rows(op, local.view(-1, 1), group).view(-1)
    return Partition(labels.cpu().numpy().astype(np.int64), int(info[0])), state, gap


def partition_edges_sharded(edges, n: int, cfg: SolverConfig, k_expected: int | None = None, *,
                            weights=None, group=None, comm: _Comm | None = None,
                            transport: str = "nccl", **kw):
    """Edge list in, labels out, rows sharded over the ranks of ``group``: each rank
    uploads the arcs and builds only its rows of W (no whole-graph CSR anywhere)."""
    src, dst, w = _device_arcs(edges, n, weights)
    g = SparseGraph(int(n), src, dst, w)
    op = RowShardedLaplacian(g, group=group, comm=comm, transport=transport)
    return partition_static_sharded(g, cfg, k_expected, group=group, op=op, **kw)
