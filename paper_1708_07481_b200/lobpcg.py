"""Block eigensolver for the smallest eigenpairs — the device LOBPCG.

Same public surface as the reference's ``specpart/lobpcg.py``:
``SolverConfig`` (lobpcg.py:38-81), ``EigenState`` (:84-129), ``DenseOperator``
(:132-151), ``random_init`` (:154-161), ``orthonormalize`` (:195-215),
``rayleigh_ritz`` (:180-192), ``lobpcg_solve`` (:263-454), ``residual_norms``
(:457-461). ``lobpcg_solve`` runs the whole soft-locked loop inside the CUDA
library (csrc/lobpcg.cu) through ``spb_lobpcg_solve``; Python only validates
arguments, owns the device buffers (torch) and bridges the three host
callbacks (per-iteration callback, Gaussian rank repair from the solve's numpy
Generator, optional preconditioner).

Precision: the six n-by-l blocks are stored in float32 (default) or float64
(``precision="float64"`` or ``SPB_PRECISION=float64``). Gram products always
accumulate in float64 and every small projected problem is solved in float64.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import os
import warnings
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _h2d
from . import _native as N
from .errors import ConditioningError, ContractError, DomainError, SolverError, SpecpartError
from .graph import DTYPES, LaplacianOperator, _device

__all__ = [
    "SolverConfig",
    "EigenState",
    "DenseOperator",
    "random_init",
    "orthonormalize",
    "rayleigh_ritz",
    "lobpcg_solve",
    "residual_norms",
    "default_precision",
]


# Below this relative tolerance float32 storage cannot converge: its residuals
# bottom out near eps32 * ||L|| (~1e-7 * scale), so the stop test would never pass.
F32_TOL_FLOOR = 1e-6


def default_precision(tol: float | None = None) -> str:
    """Storage precision when the caller did not choose one: ``SPB_PRECISION`` if set,
    else float32 -- promoted to float64 (with a warning) for a tolerance below the
    float32 residual floor, so e.g. ``SolverConfig.high_accuracy`` converges as in the
    reference instead of running max_iter iterations."""
    p = os.environ.get("SPB_PRECISION")
    if p is not None:
        if p not in DTYPES:
            raise DomainError(f"SPB_PRECISION must be one of {sorted(DTYPES)}, got {p!r}")
        return p
    if tol is not None and tol < F32_TOL_FLOOR:
        warnings.warn(f"tol={tol:g} is below the float32 residual floor ({F32_TOL_FLOOR:g}); "
                      "solving with float64 storage (pass precision='float32' to override)",
                      stacklevel=3)
        return "float64"
    return "float32"


@dataclass(frozen=True)
class SolverConfig:
    """Knobs for one eigensolve (lobpcg.py:38-81); tolerances are relative to
    max(|theta_{l-1}|, operator.scale_hint)."""

    block_size: int
    tol: float = 1e-4
    max_iter: int = 20
    seed: int = 0
    soft_lock_tol: float | None = None
    determinism: bool = False
    deflate_ones: bool = False

    def __post_init__(self):
        if self.block_size < 1:
            raise DomainError("block_size must be at least 1")
        if not (self.tol > 0):
            raise DomainError("tol must be positive")
        if self.max_iter < 1:
            raise DomainError("max_iter must be at least 1")
        if self.soft_lock_tol is not None and self.soft_lock_tol < 0:
            raise DomainError("soft_lock_tol must be non-negative")

    @property
    def lock_tol(self) -> float:
        return 0.1 * self.tol if self.soft_lock_tol is None else self.soft_lock_tol

    @classmethod
    def high_accuracy(cls, block_size: int, **overrides) -> "SolverConfig":
        defaults = dict(tol=1e-10, max_iter=500)
        defaults.update(overrides)
        return cls(block_size=block_size, **defaults)

    def replace(self, **changes) -> "SolverConfig":
        return dataclasses.replace(self, **changes)


class EigenState:
    """Result of an eigensolve and warm-start carrier (lobpcg.py:84-129).

    ``vectors`` is materialised on the host on first access; the device copy
    (storage dtype) stays available as ``device_vectors`` for the assignment
    and for warm starts without a host round trip.
    """

    def __init__(self, eigenvalues, vectors, residual_norms, iterations, converged,
                 work_blocks=0):
        self.eigenvalues = np.asarray(eigenvalues, dtype=np.float64)
        self._host = None
        self.device_vectors = None
        if isinstance(vectors, torch.Tensor):
            self.device_vectors = vectors
        else:
            self._host = np.asarray(vectors, dtype=np.float64)
        self.residual_norms = np.asarray(residual_norms, dtype=np.float64)
        self.iterations = int(iterations)
        self.converged = np.asarray(converged, dtype=bool)
        self.work_blocks = int(work_blocks)

    @property
    def vectors(self) -> np.ndarray:
        if self._host is None:
            self._host = self.device_vectors.double().cpu().numpy()
        return self._host

    @vectors.setter
    def vectors(self, v):
        self._host = np.asarray(v, dtype=np.float64)
        self.device_vectors = None

    @property
    def block_size(self) -> int:
        if self.device_vectors is not None:
            return int(self.device_vectors.shape[1])
        return int(self._host.shape[1])

    def all_converged(self, first: int | None = None) -> bool:
        return bool(np.all(self.converged[: first or len(self.converged)]))

    def save(self, path) -> None:
        np.savez(Path(path), eigenvalues=self.eigenvalues, vectors=self.vectors,
                 residual_norms=self.residual_norms, iterations=np.int64(self.iterations),
                 converged=np.asarray(self.converged, dtype=bool),
                 work_blocks=np.int64(self.work_blocks))

    @classmethod
    def load(cls, path) -> "EigenState":
        with np.load(Path(path)) as d:
            return cls(d["eigenvalues"], d["vectors"], d["residual_norms"], int(d["iterations"]),
                       np.asarray(d["converged"], dtype=bool), int(d["work_blocks"]))

    def __repr__(self):
        return (f"EigenState(block_size={self.block_size}, iterations={self.iterations}, "
                f"converged={int(self.converged.sum())}/{self.converged.size})")


class DenseOperator:
    """Dense symmetric matrix in the operator protocol (lobpcg.py:132-151), on the device."""

    def __init__(self, a):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ContractError("operator matrix must be square")
        if not np.allclose(a, a.T, atol=1e-10 * max(1.0, np.abs(a).max() if a.size else 1.0)):
            raise ContractError("operator matrix must be symmetric")
        self.a = a
        self.n = a.shape[0]
        self.scale_hint = float(np.abs(a).sum(axis=1).max()) if self.n else 1.0
        self._dev = torch.from_numpy(np.ascontiguousarray(a)).to(_device())

    def native(self, dtype: str) -> N.Operator:
        op = N.Operator()
        op.kind = N.OP_DENSE
        op.n = self.n
        op.dense = N.ptr(self._dev)
        op.scale_hint = self.scale_hint
        return op

    def apply(self, x, out=None):
        y = self.a @ np.asarray(x, dtype=np.float64)
        if out is None:
            return y
        out[...] = y
        return out

    __call__ = apply


def random_init(n: int, block_size: int, seed: int = 0) -> np.ndarray:
    """Gaussian random starting block (lobpcg.py:154-161); host numpy so the
    reference and the device path start from identical bits."""
    if block_size < 1:
        raise DomainError("block_size must be at least 1")
    if block_size > n:
        raise DomainError(f"block_size {block_size} exceeds dimension {n}")
    return np.random.default_rng(seed).standard_normal((n, block_size))


class _Bridge:
    """ctypes callbacks with exception capture (a raising callback aborts the solve)."""

    def __init__(self, callback, rng, precond, l):
        self.exc = None
        self.l = l

        def it_cb(_u, it, th, nr, ll):
            try:
                if callback is not None:
                    callback(int(it), np.ctypeslib.as_array(th, (ll,)).copy(),
                             np.ctypeslib.as_array(nr, (ll,)).copy())
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised after the solve
                self.exc = e
                return 1

        def refill_cb(_u, rows, cols, out):
            try:
                vals = rng.standard_normal((int(rows), int(cols)))
                np.ctypeslib.as_array(out, (int(rows) * int(cols),))[:] = vals.ravel()
                return 0
            except BaseException as e:  # noqa: BLE001
                self.exc = e
                return 1

        def pre_cb(_u, rows, cols, inout):
            try:
                a = np.ctypeslib.as_array(inout, (int(rows) * int(cols),)).reshape(int(rows), int(cols))
                r = np.asarray(precond(a.copy()), dtype=np.float64)
                if r.shape != a.shape:
                    raise ContractError("preconditioner changed the block shape")
                a[...] = r
                return 0
            except BaseException as e:  # noqa: BLE001
                self.exc = e
                return 1

        self.it = N.ITER_CB(it_cb)
        self.refill = N.REFILL_CB(refill_cb)
        self.pre = N.PRECOND_CB(pre_cb) if precond is not None else N.PRECOND_CB()


class _HostOperator:
    """Any object with the reference's operator protocol -- ``.n``, ``.scale_hint``,
    ``.apply(x, out=None) -> out`` (graph.py:300-317; duck-typed at lobpcg.py:273,
    :308, :374) -- bridged as an SPB_OP_HOST callback: the solve stays on the device,
    each operator apply receives a host float64 (n, cols) block."""

    def __init__(self, operator):
        self.operator = operator
        self.exc = None
        n = int(operator.n)

        def apply_cb(_u, rows, cols, x_in, y_out):
            try:
                shape = (int(rows), int(cols))
                x = np.ctypeslib.as_array(x_in, (shape[0] * shape[1],)).reshape(shape).copy()
                y = np.ctypeslib.as_array(y_out, (shape[0] * shape[1],)).reshape(shape)
                r = operator.apply(x, out=y)
                if r is not None and r is not y:
                    r = np.asarray(r, dtype=np.float64)
                    if r.shape != shape:
                        raise ContractError(f"operator.apply returned shape {r.shape}, expected {shape}")
                    y[...] = r
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised after the solve
                self.exc = e
                return 1

        self.cb = N.APPLY_CB(apply_cb)
        self.n = n

    def native(self) -> N.Operator:
        op = N.Operator()
        op.kind = N.OP_HOST
        op.n = self.n
        op.scale_hint = float(self.operator.scale_hint)
        op.apply = self.cb
        return op


def _native_operator(operator, dtype: str, cols: int):
    if isinstance(operator, LaplacianOperator):
        return operator.native(dtype, cols), dtype, None
    if isinstance(operator, DenseOperator):
        return operator.native("float64"), "float64", None
    if all(hasattr(operator, a) for a in ("n", "scale_hint", "apply")):
        host = _HostOperator(operator)
        return host.native(), dtype, host
    raise ContractError("operator must provide .n, .scale_hint and .apply(x, out=None) "
                        "(the reference's operator protocol, graph.py:300-317)")


def _x0_device(x0, n, l, precision="float64"):
    if isinstance(x0, torch.Tensor):
        t = x0.to(device=_device(), dtype=torch.float64)
        return t.contiguous()
    arr = np.ascontiguousarray(x0, dtype=np.float64)
    if precision == "float32":
        # the solver rounds x0 to float32 storage first thing (copy_block, round to
        # nearest): round on the host while staging (same bits) and move half the bytes
        return _h2d.to_device(arr, _device(), np.float32).double()
    return _h2d.to_device(arr, _device())  # multi-threaded pinned ring for large blocks


def lobpcg_solve(operator, x0, config: SolverConfig, precond=None, n_converge: int | None = None,
                 callback=None, *, precision: str | None = None) -> EigenState:
    """Smallest eigenpairs of the operator (lobpcg.py:263-454), on the GPU.

    Raises ContractError / DomainError on bad arguments, SolverError (with the
    last valid state) when the iteration cannot continue.
    """
    precision = precision or default_precision(config.tol)
    if isinstance(x0, torch.Tensor):
        shape = tuple(x0.shape)
    else:
        x0 = np.asarray(x0, dtype=np.float64)
        shape = x0.shape
    if not all(hasattr(operator, a) for a in ("n", "scale_hint", "apply")):
        raise ContractError("operator must provide .n, .scale_hint and .apply(x, out=None) "
                            "(the reference's operator protocol, graph.py:300-317)")
    n = operator.n
    if len(shape) != 2 or shape[0] != n:
        raise ContractError(f"x0 must be ({n}, block_size)")
    l = shape[1]
    if l != config.block_size:
        raise ContractError(f"x0 has {l} columns but config.block_size is {config.block_size}")
    if l > n:
        raise DomainError(f"block_size {l} exceeds operator dimension {n}")
    nc = l if n_converge is None else int(n_converge)
    if not 1 <= nc <= l:
        raise DomainError("n_converge must be in [1, block_size]")
    op, precision, host_op = _native_operator(operator, precision, l)
    code, tdt = DTYPES[precision]
    L = N.lib()
    x0_d = _x0_device(x0, n, l, precision)
    ws_bytes = L.spb_lobpcg_workspace(code, n, l)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=x0_d.device)
    cfg = N.SolverConfigC(block_size=l, max_iter=config.max_iter, tol=config.tol,
                          lock_tol=config.lock_tol, n_converge=nc,
                          deflate_ones=int(config.deflate_ones),
                          has_precond=int(precond is not None),
                          reserved=1 if os.environ.get("SPB_PROFILE_SPMM") == "1" else 0)
    bridge = _Bridge(callback, np.random.default_rng(config.seed), precond, l)
    theta = (C.c_double * l)()
    norms = (C.c_double * l)()
    conv = (C.c_uint8 * l)()
    stats = (C.c_int64 * 16)()
    status = L.spb_lobpcg_solve(C.byref(op), code, N.ptr(x0_d), C.byref(cfg), bridge.it,
                                bridge.refill, bridge.pre, None, N.ptr(ws), ws_bytes, None,
                                theta, norms, conv, stats, N.stream())
    if bridge.exc is not None:
        raise bridge.exc
    if host_op is not None and host_op.exc is not None:
        raise host_op.exc
    state = None
    if status in (N.OK, N.E_SOLVER):
        xp = C.c_void_p()
        ldx = C.c_int64()
        N.check(L.spb_lobpcg_result_block(code, n, l, N.ptr(ws), C.byref(xp), C.byref(ldx)))
        vec = torch.empty((n, l), dtype=tdt, device=ws.device)
        if op.perm:  # the solve ran in the operator's locality order: back to the caller's rows
            N.check(L.spb_permute_rows(code, xp.value, ldx.value, code, N.ptr(vec), l, n, l,
                                       op.perm, 1, N.stream()))
        else:
            N.check(L.spb_copy_block(code, xp.value, ldx.value, code, N.ptr(vec), l, n, l,
                                     N.stream()))
        state = EigenState(np.array(theta[:]), vec, np.array(norms[:]), int(stats[0]),
                           np.array(conv[:], dtype=bool), work_blocks=6)
        state.solve_stats = dict(zip(("iterations", "spmm_calls", "rr_calls", "drop_p",
                                      "rebuild"), [int(s) for s in stats[:5]]))
        state.solve_stats.update(orth_p=int(stats[5]), spmm_us=int(stats[7]), spmm_bytes=int(stats[8]),
                                 spmm_cols=int(stats[9]),
                                 gram_us=int(stats[12]), gram_calls=int(stats[13]),
                                 gram_mflop=int(stats[14]))
        state.precision = precision
    del ws
    if status == N.OK:
        return state
    msg = (L.spb_last_error() or b"").decode(errors="replace")
    if status in (N.E_SOLVER, N.E_SOLVER_NOSTATE):
        raise SolverError(msg, state=state)
    N.check(status)
    raise SpecpartError(msg)  # unreachable


def _solve_small(ga, gb, nev=None):
    """Device sygv on host matrices (float64)."""
    ga = np.ascontiguousarray(ga, dtype=np.float64)
    m = ga.shape[0]
    nev = m if nev is None else nev
    dev = _device()
    tga = torch.from_numpy(ga).to(dev)
    tgb = None if gb is None else torch.from_numpy(np.ascontiguousarray(gb, dtype=np.float64)).to(dev)
    L = N.lib()
    wsb = L.spb_sygv_workspace(m)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
    th = torch.empty(max(nev, 1), dtype=torch.float64, device=dev)
    cc = torch.empty((m, max(nev, 1)), dtype=torch.float64, device=dev)
    N.check(L.spb_sygv(N.ptr(tga), N.ptr(tgb), m, nev, N.ptr(th), N.ptr(cc), N.ptr(ws), wsb,
                       N.stream()))
    return th[:nev].cpu().numpy(), cc[:, :nev].cpu().numpy()


def rayleigh_ritz(operator, basis):
    """Ritz values and coefficients on span(basis) (lobpcg.py:180-192)."""
    basis = np.asarray(basis, dtype=np.float64)
    image = operator.apply(basis)
    return _solve_small(basis.T @ image, basis.T @ basis)


def orthonormalize(x: np.ndarray, rng=None) -> np.ndarray:
    """Orthonormalise the columns of x in place (lobpcg.py:195-215), on the device."""
    if x.shape[1] > x.shape[0]:
        raise DomainError("cannot orthonormalize: more columns than rows")
    if not np.any(x):
        raise DomainError("cannot orthonormalize an all-zero block")
    rng = np.random.default_rng(0) if rng is None else rng
    n, width = x.shape
    L = N.lib()
    dev = _device()
    xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
    wsb = L.spb_orthonormalize_workspace(N.F64, n, width)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    bridge = _Bridge(None, rng, None, width)
    status = L.spb_orthonormalize(N.F64, N.ptr(xt), width, n, width, bridge.refill, None,
                                  N.ptr(ws), wsb, N.stream())
    if bridge.exc is not None:
        raise bridge.exc
    N.check(status)
    x[...] = xt.cpu().numpy()
    return x


def residual_norms(operator, state: EigenState) -> np.ndarray:
    """||L x_i - lambda_i x_i|| recomputed from scratch (lobpcg.py:457-461)."""
    image = operator.apply(state.vectors)
    image -= state.vectors * state.eigenvalues[None, :]
    return np.linalg.norm(image, axis=0)
