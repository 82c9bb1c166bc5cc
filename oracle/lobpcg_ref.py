"""Soft-locked block LOBPCG — numpy/scipy restatement (TEST INFRASTRUCTURE ONLY).

Follows ``specpart/lobpcg.py`` of the reference:
* ``SolverConfig``        lobpcg.py:38-81  (tol 1e-4, max_iter 20, lock_tol = 0.1 tol)
* ``random_init``         lobpcg.py:154-161 (PCG64 standard_normal)
* ``_small_gen_eigh``     lobpcg.py:164-177 (finite check, cond(G_B) <= 1/sqrt(eps), dsygvd)
* ``orthonormalize``      lobpcg.py:195-215 (5 tries, Gaussian refill of dependent columns)
* ``_cholesky_orth``      lobpcg.py:218-247 (CholQR, pivoted-QR fallback)
* ``lobpcg_solve``        lobpcg.py:263-454 (setup RR, loop with soft lock, P
                          normalisation, full / drop_p / rebuild ladder, polish)

The working set is kept as six separate n-by-l blocks (X, R, P and their
operator images) rather than the reference's two packed (n, 3l) arrays; the
basis of each Rayleigh-Ritz step is the column concatenation [X | R_act | P_act].
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg

EPS = np.finfo(np.float64).eps
COND_MAX = 1.0 / np.sqrt(EPS)  # lobpcg.py:35


class OracleConditioningError(RuntimeError):
    pass


class OracleSolverError(RuntimeError):
    def __init__(self, msg, state=None):
        super().__init__(msg)
        self.state = state


@dataclass(frozen=True)
class SolverCfg:
    block_size: int
    tol: float = 1e-4
    max_iter: int = 20
    seed: int = 0
    soft_lock_tol: float | None = None
    deflate_ones: bool = False

    @property
    def lock_tol(self):
        return 0.1 * self.tol if self.soft_lock_tol is None else self.soft_lock_tol


@dataclass
class StateRef:
    eigenvalues: np.ndarray
    vectors: np.ndarray
    residual_norms: np.ndarray
    iterations: int
    converged: np.ndarray


def random_init(n, l, seed=0):
    """lobpcg.py:154-161."""
    return np.random.default_rng(seed).standard_normal((n, l))


def _sym(g):
    return 0.5 * (g + g.T)


def small_gen_eigh_ref(ga, gb):
    """lobpcg.py:168-177."""
    if not (np.isfinite(ga).all() and np.isfinite(gb).all()):
        raise OracleConditioningError("non-finite projected matrices")
    if np.linalg.cond(gb) > COND_MAX:
        raise OracleConditioningError("ill-conditioned overlap")
    try:
        return scipy.linalg.eigh(ga, gb)
    except (scipy.linalg.LinAlgError, np.linalg.LinAlgError) as exc:
        raise OracleConditioningError(str(exc)) from exc


def cholesky_orth_ref(b):
    """In-place CholQR of b; returns retained width (lobpcg.py:218-247)."""
    na = b.shape[1]
    if na == 0:
        return 0
    g = _sym(b.T @ b)
    dg = np.diag(g)
    if np.all(dg > 0) and dg.min() > (EPS * na) ** 2 * dg.max():
        try:
            c = np.linalg.cholesky(g)
            rd = np.diag(c)
            if rd.min() > np.sqrt(EPS) * rd.max():
                b[:] = b @ scipy.linalg.solve_triangular(c.T, np.eye(na), lower=False)
                return na
        except np.linalg.LinAlgError:
            pass
    q, r, _ = scipy.linalg.qr(b, mode="economic", pivoting=True)
    rd = np.abs(np.diag(r))
    if rd.size == 0 or rd[0] == 0:
        return 0
    rank = int(np.sum(rd > max(b.shape) * EPS * rd[0]))
    b[:, :rank] = q[:, :rank]
    return rank


def orthonormalize_ref(x, rng):
    """lobpcg.py:195-215."""
    if x.shape[1] > x.shape[0]:
        raise ValueError("more columns than rows")
    if not np.any(x):
        raise ValueError("all-zero block")
    width = x.shape[1]
    for _ in range(5):
        kept = cholesky_orth_ref(x)
        if kept == width:
            return x
        x[:, kept:] = rng.standard_normal((x.shape[0], width - kept))
    raise OracleConditioningError("could not build a full-rank orthonormal block")


def lobpcg_ref(op, x0, cfg: SolverCfg, n_converge=None, callback=None):
    """The soft-locked LOBPCG loop of lobpcg.py:263-454."""
    x0 = np.asarray(x0, dtype=np.float64)
    n = op.n
    l = x0.shape[1]
    nc = l if n_converge is None else int(n_converge)
    rng = np.random.default_rng(cfg.seed)

    X = x0.copy()
    if cfg.deflate_ones:
        X -= X.mean(axis=0, keepdims=True)
    orthonormalize_ref(X, rng)
    LX = op.apply(X)

    def state(theta, norms, its, scale):
        norms = np.asarray(norms, dtype=np.float64).copy()
        return StateRef(np.array(theta[:l]), X.copy(), norms, its, norms < cfg.tol * scale)

    try:
        theta, C = small_gen_eigh_ref(_sym(X.T @ LX), _sym(X.T @ X))
    except OracleConditioningError as exc:
        raise OracleSolverError(f"initial projection failed: {exc}") from exc
    X = X @ C
    LX = LX @ C

    active = np.ones(l, dtype=bool)
    P = LP = None
    iterations = 0
    norms = np.zeros(l)
    for it in range(cfg.max_iter + 1):
        R = LX - X * theta[None, :l]
        norms = np.linalg.norm(R, axis=0)
        scale = max(abs(float(theta[l - 1])), op.scale_hint, np.finfo(np.float64).tiny)
        if not np.isfinite(norms).all():
            raise OracleSolverError("residual norms not finite", state(theta, norms, iterations, scale))
        if callback is not None:
            callback(it, np.array(theta[:l]), norms.copy())
        if np.all(norms[:nc] < cfg.tol * scale) or it == cfg.max_iter:
            break
        active &= norms >= cfg.lock_tol * scale
        if not active.any():
            break
        iterations += 1
        idx = np.flatnonzero(active)
        Ra = R[:, idx].copy()
        if cfg.deflate_ones:
            Ra -= Ra.mean(axis=0, keepdims=True)
        Ra -= X @ (X.T @ Ra)  # single projection (lobpcg.py:365-369)
        na = cholesky_orth_ref(Ra)
        if na == 0:
            break
        Ra = Ra[:, :na]
        LRa = op.apply(Ra)

        Pa = LPa = None
        if P is not None:
            Pa, LPa = P[:, idx], LP[:, idx]
            pn = np.linalg.norm(Pa, axis=0)
            keep = np.flatnonzero(pn > 0)
            Pa, LPa = Pa[:, keep] / pn[keep], LPa[:, keep] / pn[keep]
            if Pa.shape[1] == 0:
                Pa = LPa = None

        got = None
        for rung in ("full", "drop_p", "rebuild"):
            if rung == "drop_p":
                if Pa is None:
                    continue
                Pa = LPa = None
            elif rung == "rebuild":
                orthonormalize_ref(X, rng)
                LX = op.apply(X)
                Ra -= X @ (X.T @ Ra)
                na = cholesky_orth_ref(Ra)
                if na == 0:
                    break
                Ra = Ra[:, :na]
                LRa = op.apply(Ra)
            B = np.concatenate([X, Ra] + ([Pa] if Pa is not None else []), axis=1)
            LB = np.concatenate([LX, LRa] + ([LPa] if LPa is not None else []), axis=1)
            try:
                got = small_gen_eigh_ref(_sym(B.T @ LB), _sym(B.T @ B))
            except OracleConditioningError:
                continue
            break
        if got is None:
            if na == 0:
                break
            raise OracleSolverError("projected eigenproblem unsolvable", state(theta, norms, iterations, scale))
        theta, Cfull = got
        C = Cfull[:, :l]
        P = B[:, l:] @ C[l:]
        LP = LB[:, l:] @ C[l:]
        X = B @ C
        LX = LB @ C

    orthonormalize_ref(X, rng)
    LX = op.apply(X)
    theta, C = small_gen_eigh_ref(_sym(X.T @ LX), np.eye(l))
    X = X @ C
    LX = LX @ C
    norms = np.linalg.norm(LX - X * theta[None, :], axis=0)
    scale = max(abs(float(theta[l - 1])), op.scale_hint, np.finfo(np.float64).tiny)
    return state(theta, norms, iterations, scale)
