"""ctypes binding of libspb200.so (the C ABI declared in include/specpart_b200.h).

There is no CPU fallback: importing this module without the built library, or
calling into it without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import (
    AssignmentError,
    ConditioningError,
    ContractError,
    DomainError,
    NativeError,
    SolverError,
)

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libspb200.so"

OK, E_CONTRACT, E_DOMAIN, E_COND, E_SOLVER, E_SOLVER_NOSTATE, E_ASSIGN, E_CUDA, E_WS, E_CB, E_PARSE = range(11)
F32, F64 = 0, 1
CSR_DIRECTED, CSR_SYMMETRIZED, CSR_AS_SYMMETRIC = 0, 1, 2
OP_LAPLACIAN, OP_DENSE, OP_HOST = 0, 1, 2

vp = C.c_void_p
i32, i64, f64, sz = C.c_int32, C.c_int64, C.c_double, C.c_size_t


APPLY_CB = C.CFUNCTYPE(C.c_int, vp, i64, i32, C.POINTER(f64), C.POINTER(f64))


class Operator(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", i32), ("row_ptr", vp), ("col", vp), ("val", vp),
                ("deg", vp), ("dense", vp), ("scale_hint", f64), ("apply", APPLY_CB),
                ("apply_user", vp), ("perm", vp)]


class Shard(C.Structure):
    _fields_ = [("comm", vp), ("nranks", i32), ("rank", i32), ("n_global", i64),
                ("row_begin", i32), ("n_max", i32)]


class SolverConfigC(C.Structure):
    _fields_ = [("block_size", i32), ("max_iter", i32), ("tol", f64), ("lock_tol", f64),
                ("n_converge", i32), ("deflate_ones", i32), ("has_precond", i32),
                ("reserved", i32)]


ITER_CB = C.CFUNCTYPE(C.c_int, vp, i32, C.POINTER(f64), C.POINTER(f64), i32)
REFILL_CB = C.CFUNCTYPE(C.c_int, vp, i64, i32, C.POINTER(f64))
PRECOND_CB = C.CFUNCTYPE(C.c_int, vp, i64, i32, C.POINTER(f64))
ALLREDUCE_CB = C.CFUNCTYPE(C.c_int, vp, C.POINTER(f64), i64)
ALLGATHER_CB = C.CFUNCTYPE(C.c_int, vp, vp, vp, i64)

_SIGS = {
    "spb_last_error": (C.c_char_p, []),
    "spb_version": (C.c_int, []),
    "spb_device_sm_count": (C.c_int, []),
    "spb_csr_build_workspace": (sz, [i64, i32, C.c_int]),
    "spb_csr_build": (C.c_int, [vp, vp, vp, i64, i32, C.c_int, vp, sz, vp, vp, vp, vp,
                                C.POINTER(i64), vp]),
    "spb_cast": (C.c_int, [vp, i64, C.c_int, vp, vp]),
    "spb_h2d_ring_bytes": (C.c_size_t, [i32]),
    "spb_h2d_staged": (C.c_int, [vp, i64, i32, i32, vp, vp, C.c_size_t, i32, vp]),
    "spb_copy_block": (C.c_int, [C.c_int, vp, i64, C.c_int, vp, i64, i64, i32, vp]),
    "spb_max_f64": (C.c_int, [vp, i64, C.POINTER(f64), vp]),
    "spb_laplacian_spmm": (C.c_int, [C.c_int, i32, i32, vp, vp, vp, vp, vp, i64, i32, vp, i64, vp]),
    "spb_vertex_order_workspace": (sz, [i32]),
    "spb_vertex_order": (C.c_int, [C.c_int, i32, vp, vp, vp, vp, i32, C.c_uint64, vp, sz, vp, vp]),
    "spb_csr_permute_workspace": (sz, [i32]),
    "spb_csr_permute": (C.c_int, [C.c_int, i32, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, vp]),
    "spb_permute_rows": (C.c_int, [C.c_int, vp, i64, C.c_int, vp, i64, i64, i32, vp, C.c_int, vp]),
    "spb_gram_workspace": (sz, [i32, i32, i64]),
    "spb_gram": (C.c_int, [C.c_int, C.c_int, vp, i64, i32, vp, i64, i32, i64, vp, i64, vp, sz, vp]),
    "spb_block_update_workspace": (sz, [i32, i32]),
    "spb_block_update": (C.c_int, [C.c_int, C.c_int, vp, i64, i32, vp, i64, i32, f64, vp, i64, vp,
                                   i64, i64, vp, sz, vp]),
    "spb_lobpcg_workspace": (sz, [C.c_int, i32, i32]),
    "spb_lobpcg_solve": (C.c_int, [C.POINTER(Operator), C.c_int, vp, C.POINTER(SolverConfigC),
                                   ITER_CB, REFILL_CB, PRECOND_CB, vp, vp, sz, vp,
                                   C.POINTER(f64), C.POINTER(f64), C.POINTER(C.c_uint8),
                                   C.POINTER(i64), vp]),
    "spb_lobpcg_result_block": (C.c_int, [C.c_int, i32, i32, vp, C.POINTER(vp), C.POINTER(i64)]),
    "spb_comm_unique_id": (C.c_int, [vp, i32]),
    "spb_comm_init": (C.c_int, [i32, i32, vp, C.POINTER(vp)]),
    "spb_comm_destroy": (C.c_int, [vp]),
    "spb_comm_selftest": (C.c_int, [vp]),
    "spb_comm_init_host": (C.c_int, [i32, i32, ALLREDUCE_CB, ALLGATHER_CB, vp, C.POINTER(vp)]),
    "spb_csr_build_rows": (C.c_int, [vp, vp, vp, i64, i32, i32, i32, vp, i32, i32, vp, sz, vp, vp,
                                     vp, vp, C.POINTER(i64), vp]),
    "spb_csr_shard": (C.c_int, [vp, vp, vp, i32, i32, vp, i32, i32, vp, vp, vp, vp]),
    "spb_lobpcg_workspace_sharded": (sz, [C.c_int, i32, i32, i32, i32]),
    "spb_lobpcg_solve_sharded": (C.c_int, [C.POINTER(Operator), C.POINTER(Shard), C.c_int, vp,
                                           C.POINTER(SolverConfigC), ITER_CB, REFILL_CB, vp, vp,
                                           sz, C.POINTER(f64), C.POINTER(f64),
                                           C.POINTER(C.c_uint8), C.POINTER(i64), vp]),
    "spb_orthonormalize_workspace": (sz, [C.c_int, i32, i32]),
    "spb_orthonormalize": (C.c_int, [C.c_int, vp, i64, i32, i32, REFILL_CB, vp, vp, sz, vp]),
    "spb_sygv_workspace": (sz, [i32]),
    "spb_sygv": (C.c_int, [vp, vp, i32, i32, vp, vp, vp, sz, vp]),
    "spb_edge_list_parse": (C.c_int, [C.c_char_p, sz, i32, i32, C.POINTER(i64), C.POINTER(i64),
                                      C.POINTER(i32), C.POINTER(i64), C.POINTER(vp)]),
    "spb_edge_list_fetch": (C.c_int, [vp, vp, vp, vp]),
    "spb_edge_list_free": (None, [vp]),
    "spb_contingency": (C.c_int, [vp, vp, i64, i32, i32, vp, vp, sz, vp]),
    "spb_kmeans_workspace": (sz, [i32, i32]),
    "spb_kmeans": (C.c_int, [C.c_int, vp, i64, i32, i32, i32, vp, i32, i32, vp, sz, vp, vp,
                             C.POINTER(i32), vp]),
    "spb_assign_workspace": (sz, [i32, i32]),
    "spb_assign_qrcp": (C.c_int, [C.c_int, vp, i64, i32, i32, vp, sz, vp, vp, C.POINTER(f64), vp]),
    "spb_assign_workspace_sharded": (sz, [i32, i32, i32]),
    "spb_assign_qrcp_sharded": (C.c_int, [C.c_int, vp, i64, i32, i32, vp, vp, sz, vp, vp,
                                          C.POINTER(f64), vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load (once) and return the CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        h = C.CDLL(str(LIB_PATH))
        missing = [name for name in _SIGS if not hasattr(h, name)]
        if missing:
            raise ImportError(f"{LIB_PATH} lacks symbols {missing}; rebuild it")
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


_EXC = {
    E_CONTRACT: ContractError,
    E_DOMAIN: DomainError,
    E_COND: ConditioningError,
    E_ASSIGN: AssignmentError,
}


def check(status: int) -> None:
    if status == OK:
        return
    msg = (lib().spb_last_error() or b"").decode(errors="replace")
    if status in _EXC:
        raise _EXC[status](msg)
    if status in (E_SOLVER, E_SOLVER_NOSTATE):
        raise SolverError(msg)
    raise NativeError(f"status {status}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream():
    import torch

    return torch.cuda.current_stream().cuda_stream
