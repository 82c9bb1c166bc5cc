"""Device-resident sparse graphs and the matrix-free Laplacian.

Mirrors the public surface of the reference's ``specpart/graph.py``
(``SparseGraph`` graph.py:35-103, ``from_edges`` :135-145, ``empty_graph``
:148-149, ``load_edge_list`` :152-209, ``write_edge_list`` :212-217,
``symmetrize`` :220-236, ``degrees`` :239-250, ``laplacian_apply`` :253-278,
``apply_delta`` :281-297, ``LaplacianOperator`` :300-317) with the data kept on
the GPU:

* the arc list (src, dst[, w]) is held on the device; the symmetrised CSR
  W = A + A' and the degree vector are built from it by the CUDA CSR builder
  (csrc/csr_build.cu) — that is what the eigensolver consumes;
* the directed CSR arrays of the reference (``row_offsets``, ``col_indices``,
  ``weights``) are built on the device on first access and returned as
  read-only numpy arrays, bit-identical to ``specpart.from_edges``.
"""

from __future__ import annotations

import io
from functools import cached_property
from pathlib import Path

import numpy as np
import torch

from . import _h2d
from . import _native as N
from .errors import ContractError, DomainError, ParseError

__all__ = [
    "SparseGraph",
    "LaplacianOperator",
    "from_edges",
    "empty_graph",
    "load_edge_list",
    "write_edge_list",
    "symmetrize",
    "degrees",
    "laplacian_apply",
    "apply_delta",
    "DTYPES",
]

DTYPES = {"float32": (N.F32, torch.float32), "float64": (N.F64, torch.float64)}


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1708_07481_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class _Csr:
    """One device CSR: int32 row_ptr/col, float64 values (+ per-dtype casts)."""

    def __init__(self, row_ptr, col, val, nnz, deg=None):
        self.row_ptr, self.col, self.val, self.nnz, self.deg = row_ptr, col, val, nnz, deg
        self._cast = {}

    def values(self, dtype: str):
        if dtype == "float64":
            return self.val
        if dtype not in self._cast:
            out = torch.empty(max(self.nnz, 1), dtype=torch.float32, device=self.val.device)
            if self.nnz:
                N.check(N.lib().spb_cast(N.ptr(self.val), self.nnz, N.F32, N.ptr(out), N.stream()))
            self._cast[dtype] = out
        return self._cast[dtype]

    def degrees(self, dtype: str):
        if dtype == "float64":
            return self.deg
        key = ("deg", dtype)
        if key not in self._cast:
            n = self.deg.numel()
            out = torch.empty(max(n, 1), dtype=torch.float32, device=self.deg.device)
            if n:
                N.check(N.lib().spb_cast(N.ptr(self.deg), n, N.F32, N.ptr(out), N.stream()))
            self._cast[key] = out
        return self._cast[key]


# Locality ordering for the SpMM (csrc/reorder.cu): used when the gathered X block
# (n x block columns) is too large to stay L2-resident (126 MB L2 on a B200).
ORDER_MIN_BYTES = 64 << 20
ORDER_STEPS = 5
ORDER_SEED = 0x5EED


class _VertexOrder:
    """perm[new] = old from spb_vertex_order on W, and W renumbered by it per dtype
    (spb_csr_permute: every row keeps its entry order, so SpMM rows are bit-identical)."""

    def __init__(self, c: _Csr, n: int):
        L = N.lib()
        dev = c.row_ptr.device
        self.n = n
        self.perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        wsb = L.spb_vertex_order_workspace(n)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        # float32 copies of W and d (the float32 solve's own; the walk computes in
        # float32 either way, the copies only halve its value traffic)
        N.check(L.spb_vertex_order(N.F32, n, N.ptr(c.row_ptr), N.ptr(c.col),
                                   N.ptr(c.values("float32")), N.ptr(c.degrees("float32")),
                                   ORDER_STEPS, ORDER_SEED, N.ptr(ws), wsb, N.ptr(self.perm),
                                   N.stream()))
        self._csr = {}

    def csr(self, c: _Csr, dtype: str):
        """(row_ptr, col, values) of P W P' in the solve dtype."""
        if dtype not in self._csr:
            L = N.lib()
            dev = c.row_ptr.device
            n = self.n
            rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
            col = torch.empty(max(c.nnz, 1), dtype=torch.int32, device=dev)
            tdt = DTYPES[dtype][1]
            val = torch.empty(max(c.nnz, 1), dtype=tdt, device=dev)
            inv = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            wsb = L.spb_csr_permute_workspace(n)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            N.check(L.spb_csr_permute(DTYPES[dtype][0], n, N.ptr(c.row_ptr), N.ptr(c.col),
                                      N.ptr(c.values(dtype)), None, N.ptr(self.perm), N.ptr(ws),
                                      wsb, N.ptr(inv), N.ptr(rp), N.ptr(col), N.ptr(val), None,
                                      N.stream()))
            self._csr[dtype] = (rp, col, val)
        return self._csr[dtype]

    def gather(self, v: torch.Tensor) -> torch.Tensor:
        """out[i] = v[perm[i]] for a device vector of the solve dtype."""
        out = torch.empty_like(v)
        code = N.F32 if v.dtype == torch.float32 else N.F64
        if self.n:
            N.check(N.lib().spb_permute_rows(code, N.ptr(v), 1, code, N.ptr(out), 1, self.n, 1,
                                             N.ptr(self.perm), 0, N.stream()))
        return out


def _build_csr(src, dst, w, m, n, mode) -> _Csr:
    dev = _device()
    L = N.lib()
    cap = max(1, (2 if mode == N.CSR_SYMMETRIZED else 1) * m)
    ws_bytes = L.spb_csr_build_workspace(m, n, mode)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    row_ptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    val = torch.empty(cap, dtype=torch.float64, device=dev)
    deg = torch.empty(max(n, 1), dtype=torch.float64, device=dev) if mode != N.CSR_DIRECTED else None
    nnz = N.C.c_int64(0)
    N.check(L.spb_csr_build(N.ptr(src), N.ptr(dst), N.ptr(w), m, n, mode, N.ptr(ws), ws_bytes,
                            N.ptr(row_ptr), N.ptr(col), N.ptr(val), N.ptr(deg),
                            N.C.byref(nnz), N.stream()))
    del ws
    return _Csr(row_ptr, col, val, int(nnz.value), deg)


class SparseGraph:
    """Directed weighted graph; immutable; arcs and CSRs live on the GPU.

    ``is_symmetric`` records that the stored arcs already form W (the
    Laplacian then skips the transpose term), as in graph.py:35-45.
    """

    def __init__(self, n_vertices: int, src, dst, weights=None, is_symmetric: bool = False):
        self.n_vertices = int(n_vertices)
        self.is_symmetric = bool(is_symmetric)
        self._src, self._dst, self._w = src, dst, weights  # device int64 / int64 / f64|None
        self._m = int(src.numel())

    # ---- device structures -------------------------------------------------
    @cached_property
    def _w_csr(self) -> _Csr:
        mode = N.CSR_AS_SYMMETRIC if self.is_symmetric else N.CSR_SYMMETRIZED
        return _build_csr(self._src, self._dst, self._w, self._m, self.n_vertices, mode)

    @cached_property
    def _a_csr(self) -> _Csr:
        return _build_csr(self._src, self._dst, self._w, self._m, self.n_vertices, N.CSR_DIRECTED)

    def device_csr(self):
        """(row_ptr, col, val64, nnz) of the symmetrised CSR W on the device."""
        c = self._w_csr
        return c.row_ptr, c.col, c.val, c.nnz

    def device_degrees(self):
        return self._w_csr.deg[: self.n_vertices]

    @cached_property
    def _vertex_order(self) -> _VertexOrder:
        return _VertexOrder(self._w_csr, self.n_vertices)

    # ---- reference-shaped host views (graph.py:35-103) ---------------------
    @cached_property
    def _host_a(self):
        c = self._a_csr
        offs = c.row_ptr.cpu().numpy().astype(np.int64)
        cols = c.col[: c.nnz].cpu().numpy().astype(np.int64)
        w = c.val[: c.nnz].cpu().numpy().astype(np.float64)
        for arr in (offs, cols, w):
            arr.setflags(write=False)
        return offs, cols, w

    @property
    def row_offsets(self) -> np.ndarray:
        return self._host_a[0]

    @property
    def col_indices(self) -> np.ndarray:
        return self._host_a[1]

    @property
    def weights(self) -> np.ndarray:
        return self._host_a[2]

    @property
    def nnz(self) -> int:
        return int(self._a_csr.nnz)

    def to_csr(self):
        import scipy.sparse as sp

        n = self.n_vertices
        return sp.csr_matrix((self.weights, self.col_indices, self.row_offsets), shape=(n, n))

    def edge_arrays(self):
        """Return (src, dst, weight) arrays of the stored directed arcs (graph.py:93-96)."""
        src = np.repeat(np.arange(self.n_vertices), np.diff(self.row_offsets))
        return src, self.col_indices.copy(), self.weights.copy()

    def to_dense(self) -> np.ndarray:
        return self.to_csr().toarray()

    def __repr__(self):
        return (f"SparseGraph(n_vertices={self.n_vertices}, arcs={self._m}, "
                f"is_symmetric={self.is_symmetric})")


def _coerce_edges(edges, weights=None):
    """Normalise edge input to (src, dst, w|None) host arrays (graph.py:106-132)."""
    if isinstance(edges, torch.Tensor):
        edges = edges.detach().cpu().numpy()
    if isinstance(edges, np.ndarray) and edges.ndim == 2:
        arr = edges
    else:
        arr = np.asarray(list(edges), dtype=np.float64)
        if arr.size == 0:
            arr = arr.reshape(0, 2)
    if arr.ndim != 2 or arr.shape[1] not in (2, 3):
        raise ContractError("edges must be (m, 2) or (m, 3)")
    src = np.ascontiguousarray(arr[:, 0], dtype=np.int64)
    dst = np.ascontiguousarray(arr[:, 1], dtype=np.int64)
    if weights is not None:
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if w.shape != (src.size,):
            raise ContractError("weights length does not match edges")
    elif arr.shape[1] == 3:
        w = np.ascontiguousarray(arr[:, 2], dtype=np.float64)
    else:
        w = None
    if w is not None and np.any(w < 0):
        raise DomainError("negative edge weight")
    return src, dst, w


def _to_device(a, dtype):
    if a is None:
        return None
    t = torch.from_numpy(np.ascontiguousarray(a))
    if t.numel() and torch.cuda.is_available():
        t = t.pin_memory() if t.numel() * t.element_size() >= (1 << 20) else t
    return t.to(device=_device(), dtype=dtype, non_blocking=True)


def from_edges(edges, n: int, weights=None, *, symmetric: bool = False) -> SparseGraph:
    """Graph from directed edges; duplicates summed, self-loops dropped (graph.py:135-145).

    ``edges`` may also be a pair of device int64 tensors ``(src, dst)``.
    """
    n = int(n)
    src, dst, w = _device_arcs(edges, n, weights)
    g = SparseGraph(n, src, dst, w, is_symmetric=symmetric)
    g._w_csr  # build W eagerly: the hot path needs it; errors surface here
    return g


def _device_arcs(edges, n: int, weights=None):
    """Arc arrays (src, dst int64, w float64|None) on the device (graph.py:106-132)."""
    if isinstance(edges, tuple) and len(edges) == 2 and isinstance(edges[0], torch.Tensor):
        src, dst = (e.to(device=_device(), dtype=torch.int64) for e in edges)
        w = None if weights is None else torch.as_tensor(weights, dtype=torch.float64, device=_device())
        if w is not None and w.numel() and bool((w < 0).any()):
            raise DomainError("negative edge weight")
    elif (weights is None and isinstance(edges, np.ndarray) and edges.ndim == 2
          and edges.shape[1] == 2 and edges.dtype == np.int64 and edges.flags.c_contiguous
          and edges.shape[0] > 0):
        # fast path: one H2D copy of the arc block (large pageable blocks through a
        # multi-threaded pinned ring, _h2d.py), columns split on the device; the
        # endpoint range check happens in the CSR build's validation pass (same
        # DomainError)
        dev = _h2d.to_device(edges, _device())
        src, dst, w = dev[:, 0].contiguous(), dev[:, 1].contiguous(), None
    else:
        hs, hd, hw = _coerce_edges(edges, weights)
        if hs.size and (min(hs.min(), hd.min()) < 0 or max(hs.max(), hd.max()) >= n):
            raise DomainError("edge endpoint out of range")
        src, dst, w = _to_device(hs, torch.int64), _to_device(hd, torch.int64), _to_device(hw, torch.float64)
    return src, dst, w


def empty_graph(n: int = 0) -> SparseGraph:
    z = torch.empty(0, dtype=torch.int64, device=_device())
    return SparseGraph(n, z, z.clone(), None)


def _read_all(source) -> bytes:
    if isinstance(source, (str, Path)):
        with open(source, "rb") as fh:
            return fh.read()
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    data = source.read()
    return data.encode("utf-8") if isinstance(data, str) else bytes(data)


def _parse_native(data: bytes, base: int, threads: int = 0):
    """Native multithreaded parse (csrc/ingest.cu); None when a line needs the
    reference's own rules (errors, or syntax outside the fast path)."""
    L = N.lib()
    m, mx, hw, bad = N.C.c_int64(0), N.C.c_int64(0), N.C.c_int32(0), N.C.c_int64(0)
    h = N.C.c_void_p()
    st = L.spb_edge_list_parse(data, len(data), base, threads, N.C.byref(m), N.C.byref(mx),
                               N.C.byref(hw), N.C.byref(bad), N.C.byref(h))
    if st == N.E_PARSE:
        return None
    N.check(st)
    src = np.empty(m.value, dtype=np.int64)
    dst = np.empty(m.value, dtype=np.int64)
    w = np.empty(m.value, dtype=np.float64) if hw.value else None
    N.check(L.spb_edge_list_fetch(h, src.ctypes.data, dst.ctypes.data,
                                  w.ctypes.data if w is not None else None))
    return src, dst, w, int(mx.value)


def _parse_python(fh, base: int):
    """The reference's line loop (graph.py:171-198): exact errors for any input."""
    src, dst, wts = [], [], []
    any_w = False
    max_idx = -1
    for line_no, raw in enumerate(fh, start=1):
        if isinstance(raw, bytes):
            raw = raw.decode("utf-8")
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) not in (2, 3):
            raise ParseError(f"expected 2 or 3 fields, got {len(parts)}", line_no)
        try:
            u = int(parts[0]) - base
            v = int(parts[1]) - base
            w = float(parts[2]) if len(parts) == 3 else 1.0
        except ValueError as exc:
            raise ParseError(str(exc), line_no) from None
        if u < 0 or v < 0:
            raise ParseError(f"vertex index below base {base}", line_no)
        if w < 0:
            raise DomainError(f"line {line_no}: negative weight {w}")
        any_w |= len(parts) == 3
        src.append(u)
        dst.append(v)
        wts.append(w)
        max_idx = max(max_idx, u, v)
    return (np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64),
            np.asarray(wts, dtype=np.float64) if (wts and any_w) else None, max_idx)


def load_edge_list(source, base: int = 1, num_vertices: int | None = None) -> SparseGraph:
    """Tab-separated ``src dst [weight]`` reader (graph.py:152-209 semantics).

    Parsed by the native multithreaded reader; a file containing a line it does
    not accept is re-read with the reference's loop, which raises the same
    ParseError / DomainError (with line number) the reference raises.
    """
    if base not in (0, 1):
        raise DomainError("base must be 0 or 1")
    data = _read_all(source)
    parsed = _parse_native(data, base)
    if parsed is None:
        parsed = _parse_python(io.BytesIO(data), base)
    src, dst, w, max_idx = parsed
    n = max_idx + 1
    if num_vertices is not None:
        if num_vertices < n:
            raise DomainError(f"num_vertices={num_vertices} below max index {max_idx}")
        n = num_vertices
    edges = np.column_stack([src, dst]) if src.size else np.empty((0, 2), dtype=np.int64)
    return from_edges(edges, n, weights=w if src.size else None)


def write_edge_list(g: SparseGraph, path, base: int = 1) -> None:
    src, dst, w = g.edge_arrays()
    with open(path, "w", encoding="utf-8") as fh:
        for u, v, x in zip(src, dst, w):
            fh.write(f"{u + base}\t{v + base}\t{format(x, '.12g')}\n")


def symmetrize(g: SparseGraph, mode: str = "algebraic") -> SparseGraph:
    """Graph holding W = A + A' (graph.py:220-236), built on the device."""
    if mode not in ("algebraic", "logical"):
        raise DomainError(f"unknown symmetrize mode {mode!r}")
    # always A + A' of the stored arcs (graph.py:227), also when g.is_symmetric: its
    # arcs are W itself, so symmetrize() doubles them, as the reference does
    c = _build_csr(g._src, g._dst, g._w, g._m, g.n_vertices, N.CSR_SYMMETRIZED)
    row_ptr, col, val, nnz = c.row_ptr, c.col, c.val, c.nnz
    rows = torch.repeat_interleave(
        torch.arange(g.n_vertices, device=row_ptr.device, dtype=torch.int64),
        (row_ptr[1:] - row_ptr[:-1]).to(torch.int64))
    dst = col[:nnz].to(torch.int64)
    w = val[:nnz].clone() if mode == "algebraic" else torch.ones(nnz, dtype=torch.float64, device=val.device)
    return SparseGraph(g.n_vertices, rows, dst, w, is_symmetric=True)


def degrees(g: SparseGraph) -> np.ndarray:
    """Row sums of W (graph.py:239-250) as a host float64 array."""
    if g.n_vertices == 0:
        return np.zeros(0)
    return g.device_degrees().cpu().numpy().copy()


def _as_device_block(x, dtype=torch.float64):
    if isinstance(x, torch.Tensor):
        return x.to(device=_device(), dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(_device(), dtype=dtype)


def _spmm(g: SparseGraph, deg_t, x_t, y_t, dtype: str):
    row_ptr, col, _, _ = g.device_csr()
    code = DTYPES[dtype][0]
    vals = g._w_csr.values(dtype)
    n = g.n_vertices
    N.check(N.lib().spb_laplacian_spmm(code, 0, n, N.ptr(row_ptr), N.ptr(col), N.ptr(vals),
                                       N.ptr(deg_t), N.ptr(x_t), x_t.stride(0), x_t.shape[1],
                                       N.ptr(y_t), y_t.stride(0), N.stream()))


def laplacian_apply(g: SparseGraph, d, x, out=None):
    """Y = diag(d) X - (A + A') X without forming L (graph.py:253-278).

    Host numpy in / out (float64). Device tensors are accepted and returned
    on the device.
    """
    on_dev = isinstance(x, torch.Tensor) and x.is_cuda
    d_np = d.detach().cpu().numpy() if isinstance(d, torch.Tensor) else np.asarray(d, dtype=np.float64)
    if d_np.shape != (g.n_vertices,):
        raise ContractError("degree vector length does not match graph")
    xs = x if on_dev else np.asarray(x, dtype=np.float64)
    squeeze = xs.ndim == 1
    if xs.ndim not in (1, 2) or xs.shape[0] != g.n_vertices:
        rows = xs.shape[0] if xs.ndim else 0
        raise ContractError(f"multivector has {rows} rows, graph has {g.n_vertices}")
    xt = _as_device_block(xs.reshape(g.n_vertices, -1) if not on_dev else xs.reshape(g.n_vertices, -1))
    yt = torch.empty_like(xt)
    if g.n_vertices and xt.shape[1]:
        dt = torch.from_numpy(np.ascontiguousarray(d_np)).to(xt.device)
        _spmm(g, dt, xt, yt, "float64")
    if on_dev:
        res = yt[:, 0] if squeeze else yt
        if out is not None:
            out.copy_(res)
            return out
        return res
    res = yt.cpu().numpy()
    res = res[:, 0] if squeeze else res
    if out is not None:
        out[...] = res
        return out
    return res


def apply_delta(g: SparseGraph, edges, new_n: int, weights=None) -> SparseGraph:
    """Add an edge delta and grow the vertex set (graph.py:281-297), on the device."""
    if new_n < g.n_vertices:
        raise DomainError("new_n below current vertex count")
    hs, hd, hw = _coerce_edges(edges, weights)
    if hs.size and (min(hs.min(), hd.min()) < 0 or max(hs.max(), hd.max()) >= new_n):
        raise DomainError("delta endpoint out of range")
    # cumulative arc list: old arcs first (already summed order is irrelevant
    # for integer weights; float weights are summed in arc order)
    src = torch.cat([g._src, _to_device(hs, torch.int64)]) if hs.size else g._src
    dst = torch.cat([g._dst, _to_device(hd, torch.int64)]) if hs.size else g._dst
    if g._w is None and hw is None:
        w = None
    else:
        old = g._w if g._w is not None else torch.ones(g._m, dtype=torch.float64, device=src.device)
        new = _to_device(hw, torch.float64) if hw is not None else torch.ones(hs.size, dtype=torch.float64, device=src.device)
        w = torch.cat([old, new]) if hs.size else old
    out = SparseGraph(new_n, src, dst, w)
    out._w_csr
    return out


class LaplacianOperator:
    """Matrix-free handle for L = D - (A + A') (graph.py:300-317), device-resident.

    ``apply`` accepts host numpy blocks (float64 round trip) or device tensors.
    The eigensolver uses the device CSR directly (no host round trip).
    """

    def __init__(self, g: SparseGraph, d=None, *, vertex_order="auto"):
        if vertex_order not in ("auto", True, False):
            raise ContractError("vertex_order must be 'auto', True or False")
        self.graph = g
        self.n = g.n_vertices
        self.vertex_order = vertex_order
        self._deg_perm = {}
        if d is None:
            self._deg64 = g.device_degrees() if self.n else torch.zeros(1, dtype=torch.float64, device=_device())
            self._own_deg = False
        else:
            self._deg64 = _as_device_block(np.asarray(d, dtype=np.float64).reshape(-1, 1)).reshape(-1)
            self._own_deg = True
        if self.n:
            mx = N.C.c_double(0.0)
            N.check(N.lib().spb_max_f64(N.ptr(self._deg64), self.n, N.C.byref(mx), N.stream()))
            self.scale_hint = float(mx.value)
        else:
            self.scale_hint = 1.0
        self._deg_cast = {}

    @property
    def degrees(self) -> np.ndarray:
        return self._deg64[: self.n].cpu().numpy()

    def device_degrees(self, dtype: str):
        if dtype == "float64":
            return self._deg64
        if dtype not in self._deg_cast:
            out = torch.empty(max(self.n, 1), dtype=torch.float32, device=self._deg64.device)
            if self.n:
                N.check(N.lib().spb_cast(N.ptr(self._deg64), self.n, N.F32, N.ptr(out), N.stream()))
            self._deg_cast[dtype] = out
        return self._deg_cast[dtype]

    def uses_vertex_order(self, cols: int, dtype: str) -> bool:
        """Whether a solve with ``cols`` block columns runs in the locality order:
        'auto' when the gathered X block (n x cols) would not stay L2-resident."""
        if self.vertex_order == "auto":
            esz = 4 if dtype == "float32" else 8
            return self.n * cols * esz >= ORDER_MIN_BYTES
        return bool(self.vertex_order) and self.n > 0

    def native(self, dtype: str, cols: int | None = None) -> N.Operator:
        """Operator handle for the device solver; with ``cols`` (the block width)
        the CSR may be the locality-ordered one (op.perm set, see reorder.cu)."""
        op = N.Operator()
        op.kind = N.OP_LAPLACIAN
        op.n = self.n
        op.dense = None
        op.scale_hint = self.scale_hint
        if cols is not None and self.uses_vertex_order(cols, dtype):
            order = self.graph._vertex_order
            row_ptr, col, val = order.csr(self.graph._w_csr, dtype)
            if dtype not in self._deg_perm:
                self._deg_perm[dtype] = order.gather(self.device_degrees(dtype)[: max(self.n, 1)])
            deg = self._deg_perm[dtype]
            op.perm = N.ptr(order.perm)
            op._keep = (row_ptr, col, val, deg, order.perm)
        else:
            row_ptr, col, _, _ = self.graph.device_csr()
            val = self.graph._w_csr.values(dtype)
            deg = self.device_degrees(dtype)
            op.perm = None
            op._keep = (row_ptr, col)
        op.row_ptr = N.ptr(row_ptr)
        op.col = N.ptr(col)
        op.val = N.ptr(val)
        op.deg = N.ptr(deg)
        return op

    def apply(self, x, out=None):
        return laplacian_apply(self.graph, self._deg64[: self.n], x, out=out)

    __call__ = apply
