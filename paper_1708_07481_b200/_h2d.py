"""Host -> device copies of the public API's pageable numpy inputs.

A pageable ``cudaMemcpy`` runs at ~11 GB/s on the B200 hosts (the driver stages it
through its own pinned buffer on one thread). Large inputs (the C3 x0 block is
432 MB, its arc list 160 MB) go through a ring of three 32 MB pinned buffers from
torch's caching host allocator instead: the next chunk is copied into a free buffer
by several host threads while the previous chunk's DMA runs (34 GB/s measured,
tools/h2d_bench.py). The returned tensor is ordered on the current stream.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

_CHUNK = 32 << 20
_SMALL = 16 << 20
_THREADS = max(1, min(8, os.cpu_count() or 1))
_pool: ThreadPoolExecutor | None = None


def _executor() -> ThreadPoolExecutor:
    global _pool
    if _pool is None:
        _pool = ThreadPoolExecutor(_THREADS, thread_name_prefix="spb-h2d")
    return _pool


def to_device(arr: np.ndarray, device, dtype=None) -> torch.Tensor:
    """Copy a C-contiguous numpy array to ``device``; with ``dtype`` (a numpy dtype)
    the host threads convert while staging (round to nearest, as numpy's astype), so
    only the converted bytes cross the link."""
    if dtype is not None and np.dtype(dtype) != arr.dtype:
        if arr.nbytes < _SMALL or not arr.flags.c_contiguous:
            return torch.from_numpy(arr.astype(dtype)).to(device, non_blocking=True)
        return _staged(arr, device, np.dtype(dtype))
    src = torch.from_numpy(arr)
    if arr.nbytes < _SMALL or not arr.flags.c_contiguous:
        return src.to(device, non_blocking=True)
    return _staged(arr, device, arr.dtype)


def _staged(arr: np.ndarray, device, dtype: np.dtype) -> torch.Tensor:
    out = torch.empty(arr.shape, dtype=torch.from_numpy(np.empty(0, dtype)).dtype, device=device)
    esz_out = dtype.itemsize
    flat = arr.reshape(-1)
    dflat = out.view(-1).view(torch.uint8)
    stream = torch.cuda.current_stream(device)
    bufs = [torch.empty(_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
    done = [None, None, None]
    pool = _executor()
    per = _CHUNK // esz_out  # elements per chunk
    n = flat.size
    for i, off in enumerate(range(0, n, per)):
        b = i % 3
        if done[b] is not None:
            done[b].synchronize()  # the DMA that last read this buffer has finished
        m = min(per, n - off)
        hb = bufs[b].numpy().view(dtype)
        step = -(-m // _THREADS)
        list(pool.map(lambda j: np.copyto(hb[j * step:min(m, (j + 1) * step)],
                                          flat[off + j * step:off + min(m, (j + 1) * step)],
                                          casting="unsafe"),
                      range(_THREADS)))
        dflat[off * esz_out:(off + m) * esz_out].copy_(bufs[b][:m * esz_out], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        done[b] = ev
    return out
