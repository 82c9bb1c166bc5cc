"""Host -> device copies of the public API's pageable numpy inputs.

A pageable ``cudaMemcpy`` runs at ~11 GB/s on the B200 hosts (the driver stages it
through its own pinned buffer on one thread). Large inputs (the C3 x0 block is
432 MB, its arc list 160 MB) go through a pinned ring from torch's caching host
allocator instead, filled by several native host threads that each own their chunks
and ring slots (csrc/h2d.cu; tools/stage_bench.py, tools/h2d_bench.py). The
returned tensor is ordered on the current stream.
"""

from __future__ import annotations

import os
import threading

import numpy as np
import torch

_SMALL = 16 << 20
_THREADS = max(1, min(12, os.cpu_count() or 1))  # 8: 8.9 ms, 12: 7.2 ms, 16: 7.4 ms for the C3 x0


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


_ring: dict = {}
_ring_lock = threading.Lock()  # one staged upload at a time shares the pinned ring


def _staged(arr: np.ndarray, device, dtype: np.dtype) -> torch.Tensor:
    """spb_h2d_staged (csrc/h2d.cu): _THREADS host threads, each copying (or narrowing
    float64 -> float32) its chunks into its own slots of a pinned ring and enqueueing the
    DMAs on the current stream; the ring comes from torch's caching host allocator."""
    from . import _native as N

    out = torch.empty(arr.shape, dtype=torch.from_numpy(np.empty(0, dtype)).dtype, device=device)
    L = N.lib()
    narrow = arr.dtype == np.float64 and dtype == np.float32
    if arr.dtype != dtype and not narrow:
        return torch.from_numpy(arr.astype(dtype)).to(device, non_blocking=True)
    need = int(L.spb_h2d_ring_bytes(_THREADS))
    with _ring_lock, torch.cuda.device(device):
        ring = _ring.get(need)
        if ring is None:
            ring = _ring[need] = torch.empty(need, dtype=torch.uint8, pin_memory=True)
        N.check(L.spb_h2d_staged(arr.ctypes.data, arr.size, arr.dtype.itemsize, dtype.itemsize,
                                 out.data_ptr(), ring.data_ptr(), need, _THREADS,
                                 torch.cuda.current_stream(device).cuda_stream))
    return out
