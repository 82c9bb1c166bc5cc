"""Host->device strategies for the public API's pageable numpy inputs (C3: 432 MB x0,
160 MB arcs). Prints ms and GB/s per strategy.

    python tools/h2d_bench.py
"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return min(ts), float(np.median(ts))


def main():
    dev = torch.device("cuda", 0)
    x = np.random.default_rng(0).standard_normal((500_000, 108))
    nb = x.nbytes
    dst = torch.empty(x.shape, dtype=torch.float64, device=dev)
    flat = x.reshape(-1)
    pool = ThreadPoolExecutor(16)

    def pageable():
        dst.copy_(torch.from_numpy(x))

    chunk = 32 << 20
    bufs = [torch.empty(chunk // 8, dtype=torch.float64).pin_memory() for _ in range(3)]
    evs = [torch.cuda.Event() for _ in range(3)]
    dflat = dst.view(-1)

    def staged(threads):
        n = flat.size
        per = chunk // 8
        s = torch.cuda.current_stream()
        for i, off in enumerate(range(0, n, per)):
            b = i % 3
            evs[b].synchronize()  # the copy that last used this buffer is done
            m = min(per, n - off)
            hb = bufs[b].numpy()
            if threads > 1:
                step = (m + threads - 1) // threads
                list(pool.map(lambda j: np.copyto(hb[j * step:min(m, (j + 1) * step)],
                                                  flat[off + j * step:off + min(m, (j + 1) * step)]),
                              range(threads)))
            else:
                np.copyto(hb[:m], flat[off:off + m])
            dflat[off:off + m].copy_(bufs[b][:m], non_blocking=True)
            evs[b].record(s)

    def registered():
        cr = torch.cuda.cudart()
        ptr = x.ctypes.data
        assert cr.cudaHostRegister(ptr, nb, 0) == 0
        try:
            dst.copy_(torch.from_numpy(x), non_blocking=True)
            torch.cuda.synchronize()
        finally:
            cr.cudaHostUnregister(ptr)

    for name, fn in [("pageable torch copy", pageable), ("staged 32 MB x3, 1 thread", lambda: staged(1)),
                     ("staged 32 MB x3, 4 threads", lambda: staged(4)),
                     ("staged 32 MB x3, 8 threads", lambda: staged(8)),
                     ("staged 32 MB x3, 16 threads", lambda: staged(16)),
                     ("cudaHostRegister + copy + unregister", registered)]:
        best, med = timeit(fn)
        ok = torch.equal(dst.view(-1)[:1000].cpu(), torch.from_numpy(flat[:1000]))
        print(f"{name:40s} best {best * 1e3:7.1f} ms  median {med * 1e3:7.1f} ms  "
              f"{nb / best / 1e9:6.1f} GB/s  ok={ok}", flush=True)


if __name__ == "__main__":
    main()
