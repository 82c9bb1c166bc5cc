"""Block update out = init + scale * A C (lobpcg.py:436-439) through the C-ABI:
the float32 CUDA-core kernels (mode 0) and the 3xTF32 tensor-core kernel
(mode 1) against a float64 product of the same float32 inputs. Bound: the
error relative to sum_k |a_k||c_k| per output (the float32 dot-product scale)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(mode, a, c, scale, init, ld_out):
    from paper_1708_07481_b200 import _native as N

    L = N.lib()
    n, w = a.shape[0], c.shape[0]
    q = c.shape[1]
    out = torch.full((n, ld_out), float("nan"), dtype=a.dtype, device="cuda")
    wsb = L.spb_block_update_workspace(w, q)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    code = N.F32 if a.dtype == torch.float32 else N.F64
    N.check(L.spb_block_update(code, mode, N.ptr(a), a.stride(0), w, N.ptr(c), c.stride(0), q, scale,
                               N.ptr(init) if init is not None else None,
                               init.stride(0) if init is not None else 0, N.ptr(out), ld_out, n,
                               N.ptr(ws), wsb, N.stream()))
    torch.cuda.synchronize()
    return out[:, :q]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n,w,q", [(1000, 49, 49), (5003, 147, 49), (20000, 108, 108),
                                   (777, 32, 16), (4096, 324, 108), (3000, 200, 256),
                                   (3001, 528, 176), (2048, 176, 144), (1500, 96, 192)])
@pytest.mark.parametrize("with_init", [False, True])
def test_update_accuracy(mode, n, w, q, with_init):
    g = torch.Generator(device="cuda").manual_seed(n + w + q)
    ld = ((w + 7) // 8) * 8
    a_full = torch.randn((n, ld), device="cuda", generator=g, dtype=torch.float32)
    a = a_full[:, :w]
    c = torch.randn((w, q), device="cuda", generator=g, dtype=torch.float64) / np.sqrt(w)
    init = torch.randn((n, ((q + 7) // 8) * 8), device="cuda", generator=g, dtype=torch.float32) \
        if with_init else None
    scale = -1.0 if with_init else 1.0
    got = _run(mode, a_full, c, scale, init, ((q + 7) // 8) * 8)
    c32 = c.float().double()  # the kernels compute with the float32-rounded coefficients
    want = scale * (a.double() @ c32)
    mag = a.double().abs() @ c32.abs()
    if init is not None:
        want = want + init[:, :q].double()
        mag = mag + init[:, :q].double().abs()
    err = ((got.double() - want).abs() / mag).max().item()
    assert torch.isfinite(got).all()
    assert err < (2e-6 if mode == 1 else 1e-6), err


def test_update_in_place_and_f64():
    from paper_1708_07481_b200 import _native as N

    g = torch.Generator(device="cuda").manual_seed(5)
    n, w = 3000, 49
    a = torch.randn((n, 56), device="cuda", generator=g)
    c = torch.randn((w, w), device="cuda", generator=g, dtype=torch.float64)
    want = a[:, :w].double() @ c.float().double()
    L = N.lib()
    wsb = L.spb_block_update_workspace(w, w)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    for mode in (0, 1):
        b = a.clone()
        N.check(L.spb_block_update(N.F32, mode, N.ptr(b), 56, w, N.ptr(c), w, w, 1.0, None, 0,
                                   N.ptr(b), 56, n, N.ptr(ws), wsb, N.stream()))
        torch.cuda.synchronize()
        assert ((b[:, :w].double() - want).abs() / (a[:, :w].double().abs() @ c.abs())).max() < 2e-6
    ad = a.double()
    out = torch.empty_like(ad)
    N.check(L.spb_block_update(N.F64, -1, N.ptr(ad), 56, w, N.ptr(c), w, w, 1.0, None, 0,
                               N.ptr(out), 56, n, N.ptr(ws), wsb, N.stream()))
    torch.cuda.synchronize()
    assert ((out[:, :w] - ad[:, :w] @ c).abs().max() / (ad[:, :w].abs() @ c.abs()).max()) < 1e-14
    with pytest.raises(Exception):
        N.check(L.spb_block_update(N.F64, 1, N.ptr(ad), 56, w, N.ptr(c), w, w, 1.0, None, 0,
                                   N.ptr(out), 56, n, N.ptr(ws), wsb, N.stream()))
