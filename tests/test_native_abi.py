"""CPU checks of the C ABI: the library builds/loads and exports every symbol
declared in include/specpart_b200.h; the ctypes binding covers all of them.
No compute calls (there is no GPU in the build container)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "specpart_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"SPB_API\s+[\w\s\*]*?\b(spb_\w+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for must in ("spb_csr_build", "spb_laplacian_spmm", "spb_lobpcg_solve", "spb_sygv",
                 "spb_assign_qrcp", "spb_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1708_07481_b200 import _native as N

    if not N.LIB_PATH.exists():
        pytest.fail("libspb200.so not built: run __graft_entry__.build()")
    lib = ctypes.CDLL(str(N.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_1708_07481_b200 import _native as N

    assert sorted(N.EXPORTED) == declared_symbols()
    N.lib()  # loads and sets argtypes without touching the device


def test_pure_host_queries():
    from paper_1708_07481_b200 import _native as N

    lib = N.lib()
    assert lib.spb_version() >= 100
    assert lib.spb_csr_build_workspace(1000, 100, N.CSR_SYMMETRIZED) > 2000 * 12
    assert lib.spb_sygv_workspace(63) > 63 * 63 * 8


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_1708_07481_b200 as spb

    with pytest.raises(RuntimeError, match="CUDA device"):
        spb.from_edges([(0, 1)], 2)
