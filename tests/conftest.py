import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_graph():
    return load_golden("graph")


@pytest.fixture(scope="session")
def golden_solve():
    return load_golden("solve")


@pytest.fixture(scope="session")
def golden_partition():
    return load_golden("partition")


@pytest.fixture(scope="session")
def golden_qrcp():
    return load_golden("qrcp")
