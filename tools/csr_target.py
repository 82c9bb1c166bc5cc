"""ncu target: the device CSR build (from_edges) of a config's arc list, N times.

    python tools/csr_target.py [c3] [reps]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = CONFIGS[cfg]
edges, _ = generate_dcsbm(spec)
src = torch.from_numpy(np.ascontiguousarray(edges[:, 0])).cuda()
dst = torch.from_numpy(np.ascontiguousarray(edges[:, 1])).cuda()
for _ in range(reps):
    g = spb.from_edges((src, dst), spec.n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g = spb.from_edges((src, dst), spec.n)
e1.record()
torch.cuda.synchronize()
print(f"{cfg}: from_edges {e0.elapsed_time(e1) / 5:.3f} ms")
