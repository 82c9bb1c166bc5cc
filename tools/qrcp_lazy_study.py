"""Study: how many QRCP columns would a lazy (deferred) downdate ever touch at C3?

Runs the C3 partition on the device, takes the k-column embedding, and with scipy's
dgeqp3 R factor computes every column's partial norm at every step. For a deferral
rule "defer when norm < alpha * pivot norm of this step" it reports the fraction of
column-steps the per-step pass would still read and how many deferred columns come
back (bound >= a later pivot norm)."""
import sys
from pathlib import Path

import numpy as np
import scipy.linalg as sl
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1708_07481_b200 as spb  # noqa: E402
from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm  # noqa: E402

cfgn = sys.argv[1] if len(sys.argv) > 1 else "c3"
spec = CONFIGS[cfgn]
edges, _ = generate_dcsbm(spec)
k = spec.blocks
l = spb.block_size_for(k)
x0 = np.random.default_rng(0).standard_normal((spec.n, l))
g = spb.from_edges(edges, spec.n)
cfg = spb.SolverConfig(block_size=l, tol=bench.golden_tol(cfgn) or 1e-12, max_iter=30, seed=0)
part, st, _ = spb.partition_static(g, cfg, k, fix_k=True, x0=x0, precision="float32")
X = st.vectors[:, :k].astype(np.float64)
R, piv = sl.qr(X.T, mode="r", pivoting=True)
R = R[:k]
n = X.shape[0]
# partial norms: column c (original index piv[c] order) at step j = ||R[j:, c]||
sq = R ** 2
tail = np.cumsum(sq[::-1], axis=0)[::-1]  # tail[j, c] = sum_{i >= j} R[i, c]^2
pn = np.sqrt(tail)  # k x n
pv = np.abs(np.diag(R))
print("pivot norms: first", pv[:3], "last", pv[-3:], "min", pv.min())
for alpha in (0.9, 0.7, 0.5, 0.3):
    reads = 0
    back = 0
    deferred = np.zeros(n, dtype=bool)
    bound = np.zeros(n)
    for j in range(k):
        active = ~deferred
        reads += active.sum()
        # deferred columns whose bound reaches this step's pivot norm come back
        ret = deferred & (bound >= pv[j])
        back += ret.sum()
        deferred &= ~ret
        # after this step's downdate (norm at step j+1), defer the small ones
        if j + 1 < k:
            nj = pn[j + 1]
            newd = (~deferred) & (nj < alpha * pv[j]) & (np.arange(n) > j)
            deferred |= newd
            bound[newd] = nj[newd]
    print(f"alpha {alpha}: column reads {reads / (k * n):.3f} of the full passes, "
          f"returns {back} ({back / n:.4f} of n)")
