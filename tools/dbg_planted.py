import sys, numpy as np
sys.path.insert(0, '.')
import paper_1708_07481_b200 as spb
from paper_1708_07481_b200.dcsbm import DcsbmSpec, generate_dcsbm
spec = DcsbmSpec(n=900, blocks=4, arcs=18000, alpha=30.0, ratio=30.0, seed=2)
e, truth = generate_dcsbm(spec)
g = spb.from_edges(e, spec.n)
hist = []
def cb(it, th, nr):
    hist.append((it, th.copy(), nr.copy()))
l = 6
x0 = np.random.default_rng(0).standard_normal((spec.n, l))
op = spb.LaplacianOperator(g) if hasattr(spb, 'LaplacianOperator') else None
import os
st = spb.lobpcg_solve(op, x0, spb.SolverConfig(block_size=6, tol=1e-6, max_iter=300, seed=0), n_converge=5, callback=cb, precision=os.environ.get("PREC", "float32"))
for it, th, nr in hist[54:140:4]:
    print(it, np.array2string(th[:3], precision=6), np.array2string(nr.max(keepdims=True), precision=3))
print("iters", st.iterations, getattr(st, "work_blocks", None))
