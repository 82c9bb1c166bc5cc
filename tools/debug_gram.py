import sys
import numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_gram import _gram

def probe(n, p, q, k, a, b):
    u = np.zeros((n, p), np.float32); v = np.zeros((n, q), np.float32)
    u[k, a] = 1.0; v[k, b] = 1.0
    g = _gram(u, v, 1)
    nz = np.argwhere(np.abs(g) > 1e-6)
    return [tuple(x) + (float(g[tuple(x)]),) for x in nz[:6]]

n, p, q = 32, 128, 64
for (k, a, b) in [(0, 0, 0), (0, 1, 0), (0, 0, 1), (0, 5, 3), (0, 33, 0), (0, 0, 33), (1, 0, 0), (1, 2, 3), (3, 7, 9), (8, 0, 0), (9, 4, 4), (0, 70, 40), (15, 100, 50)]:
    print((k, a, b), '->', probe(n, p, q, k, a, b), flush=True)
rng = np.random.default_rng(0)
u = rng.standard_normal((64, 128)).astype(np.float32); v = rng.standard_normal((64, 64)).astype(np.float32)
g = _gram(u, v, 1); ex = u.T.astype(np.float64) @ v
print('rand err', np.abs(g-ex).max())
