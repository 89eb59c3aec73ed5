"""A few align steps at config 3 sizes (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2505_04612_b200 import translation as T
rng = np.random.default_rng(0)
n, m = 2000, 200_000
c = rng.normal(size=(n, 3))
e = set()
while len(e) < m:
    a = rng.integers(0, n, size=(m, 2))
    for i, j in a:
        if i != j: e.add((min(i, j), max(i, j)))
        if len(e) >= m: break
e = np.array(sorted(e))
d = c[e[:, 1]] - c[e[:, 0]]; d /= np.linalg.norm(d, axis=1, keepdims=True)
g = T.DirectionGraph(n=n, edges_i=e[:, 0], edges_j=e[:, 1], directions=d)
class C:
    translation_lr, translation_steps, translation_inits = 1e-3, 6000, 16
    adam_beta1, adam_beta2, adam_eps = 0.9, 0.999, 1e-8
C.translation_steps = 6
if len(sys.argv) > 1 and sys.argv[1] == "multi":
    T.multi_init_align(g, C, seed=0)
else:
    T.align_centers(g, C, seed=0, steps=9)
torch.cuda.synchronize()
