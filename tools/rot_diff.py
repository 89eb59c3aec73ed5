import sys, numpy as np
sys.path.insert(0, "/root/repo")
from tests.test_rotation_gpu import _Graph, _Cfg
import paper_2505_04612_b200.rotation as Rm
g = dict(np.load("/root/repo/tests/golden/golden_rotation.npz"))
for k in range(3):
    pre = f"r{k}_"
    graph = _Graph(int(g[pre + "n"][0]), g[pre + "ei"], g[pre + "ej"], g[pre + "rel"])
    out, hist = Rm.refine_rotations(g[pre + "init"], graph, _Cfg(g[pre + "steps"][0], g[pre + "cfg"]))
    ref = g[pre + "hist"]; h = np.array(hist)
    rel = np.abs(h - ref) / np.abs(ref)
    print(k, [f"{s}:{rel[s]:.1e}" for s in [0, 1, 5, 10, 50, 100, 200, 500, 1000, len(ref) - 1] if s < len(ref)])
