"""A few batched align steps on the C3 direction graph (for ncu).
    python tools/tr_one.py [B] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_04612_b200 import translation as T  # noqa: E402
from paper_2505_04612_b200.scenes import translation_graph_c3  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ei, ej, d, _ = translation_graph_c3()
g = T.DirectionGraph(n=2000, edges_i=ei, edges_j=ej, directions=d)


class C:
    translation_lr, translation_steps, translation_inits = 1e-3, steps, B
    adam_beta1, adam_beta2, adam_eps = 0.9, 0.999, 1e-8


dg = T.device_graph(g)
init = np.stack([np.random.default_rng(k).standard_normal((g.n, 3)) for k in range(B)], axis=1)
T._align(dg, init, C, steps)
torch.cuda.synchronize()
def timed(k):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    T._align(dg, init, C, k)
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) * 1e3


t200, t1000 = timed(200), timed(1000)
print(f"B={B}: {t1000 / 1000:.1f} us/step over 1000 steps; marginal {(t1000 - t200) / 800:.1f} us/step; "
      f"fixed per call {t200 - 200 * (t1000 - t200) / 800:.0f} us")
