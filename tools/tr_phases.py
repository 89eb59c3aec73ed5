"""multi_init_align at C3 split into its phases: the batched 16-start
descent (init_runs) and the merge + final single-run descent."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_04612_b200 import translation as T
from paper_2505_04612_b200.scenes import translation_graph_c3
n, m = 2000, 200_000
ei, ej, d, _ = translation_graph_c3(n, m)
g = T.DirectionGraph(n=n, edges_i=ei, edges_j=ej, directions=d)
class C:
    translation_lr, translation_steps, translation_inits = 1e-3, 6000, 16
    adam_beta1, adam_beta2, adam_eps = 0.9, 0.999, 1e-8
dg = T.device_graph(g)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    runs = T.init_runs(g, C, 0, range(16), dg)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    c, loss = T.merge_and_finish(g, C, runs, dg)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"batched 16 x 6000: {t1 - t0:.3f} s ({1e6 * (t1 - t0) / 6000:.1f} us/step); "
          f"merge + final 6000: {t2 - t1:.3f} s ({1e6 * (t2 - t1) / 6000:.1f} us/step)")
