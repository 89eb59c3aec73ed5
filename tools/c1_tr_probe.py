"""C1 translation: one 3-run 6000-step descent (translation._align) timed
with CUDA events and wall clock, repeated; A/B the cluster-persistent path
with FM_TR_NOCLUSTER=1 / FM_TRC_R / FM_TRC_CLUSTER."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2505_04612_b200 import epipolar as E, translation as T
from paper_2505_04612_b200.config import HotPathConfig
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g, pairs, graph = bench.c1_problem(E.EpipolarPair, T.DirectionGraph)
dg = T.device_graph(graph)
cfg = HotPathConfig()
init = np.stack([np.random.default_rng(k).standard_normal((graph.n, 3)) for k in range(3)], axis=1)
ev, wall = [], []
for r in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record()
    c, loss = T._align(dg, init, cfg, cfg.translation_steps)
    b.record()
    torch.cuda.synchronize()
    wall.append(time.perf_counter() - t0)
    ev.append(a.elapsed_time(b) / 1e3)
print("event ms", " ".join(f"{1e3 * t:.1f}" for t in ev), "| wall ms", " ".join(f"{1e3 * t:.1f}" for t in wall),
      "| loss", loss)
