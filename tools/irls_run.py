"""One irls_refine schedule at a BASELINE config on device-generated data
(for ncu launch lists / step-kernel profiling)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_04612_b200 import scenes, epipolar as E
from paper_2505_04612_b200.config import HotPathConfig

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
use_graph = (sys.argv[3] != "nograph") if len(sys.argv) > 3 else True
dev = torch.device("cuda")
sc = scenes.generate(scenes.CONFIGS[cfgname], dev)
store = scenes.device_store(sc, dev)
graph, ids = scenes.device_graph(sc, dev)
for rep in range(2):
    store.reset_active()
    params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
    eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision=prec, use_graph=use_graph)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    l1 = eng.run()
    torch.cuda.synchronize()
    print(f"{cfgname} {prec} graph={use_graph} irls_refine {time.perf_counter() - t0:.4f}s l1 {l1}")
