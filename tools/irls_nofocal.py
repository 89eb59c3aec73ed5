"""irls_refine at C2 with and without focal refinement (camera role cost)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_04612_b200 import scenes, epipolar as E
from paper_2505_04612_b200.config import HotPathConfig
dev = torch.device("cuda")
sc = scenes.generate(scenes.CONFIGS["c2"], dev)
store = scenes.device_store(sc, dev)
for rf in (True, False):
    graph, ids = scenes.device_graph(sc, dev, refine_focal=rf)
    cfg = HotPathConfig(refine_focal=rf)
    for rep in range(2):
        store.reset_active()
        params = torch.as_tensor(scenes.initial_params(sc, ids, refine_focal=rf), device=dev)
        eng = E.IrlsEngine(store, graph, params, cfg)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        eng.run()
        torch.cuda.synchronize()
        print(f"refine_focal={rf}: irls_refine {1e3 * (time.perf_counter() - t0):.2f} ms")
