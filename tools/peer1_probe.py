"""irls_refine at C2 through the fused peer-exchange step over a one-rank
group, vs the single engine."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_04612_b200 import scenes, parallel as P_, epipolar as E
from paper_2505_04612_b200.config import HotPathConfig
dev = torch.device("cuda")
sc = scenes.generate(scenes.CONFIGS["c2"], dev)
store = scenes.device_store(sc, dev)
graph, ids = scenes.device_graph(sc, dev)
comm = P_.PeerComm.local_group(graph.struct(), 1, dev)[0]
for rep in range(3):
    for name in ("single", "peer1"):
        store.reset_active()
        params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
        eng = (E.IrlsEngine(store, graph, params, HotPathConfig()) if name == "single" else
               P_.ShardedIrlsEngine([P_.Shard(store, graph, "fp32")], params, HotPathConfig(), comm=comm))
        torch.cuda.synchronize(); t0 = time.perf_counter()
        eng.run()
        torch.cuda.synchronize()
        print(f"{name} irls_refine {1e3 * (time.perf_counter() - t0):.2f} ms")
comm.close()
