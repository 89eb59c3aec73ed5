"""irls_refine at C2 through ShardedIrlsEngine over a one-rank NCCL
communicator (the multi-GPU step graph), for launch lists."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_04612_b200 import scenes, parallel as P_
from paper_2505_04612_b200.config import HotPathConfig
dev = torch.device("cuda")
sc = scenes.generate(scenes.CONFIGS["c2"], dev)
store = scenes.device_store(sc, dev)
graph, ids = scenes.device_graph(sc, dev)
comm = P_.NcclComm()
for rep in range(2):
    store.reset_active()
    params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
    eng = P_.ShardedIrlsEngine([P_.Shard(store, graph, "fp32")], params, HotPathConfig(), comm=comm)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.run()
    torch.cuda.synchronize()
    print(f"nccl1 irls_refine {1e3 * (time.perf_counter() - t0):.2f} ms")
comm.close()
