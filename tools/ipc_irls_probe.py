"""Two processes on one GPU: sharded irls_refine (config 1, short epochs)
over PeerComm (CUDA IPC between the processes) vs the two-shard engine in
one process.  Prints whether both ranks match it bitwise."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
from paper_2505_04612_b200 import parallel as P_
from tests.helpers import Cfg
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
dev = torch.device("cuda")
g = dict(np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "golden_config1.npz")))
lengths = g["c1_len"].astype(np.int64); ij = g["c1_ij"].astype(np.int64)
x1 = np.column_stack([g["c1_x1"].astype(np.float64), np.ones(len(g["c1_x1"]))])
x2 = np.column_stack([g["c1_x2"].astype(np.float64), np.ones(len(g["c1_x2"]))])
R = g["c1_R_in"]
p0 = np.concatenate([np.concatenate([R[:, :, 0], R[:, :, 1]], 1).ravel(), g["c1_c_in"].ravel(), [0.0]])
n = int(ij.max()) + 1
cfg = Cfg(epipolar_epoch_steps=10)
bounds = P_.partition_pairs(lengths, world)
sh = P_.make_shards(x1, x2, lengths, ij, np.zeros_like(ij), n, 1, True, bounds, dev, ranks=[rank])
comm = P_.PeerComm.from_process_group(sh[0].graph.struct(), dev)
p = torch.as_tensor(p0.copy(), device=dev)
eng = P_.ShardedIrlsEngine(sh, p, cfg, comm=comm)
t0 = time.perf_counter()
try:
    l1 = eng.run()
    err = None
except Exception as exc:
    l1, err = None, repr(exc)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
comm.close()
ok = None
if rank == 0 and err is None:
    ref_sh = P_.make_shards(x1, x2, lengths, ij, np.zeros_like(ij), n, 1, True, bounds, dev)
    pr = torch.as_tensor(p0.copy(), device=dev)
    lr = P_.ShardedIrlsEngine(ref_sh, pr, cfg).run()
    ok = bool(lr == l1 and torch.equal(pr, p))
print(f"rank {rank}: {dt:.2f}s err={err} l1={l1} bitwise_vs_two_shard_engine={ok}", flush=True)
dist.destroy_process_group()
