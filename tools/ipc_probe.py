"""Two processes on one GPU (gloo for the handle exchange): PeerSum over
CUDA IPC-mapped buffers.  Kernels of two processes are time-sliced, so an
exchange either completes slowly or ends in the bounded wait (err set)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2505_04612_b200 import parallel as P_
dist.init_process_group("gloo")
rank = dist.get_rank()
torch.cuda.set_device(0)
comm = P_.PeerSum.from_process_group(3)
t = torch.tensor([1.0 + rank, 10.0 * (rank + 1), 100.0], dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
comm.allreduce_(t)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"rank {rank}: {t.tolist()} err={comm.err.item()} {dt:.3f}s", flush=True)
comm.close()
dist.destroy_process_group()
