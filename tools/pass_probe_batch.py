"""Pass time without event quantisation: B back-to-back fused passes per
event pair (no L2 flush between them; C2's 161 MB store exceeds L2), R
repetitions; prints the per-pass mean.  CUDA event timestamps on this
GPU move in ~2 us steps, so single-pass A/B differences below that are
invisible to per-step events.
    FASTMAP_B200_LIB=... python tools/pass_probe_batch.py [config] [B] [R]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_04612_b200 import scenes  # noqa: E402
from paper_2505_04612_b200.config import HotPathConfig  # noqa: E402


class A:
    pass


cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 20
R = int(sys.argv[3]) if len(sys.argv) > 3 else 10
args = A()
args.cfg = HotPathConfig()
args.precision = "fp32"
dev = torch.device("cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    sc, store, graph, ids, eng = bench.make_engine(scenes.CONFIGS[cfg], dev, args)
    eng._ghat()
    eng.buf.n_active[0].fill_(1)
    eng.point_pass(bench.HOT_MODE(), bench.TH, 0, 0)
torch.cuda.synchronize()
res = []
with torch.cuda.stream(st):
    for r in range(R + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(400_000)
        e0.record(st)
        for _ in range(B):
            if os.environ.get("KERNEL_ONLY"):
                bench.pass_kernel_only(eng)
            else:
                eng.point_pass(bench.HOT_MODE(), bench.TH, 0, 0)
        e1.record(st)
        torch.cuda.synchronize()
        if r:
            res.append(1e3 * e0.elapsed_time(e1) / B)
print(json.dumps({"config": cfg, "per_pass_us_mean": float(np.mean(res)),
                  "per_pass_us_min": float(np.min(res)), "per_pass_us_max": float(np.max(res))}))
