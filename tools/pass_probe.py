"""Time the C2 fused pass (bench.py's step) under environment variants.
    python tools/pass_probe.py [config] [VAR=val,VAR2=val ...]
Each argument after the config is one variant (comma-separated env
assignments, "-" for none); every variant runs in its own subprocess."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, os, json
sys.path.insert(0, %r)
import numpy as np, torch, bench
from paper_2505_04612_b200 import scenes
from paper_2505_04612_b200.config import HotPathConfig
class A: pass
args = A(); args.cfg = HotPathConfig(); args.precision = os.environ.get("PREC", "fp32")
spec = scenes.CONFIGS[%r]
dev = torch.device("cuda"); st = torch.cuda.Stream()
with torch.cuda.stream(st):
    sc, store, graph, ids, eng = bench.make_engine(spec, dev, args)
    eng._ghat(); eng.buf.n_active[0].fill_(1)
    eng.point_pass(bench.HOT_MODE(), bench.TH, 0, 0)
torch.cuda.synchronize()
bench.time_passes(eng, st, 5, lambda: None)
ms = bench.time_passes(eng, st, 30, lambda: None)
print(json.dumps({"median_us": 1e3 * float(np.median(ms)), "mean_us": 1e3 * float(np.mean(ms)),
                  "min_us": 1e3 * float(np.min(ms)), "tot": eng.buf.tot.cpu().tolist()}))
"""


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    variants = sys.argv[2:] or ["-"]
    for v in variants:
        env = dict(os.environ)
        if v != "-":
            for kv in v.split(","):
                k, val = kv.split("=", 1)
                env[k] = val
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env,
                           capture_output=True, text=True, timeout=600)
        out = r.stdout.strip().splitlines()
        print(f"{cfg} {v}: {out[-1] if out else r.stderr[-800:]}", flush=True)


if __name__ == "__main__":
    main()
