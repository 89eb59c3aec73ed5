"""cProfile of the drop-in irls_refine on C2's 25,000 EpipolarPair objects
(host-side store preparation vs the device schedule)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2505_04612_b200 import scenes
from paper_2505_04612_b200.config import HotPathConfig
class A: pass
args = A(); args.cfg = HotPathConfig(); args.precision = "fp32"
dev = torch.device("cuda")
sc = scenes.generate(scenes.CONFIGS["c2"], dev)
bench.api_irls_bench(args, sc, dev, torch.cuda.current_stream())  # warm-up
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
out = bench.api_irls_bench(args, sc, dev, torch.cuda.current_stream())
pr.disable()
print("api irls_refine (incl. pair construction)", time.perf_counter() - t0, out["irls_refine_api_s"])
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
