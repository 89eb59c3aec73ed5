"""BASELINE config 1 through the drop-in API: irls_refine + multi_init_align
wall times per call (bench.c1_sfm_optimize), for launch lists / ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2505_04612_b200 import epipolar as E, translation as T
from paper_2505_04612_b200.config import HotPathConfig
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
out = bench.c1_sfm_optimize(E, T, HotPathConfig(), bench.Poses, reps, torch.cuda.synchronize)
print("irls_s", ["%.4f" % t for t in out["irls_s"]], "translation_s", ["%.4f" % t for t in out["translation_s"]])
