"""Time multi_init_align at BASELINE config 3 (2k nodes, 200k edges, 16 inits)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
print(json.dumps(bench.translation_bench(torch.device("cuda"), torch.cuda.Stream())))
