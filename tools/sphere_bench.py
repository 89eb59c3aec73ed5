"""Per-pair sphere search (reestimate_relative) on the recorded NOISY_SPEC
pipeline inputs: device path vs the reference's per-call time recorded with
the fixture (tests/golden/make_pipeline_golden.py)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_04612_b200 import translation as T
g = dict(np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "golden_pipeline.npz")))
class C: sphere_samples, sphere_refine_levels = (int(v) for v in g["rr_cfg"])
L = g["rr_len"].astype(np.int64); st = np.concatenate([[0], np.cumsum(L)])
for k in range(5): T.reestimate_relative(g["rr_x1"][st[k]:st[k+1]], g["rr_x2"][st[k]:st[k+1]], g["rr_R"][k], C)
torch.cuda.synchronize(); t0 = time.perf_counter()
for k in range(len(L)): T.reestimate_relative(g["rr_x1"][st[k]:st[k+1]], g["rr_x2"][st[k]:st[k+1]], g["rr_R"][k], C)
dt = (time.perf_counter() - t0) / len(L)
# batched: the 80 pairs tiled to config-1 size (1225 image pairs)
reps = 1225 // len(L) + 1
x1s = [g["rr_x1"][st[k]:st[k+1]] for k in range(len(L))] * reps
x2s = [g["rr_x2"][st[k]:st[k+1]] for k in range(len(L))] * reps
Rs = list(g["rr_R"]) * reps
x1s, x2s, Rs = x1s[:1225], x2s[:1225], Rs[:1225]
T.reestimate_relative_batch(x1s[:50], x2s[:50], Rs[:50], C)
torch.cuda.synchronize(); t0 = time.perf_counter()
T.reestimate_relative_batch(x1s, x2s, Rs, C)
torch.cuda.synchronize(); tb = time.perf_counter() - t0
print(json.dumps({"pairs": len(L), "mean_points": float(L.mean()), "device_ms_per_call": dt * 1e3,
                  "reference_ms_per_call": float(g["rr_ref_seconds_per_call"][0]) * 1e3,
                  "batch_pairs": len(x1s), "batch_s": tb, "batch_ms_per_pair": tb * 1e3 / len(x1s)}))
