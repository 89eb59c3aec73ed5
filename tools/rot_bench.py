"""refine_rotations at a C2-like scale (500 images, ring band 50: 25k edges,
2000 Adam steps) on the device; with --reference, the reference's per-step
time on this host (numpy, 20 steps) for comparison."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scipy.spatial.transform import Rotation
n, band = 500, 50
rng = np.random.default_rng(0)
gt = Rotation.random(n, random_state=0).as_matrix()
ei = np.array([i for i in range(n) for d in range(1, band + 1)])
ej = np.array([(i + d) % n for i in range(n) for d in range(1, band + 1)])
noise = Rotation.from_rotvec(rng.normal(size=(len(ei), 3)) * np.radians(1.0) / np.sqrt(3)).as_matrix()
rel = noise @ gt[ej] @ np.transpose(gt[ei], (0, 2, 1))
init = Rotation.from_rotvec(rng.normal(size=(n, 3)) * 0.05).as_matrix() @ gt
class E:
    def __init__(s, i, j, r): s.i, s.j, s.rel_rotation = int(i), int(j), r
class G:
    n_images = n; registered = np.ones(n, bool)
    edges = [E(i, j, r) for i, j, r in zip(ei, ej, rel)]
class C:
    rotation_steps, rotation_lr, adam_beta1, adam_beta2, adam_eps = 2000, 1e-4, 0.9, 0.999, 1e-8
if "--reference" in sys.argv:
    sys.path.insert(0, "/root/reference/pkg/src")
    from fastmap import rotation as R
    from fastmap.optim import matrix_to_rot6d
    p = matrix_to_rot6d(init)
    t0 = time.perf_counter()
    for _ in range(20): R.rotation_loss_and_grad(p, ei, ej, rel)
    print(json.dumps({"edges": len(ei), "reference_step_ms": (time.perf_counter() - t0) / 20 * 1e3}))
else:
    import torch
    from paper_2505_04612_b200 import rotation as Rm
    C.rotation_steps = 200; Rm.refine_rotations(init, G, C); C.rotation_steps = 2000
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out, hist = Rm.refine_rotations(init, G, C)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(json.dumps({"edges": len(ei), "steps": len(hist), "device_s": dt,
                      "device_step_us": dt / len(hist) * 1e6, "final_loss": hist[-1]}))
