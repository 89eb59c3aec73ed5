"""Golden vectors of the rotation refinement (ref/rotation.py:162-230,
SURVEY 8f "next" #3) from the REFERENCE implementation (read-only import):
the loss / 6D gradient at random parameters and full refine_rotations runs
(early-stopped and step-capped) on seeded relative-rotation graphs.

    python tests/golden/make_rotation_golden.py      (seconds; not run by pytest)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fastmap import rotation  # noqa: E402
from fastmap.config import PipelineConfig  # noqa: E402
from fastmap.optim import matrix_to_rot6d  # noqa: E402
from scipy.spatial.transform import Rotation  # noqa: E402


def graph(n, extra, noise_deg, seed):
    rng = np.random.default_rng(seed)
    gt = Rotation.random(n, random_state=seed).as_matrix()
    pairs = {(k, k + 1) for k in range(n - 1)}
    while len(pairs) < n - 1 + extra:
        i, j = sorted(rng.integers(0, n, size=2))
        if i != j:
            pairs.add((int(i), int(j)))
    edges = []
    for i, j in sorted(pairs):
        noise = Rotation.from_rotvec(rng.normal(size=3) * np.radians(noise_deg) / np.sqrt(3)).as_matrix()
        edges.append(rotation.RelPoseEdge(i=i, j=j, rel_rotation=noise @ gt[j] @ gt[i].T, inlier_count=50))
    init = np.stack([Rotation.from_rotvec(rng.normal(size=3) * 0.05).as_matrix() @ R for R in gt])
    return rotation.RelPoseGraph(n_images=n, edges=edges), gt, init


def main():
    d = {}
    for k, (n, extra, noise, steps) in enumerate([(12, 20, 1.0, 2000), (30, 60, 0.5, 300),
                                                  (8, 6, 0.0, 2000)]):
        g, gt, init = graph(n, extra, noise, seed=k)
        ei = np.array([e.i for e in g.edges])
        ej = np.array([e.j for e in g.edges])
        rel = np.stack([e.rel_rotation for e in g.edges])
        p = matrix_to_rot6d(init)
        loss, grad = rotation.rotation_loss_and_grad(p, ei, ej, rel)
        cfg = PipelineConfig()
        cfg.rotation_steps = steps
        out, hist = rotation.refine_rotations(init, g, cfg)
        pre = f"r{k}_"
        d.update({pre + "n": np.array([n]), pre + "ei": ei, pre + "ej": ej, pre + "rel": rel,
                  pre + "init": init, pre + "gt": gt, pre + "p": p, pre + "loss": np.array([loss]),
                  pre + "grad": grad, pre + "steps": np.array([steps]), pre + "out": out,
                  pre + "hist": np.array(hist),
                  pre + "cfg": np.array([cfg.rotation_lr, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps])})
        print(f"graph {k}: n={n} m={len(ei)} loss {loss:.4e}, refine {len(hist)} steps, "
              f"final {hist[-1]:.4e}")
    np.savez_compressed(os.path.join(HERE, "golden_rotation.npz"), **d)


if __name__ == "__main__":
    main()
