"""Generate the golden vectors that pin the oracle and the CUDA path.

Runs the REFERENCE implementation (/root/reference/pkg/src/fastmap, imported
read-only) on seeded inputs and stores inputs + reference outputs as .npz
fixtures next to this script.  Point coordinates are rounded to fp32 BEFORE
the reference sees them, so the reference, the oracle and the device store
all read bit-identical inputs.

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --small    # skip the config-1 scene

Not run by the test suite (the reference does not exist on the GPU box).
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from fastmap import epipolar as E  # noqa: E402
from fastmap import optim as O  # noqa: E402
from fastmap import translation as T  # noqa: E402
from fastmap.config import PipelineConfig  # noqa: E402
from fastmap.model import PoseState, project_to_so3  # noqa: E402
from scipy.spatial.transform import Rotation  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def arc_scene(n_images, n_points, seed, noise=0.0, n_cams=1):
    """Cameras on an arc looking at a point cloud; normalized observations."""
    rng = np.random.default_rng(seed)
    ang = np.linspace(0.0, 1.3, n_images)
    centers = np.stack([2.5 * np.cos(ang), 2.5 * np.sin(ang), 0.3 * ang - 0.2], axis=1)
    rots = []
    for c in centers:
        fwd = -c / np.linalg.norm(c)
        right = np.cross(fwd, [0.0, 0.0, 1.0])
        right /= np.linalg.norm(right)
        rots.append(np.stack([right, np.cross(fwd, right), fwd]))
    rots = np.stack(rots)
    pts = rng.uniform(-0.6, 0.6, size=(n_points, 3))
    pairs = []
    for i in range(n_images):
        for j in range(i + 1, n_images):
            m = rng.integers(n_points // 2, n_points + 1)
            sel = rng.choice(n_points, size=m, replace=False)
            xi = (pts[sel] - centers[i]) @ rots[i].T
            xj = (pts[sel] - centers[j]) @ rots[j].T
            xi = xi / xi[:, 2:3]
            xj = xj / xj[:, 2:3]
            if noise:
                xi[:, :2] += rng.normal(scale=noise, size=(m, 2))
                xj[:, :2] += rng.normal(scale=noise, size=(m, 2))
            xi[:, :2] = f32(xi[:, :2])
            xj[:, :2] = f32(xj[:, :2])
            pairs.append(E.EpipolarPair(i=i, j=j, cam_i=i % n_cams, cam_j=j % n_cams, x1=xi, x2=xj))
    poses = PoseState(rotations=rots, centers=centers, registered=np.ones(n_images, dtype=bool))
    return poses, pairs


def perturb(poses, rng, rot_deg, center_sigma):
    out = PoseState(rotations=poses.rotations.copy(), centers=poses.centers.copy(),
                    registered=poses.registered.copy())
    for k in range(1, len(out.rotations)):
        rv = rng.normal(size=3)
        rv *= np.radians(rot_deg) / np.linalg.norm(rv)
        out.rotations[k] = Rotation.from_rotvec(rv).as_matrix() @ out.rotations[k]
        out.centers[k] += rng.normal(scale=center_sigma, size=3)
    return out


def flat_pairs(prefix, pairs, d):
    d[prefix + "x1"] = np.concatenate([p.x1 for p in pairs])
    d[prefix + "x2"] = np.concatenate([p.x2 for p in pairs])
    d[prefix + "len"] = np.array([len(p.x1) for p in pairs])
    d[prefix + "ij"] = np.array([[p.i, p.j] for p in pairs])
    d[prefix + "cams"] = np.array([[p.cam_i, p.cam_j] for p in pairs])
    d[prefix + "active"] = np.concatenate([p.active for p in pairs])


def epipolar_cases(d):
    """API-level vectors: residuals, weights, losses, gradients."""
    cases = [
        dict(n=4, pts=40, seed=2, noise=1e-3, cams=1, rf=False, shuffle=False, mask=False),
        dict(n=5, pts=60, seed=3, noise=2e-3, cams=2, rf=True, shuffle=True, mask=True),
        dict(n=6, pts=30, seed=4, noise=5e-4, cams=3, rf=True, shuffle=True, mask=False),
    ]
    for k, c in enumerate(cases):
        rng = np.random.default_rng(100 + k)
        poses, pairs = arc_scene(c["n"], c["pts"], c["seed"], c["noise"], c["cams"])
        if c["shuffle"]:
            perm = rng.permutation(len(pairs))
            pairs = [pairs[q] for q in perm]
        if c["mask"]:
            for p in pairs:
                p.active = rng.random(len(p.x1)) > 0.2
        ids = list(range(c["n"]))
        state = E.AdjustmentState.from_poses(poses, ids, c["cams"], c["rf"])
        packed = state.pack() + rng.normal(scale=0.02, size=state.pack().shape)
        state.unpack(packed.copy())
        pre = f"e{k}_"
        flat_pairs(pre, pairs, d)
        d[pre + "params"] = packed
        d[pre + "meta"] = np.array([c["n"], c["cams"], int(c["rf"])])
        res = E.current_residuals(state, pairs)
        d[pre + "residuals"] = np.concatenate(res)
        W1 = [E.precompute_weights(p.x1[p.active], p.x2[p.active]) for p in pairs]
        W2 = [E.precompute_weights(p.x1[p.active], p.x2[p.active], residuals=r[p.active])
              for p, r in zip(pairs, res)]
        d[pre + "W_unweighted"] = np.stack(W1)
        d[pre + "W_irls"] = np.stack(W2)
        l2, Z = E.epipolar_loss(state, pairs, mode="l2")
        l1, _ = E.epipolar_loss(state, pairs, mode="l1")
        d[pre + "loss_l2"] = np.array([l2, Z])
        d[pre + "loss_l1"] = np.array([l1, Z])
        loss, grad = E.quadratic_loss_and_grad(state, pairs, W2, Z)
        d[pre + "quad_loss"] = np.array([loss])
        d[pre + "quad_grad"] = grad


def irls_case(d):
    poses, pairs = arc_scene(5, 60, seed=5, noise=1e-3, n_cams=1)
    noisy = perturb(poses, np.random.default_rng(5), 0.6, 0.01)
    flat_pairs("irls_", pairs, d)
    d["irls_R_in"] = noisy.rotations
    d["irls_c_in"] = noisy.centers
    cfg = PipelineConfig(epipolar_lr=1e-3)
    out, fs, rep = E.irls_refine(noisy, pairs, cfg, n_cameras=1)
    d["irls_R_out"] = out.rotations
    d["irls_c_out"] = out.centers
    d["irls_focal"] = fs
    d["irls_l1"] = np.array(rep["l1_history"])
    d["irls_counts"] = np.array([rep["dropped_pairs"], rep["active_pairs"]])
    d["irls_active_out"] = np.concatenate([p.active for p in pairs])


def optim_cases(d):
    rng = np.random.default_rng(7)
    v = rng.normal(size=(16, 6))
    d["rot6d_in"] = v
    d["rot6d_R"] = O.rot6d_to_matrix(v)
    d["rot6d_J"] = O.rot6d_jacobian(v)
    M = rng.normal(size=(16, 3, 3))
    d["so3_in"] = M
    d["so3_out"] = np.stack([project_to_so3(m) for m in M])
    p0 = rng.normal(size=11)
    grads = rng.normal(size=(25, 11))
    opt = O.Adam(p0, lr=0.05)
    traj = []
    for g in grads:
        traj.append(opt.step(g).copy())
    d["adam_p0"] = p0
    d["adam_grads"] = grads
    d["adam_traj"] = np.stack(traj)


def ring(n, seed, extra):
    rng = np.random.default_rng(seed)
    a = np.linspace(0, 2 * np.pi, n, endpoint=False)
    c = np.stack([np.cos(a), np.sin(a), 0.25 * np.cos(3 * a)], axis=1)
    edges = {(i, (i + 1) % n) if i < (i + 1) % n else ((i + 1) % n, i) for i in range(n)}
    while len(edges) < n + extra:
        i, j = sorted(rng.integers(0, n, 2))
        if i != j:
            edges.add((int(i), int(j)))
    edges = sorted(edges)
    ei = np.array([e[0] for e in edges])
    ej = np.array([e[1] for e in edges])
    dirs = c[ej] - c[ei]
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return T.DirectionGraph(n=n, edges_i=ei, edges_j=ej, directions=dirs), c


def translation_cases(d):
    g, c = ring(12, 3, 14)
    rng = np.random.default_rng(9)
    start = c + rng.normal(scale=0.3, size=c.shape)
    d["tr_n"] = np.array([g.n])
    d["tr_ei"], d["tr_ej"], d["tr_dirs"] = g.edges_i, g.edges_j, g.directions
    d["tr_gt"] = c
    d["tr_start"] = start
    loss, grad = T.translation_loss_and_grad(start, g)
    d["tr_loss"] = np.array([loss])
    d["tr_grad"] = grad
    d["tr_node_res"] = T.per_node_residuals(start, g)
    d["tr_canon"] = T.canonicalize(start * 3 + 1)
    cfg = PipelineConfig(translation_steps=300)
    ac, al = T.align_centers(g, cfg, seed=4)
    d["tr_align"] = ac
    d["tr_align_loss"] = np.array([al])
    cfg = PipelineConfig(translation_steps=400, translation_inits=3)
    mc, ml = T.multi_init_align(g, cfg, seed=1)
    d["tr_multi"] = mc
    d["tr_multi_loss"] = np.array([ml])


def config1(d):
    """BASELINE config 1: SURVEY.md section 8d C1 scene, GT-seeded inputs."""
    from fastmap import synth
    from fastmap.distortion import undistort_pixels
    spec = synth.SynthSpec(n_images=50, n_points=5000, layout="ring", fov_deg=13.0, alpha=-0.1,
                           noise_px=0.5, outlier_frac=0.02, seed=0, min_visible_per_image=20,
                           min_pair_corrs=16)
    ms, gt = synth.generate(spec)
    norm = []
    for im in ms.images:
        cam = gt.cameras[im.camera_id]
        und = undistort_pixels(ms.keypoints[im.image_id], cam)
        norm.append((und - np.array([cam.cx, cam.cy])) / cam.focal)
    pairs = []
    for pr in ms.pairs:
        x1 = norm[pr.i][pr.correspondences[:, 0]]
        x2 = norm[pr.j][pr.correspondences[:, 1]]
        ok = np.all(np.isfinite(x1), axis=1) & np.all(np.isfinite(x2), axis=1)
        x1 = np.column_stack([f32(x1[ok]), np.ones(ok.sum())])
        x2 = np.column_stack([f32(x2[ok]), np.ones(ok.sum())])
        pairs.append(E.EpipolarPair(i=pr.i, j=pr.j, cam_i=0, cam_j=0, x1=x1, x2=x2))
    noisy = perturb(gt.poses, np.random.default_rng(0), 0.5, 0.01)
    d["c1_x1"] = np.concatenate([p.x1[:, :2] for p in pairs]).astype(np.float32)
    d["c1_x2"] = np.concatenate([p.x2[:, :2] for p in pairs]).astype(np.float32)
    d["c1_len"] = np.array([len(p.x1) for p in pairs], dtype=np.int32)
    d["c1_ij"] = np.array([[p.i, p.j] for p in pairs], dtype=np.int32)
    d["c1_R_gt"], d["c1_c_gt"] = gt.poses.rotations, gt.poses.centers
    d["c1_R_in"], d["c1_c_in"] = noisy.rotations, noisy.centers
    t0 = time.perf_counter()
    out, fs, rep = E.irls_refine(noisy, pairs, PipelineConfig(), n_cameras=1)
    d["c1_ref_seconds"] = np.array([time.perf_counter() - t0])
    d["c1_R_out"], d["c1_c_out"] = out.rotations, out.centers
    d["c1_focal"] = fs
    d["c1_l1"] = np.array(rep["l1_history"])
    d["c1_counts"] = np.array([rep["dropped_pairs"], rep["active_pairs"]])
    d["c1_active_count"] = np.array([int(p.active.sum()) for p in pairs], dtype=np.int32)
    # translation on the same scene: GT directions + 1 degree noise + 5% outliers
    rng = np.random.default_rng(1)
    ei = d["c1_ij"][:, 0].astype(np.int64)
    ej = d["c1_ij"][:, 1].astype(np.int64)
    c = gt.poses.centers
    dirs = c[ej] - c[ei]
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    dirs = dirs + rng.normal(scale=np.radians(1.0), size=dirs.shape)
    bad = rng.random(len(dirs)) < 0.05
    dirs[bad] = rng.normal(size=(bad.sum(), 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    g = T.DirectionGraph(n=len(c), edges_i=ei, edges_j=ej, directions=dirs)
    d["c1_dirs"] = dirs
    t0 = time.perf_counter()
    mc, ml = T.multi_init_align(g, PipelineConfig(), seed=0)
    d["c1_tr_seconds"] = np.array([time.perf_counter() - t0])
    d["c1_tr_centers"] = mc
    d["c1_tr_loss"] = np.array([ml])
    print(f"config1: {len(pairs)} pairs, {int(d['c1_len'].sum())} point pairs, "
          f"irls {d['c1_ref_seconds'][0]:.1f}s, translation {d['c1_tr_seconds'][0]:.1f}s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true")
    args = ap.parse_args()
    d = {}
    epipolar_cases(d)
    irls_case(d)
    optim_cases(d)
    translation_cases(d)
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **d)
    print("wrote golden_small.npz", len(d), "arrays")
    if not args.small:
        d = {}
        config1(d)
        np.savez_compressed(os.path.join(HERE, "golden_config1.npz"), **d)
        print("wrote golden_config1.npz")


if __name__ == "__main__":
    main()
