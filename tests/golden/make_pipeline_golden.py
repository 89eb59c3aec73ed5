"""Golden vectors of the hot path inside the REFERENCE pipeline on NOISY_SPEC
(acceptance criterion 5, pkg/tests/test_acceptance.py:70-72, :240-250).

Runs fastmap.run_pipeline (/root/reference, read-only) with two recording
wrappers at the exact call sites of the hot path:
  * ref/pipeline.py:233  translation.multi_init_align(dir_graph, cfg, seed)
  * ref/pipeline.py:248  irls_refine(poses, epi_pairs, cfg, n_cameras)
The epipolar pairs are rebuilt with fp32-rounded coordinates before the
reference adjustment sees them (the device store holds fp32), so the
reference and the CUDA path read bit-identical inputs.  Stores the stage
inputs, the reference stage outputs, the GT poses and the final metrics.

    python tests/golden/make_pipeline_golden.py     (~40 s; not run by pytest)
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fastmap import epipolar, metrics, pipeline, synth, translation  # noqa: E402
from fastmap.config import PipelineConfig  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    spec = synth.SynthSpec(n_images=30, n_points=500, fov_deg=60.0, alpha=-0.15, noise_px=0.5,
                           outlier_frac=0.02, seed=0)
    match_set, gt = synth.generate(spec)
    d = {}
    orig_mia, orig_irls = translation.multi_init_align, pipeline.irls_refine
    orig_rr = translation.reestimate_relative
    rr_calls = []
    rr_seconds = []

    def rr(x1, x2, rel_rotation, cfg):
        # ref/pipeline.py:209 -- the sphere search of every candidate pair
        try:
            t0 = time.perf_counter()
            t = orig_rr(x1, x2, rel_rotation, cfg)
            rr_seconds.append(time.perf_counter() - t0)
            rr_calls.append((np.asarray(x1), np.asarray(x2), np.asarray(rel_rotation), t, ""))
            return t
        except translation.PairRejected as exc:
            rr_calls.append((np.asarray(x1), np.asarray(x2), np.asarray(rel_rotation), np.zeros(3),
                             str(exc)))
            raise

    def mia(graph, cfg, seed=0):
        t0 = time.perf_counter()
        c, loss = orig_mia(graph, cfg, seed=seed)
        d.update(tr_n=np.array([graph.n]), tr_ei=np.asarray(graph.edges_i),
                 tr_ej=np.asarray(graph.edges_j), tr_dirs=np.asarray(graph.directions),
                 tr_seed=np.array([seed]), tr_centers=c, tr_loss=np.array([loss]),
                 tr_cfg=np.array([cfg.translation_lr, cfg.translation_steps, cfg.translation_inits,
                                  cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps]),
                 tr_seconds=np.array([time.perf_counter() - t0]))
        return c, loss

    def irls(poses, pairs, cfg, n_cameras=1):
        p32 = [epipolar.EpipolarPair(i=p.i, j=p.j, cam_i=p.cam_i, cam_j=p.cam_j, x1=f32(p.x1),
                                     x2=f32(p.x2), active=p.active.copy()) for p in pairs]
        d.update(ep_R_in=poses.rotations.copy(), ep_c_in=poses.centers.copy(),
                 ep_reg=np.asarray(poses.registered).copy(),
                 ep_ij=np.array([[p.i, p.j] for p in pairs], dtype=np.int32),
                 ep_cams=np.array([[p.cam_i, p.cam_j] for p in pairs], dtype=np.int32),
                 ep_len=np.array([len(p.x1) for p in pairs], dtype=np.int32),
                 ep_x1=np.concatenate([p.x1[:, :2] for p in p32]).astype(np.float32),
                 ep_x2=np.concatenate([p.x2[:, :2] for p in p32]).astype(np.float32),
                 ep_active_in=np.concatenate([p.active for p in p32]),
                 ep_n_cameras=np.array([n_cameras]),
                 ep_cfg=np.array([cfg.epipolar_lr, cfg.lr_decay, cfg.prune_threshold_start,
                                  cfg.prune_threshold_end, cfg.prune_rounds,
                                  cfg.irls_iters_between_prunes, cfg.epipolar_epoch_steps,
                                  float(cfg.refine_focal)]))
        t0 = time.perf_counter()
        out, fs, rep = orig_irls(poses, p32, cfg, n_cameras=n_cameras)
        d.update(ep_seconds=np.array([time.perf_counter() - t0]), ep_R_out=out.rotations,
                 ep_c_out=out.centers, ep_focal=np.asarray(fs), ep_l1=np.array(rep["l1_history"]),
                 ep_counts=np.array([rep["dropped_pairs"], rep["active_pairs"]]),
                 ep_active_out=np.concatenate([p.active for p in p32]))
        for p, q in zip(pairs, p32):
            p.active[...] = q.active
        return out, fs, rep

    translation.multi_init_align, pipeline.irls_refine = mia, irls
    translation.reestimate_relative = rr
    try:
        t0 = time.perf_counter()
        scene, _ = pipeline.run_pipeline(match_set, PipelineConfig(), seed=0)
        total = time.perf_counter() - t0
    finally:
        translation.multi_init_align, pipeline.irls_refine = orig_mia, orig_irls
        translation.reestimate_relative = orig_rr
    # sphere-search calls: all outcomes; the points of the first 80 calls
    keep = rr_calls[:80]
    cfg = PipelineConfig()
    d.update(rr_len=np.array([len(c[0]) for c in keep], dtype=np.int32),
             rr_x1=np.concatenate([c[0] for c in keep]), rr_x2=np.concatenate([c[1] for c in keep]),
             rr_R=np.stack([c[2] for c in keep]), rr_t=np.stack([c[3] for c in keep]),
             rr_msg=np.array([c[4] for c in keep]),
             rr_cfg=np.array([cfg.sphere_samples, cfg.sphere_refine_levels]),
             rr_n_calls=np.array([len(rr_calls)]),
             rr_n_rejected=np.array([sum(1 for c in rr_calls if c[4])]),
             rr_ref_seconds_per_call=np.array([np.mean(rr_seconds)]))
    table = metrics.evaluate(scene.poses, gt.poses)
    d.update(gt_R=gt.poses.rotations, gt_c=gt.poses.centers,
             final_metrics=np.array([table["ATE"], table["RRA@1"], table["RTA@3"]]),
             pipeline_seconds=np.array([total]))
    # synthetic sphere-search cases for the rejection paths: a noise-free pure
    # rotation (flat landscape) and a small generic pair
    rng = np.random.default_rng(11)
    ang = 0.3
    Rz = np.array([[np.cos(ang), -np.sin(ang), 0.0], [np.sin(ang), np.cos(ang), 0.0], [0.0, 0.0, 1.0]])
    X = rng.uniform(-1, 1, size=(60, 3)) + np.array([0.0, 0.0, 4.0])
    x1 = X / X[:, 2:3]
    y = X @ Rz.T
    x2 = y / y[:, 2:3]
    xs = []
    for name, (a, b, R) in {"rot": (x1, x2, Rz),
                            "gen": (x1, (X @ Rz.T + [0.4, -0.1, 0.2]) / (X @ Rz.T + [0.4, -0.1, 0.2])[:, 2:3],
                                    Rz)}.items():
        try:
            t, msg = translation.reestimate_relative(a, b, R, cfg), ""
        except translation.PairRejected as exc:
            t, msg = np.zeros(3), str(exc)
        xs.append((a, b, R, t, msg))
    d.update(rrx_x1=np.stack([c[0] for c in xs]), rrx_x2=np.stack([c[1] for c in xs]),
             rrx_R=np.stack([c[2] for c in xs]), rrx_t=np.stack([c[3] for c in xs]),
             rrx_msg=np.array([c[4] for c in xs]))
    print("synthetic sphere cases:", [c[4] or "ok" for c in xs])
    np.savez_compressed(os.path.join(HERE, "golden_pipeline.npz"), **d)
    print(f"sphere search: {len(rr_calls)} calls, {int(d['rr_n_rejected'][0])} rejected, "
          f"{1e3 * np.mean(rr_seconds):.2f} ms per call (reference, this host)")
    print(f"pipeline {total:.1f}s: translation {d['tr_seconds'][0]:.1f}s ({len(d['tr_ei'])} edges), "
          f"irls {d['ep_seconds'][0]:.1f}s ({int(d['ep_len'].sum())} point pairs, "
          f"{len(d['ep_len'])} image pairs); ATE {table['ATE']:.3e} RRA@1 {table['RRA@1']} "
          f"RTA@3 {table['RTA@3']}")


if __name__ == "__main__":
    main()
