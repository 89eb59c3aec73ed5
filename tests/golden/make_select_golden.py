"""Golden vectors of the epipolar-pair / direction-graph selection inside the
REFERENCE pipeline (ref/pipeline.py:188-228) on NOISY_SPEC (acceptance
criterion 5, pkg/tests/test_acceptance.py:70-72).

Runs fastmap.run_pipeline (/root/reference, read-only) with a recording
_Report.start: at "translation.relative" it snapshots the stage inputs (the
completed match set, the verified inlier pairs behind pair_points, the
normalised keypoints, the rotations, the registered mask), at
"translation.align" the stage outputs (the DirectionGraph and the
EpipolarPair list), then stops the pipeline.  Points are stored as keypoint
row indices; the script checks that gathering the rows reproduces the
reference's arrays exactly.

    python tests/golden/make_select_golden.py     (~30 s; not run by pytest)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fastmap import pipeline, synth  # noqa: E402
from fastmap.config import PipelineConfig  # noqa: E402


class _Stop(Exception):
    pass


def main():
    spec = synth.SynthSpec(n_images=30, n_points=500, fov_deg=60.0, alpha=-0.15, noise_px=0.5,
                           outlier_frac=0.02, seed=0)
    match_set, _ = synth.generate(spec)
    snap = {}
    orig = pipeline._Report.start

    def start(self, name):
        if name in ("translation.relative", "translation.align"):
            snap[name] = dict(sys._getframe(1).f_locals)
            if name == "translation.align":
                raise _Stop
        return orig(self, name)

    pipeline._Report.start = start
    try:
        pipeline.run_pipeline(match_set, PipelineConfig(), seed=0)
    except (_Stop, pipeline.StageError) as exc:
        if not isinstance(exc, _Stop) and not isinstance(exc.cause, _Stop):
            raise
    finally:
        pipeline._Report.start = orig

    a, b = snap["translation.relative"], snap["translation.align"]
    norm_kps = a["norm_kps"]
    kp_off = np.concatenate([[0], np.cumsum([len(k) for k in norm_kps])]).astype(np.int64)
    kp = np.concatenate(norm_kps)
    completed = a["completed"].pairs
    corr = [np.asarray(p.correspondences, dtype=np.int64) for p in completed]
    # pair_points[(i, j)] = verified inlier rows (ref/pipeline.py:130-145)
    pp = a["pair_points"]
    vmap = {(p.i, p.j): np.asarray(p.correspondences, dtype=np.int64) for p in a["verified"].pairs}
    pp_keys = sorted(pp)
    for key in pp_keys:
        c = vmap[key]
        assert np.array_equal(norm_kps[key[0]][c[:, 0]], pp[key][0])
        assert np.array_equal(norm_kps[key[1]][c[:, 1]], pp[key][1])
    # expected outputs as keypoint rows (checked against the reference's arrays)
    epi = b["epi_pairs"]
    rows1, rows2 = [], []
    for p in epi:
        key = (p.i, p.j)
        src = next(q for q in completed if (q.i, q.j) == key)
        if src.synthetic_from_tracks or key not in pp:
            c = np.asarray(src.correspondences, dtype=np.int64)
            x1 = norm_kps[p.i][c[:, 0]]
            x2 = norm_kps[p.j][c[:, 1]]
            ok = np.all(np.isfinite(x1), axis=1) & np.all(np.isfinite(x2), axis=1)
            c = c[ok]
        else:
            c = vmap[key]
        r1, r2 = kp_off[p.i] + c[:, 0], kp_off[p.j] + c[:, 1]
        assert np.array_equal(kp[r1], p.x1) and np.array_equal(kp[r2], p.x2)
        rows1.append(r1)
        rows2.append(r2)
    dg = b["dir_graph"]
    images = a["match_set"].images
    d = dict(
        kp_off=kp_off, kp=kp,
        cp_ij=np.array([[p.i, p.j] for p in completed], dtype=np.int64),
        cp_synth=np.array([bool(p.synthetic_from_tracks) for p in completed]),
        cp_off=np.concatenate([[0], np.cumsum([len(c) for c in corr])]).astype(np.int64),
        cp_corr=np.concatenate(corr).astype(np.int32),
        pp_ij=np.array(pp_keys, dtype=np.int64),
        pp_off=np.concatenate([[0], np.cumsum([len(vmap[k]) for k in pp_keys])]).astype(np.int64),
        pp_corr=np.concatenate([vmap[k] for k in pp_keys]).astype(np.int32),
        rotations=np.asarray(a["rotations"]), registered=np.asarray(a["graph"].registered).astype(bool),
        cams=np.array([im.camera_id for im in images], dtype=np.int64),
        cfg=np.array([a["cfg"].sphere_samples, a["cfg"].sphere_refine_levels]),
        out_n=np.array([dg.n]), out_ei=np.asarray(dg.edges_i), out_ej=np.asarray(dg.edges_j),
        out_dirs=np.asarray(dg.directions),
        out_ij=np.array([[p.i, p.j] for p in epi], dtype=np.int64),
        out_cams=np.array([[p.cam_i, p.cam_j] for p in epi], dtype=np.int64),
        out_len=np.array([len(p.x1) for p in epi], dtype=np.int64),
        out_rows1=np.concatenate(rows1).astype(np.int32),
        out_rows2=np.concatenate(rows2).astype(np.int32),
    )
    np.savez_compressed(os.path.join(HERE, "golden_select.npz"), **d)
    n_synth = int(d["cp_synth"].sum())
    print(f"{len(completed)} completed pairs ({n_synth} synthetic), {len(pp_keys)} with verified "
          f"inliers, {len(epi)} epipolar pairs / {len(dg.edges_i)} edges, "
          f"{int(d['out_len'].sum())} point pairs")


if __name__ == "__main__":
    main()
