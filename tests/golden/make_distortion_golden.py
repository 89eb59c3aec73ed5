"""Golden vectors of the distortion candidate search (ref/distortion.py:90-193,
SURVEY 8f "next" #4) from the REFERENCE implementation (read-only import):
the synthetic match sets of the reference's own distortion tests
(pkg/tests/test_distortion.py:43-80), the scores score_alpha gives every
candidate of every search level, the search_alpha result, and the
schedule_cameras result of the two-camera scene, a subset-sized pair set
(M < 16, the non-LMedS branch), and undistorted_fundamentals + the focal
vote (ref/focal.py:51-172) on both scenes, and apply_calibration
(ref/focal.py:175-203) on those and on a planar scene (homography pairs), and
build_tracks + complete_matches (ref/tracks.py:38-106).

    python tests/golden/make_distortion_golden.py      (a minute; not run by pytest)
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fastmap import distortion, focal, synth, tracks  # noqa: E402
from fastmap.config import PipelineConfig  # noqa: E402
from fastmap.model import CameraModel, GeometryClass  # noqa: E402


def pack(prefix, ms, out):
    out[prefix + "img"] = np.array([[im.camera_id, im.width, im.height] for im in ms.images],
                                   dtype=np.int64)
    out[prefix + "kp_len"] = np.array([len(k) for k in ms.keypoints], dtype=np.int64)
    out[prefix + "kp"] = np.concatenate(ms.keypoints)
    out[prefix + "pair_ij"] = np.array([[p.i, p.j] for p in ms.pairs], dtype=np.int64)
    out[prefix + "pair_len"] = np.array([len(p.correspondences) for p in ms.pairs], dtype=np.int64)
    out[prefix + "corr"] = np.concatenate([p.correspondences for p in ms.pairs]).astype(np.int64)


def m_cams(ms):
    return max(im.camera_id for im in ms.images) + 1


def main():
    out = {}
    cfg = PipelineConfig()
    # scene A: single camera, alpha = -0.2 (test_recovers_alpha_on_synthetic_scene)
    ms, _ = synth.generate(synth.SynthSpec(n_images=8, n_points=200, fov_deg=70.0, alpha=-0.2,
                                           seed=0))
    pack("a_", ms, out)
    out["a_homography"] = np.array([p.geometry_class is GeometryClass.HOMOGRAPHY for p in ms.pairs])
    pairs = distortion.ready_fundamental_pairs(ms)
    ready = [ms.pairs.index(p) for p in pairs]
    out["a_ready"] = np.array(ready, dtype=np.int64)
    lo, hi, n = cfg.distortion_min, cfg.distortion_max, cfg.distortion_samples_per_level
    cands, scores = [], []
    t0 = time.perf_counter()
    for _ in range(cfg.distortion_levels):
        c = np.linspace(lo, hi, n)
        s = np.array([distortion.score_alpha(a, ms, pairs) for a in c])
        k = int(np.argmin(s))
        cands.append(c)
        scores.append(s)
        lo, hi = c[max(k - 1, 0)], c[min(k + 1, n - 1)]
    out["a_ref_seconds"] = np.array(time.perf_counter() - t0)
    out["a_cands"] = np.stack(cands)
    out["a_scores"] = np.stack(scores)
    out["a_alpha"] = np.array(distortion.search_alpha(ms, pairs, cfg))
    # small pairs: every ready pair cut to its first 12 correspondences (M < 16)
    small = [type(p)(p.i, p.j, p.geometry_class, p.correspondences[:12]) for p in pairs]
    out["a_small_scores"] = np.array([distortion.score_alpha(a, ms, small)
                                      for a in (-0.3, 0.0, 0.25)])
    # scene B: two cameras (test_multi_camera_scheduling)
    ms_b, _ = synth.generate(synth.SynthSpec(n_images=10, n_points=250, seed=3, n_cameras=2,
                                             alpha=(-0.15, 0.1)))
    pack("b_", ms_b, out)
    out["b_homography"] = np.array([p.geometry_class is GeometryClass.HOMOGRAPHY for p in ms_b.pairs])
    alphas, unest = distortion.schedule_cameras(ms_b, cfg)
    out["b_alphas"] = np.array([alphas[c] for c in sorted(alphas)])
    out["b_unestimated"] = np.array(unest, dtype=np.int64)
    # undistorted_fundamentals + the focal vote (ref/focal.py:51-172) on both scenes
    for pre, m, al in (("a_", ms, {0: float(out["a_alpha"])}), ("b_", ms_b, alphas)):
        t0 = time.perf_counter()
        fund = focal.undistorted_fundamentals(m, al)
        out[pre + "fund_seconds"] = np.array(time.perf_counter() - t0)
        out[pre + "fund_idx"] = np.array([m.pairs.index(p) for p, _ in fund], dtype=np.int64)
        out[pre + "fund_F"] = np.stack([F for _, F in fund])
        foc, fb = focal.vote_focal_multi(m, fund, cfg)
        out[pre + "focals"] = np.array([foc[c] for c in sorted(foc)])
        im0 = m.images[0]
        out[pre + "votes"] = focal.vote_focal(fund, im0.width, im0.height, cfg)[2]
        if pre == "b_":  # the cross-camera form: camera 1 against camera 0's focal
            out[pre + "votes_cam1"] = focal.vote_focal(
                focal._pairs_for_camera(fund, m.images, 1, {0: foc[0]}), m.images[0].width,
                m.images[0].height, cfg, known={0: foc[0]}, images=m.images, camera_id=1)[2]
    # apply_calibration (ref/focal.py:175-203) on A, B and a planar
    # scene C (homography pairs), with the cameras the pipeline would build
    ms_c, _ = synth.generate(synth.SynthSpec(n_images=8, n_points=200, seed=2,
                                             planar_fraction=1.0))
    pack("c_", ms_c, out)
    out["c_homography"] = np.array([p.geometry_class is GeometryClass.HOMOGRAPHY for p in ms_c.pairs])
    for pre, m, foc, al in (("a_", ms, out["a_focals"], {0: float(out["a_alpha"])}),
                            ("b_", ms_b, out["b_focals"], alphas),
                            ("c_", ms_c, [500.0] * m_cams(ms_c), {})):
        dims = {im.camera_id: (im.width, im.height) for im in m.images}
        cams = {c: CameraModel(float(foc[c]), dims[c][0], dims[c][1], float(al.get(c, 0.0)))
                for c in sorted(dims)}
        t0 = time.perf_counter()
        nk, geo = focal.apply_calibration(m, cams)
        out[pre + "calib_seconds"] = np.array(time.perf_counter() - t0)
        out[pre + "cam"] = np.array([[cams[c].focal, cams[c].alpha] for c in sorted(cams)])
        out[pre + "norm_kps"] = np.concatenate(nk)
        out[pre + "calib_mats"] = np.stack([np.full((3, 3), np.nan) if g is None else g
                                            for _, g in geo])
    # build_tracks + complete_matches (ref/tracks.py:38-106) on A and B, and on
    # B with a small completion cap (oversized tracks keep their edges)
    # scene D: scene B thinned (60% of each pair's correspondences, every 4th
    # pair dropped) plus cross links that merge tracks into same-image
    # conflicts, so completion has pairs and correspondences to add
    from fastmap.model import ImagePairMatches, MatchSet
    rng = np.random.default_rng(7)
    thin = []
    for q, p in enumerate(ms_b.pairs):
        if q % 4 == 3:
            continue
        c = p.correspondences[np.sort(rng.choice(len(p.correspondences),
                                                 int(0.6 * len(p.correspondences)), replace=False))]
        if q % 5 == 0 and len(c) > 2:
            c = np.concatenate([c, [[c[0, 0], c[1, 1]]]])
        thin.append(ImagePairMatches(p.i, p.j, p.geometry_class, c))
    ms_d = MatchSet(images=ms_b.images, keypoints=ms_b.keypoints, pairs=thin)
    pack("d_", ms_d, out)
    out["d_homography"] = np.array([p.geometry_class is GeometryClass.HOMOGRAPHY for p in thin])
    for pre, m, cap in (("a_", ms, 200), ("b_", ms_b, 200), ("d_", ms_d, 200), ("d3_", ms_d, 4)):
        t0 = time.perf_counter()
        ts = tracks.build_tracks(m)
        done = tracks.complete_matches(ts, m, max_track_size=cap)
        out[pre + "tracks_seconds"] = np.array(time.perf_counter() - t0)
        out[pre + "track_len"] = np.array([len(t) for t in ts.tracks], dtype=np.int64)
        out[pre + "track_nodes"] = np.array([x for t in ts.tracks for x in t], dtype=np.int64)
        out[pre + "done_ij"] = np.array([[p.i, p.j] for p in done.pairs], dtype=np.int64)
        out[pre + "done_len"] = np.array([len(p.correspondences) for p in done.pairs], dtype=np.int64)
        out[pre + "done_corr"] = np.concatenate([p.correspondences for p in done.pairs]).astype(np.int64)
        out[pre + "done_synth"] = np.array([p.synthetic_from_tracks for p in done.pairs])
        out[pre + "done_homog"] = np.array([p.geometry_class is GeometryClass.HOMOGRAPHY
                                            for p in done.pairs])
    np.savez_compressed(os.path.join(HERE, "golden_distortion.npz"), **out)
    print({k: v.shape for k, v in out.items()})
    print("scene A alpha", out["a_alpha"], "ref search seconds", out["a_ref_seconds"],
          "scene B alphas", out["b_alphas"])


if __name__ == "__main__":
    main()
