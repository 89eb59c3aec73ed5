"""Distortion candidate search (SURVEY 8f "next" #4) against the reference's
own outputs recorded in tests/golden/golden_distortion.npz
(make_distortion_golden.py): every candidate score of the three search
levels, the searched alpha, the M < 16 (non-LMedS) branch, and the
two-camera schedule of pkg/tests/test_distortion.py:70-80."""

import os
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_distortion.npz")


def _match_set(g, p):
    img = g[p + "img"]
    kp = np.split(g[p + "kp"], np.cumsum(g[p + "kp_len"])[:-1])
    corr = np.split(g[p + "corr"], np.cumsum(g[p + "pair_len"])[:-1])
    homog = g[p + "homography"]
    images = [SimpleNamespace(image_id=k, camera_id=int(c), width=int(w), height=int(h))
              for k, (c, w, h) in enumerate(img)]
    pairs = [SimpleNamespace(i=int(i), j=int(j), correspondences=c,
                             geometry_class=SimpleNamespace(name="HOMOGRAPHY" if h else "FUNDAMENTAL"))
             for (i, j), c, h in zip(g[p + "pair_ij"], corr, homog)]
    return SimpleNamespace(images=images, keypoints=kp, pairs=pairs)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _cfg():
    from paper_2505_04612_b200.config import HotPathConfig
    c = HotPathConfig()
    for k, v in dict(distortion_levels=3, distortion_samples_per_level=10, distortion_min=-1.0,
                     distortion_max=1.0, distortion_max_pairs=120).items():
        setattr(c, k, v)
    return c


def test_candidate_scores_match_reference(golden):
    """All 30 candidate scores of the reference's 3-level search (LMedS
    branch, M = 200): the fit is the same algorithm with the same seeded
    samples; only summation orders and the eigen-solver differ."""
    from paper_2505_04612_b200 import distortion as D
    ms = _match_set(golden, "a_")
    pairs = [ms.pairs[k] for k in golden["a_ready"]]
    assert [id(p) for p in D.ready_fundamental_pairs(ms)] == [id(p) for p in pairs]
    for cands, ref in zip(golden["a_cands"], golden["a_scores"]):
        got = D.score_alpha_batch(cands, ms, pairs)
        np.testing.assert_allclose(got, ref, rtol=1e-8)
        assert int(np.argmin(got)) == int(np.argmin(ref))


def test_search_alpha_matches_reference(golden):
    from paper_2505_04612_b200 import distortion as D
    ms = _match_set(golden, "a_")
    pairs = [ms.pairs[k] for k in golden["a_ready"]]
    assert D.search_alpha(ms, pairs, _cfg()) == float(golden["a_alpha"])
    assert D.score_alpha(float(golden["a_cands"][0, 3]), ms, pairs) == pytest.approx(
        float(golden["a_scores"][0, 3]), rel=1e-8)


def test_small_pairs_use_the_plain_fit(golden):
    """12 correspondences per pair: no LMedS (M < 16), least squares + refit."""
    from paper_2505_04612_b200 import distortion as D
    ms = _match_set(golden, "a_")
    small = [SimpleNamespace(i=p.i, j=p.j, correspondences=p.correspondences[:12],
                             geometry_class=p.geometry_class)
             for p in (ms.pairs[k] for k in golden["a_ready"])]
    got = D.score_alpha_batch([-0.3, 0.0, 0.25], ms, small)
    np.testing.assert_allclose(got, golden["a_small_scores"], rtol=1e-8)


def test_two_camera_schedule_matches_reference(golden):
    from paper_2505_04612_b200 import distortion as D
    ms = _match_set(golden, "b_")
    alphas, unest = D.schedule_cameras(ms, _cfg())
    assert [alphas[c] for c in sorted(alphas)] == list(golden["b_alphas"])
    assert unest == list(golden["b_unestimated"])


def test_degenerate_inputs_raise_like_reference(golden):
    from paper_2505_04612_b200 import distortion as D
    ms = _match_set(golden, "a_")
    with pytest.raises(D.DegenerateGeometryError):
        D.score_alpha(0.0, ms, [])
    tiny = [SimpleNamespace(i=p.i, j=p.j, correspondences=p.correspondences[:7],
                            geometry_class=p.geometry_class) for p in ms.pairs[:3]]
    with pytest.raises(D.DegenerateGeometryError):  # every pair below 8 points: none scored
        D.score_alpha(0.0, ms, tiny)


@pytest.mark.parametrize("scene", ["a_", "b_"])
def test_undistorted_fundamentals_match_reference(golden, scene):
    """ref/focal.py:51-78 on both scenes with the searched alphas: the same
    pairs survive, and every F equals the reference's up to its sign (the
    eigenvector sign is solver-dependent; the focal vote uses singular
    values only)."""
    from paper_2505_04612_b200 import focal
    ms = _match_set(golden, scene)
    al = ({0: float(golden["a_alpha"])} if scene == "a_"
          else {c: float(a) for c, a in enumerate(golden["b_alphas"])})
    got = focal.undistorted_fundamentals(ms, al)
    assert [ms.pairs.index(p) for p, _ in got] == list(golden[scene + "fund_idx"])
    for (_, F), R in zip(got, golden[scene + "fund_F"]):
        d = min(np.abs(F - R).max(), np.abs(F + R).max())
        assert d < 1e-7, d


@pytest.mark.parametrize("scene", ["a_", "b_", "c_"])
def test_apply_calibration_matches_reference(golden, scene):
    """ref/focal.py:175-203 with the pipeline's cameras: normalised keypoints
    bit-identical (same numpy expressions), every pair's refit essential
    matrix (scenes a, b) or homography (scene c: all pairs planar) within
    1e-7 -- E up to sign, H exactly signed (positive trace)."""
    from paper_2505_04612_b200 import focal
    ms = _match_set(golden, scene)
    cams = {}
    for c, (f, a) in enumerate(golden[scene + "cam"]):
        im = next(i for i in ms.images if i.camera_id == c)
        w, h = im.width, im.height
        cams[c] = SimpleNamespace(focal=float(f), alpha=float(a), cx=w / 2.0, cy=h / 2.0,
                                  half_diagonal=0.5 * float(np.hypot(w, h)))
    nk, geo = focal.apply_calibration(ms, cams)
    assert np.array_equal(np.concatenate(nk), golden[scene + "norm_kps"])
    ref = golden[scene + "calib_mats"]
    assert len(geo) == len(ref)
    homog = golden[scene + "homography"]
    for (pair, m), r, hg in zip(geo, ref, homog):
        assert (m is None) == bool(np.isnan(r).any())
        if m is None:
            continue
        d = np.abs(m - r).max() if hg else min(np.abs(m - r).max(), np.abs(m + r).max())
        assert d < 1e-7, (pair.i, pair.j, d)


def test_focal_votes_match_reference(golden):
    """ref/focal.py:81-120: all 100 FoV candidate votes within 1e-9 and the
    same winner -- one camera (scene a) and the cross-camera form (scene b,
    camera 1 voted against camera 0's known focal)."""
    from paper_2505_04612_b200 import focal
    cfg = SimpleNamespace(fov_min_deg=20.0, fov_max_deg=160.0, focal_samples=100, tau=0.01)
    ms = _match_set(golden, "a_")
    fund = focal.undistorted_fundamentals(ms, {0: float(golden["a_alpha"])})
    im0 = ms.images[0]
    f, fov, votes = focal.vote_focal(fund, im0.width, im0.height, cfg)
    np.testing.assert_allclose(votes, golden["a_votes"], rtol=1e-9, atol=1e-300)
    assert f == pytest.approx(float(golden["a_focals"][0]), rel=1e-15)
    ms = _match_set(golden, "b_")
    al = {c: float(a) for c, a in enumerate(golden["b_alphas"])}
    fund = focal.undistorted_fundamentals(ms, al)
    f0 = float(golden["b_focals"][0])
    mine = [(p, F) for p, F in fund
            if {ms.images[p.i].camera_id, ms.images[p.j].camera_id} <= {0, 1}
            and 1 in (ms.images[p.i].camera_id, ms.images[p.j].camera_id)]
    _, _, votes = focal.vote_focal(mine, ms.images[0].width, ms.images[0].height, cfg,
                                   known={0: f0}, images=ms.images, camera_id=1)
    np.testing.assert_allclose(votes, golden["b_votes_cam1"], rtol=1e-9, atol=1e-300)
    assert int(np.argmax(votes)) == int(np.argmax(golden["b_votes_cam1"]))
    with pytest.raises(focal.FocalUnderdeterminedError):
        focal.vote_focal([], 640, 480, cfg)


def test_empty_and_short_pairs_are_skipped(golden):
    """Pairs with 0 or < 8 valid correspondences contribute nothing (as the
    reference's `ok.sum() < 8: continue`), wherever they sit in the list."""
    from paper_2505_04612_b200 import distortion as D
    ms = _match_set(golden, "a_")
    pairs = [ms.pairs[k] for k in golden["a_ready"]]
    empty = SimpleNamespace(i=pairs[0].i, j=pairs[0].j, geometry_class=pairs[0].geometry_class,
                            correspondences=np.zeros((0, 2), dtype=np.int64))
    short = SimpleNamespace(i=pairs[1].i, j=pairs[1].j, geometry_class=pairs[1].geometry_class,
                            correspondences=pairs[1].correspondences[:5])
    cands = golden["a_cands"][0]
    got = D.score_alpha_batch(cands, ms, [empty] + pairs + [short, empty])
    np.testing.assert_allclose(got, golden["a_scores"][0], rtol=1e-8)
