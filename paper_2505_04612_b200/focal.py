"""Drop-in for the per-pair geometry refits of ``fastmap.focal``
(ref/focal.py:51-78 and :175-203, reached from ref/pipeline.py:105 and
:123; SURVEY 8f "next" #2/#4).

``undistorted_fundamentals`` undistorts every fundamental pair's keypoints
with its camera's alpha (the reference's numpy expressions) and fits all
pairs' robust fundamental matrices in one device launch
(``distortion.estimate_fundamental_batch`` -> ``fm_fund_score``).
``vote_focal`` scores every FoV candidate against every fundamental matrix
in one launch (``fm_focal_votes``); the candidate focals are computed with
the reference's numpy expressions.  ``apply_calibration`` refits all pairs
in two launches (F and H).
"""


class FocalUnderdeterminedError(ValueError):
    """ref/focal.py:16-17 (install() rebinds it to the reference class)."""


def fov_to_focal(fov_deg, width):
    """ref/focal.py:20-21."""
    return (width / 2.0) / np.tan(np.radians(fov_deg) / 2.0)


def vote_focal(fundamentals, width, height, cfg, known=None, images=None, camera_id=None):
    """ref/focal.py:81-120: (focal_px, fov_deg, votes) -- the FoV candidate
    whose K makes the fundamentals most essential-like, summed validity
    exp((1 - s0/s1) / tau) per candidate."""
    if not fundamentals:
        raise FocalUnderdeterminedError("focal underdetermined: no fundamental matrices")
    fovs = np.linspace(cfg.fov_min_deg, cfg.fov_max_deg, cfg.focal_samples)
    known = known or {}
    C, P = len(fovs), len(fundamentals)
    focal = np.empty((C, P, 2))
    principal = np.empty((P, 4))
    for q, (pair, _) in enumerate(fundamentals):
        if images is None or camera_id is None:
            focal[:, q, 0] = focal[:, q, 1] = fov_to_focal(fovs, width)
            principal[q] = (width / 2.0, height / 2.0, width / 2.0, height / 2.0)
            continue
        for side, img_id in enumerate((pair.i, pair.j)):
            im = images[img_id]
            if im.camera_id == camera_id:
                focal[:, q, side] = fov_to_focal(fovs, im.width)
            else:
                focal[:, q, side] = known[im.camera_id]
            principal[q, 2 * side:2 * side + 2] = (im.width / 2.0, im.height / 2.0)
    device = N.require_cuda()
    F = torch.as_tensor(np.ascontiguousarray(np.stack([F for _, F in fundamentals]), dtype=np.float64),
                        device=device)
    foc = torch.as_tensor(focal, device=device)
    pp = torch.as_tensor(principal, device=device)
    votes = torch.empty(C, dtype=torch.float64, device=device)
    N.check(N.lib().fm_focal_votes(C, P, N.ptr(F), N.ptr(foc), N.ptr(pp), float(cfg.tau),
                                   N.ptr(votes), N.stream_handle()))
    votes = votes.cpu().numpy()
    best = int(np.argmax(votes))
    return float(fov_to_focal(fovs[best], width)), float(fovs[best]), votes


import numpy as np
import torch

from . import _native as N
from .distortion import (_is_homography, estimate_fundamental_batch, estimate_homography_batch,
                         undistort_normalized)


def undistorted_fundamentals(match_set, alphas):
    """ref/focal.py:51-78: (pair, F) for every fundamental pair with >= 8
    valid undistorted points and a non-degenerate fit, in pair order; F is
    fitted on the undistorted pixel coordinates."""
    cand, p1s, p2s = [], [], []
    for pair in match_set.pairs:
        if _is_homography(pair) or len(pair.correspondences) < 8:
            continue
        im_i, im_j = match_set.images[pair.i], match_set.images[pair.j]
        u = []
        for im, kp in ((im_i, match_set.keypoints[pair.i][pair.correspondences[:, 0]]),
                       (im_j, match_set.keypoints[pair.j][pair.correspondences[:, 1]])):
            s = 0.5 * float(np.hypot(im.width, im.height))
            center = np.array([im.width / 2.0, im.height / 2.0])
            xn = (np.asarray(kp, dtype=np.float64) - center) / s
            u.append(undistort_normalized(xn, alphas.get(im.camera_id, 0.0)) * s + center)
        ok = np.all(np.isfinite(u[0]), axis=1) & np.all(np.isfinite(u[1]), axis=1)
        if ok.sum() < 8:
            continue
        cand.append(pair)
        p1s.append(u[0][ok])
        p2s.append(u[1][ok])
    Fs = estimate_fundamental_batch(p1s, p2s)
    return [(pair, F) for pair, F in zip(cand, Fs) if F is not None]


def apply_calibration(match_set, cameras):
    """ref/focal.py:175-203: normalised homogeneous keypoints per image
    (undistort with the camera's alpha, subtract the principal point, divide
    by the focal -- the reference's numpy expressions) and every pair's
    geometry refit in normalised coordinates, all fundamental pairs in one
    device launch and all homography pairs in another.  Returns
    (norm_kps, [(pair, matrix or None)]) in pair order."""
    norm_kps = []
    for im in match_set.images:
        cam = cameras[im.camera_id]
        s = cam.half_diagonal
        center = np.array([cam.cx, cam.cy])
        xn = (np.asarray(match_set.keypoints[im.image_id], dtype=np.float64) - center) / s
        und = undistort_normalized(xn, cam.alpha) * s + center
        xy = (und - np.array([cam.cx, cam.cy])) / cam.focal
        norm_kps.append(np.concatenate([xy, np.ones(xy.shape[:-1] + (1,))], axis=-1))
    fund, homog = [], []
    for q, pair in enumerate(match_set.pairs):
        x1 = norm_kps[pair.i][pair.correspondences[:, 0]][:, :2]
        x2 = norm_kps[pair.j][pair.correspondences[:, 1]][:, :2]
        ok = np.all(np.isfinite(x1), axis=1) & np.all(np.isfinite(x2), axis=1)
        (homog if _is_homography(pair) else fund).append((q, x1[ok], x2[ok]))
    mats = [None] * len(match_set.pairs)
    for group, fit in ((fund, estimate_fundamental_batch), (homog, estimate_homography_batch)):
        if group:
            res = fit([a for _, a, _ in group], [b for _, _, b in group])
            for (q, _, _), m in zip(group, res):
                mats[q] = m
    return norm_kps, [(pair, m) for pair, m in zip(match_set.pairs, mats)]


__all__ = ["FocalUnderdeterminedError", "fov_to_focal", "vote_focal", "undistorted_fundamentals",
           "apply_calibration"]
