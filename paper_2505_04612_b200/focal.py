"""Drop-in for the per-pair fundamental refits of ``fastmap.focal``
(ref/focal.py:51-78, reached from ref/pipeline.py:105; SURVEY 8f "next" #4).

``undistorted_fundamentals`` undistorts every fundamental pair's keypoints
with its camera's alpha (the reference's numpy expressions) and fits all
pairs' robust fundamental matrices in one device launch
(``distortion.estimate_fundamental_batch`` -> ``fm_fund_score``).  The
focal vote itself (``vote_focal``, a few 3x3 SVDs per candidate) stays the
reference's.
"""

import numpy as np

from .distortion import _is_homography, estimate_fundamental_batch, undistort_normalized


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


__all__ = ["undistorted_fundamentals"]
