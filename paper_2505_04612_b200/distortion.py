"""Drop-in for the distortion candidate search of ``fastmap.distortion``
(ref/distortion.py:90-161, SURVEY 8f "next" #4) on the B200.

``score_alpha`` undistorts every pair's keypoints with the candidate alpha
(the reference's numpy expressions, ref/distortion.py:18-55), then runs the
robust fundamental-matrix fit and error sum of every pair on the device in
one launch (``fm_fund_score``: one CTA per (candidate, pair) job).
``search_alpha`` scores all candidates of a level in that single launch.
The LMedS minimal samples are the reference's own seeded numpy draws
(ref/twoview.py:86-88), generated once per point count M and cached.

Semantics follow the reference: pairs with fewer than 8 valid points or a
degenerate fit are skipped; a candidate with no usable pair raises
``DegenerateGeometryError`` (install() rebinds the name to the reference's
class).
"""

import functools

import numpy as np
import torch

from . import _native as N

_DENOM_EPS = 1e-6        # ref/distortion.py:15
_LMEDS_ITERS = 64        # ref/twoview.py:44
_LMEDS_SEED = 12345      # ref/twoview.py:45


class DegenerateGeometryError(ValueError):
    """ref/twoview.py:14-15 (install() rebinds it to the reference class)."""


def undistort_normalized(xy, alpha):
    """ref/distortion.py:18-28 (same numpy expressions)."""
    xy = np.asarray(xy, dtype=np.float64)
    r2 = np.sum(xy ** 2, axis=-1, keepdims=True)
    denom = 1.0 + alpha * r2
    denom = np.where(denom > _DENOM_EPS, denom, np.nan)
    return xy / denom


def _geom(match_set, image_id):
    """(cx, cy, half_diagonal) of the geometry-only camera of ref/distortion.py:129-134."""
    im = match_set.images[image_id]
    return np.array([im.width / 2.0, im.height / 2.0]), 0.5 * float(np.hypot(im.width, im.height))


def _undistort_pixels(px, center, s, alpha):
    """ref/distortion.py:58-64 with the geometry-only camera."""
    xn = (np.asarray(px, dtype=np.float64) - center) / s
    return undistort_normalized(xn, alpha) * s + center


@functools.lru_cache(maxsize=4096)
def lmeds_samples(M):
    """The reference's 64 minimal samples for M points (ref/twoview.py:86-88):
    rng(12345).choice(M, 8, replace=False), 64 times -> (64, 8) int32."""
    rng = np.random.default_rng(_LMEDS_SEED)
    return np.stack([rng.choice(M, 8, replace=False) for _ in range(_LMEDS_ITERS)]).astype(np.int32)


def _jobs(alphas, match_set, pairs, camera_id, known_alphas):
    """Host side of score_alpha (ref/distortion.py:99-118) for every
    candidate, vectorised over all pairs (the same elementwise numpy
    expressions, so every value equals the per-pair computation): the scaled
    undistorted point pairs of each (candidate, pair) job with >= 8 valid
    points, concatenated.  Returns (candidate of each job, lengths, p1, p2)."""
    known_alphas = known_alphas or {}
    kp_i = np.concatenate([match_set.keypoints[p.i][p.correspondences[:, 0]] for p in pairs])
    kp_j = np.concatenate([match_set.keypoints[p.j][p.correspondences[:, 1]] for p in pairs])
    kp_i = np.asarray(kp_i, dtype=np.float64)
    kp_j = np.asarray(kp_j, dtype=np.float64)
    lens = np.array([len(p.correspondences) for p in pairs], dtype=np.int64)
    seg = np.repeat(np.arange(len(pairs)), lens)  # pair of every point
    geo_i = [_geom(match_set, p.i) for p in pairs]
    geo_j = [_geom(match_set, p.j) for p in pairs]
    c_i = np.repeat(np.stack([g[0] for g in geo_i]), lens, axis=0)
    c_j = np.repeat(np.stack([g[0] for g in geo_j]), lens, axis=0)
    s_i = np.repeat(np.array([g[1] for g in geo_i]), lens)[:, None]
    s_j = np.repeat(np.array([g[1] for g in geo_j]), lens)[:, None]
    cam_i = np.array([match_set.images[p.i].camera_id for p in pairs])
    cam_j = np.array([match_set.images[p.j].camera_id for p in pairs])
    xn_i = (kp_i - c_i) / s_i
    xn_j = (kp_j - c_j) / s_j
    # all candidates at once: (C, n, 2); every element sees the same operations
    def alpha_for(alpha, cam):
        if camera_id is None or cam == camera_id:
            return alpha
        return known_alphas[cam]

    a_i = np.array([[alpha_for(a, k) for k in cam_i] for a in alphas], dtype=np.float64)
    a_j = np.array([[alpha_for(a, k) for k in cam_j] for a in alphas], dtype=np.float64)
    a_i = np.repeat(a_i, lens, axis=1)[:, :, None]
    a_j = np.repeat(a_j, lens, axis=1)[:, :, None]
    u_i = undistort_normalized(xn_i[None], a_i) * s_i[None] + c_i[None]
    u_j = undistort_normalized(xn_j[None], a_j) * s_j[None] + c_j[None]
    ok = np.all(np.isfinite(u_i), axis=2) & np.all(np.isfinite(u_j), axis=2)  # (C, n)
    C, P = len(alphas), len(pairs)
    n_ok = np.bincount((np.arange(C)[:, None] * P + seg[None, :]).ravel(), weights=ok.ravel(),
                       minlength=C * P).astype(np.int64).reshape(C, P)
    good = n_ok >= 8
    use = ok & np.repeat(good, lens, axis=1)
    s_full = np.broadcast_to(s_i[None], (C,) + s_i.shape)
    return (np.nonzero(good)[0].astype(np.int64), n_ok[good], u_i[use] / s_full[use],
            u_j[use] / s_full[use])


def fit_jobs(lens, p1, p2, want_F=False):
    """One fm_fund_score launch over concatenated jobs (lens[k] >= 8 point
    pairs each, p1/p2 (sum lens, 2) fp64).  Returns (error sums, point counts
    (0 = degenerate fit), F (n_jobs, 3, 3) or None)."""
    device = N.require_cuda()
    lib = N.lib()
    lens = np.asarray(lens, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)])
    tables, s_off, at = [], [], 0
    seen = {}
    for M in lens:
        if M < 16:
            s_off.append(-1)
            continue
        if M not in seen:
            seen[M] = at
            tables.append(lmeds_samples(int(M)).ravel())
            at += 8 * _LMEDS_ITERS
        s_off.append(seen[M])
    samples = np.concatenate(tables) if tables else np.zeros(1, dtype=np.int32)
    n_pts = int(off[-1])
    P1 = torch.as_tensor(np.ascontiguousarray(p1, dtype=np.float64), device=device)
    P2 = torch.as_tensor(np.ascontiguousarray(p2, dtype=np.float64), device=device)
    off_d = torch.as_tensor(off, device=device)
    samp_d = torch.as_tensor(samples, device=device)
    soff_d = torch.as_tensor(np.array(s_off, dtype=np.int64), device=device)
    err = torch.empty(len(lens), dtype=torch.float64, device=device)
    nerr = torch.empty(len(lens), dtype=torch.int32, device=device)
    F = torch.empty((len(lens), 9), dtype=torch.float64, device=device) if want_F else None
    nbytes = int(lib.fm_fund_scratch_bytes(n_pts))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=device)
    N.check(lib.fm_fund_score(len(lens), N.ptr(off_d), N.ptr(P1), N.ptr(P2), N.ptr(samp_d),
                              N.ptr(soff_d), N.ptr(err), N.ptr(nerr),
                              N.ptr(F) if want_F else None, N.ptr(scratch), nbytes, n_pts,
                              N.stream_handle()))
    return (err.cpu().numpy(), nerr.cpu().numpy(),
            F.cpu().numpy().reshape(-1, 3, 3) if want_F else None)


def estimate_fundamental_batch(p1s, p2s):
    """estimate_fundamental (ref/twoview.py:58-76) for many point sets in one
    launch: a list of F (Frobenius-normalised, rank 2) or None where the
    reference raises DegenerateGeometryError (fewer than 8 points or a
    degenerate fit)."""
    out = [None] * len(p1s)
    keep = [k for k in range(len(p1s)) if len(p1s[k]) >= 8]
    if not keep:
        return out
    lens = [len(p1s[k]) for k in keep]
    _, nerr, F = fit_jobs(lens, np.concatenate([np.asarray(p1s[k], np.float64) for k in keep]),
                          np.concatenate([np.asarray(p2s[k], np.float64) for k in keep]),
                          want_F=True)
    for q, k in enumerate(keep):
        if nerr[q]:
            out[k] = F[q]
    return out


@functools.lru_cache(maxsize=4096)
def lmeds_samples4(M):
    """The reference's homography samples for M points (ref/twoview.py:157-161):
    one rng(12345), 64 sequential choice(M, 4, replace=False) -> (64, 4) int32."""
    rng = np.random.default_rng(_LMEDS_SEED)
    return np.stack([rng.choice(M, 4, replace=False) for _ in range(_LMEDS_ITERS)]).astype(np.int32)


def estimate_homography_batch(p1s, p2s):
    """estimate_homography (ref/twoview.py:136-153) for many point sets in one
    launch (fm_homog_fit): a list of H (Frobenius-normalised, positive trace)
    or None where the reference raises DegenerateGeometryError."""
    out = [None] * len(p1s)
    keep = [k for k in range(len(p1s)) if len(p1s[k]) >= 4]
    if not keep:
        return out
    device = N.require_cuda()
    lib = N.lib()
    lens = np.array([len(p1s[k]) for k in keep], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)])
    tables, s_off, at, seen = [], [], 0, {}
    for M in lens:
        if M < 12:
            s_off.append(-1)
            continue
        if M not in seen:
            seen[M] = at
            tables.append(lmeds_samples4(int(M)).ravel())
            at += 4 * _LMEDS_ITERS
        s_off.append(seen[M])
    samples = np.concatenate(tables) if tables else np.zeros(1, dtype=np.int32)
    n_pts = int(off[-1])
    P1 = torch.as_tensor(np.concatenate([np.asarray(p1s[k], np.float64) for k in keep]), device=device)
    P2 = torch.as_tensor(np.concatenate([np.asarray(p2s[k], np.float64) for k in keep]), device=device)
    off_d = torch.as_tensor(off, device=device)
    samp_d = torch.as_tensor(samples, device=device)
    soff_d = torch.as_tensor(np.array(s_off, dtype=np.int64), device=device)
    H = torch.empty((len(keep), 9), dtype=torch.float64, device=device)
    nbytes = int(lib.fm_fund_scratch_bytes(n_pts))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=device)
    N.check(lib.fm_homog_fit(len(keep), N.ptr(off_d), N.ptr(P1), N.ptr(P2), N.ptr(samp_d),
                             N.ptr(soff_d), N.ptr(H), N.ptr(scratch), nbytes, n_pts,
                             N.stream_handle()))
    H = H.cpu().numpy().reshape(-1, 3, 3)
    for q, k in enumerate(keep):
        if np.all(np.isfinite(H[q])):
            out[k] = H[q]
    return out


def score_alpha_batch(alphas, match_set, pairs, camera_id=None, known_alphas=None):
    """score_alpha (ref/distortion.py:90-126) for several candidates in one
    device launch.  Returns the scores in candidate order; raises like the
    reference at the first candidate without a usable pair."""
    if not pairs:
        raise DegenerateGeometryError("no usable fundamental-matrix pairs")
    alphas = [float(a) for a in alphas]
    job_cand, lens, p1, p2 = _jobs(alphas, match_set, pairs, camera_id, known_alphas)
    total = np.zeros(len(alphas))
    count = np.zeros(len(alphas), dtype=np.int64)
    if len(lens):
        err, nerr, _ = fit_jobs(lens, p1, p2)
        for q, c in enumerate(job_cand):  # pair order within a candidate, as the reference
            if nerr[q]:
                total[c] += float(err[q])
                count[c] += int(nerr[q])
    scores = []
    for c in range(len(alphas)):
        if count[c] == 0:
            raise DegenerateGeometryError("no pair could be scored")
        scores.append(total[c] / count[c])
    return np.array(scores)


def score_alpha(alpha, match_set, pairs, camera_id=None, known_alphas=None):
    """ref/distortion.py:90-126: mean epipolar error after undistorting with
    ``alpha`` and re-fitting each pair's fundamental matrix."""
    return float(score_alpha_batch([alpha], match_set, pairs, camera_id, known_alphas)[0])


def search_alpha(match_set, pairs, cfg, camera_id=None, known_alphas=None):
    """ref/distortion.py:137-161: hierarchical interval search, every level's
    candidates scored in one device launch."""
    lo, hi = cfg.distortion_min, cfg.distortion_max
    n = cfg.distortion_samples_per_level
    if len(pairs) > cfg.distortion_max_pairs:
        idx = np.linspace(0, len(pairs) - 1, cfg.distortion_max_pairs)
        pairs = [pairs[int(k)] for k in idx]
    best_alpha = 0.0
    for _ in range(cfg.distortion_levels):
        candidates = np.linspace(lo, hi, n)
        scores = score_alpha_batch(candidates, match_set, pairs, camera_id, known_alphas)
        k = int(np.argmin(scores))
        best_alpha = float(candidates[k])
        lo = candidates[max(k - 1, 0)]
        hi = candidates[min(k + 1, n - 1)]
    return best_alpha


def _is_homography(pair):
    gc = pair.geometry_class
    return getattr(gc, "name", str(gc)) == "HOMOGRAPHY"


def ready_fundamental_pairs(match_set, camera_id=None, known_alphas=None):
    """ref/distortion.py:67-87 (host logic, same rules and order)."""
    known_alphas = known_alphas or {}
    out = []
    for pair in match_set.pairs:
        if _is_homography(pair) or len(pair.correspondences) < 8:
            continue
        if camera_id is None:
            out.append(pair)
            continue
        cam_i = match_set.images[pair.i].camera_id
        cam_j = match_set.images[pair.j].camera_id
        if (cam_i == camera_id and cam_j == camera_id) or \
                (cam_i == camera_id and cam_j in known_alphas) or \
                (cam_j == camera_id and cam_i in known_alphas):
            out.append(pair)
    return out


def schedule_cameras(match_set, cfg):
    """ref/distortion.py:164-193 (host scheduling around the device search):
    cameras by descending ready-pair count; never-ready cameras get 0."""
    n_cameras = max(im.camera_id for im in match_set.images) + 1 if match_set.images else 0
    if n_cameras == 1:
        pairs = ready_fundamental_pairs(match_set)
        if not pairs:
            return {0: 0.0}, [0]
        return {0: search_alpha(match_set, pairs, cfg, None)}, []
    alphas, unestimated = {}, []
    remaining = set(range(n_cameras))
    while remaining:
        ready = {cam: ready_fundamental_pairs(match_set, cam, alphas) for cam in remaining}
        cam = max(remaining, key=lambda c: (len(ready[c]), -c))
        if not ready[cam]:
            unestimated.extend(sorted(remaining))
            for c in remaining:
                alphas[c] = 0.0
            break
        alphas[cam] = search_alpha(match_set, ready[cam], cfg, cam, alphas)
        remaining.discard(cam)
    return alphas, unestimated


__all__ = ["DegenerateGeometryError", "undistort_normalized", "lmeds_samples", "fit_jobs",
           "estimate_fundamental_batch", "lmeds_samples4", "estimate_homography_batch", "score_alpha",
           "score_alpha_batch", "search_alpha", "ready_fundamental_pairs", "schedule_cameras"]
