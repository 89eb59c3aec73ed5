"""CPU oracle of the FastMap hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (FastMap, arXiv 2505.04612,
reference package /root/reference/pkg/src/fastmap) for the two gradient
stages the B200 library replaces.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg may import this module, and only as the
checker / the timed CPU path -- never as part of the product.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports /root/reference and writes
``tests/golden/*.npz``).

Formulation differences from the reference (same mathematics):
* point pairs live in one flat array with a per-point pair index instead of
  per-pair Python objects; per-pair sums are segment sums (np.add.reduceat);
* the Jacobian of the 6D map is applied as a vector-Jacobian product;
* epipolar scatters use np.bincount instead of np.add.at; the translation
  functions keep the reference's np.add.at calls in the reference's order, so
  they are bitwise the reference (the CUDA translation path is held to that).
"""

import numpy as np

HUBER_EPS = 1e-6   # ref/epipolar.py:16
NORM_EPS = 1e-8    # ref/translation.py:15


# --------------------------------------------------------------- optimizer
class Adam:
    """Bias-corrected Adam on a flat fp64 vector (ref/optim.py:11-36)."""

    def __init__(self, params, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        self.params = np.array(params, dtype=np.float64, copy=True)
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.m = np.zeros_like(self.params)
        self.v = np.zeros_like(self.params)
        self.t = 0

    def step(self, g):
        g = np.asarray(g, dtype=np.float64)
        if g.shape != self.params.shape:
            raise ValueError("gradient shape mismatch")
        if not np.isfinite(g).all():
            raise FloatingPointError("non-finite gradients")
        self.t += 1
        self.m = self.beta1 * self.m + (1.0 - self.beta1) * g
        self.v = self.beta2 * self.v + (1.0 - self.beta2) * g ** 2
        mh = self.m / (1.0 - self.beta1 ** self.t)
        vh = self.v / (1.0 - self.beta2 ** self.t)
        self.params -= self.lr * mh / (np.sqrt(vh) + self.eps)
        return self.params


# ------------------------------------------------------------ 6D rotations
def rot6d_to_matrix(v):
    """Gram-Schmidt 6D -> SO(3), columns (b1, b2, b1 x b2) (ref/optim.py:39-59)."""
    v = np.asarray(v, dtype=np.float64)
    a, b = v[..., :3], v[..., 3:]
    na = np.sqrt(np.sum(a * a, axis=-1, keepdims=True))
    if np.any(na < 1e-12):
        raise ValueError("degenerate 6D rotation input: zero first half")
    e = a / na
    u = b - np.sum(e * b, axis=-1, keepdims=True) * e
    nu = np.sqrt(np.sum(u * u, axis=-1, keepdims=True))
    if np.any(nu < 1e-12):
        raise ValueError("degenerate 6D rotation input: collinear halves")
    f = u / nu
    return np.stack([e, f, np.cross(e, f)], axis=-1)


def rot6d_vjp(v, gR):
    """J(v)^T vec(gR) for the 6D map, batched (..., 6), (..., 3, 3)."""
    v = np.asarray(v, dtype=np.float64)
    a, b = v[..., :3], v[..., 3:]
    na = np.linalg.norm(a, axis=-1, keepdims=True)
    e = a / na
    d = np.sum(e * b, axis=-1, keepdims=True)
    u = b - d * e
    nu = np.linalg.norm(u, axis=-1, keepdims=True)
    f = u / nu
    ge = gR[..., :, 0] + np.cross(f, gR[..., :, 2])
    gf = gR[..., :, 1] + np.cross(gR[..., :, 2], e)
    gu = (gf - f * np.sum(f * gf, axis=-1, keepdims=True)) / nu
    eg = np.sum(e * gu, axis=-1, keepdims=True)
    gb = gu - e * eg
    ge = ge - eg * b - d * gu
    ga = (ge - e * np.sum(e * ge, axis=-1, keepdims=True)) / na
    return np.concatenate([ga, gb], axis=-1)


def rot6d_jacobian(v):
    """(…, 9, 6) Jacobian, rows = row-major flat R (ref/optim.py:68-110)."""
    v = np.asarray(v, dtype=np.float64)
    rows = []
    for k in range(9):
        gR = np.zeros(v.shape[:-1] + (3, 3))
        gR[..., k // 3, k % 3] = 1.0
        rows.append(rot6d_vjp(v, gR))
    return np.stack(rows, axis=-2)


def project_to_so3(R):
    """U diag(1, 1, sign det(U V^T)) V^T (ref/model.py:112-116)."""
    U, _, Vt = np.linalg.svd(np.asarray(R, dtype=np.float64))
    s = np.sign(np.linalg.det(U @ Vt))
    D = np.zeros(U.shape[:-2] + (3, 3))
    D[..., 0, 0] = 1.0
    D[..., 1, 1] = 1.0
    D[..., 2, 2] = s
    return U @ D @ Vt


def skew(t):
    t = np.asarray(t, dtype=np.float64)
    z = np.zeros(t.shape[:-1])
    return np.stack([np.stack([z, -t[..., 2], t[..., 1]], -1),
                     np.stack([t[..., 2], z, -t[..., 0]], -1),
                     np.stack([-t[..., 1], t[..., 0], z], -1)], -2)


# ------------------------------------------------------- epipolar geometry
def unpack(params, n, refine_focal):
    """Packed [rot6d | centers | log_focal] (ref/epipolar.py:95-106)."""
    params = np.asarray(params, dtype=np.float64)
    rot6d = params[:6 * n].reshape(n, 6)
    centers = params[6 * n:9 * n].reshape(n, 3)
    log_focal = params[9 * n:] if refine_focal else None
    return rot6d, centers, log_focal


def pair_forward(params, n, idx_i, idx_j, cam_i, cam_j, refine_focal):
    """Normalised per-pair G (ref/epipolar.py:109-138) and intermediates."""
    rot6d, centers, log_focal = unpack(params, n, refine_focal)
    R = rot6d_to_matrix(rot6d)
    Ri, Rj = R[idx_i], R[idx_j]
    dc = centers[idx_j] - centers[idx_i]
    t = -np.einsum("pab,pb->pa", Rj, dc)
    Rrel = Rj @ np.swapaxes(Ri, 1, 2)
    E = skew(t) @ Rrel
    if refine_focal:
        di = np.exp(-log_focal[cam_i])
        dj = np.exp(-log_focal[cam_j])
        sj = np.stack([dj, dj, np.ones_like(dj)], -1)[:, :, None]
        si = np.stack([di, di, np.ones_like(di)], -1)[:, None, :]
        G = sj * E * si
    else:
        di = dj = si = sj = None
        G = E
    g = G.reshape(-1, 9)
    nrm = np.maximum(np.linalg.norm(g, axis=1, keepdims=True), 1e-15)
    return dict(R=R, Ri=Ri, Rj=Rj, dc=dc, t=t, Rrel=Rrel, E=E, G=G, di=di, dj=dj,
                si=si, sj=sj, nrm=nrm, ghat=g / nrm)


class FlatPairs:
    """All point pairs of a pair list in one flat array (pairs in caller order)."""

    def __init__(self, x1, x2, lengths, active=None):
        self.x1 = np.asarray(x1, dtype=np.float64)
        self.x2 = np.asarray(x2, dtype=np.float64)
        self.lengths = np.asarray(lengths, dtype=np.int64)
        self.start = np.concatenate([[0], np.cumsum(self.lengths)])
        self.seg = np.repeat(np.arange(len(self.lengths)), self.lengths)
        self.active = (np.ones(len(self.x1), dtype=bool) if active is None
                       else np.asarray(active, dtype=bool).copy())

    @classmethod
    def from_pairs(cls, pairs):
        return cls(np.concatenate([p.x1 for p in pairs]), np.concatenate([p.x2 for p in pairs]),
                   [len(p.x1) for p in pairs], np.concatenate([p.active for p in pairs]))

    def split(self, flat):
        return [flat[self.start[k]:self.start[k + 1]] for k in range(len(self.lengths))]


def segment_sum(values, seg, n_seg):
    """Sum rows of values per segment id (values: (Z,) or (Z, K))."""
    values = np.asarray(values, dtype=np.float64)
    if values.ndim == 1:
        return np.bincount(seg, weights=values, minlength=n_seg)
    return np.stack([np.bincount(seg, weights=values[:, k], minlength=n_seg)
                     for k in range(values.shape[1])], axis=1)


def terms_of(x1, x2):
    """flatten(x2 x1^T) per point (ref/epipolar.py:34, :39-43)."""
    return (x2[:, :, None] * x1[:, None, :]).reshape(len(x1), 9)


def signed_residuals(flat, ghat):
    """t_m . ghat_n for every point (ref/epipolar.py:251-255, signed)."""
    return np.einsum("zk,zk->z", terms_of(flat.x1, flat.x2), ghat[flat.seg])


def weights_per_pair(flat, w, chunk=1 << 18):
    """W_n = sum_m w_m t_m t_m^T (ref/epipolar.py:46-59), (P, 9, 9)."""
    P = len(flat.lengths)
    out = np.zeros((P, 81))
    for s in range(0, len(flat.x1), chunk):
        sl = slice(s, s + chunk)
        T = terms_of(flat.x1[sl], flat.x2[sl])
        outer = (T[:, :, None] * (w[sl, None] * T)[:, None, :]).reshape(-1, 81)
        out += segment_sum(outer, flat.seg[sl], P)
    return out.reshape(P, 9, 9)


def irls_weights(res, mask):
    """1 / max(|r|, eps) on active points, 0 elsewhere (ref/epipolar.py:58)."""
    return np.where(mask, 1.0 / np.maximum(np.abs(res), HUBER_EPS), 0.0)


def point_pass(flat, ghat, threshold=None, irls=True):
    """One fused sweep: prune (optional), L1 over pre-prune active points,
    IRLS W, linearisation terms.  Mutates flat.active when pruning."""
    P = len(flat.lengths)
    r = signed_residuals(flat, ghat)
    ar = np.abs(r)
    pre = flat.active.copy()
    l1 = segment_sum(np.where(pre, ar, 0.0), flat.seg, P)
    if threshold is not None:
        flat.active &= ar <= threshold
    act = flat.active
    w = irls_weights(r, act) if irls else act.astype(np.float64)
    W = weights_per_pair(flat, w)
    T = terms_of(flat.x1, flat.x2)
    vgrad = segment_sum((w * r)[:, None] * T, flat.seg, P)
    s0 = segment_sum(w * r * r, flat.seg, P)
    n_active = np.bincount(flat.seg, weights=act, minlength=P).astype(np.int64)
    return dict(residual=ar, l1=l1, W=W, vgrad=vgrad, s0=s0, n_active=n_active)


def quad_loss_grad(params, n, idx_i, idx_j, cam_i, cam_j, refine_focal, n_cams, W, Z):
    """(2/Z) sum ghat^T W ghat and the packed gradient
    (ref/epipolar.py:172-232, focal terms :235-248)."""
    f = pair_forward(params, n, idx_i, idx_j, cam_i, cam_j, refine_focal)
    gh = f["ghat"]
    Wg = np.einsum("pkl,pl->pk", W, gh)
    loss = float(2.0 / Z * np.einsum("pk,pk->", gh, Wg))
    gg = 4.0 / Z * Wg
    gG = ((gg - gh * np.sum(gh * gg, axis=1, keepdims=True)) / f["nrm"]).reshape(-1, 3, 3)
    P = len(idx_i)
    if refine_focal:
        E, si, sj = f["E"], f["si"], f["sj"]
        gE = sj * gG * si
        gphi_i = -f["di"] * np.einsum("pab,pab->p", gG[:, :, :2], (sj * E)[:, :, :2])
        gphi_j = -f["dj"] * np.einsum("pab,pab->p", gG[:, :2, :], (E * si)[:, :2, :])
        gfoc = (np.bincount(cam_i, weights=gphi_i, minlength=n_cams) +
                np.bincount(cam_j, weights=gphi_j, minlength=n_cams))
    else:
        gE = gG
    t, Rrel, Ri, Rj, dc = f["t"], f["Rrel"], f["Ri"], f["Rj"], f["dc"]
    Mrel = np.swapaxes(skew(t), 1, 2) @ gE
    Pm = gE @ np.swapaxes(Rrel, 1, 2)
    gt = np.stack([Pm[:, 2, 1] - Pm[:, 1, 2], Pm[:, 0, 2] - Pm[:, 2, 0],
                   Pm[:, 1, 0] - Pm[:, 0, 1]], axis=1)
    gdc = -np.einsum("pba,pb->pa", Rj, gt)
    gRj = Mrel @ Ri - gt[:, :, None] * dc[:, None, :]
    gRi = np.swapaxes(Mrel, 1, 2) @ Rj
    gR = (segment_sum(gRi.reshape(P, 9), idx_i, n) + segment_sum(gRj.reshape(P, 9), idx_j, n))
    gc = segment_sum(gdc, idx_j, n) - segment_sum(gdc, idx_i, n)
    rot6d = np.asarray(params[:6 * n]).reshape(n, 6)
    g6 = rot6d_vjp(rot6d, gR.reshape(n, 3, 3))
    parts = [g6.ravel(), gc.ravel()]
    if refine_focal:
        parts.append(gfoc)
    return loss, np.concatenate(parts)


def prune_thresholds(cfg):
    if cfg.prune_rounds == 1:
        return [cfg.prune_threshold_start]
    return list(np.linspace(cfg.prune_threshold_start, cfg.prune_threshold_end, cfg.prune_rounds))


def irls_refine(rotations, centers, pairs_ij, cams_ij, flat, cfg, n_cameras=1):
    """Schedule of ref/epipolar.py:265-319 on a FlatPairs store.

    rotations/centers: per-image arrays indexed by image id; pairs_ij (P, 2)
    image ids, cams_ij (P, 2) camera ids.  Returns (rotations, centers,
    focal_scale, report) with flat.active pruned in place.
    """
    pairs_ij = np.asarray(pairs_ij, dtype=np.int64)
    cams_ij = np.asarray(cams_ij, dtype=np.int64)
    ids = np.unique(pairs_ij)
    n = len(ids)
    idx_i = np.searchsorted(ids, pairs_ij[:, 0])
    idx_j = np.searchsorted(ids, pairs_ij[:, 1])
    ci, cj = cams_ij[:, 0], cams_ij[:, 1]
    rf = bool(cfg.refine_focal)
    R0 = np.asarray(rotations, dtype=np.float64)[ids]
    parts = [np.concatenate([R0[:, :, 0], R0[:, :, 1]], axis=1).ravel(),
             np.asarray(centers, dtype=np.float64)[ids].ravel()]
    if rf:
        parts.append(np.zeros(n_cameras))
    params = np.concatenate(parts)
    P = len(pairs_ij)
    kept = np.ones(P, dtype=bool)
    l1_history, dropped = [], 0
    lr = cfg.epipolar_lr
    Z = None
    for th in prune_thresholds(cfg):
        gh = pair_forward(params, n, idx_i, idx_j, ci, cj, rf)["ghat"]
        out = point_pass(flat, gh, threshold=th)
        now = out["n_active"] > 0
        dropped += int(np.sum(kept & ~now))
        kept &= now
        if not kept.any():
            raise ValueError("all pairs pruned away")
        Z = int(out["n_active"].sum())
        opt = Adam(params, lr=lr, beta1=cfg.adam_beta1, beta2=cfg.adam_beta2, eps=cfg.adam_eps)
        for it in range(cfg.irls_iters_between_prunes):
            if it > 0:
                gh = pair_forward(opt.params, n, idx_i, idx_j, ci, cj, rf)["ghat"]
                out = point_pass(flat, gh)
            W = out["W"]
            for _ in range(cfg.epipolar_epoch_steps):
                loss, g = quad_loss_grad(opt.params, n, idx_i[kept], idx_j[kept], ci[kept],
                                         cj[kept], rf, n_cameras, W[kept], Z)
                if not np.isfinite(loss):
                    raise FloatingPointError("non-finite epipolar loss")
                opt.step(g)
        params = opt.params
        gh = pair_forward(params, n, idx_i, idx_j, ci, cj, rf)["ghat"]
        r = np.abs(signed_residuals(flat, gh))
        l1_history.append(float(np.sum(np.where(flat.active, r, 0.0)) / Z))
        lr /= cfg.lr_decay
    rot6d, cen, logf = unpack(params, n, rf)
    Rout = np.array(rotations, dtype=np.float64, copy=True)
    Cout = np.array(centers, dtype=np.float64, copy=True)
    Rout[ids] = project_to_so3(rot6d_to_matrix(rot6d))
    Cout[ids] = cen
    focal_scale = np.exp(logf) if rf else np.ones(n_cameras)
    report = {"l1_history": l1_history, "dropped_pairs": dropped,
              "active_pairs": int(kept.sum())}
    return Rout, Cout, focal_scale, report


# ------------------------------------------------------ global translation
def translation_loss_grad(centers, ei, ej, dirs):
    """Mean per-edge L1 direction loss and gradient (ref/translation.py:112-125)."""
    centers = np.asarray(centers, dtype=np.float64)
    delta = centers[ej] - centers[ei]
    length = np.maximum(np.linalg.norm(delta, axis=1, keepdims=True), NORM_EPS)
    u = delta / length
    r = u - dirs
    m = len(dirs)
    gu = np.sign(r) / m
    gd = (gu - u * np.sum(u * gu, axis=1, keepdims=True)) / length
    grad = np.zeros_like(centers)
    np.add.at(grad, ej, gd)       # ref/translation.py:123-124 order
    np.add.at(grad, ei, -gd)
    return float(np.abs(r).sum() / m), grad


def canonicalize(c):
    """Centroid to 0, unit mean norm (ref/translation.py:128-134)."""
    out = c - c.mean(axis=0)
    s = np.linalg.norm(out, axis=1).mean()
    return out / s if s > NORM_EPS else out


def align_centers(n, ei, ej, dirs, cfg, seed=0, init=None, steps=None):
    """Adam descent from seeded init (ref/translation.py:137-152)."""
    rng = np.random.default_rng(seed)
    if init is None:
        init = rng.standard_normal((n, 3))
    opt = Adam(np.asarray(init, dtype=np.float64).ravel(), lr=cfg.translation_lr,
               beta1=cfg.adam_beta1, beta2=cfg.adam_beta2, eps=cfg.adam_eps)
    loss = np.inf
    for _ in range(cfg.translation_steps if steps is None else steps):
        loss, g = translation_loss_grad(opt.params.reshape(n, 3), ei, ej, dirs)
        if not np.isfinite(loss):
            raise FloatingPointError("non-finite translation loss")
        opt.step(g.ravel())
    return opt.params.reshape(n, 3).copy(), loss


def per_node_residuals(c, ei, ej, dirs):
    """Mean incident L1 residual per node (ref/translation.py:155-166)."""
    delta = c[ej] - c[ei]
    length = np.maximum(np.linalg.norm(delta, axis=1, keepdims=True), NORM_EPS)
    r = np.abs(delta / length - dirs).sum(axis=1)
    n = len(c)
    tot = np.zeros(n)
    cnt = np.zeros(n)
    np.add.at(tot, ei, r)         # ref/translation.py:161-164 order
    np.add.at(tot, ej, r)
    np.add.at(cnt, ei, 1.0)
    np.add.at(cnt, ej, 1.0)
    return tot / np.maximum(cnt, 1.0)


def multi_init_align(n, ei, ej, dirs, cfg, seed=0):
    """Runs seed..seed+B-1, canonicalize, per-node argmin merge, final run
    (ref/translation.py:169-186)."""
    if cfg.translation_inits == 1:
        return align_centers(n, ei, ej, dirs, cfg, seed=seed)
    runs = [canonicalize(align_centers(n, ei, ej, dirs, cfg, seed=seed + k)[0])
            for k in range(cfg.translation_inits)]
    res = np.stack([per_node_residuals(c, ei, ej, dirs) for c in runs])
    choice = np.argmin(res, axis=0)
    merged = np.stack([runs[choice[v]][v] for v in range(n)])
    return align_centers(n, ei, ej, dirs, cfg, seed=seed, init=merged)


# ------------------------------------------------------------ pose metrics
def umeyama(src, dst):
    """Similarity (s, R, t) minimising sum |s R src + t - dst|^2
    (ref/metrics.py:20-43)."""
    mu_s, mu_d = src.mean(0), dst.mean(0)
    xs, xd = src - mu_s, dst - mu_d
    var_s = np.mean(np.sum(xs ** 2, axis=1))
    U, d, Vt = np.linalg.svd(xd.T @ xs / len(src))
    S = np.eye(3)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        S[2, 2] = -1.0
    R = U @ S @ Vt
    s = float(np.trace(np.diag(d) @ S) / var_s)
    return s, R, mu_d - s * R @ mu_s


def pose_metrics(R_est, c_est, R_gt, c_gt, deltas=(1.0, 3.0)):
    """ATE (RMSE after similarity alignment to unit-normalised GT centres)
    and RRA/RTA@delta in percent over all image pairs (ref/metrics.py:46-165,
    all images registered)."""
    g = c_gt - c_gt.mean(axis=0)
    g = g / np.linalg.norm(g, axis=1).mean()
    s, R, t = umeyama(c_est, g)
    aligned = c_est @ (s * R).T + t
    out = {"ATE": float(np.sqrt(np.mean(np.sum((aligned - g) ** 2, axis=1))))}
    n = len(R_gt)
    rerr, terr = [], []
    for i in range(n):
        for j in range(i + 1, n):
            Re = R_est[j] @ R_est[i].T
            Rg = R_gt[j] @ R_gt[i].T
            cosv = np.clip((np.trace(Re.T @ Rg) - 1.0) / 2.0, -1.0, 1.0)
            rerr.append(np.degrees(np.arccos(cosv)))
            dg = c_gt[j] - c_gt[i]
            de = c_est[j] - c_est[i]
            ug = R_gt[i] @ (dg / np.linalg.norm(dg))
            ue = R_est[i] @ (de / max(np.linalg.norm(de), 1e-300))
            terr.append(np.degrees(np.arccos(np.clip(ug @ ue, -1.0, 1.0))))
    rerr, terr = np.array(rerr), np.array(terr)
    for dl in deltas:
        k = int(dl) if float(dl).is_integer() else dl
        out[f"RRA@{k}"] = 100.0 * float(np.mean(rerr < dl))
        out[f"RTA@{k}"] = 100.0 * float(np.mean(terr < dl))
    return out
