"""Synthetic workloads of BASELINE.json, generated on
the device so the 10M-1B point-pair configs never touch host memory.

Ring of cameras looking at a unit ball of points; image pair (i, i+d mod n)
for d = 1..band; every pair observes its own ``points_per_pair`` points
(epipolar adjustment never uses tracks), projected with a pinhole of 60
degree FoV at 640 px (f = 554.3 px), 0.5 px noise, 2% outliers (x2 swapped
within the pair), poses perturbed by 0.5 degree / 0.01 (image 0 fixed).
Pairs come out already in (i, j) order, so the store needs no sort.
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from .store import PairGraph, PointPairStore, slot_layout


@dataclass
class SceneSpec:
    n_images: int = 500
    band: int = 50
    points_per_pair: int = 400
    fov_deg: float = 60.0
    width: int = 640
    noise_px: float = 0.5
    outlier_frac: float = 0.02
    rot_noise_deg: float = 0.5
    center_noise: float = 0.01
    seed: int = 0

    @property
    def n_pairs(self):
        return self.n_images * self.band if 2 * self.band < self.n_images else \
            self.n_images * (self.n_images - 1) // 2

    @property
    def focal_px(self):
        return (self.width / 2.0) / math.tan(math.radians(self.fov_deg) / 2.0)


CONFIGS = {
    "c2": SceneSpec(n_images=500, band=50, points_per_pair=400),        # ~10M point pairs
    "c4": SceneSpec(n_images=2000, band=50, points_per_pair=1000),      # ~100M
    "c5": SceneSpec(n_images=10000, band=50, points_per_pair=2000),     # ~1B
}


def ring_poses(n, radius=4.0):
    """World-to-camera rotations (rows right, down, forward) looking at 0."""
    a = np.linspace(0.0, 2 * np.pi, n, endpoint=False)
    centers = np.stack([radius * np.cos(a), radius * np.sin(a), 0.3 * np.sin(3 * a)], axis=1)
    rots = np.empty((n, 3, 3))
    for k, c in enumerate(centers):
        fwd = -c / np.linalg.norm(c)
        right = np.cross(fwd, [0.0, 0.0, 1.0])
        right /= np.linalg.norm(right)
        rots[k] = np.stack([right, np.cross(fwd, right), fwd])
    return rots, centers


def _rotvec_to_matrix(rv):
    th = np.linalg.norm(rv, axis=-1, keepdims=True)
    k = rv / np.maximum(th, 1e-300)
    K = np.zeros(rv.shape[:-1] + (3, 3))
    K[..., 0, 1], K[..., 0, 2], K[..., 1, 2] = -k[..., 2], k[..., 1], -k[..., 0]
    K[..., 1, 0], K[..., 2, 0], K[..., 2, 1] = k[..., 2], -k[..., 1], k[..., 0]
    s, c = np.sin(th)[..., None], np.cos(th)[..., None]
    return np.eye(3) + s * K + (1 - c) * (K @ K)


def perturb_poses(rots, centers, spec, rng):
    n = len(rots)
    rv = rng.normal(size=(n, 3))
    rv *= math.radians(spec.rot_noise_deg) / np.linalg.norm(rv, axis=1, keepdims=True)
    R = _rotvec_to_matrix(rv) @ rots
    c = centers + rng.normal(scale=spec.center_noise, size=centers.shape)
    R[0], c[0] = rots[0], centers[0]
    return R, c


def pair_list(spec):
    n, band = spec.n_images, spec.band
    if 2 * band >= n:
        ij = np.array([(i, j) for i in range(n) for j in range(i + 1, n)], dtype=np.int64)
    else:
        i = np.repeat(np.arange(n), band)
        j = (i + np.tile(np.arange(1, band + 1), n)) % n
        ij = np.stack([np.minimum(i, j), np.maximum(i, j)], axis=1)
    order = np.lexsort((ij[:, 1], ij[:, 0]))
    return ij[order]


def generate_poses(spec):
    """The scene's GT and perturbed poses alone (host; as generate() draws them)."""
    rng = np.random.default_rng(spec.seed)
    rots, centers = ring_poses(spec.n_images)
    R_in, c_in = perturb_poses(rots, centers, spec, rng)
    return dict(R_gt=rots, c_gt=centers, R_in=R_in, c_in=c_in)


def generate(spec, device, pair_slice=None):
    """Device tensors of a scene: x1, x2 (Z, 2) float32 in (i, j) pair order,
    per-pair lengths (host int64), pair ids (host), GT and perturbed poses."""
    rng = np.random.default_rng(spec.seed)
    rots, centers = ring_poses(spec.n_images)
    R_in, c_in = perturb_poses(rots, centers, spec, rng)
    ij = pair_list(spec)
    if pair_slice is not None:
        ij = ij[pair_slice]
    P, M = len(ij), spec.points_per_pair
    g = torch.Generator(device=device)
    g.manual_seed(spec.seed + 12345)
    Rt = torch.as_tensor(rots, device=device)
    Ct = torch.as_tensor(centers, device=device)
    ii = torch.as_tensor(ij[:, 0], device=device)
    jj = torch.as_tensor(ij[:, 1], device=device)
    x1 = torch.empty((P * M, 2), dtype=torch.float32, device=device)
    x2 = torch.empty((P * M, 2), dtype=torch.float32, device=device)
    sigma = spec.noise_px / spec.focal_px
    step = max(1, (1 << 24) // M)
    for s in range(0, P, step):
        e = min(P, s + step)
        n = e - s
        # uniform points in the unit ball
        d = torch.randn((n, M, 3), generator=g, device=device, dtype=torch.float64)
        d = d / d.norm(dim=-1, keepdim=True)
        r = torch.rand((n, M, 1), generator=g, device=device, dtype=torch.float64) ** (1.0 / 3.0)
        X = d * r
        out = []
        for idx in (ii[s:e], jj[s:e]):
            xc = torch.einsum("pab,pmb->pma", Rt[idx], X - Ct[idx][:, None, :])
            uv = xc[..., :2] / xc[..., 2:3]
            uv = uv + sigma * torch.randn(uv.shape, generator=g, device=device, dtype=torch.float64)
            out.append(uv)
        a, b = out
        if spec.outlier_frac > 0:
            bad = torch.rand((n, M), generator=g, device=device) < spec.outlier_frac
            shuffled = b.roll(shifts=M // 2, dims=1)
            b = torch.where(bad[..., None], shuffled, b)
        x1[s * M:e * M] = a.reshape(-1, 2).float()
        x2[s * M:e * M] = b.reshape(-1, 2).float()
    lengths = np.full(P, M, dtype=np.int64)
    return dict(x1=x1, x2=x2, lengths=lengths, ij=ij, R_gt=rots, c_gt=centers, R_in=R_in, c_in=c_in)


def device_store(scene, device, chunk=None):
    """PointPairStore straight from device tensors (pairs already sorted)."""
    from .store import CHUNK
    return PointPairStore.from_device(scene["x1"], scene["x2"], scene["lengths"], device=device,
                                      chunk=chunk or CHUNK)


def device_graph(scene, device, refine_focal=True):
    ij = scene["ij"]
    ids = np.unique(ij)
    ii = np.searchsorted(ids, ij[:, 0])
    jj = np.searchsorted(ids, ij[:, 1])
    zeros = np.zeros(len(ij), dtype=np.int64)
    return PairGraph(ii, jj, zeros, zeros, len(ids), 1, refine_focal, device=device), ids


def initial_params(scene, ids, refine_focal=True):
    R = scene["R_in"][ids]
    parts = [np.concatenate([R[:, :, 0], R[:, :, 1]], axis=1).ravel(), scene["c_in"][ids].ravel()]
    if refine_focal:
        parts.append(np.zeros(1))
    return np.concatenate(parts)


__all__ = ["SceneSpec", "CONFIGS", "generate", "device_store", "device_graph", "initial_params",
           "slot_layout", "pair_list"]


def translation_graph_c3(n=2000, m=200_000, seed=0):
    """BASELINE configs[2] direction graph (SURVEY 8d "C3"): n GT centres
    from default_rng(seed).normal, a ring backbone plus uniform random pairs
    up to m edges (i < j, sorted), directions = unit GT differences + 1 degree
    noise, 5% replaced by random unit vectors.  Host numpy (deterministic on
    every machine).  Returns (edges_i, edges_j, directions, gt_centers)."""
    rng = np.random.default_rng(seed)
    c = rng.normal(size=(n, 3))
    ring = np.stack([np.arange(n), (np.arange(n) + 1) % n], axis=1)
    extra = set()
    while len(extra) < m - n:
        a = rng.integers(0, n, size=(m, 2))
        for i, j in a:
            if i != j:
                extra.add((min(i, j), max(i, j)))
            if len(extra) >= m - n:
                break
    e = np.concatenate([np.sort(ring, axis=1), np.array(sorted(extra))])
    d = c[e[:, 1]] - c[e[:, 0]]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d += rng.normal(scale=np.radians(1.0), size=d.shape)
    bad = rng.random(m) < 0.05
    d[bad] = rng.normal(size=(bad.sum(), 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return e[:, 0].astype(np.int64), e[:, 1].astype(np.int64), d, c
