"""Shared test helpers: rebuild pair lists and graphs from golden arrays."""

import numpy as np


class Cfg:
    """Hot-path config with the reference defaults (ref/config.py:37-54)."""

    def __init__(self, **kw):
        self.translation_lr = 1e-3
        self.translation_steps = 6000
        self.translation_inits = 3
        self.epipolar_lr = 1e-4
        self.lr_decay = 2.0
        self.prune_rounds = 3
        self.prune_threshold_start = 0.01
        self.prune_threshold_end = 0.005
        self.irls_iters_between_prunes = 3
        self.epipolar_epoch_steps = 100
        self.refine_focal = True
        self.adam_beta1 = 0.9
        self.adam_beta2 = 0.999
        self.adam_eps = 1e-8
        for k, v in kw.items():
            setattr(self, k, v)


def split(flat, lengths):
    start = np.concatenate([[0], np.cumsum(lengths)])
    return [flat[start[k]:start[k + 1]] for k in range(len(lengths))]


def pairs_from(g, prefix, cls):
    """EpipolarPair objects (class cls) from golden arrays."""
    lengths = g[prefix + "len"]
    x1 = split(g[prefix + "x1"], lengths)
    x2 = split(g[prefix + "x2"], lengths)
    act = split(g[prefix + "active"], lengths)
    out = []
    for k, (i, j) in enumerate(g[prefix + "ij"]):
        ci, cj = g[prefix + "cams"][k]
        out.append(cls(i=int(i), j=int(j), cam_i=int(ci), cam_j=int(cj), x1=x1[k].copy(),
                       x2=x2[k].copy(), active=act[k].astype(bool).copy()))
    return out


def c1_pairs(g, cls):
    lengths = g["c1_len"].astype(np.int64)
    x1 = split(g["c1_x1"].astype(np.float64), lengths)
    x2 = split(g["c1_x2"].astype(np.float64), lengths)
    out = []
    for k, (i, j) in enumerate(g["c1_ij"]):
        a = np.column_stack([x1[k], np.ones(len(x1[k]))])
        b = np.column_stack([x2[k], np.ones(len(x2[k]))])
        out.append(cls(i=int(i), j=int(j), cam_i=0, cam_j=0, x1=a, x2=b))
    return out


class SimplePair:
    """Minimal EpipolarPair stand-in for the oracle tests."""

    def __init__(self, i, j, cam_i, cam_j, x1, x2, active=None):
        self.i, self.j, self.cam_i, self.cam_j = i, j, cam_i, cam_j
        self.x1, self.x2 = x1, x2
        self.active = np.ones(len(x1), dtype=bool) if active is None else active


class Poses:
    """PoseState stand-in (same constructor keywords as ref/model.py:129-135)."""

    def __init__(self, rotations, centers, registered=None):
        self.rotations = rotations
        self.centers = centers
        self.registered = np.ones(len(rotations), dtype=bool) if registered is None else registered
