"""Drop-in for ``fastmap.tracks`` (ref/tracks.py:38-106, reached from
ref/pipeline.py:178-181; SURVEY 8f "next" #2): track building and match
completion.

``build_tracks``: the components of the (image, keypoint) match graph come
from the device (``fm_cc_labels``, hook-and-compress); grouping, the
same-image conflict rule and the track order are integer numpy on the host.
Each component is labelled by its smallest node id, and node ids follow
(image, keypoint) order, so sorting the nodes by (label, id) yields every
track already sorted.  Tracks are disjoint, so the reference's lexicographic
track sort reduces to ordering by first member.

``complete_matches``: every track's implied pairs, expanded with numpy by
track size, minus the existing correspondences (an int64 key per
correspondence), deduplicated and sorted like the reference's sets.

install() rebinds ``TrackSet`` to the reference's class; the match-set and
pair objects are built with the caller's own classes.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N


@dataclass
class TrackSet:
    """ref/model.py:159-170 (install() rebinds this name to the reference class)."""
    tracks: list
    index: dict = field(default_factory=dict)

    def __post_init__(self):
        if not self.index:
            self.index = {obs: t for t, members in enumerate(self.tracks) for obs in members}


def _sorted_unique(a):
    """np.unique by sorting (numpy 2.x's hash-based unique is slower here)."""
    a = np.sort(a)
    return a[np.r_[True, a[1:] != a[:-1]]] if len(a) else a


def _node_offsets(match_set):
    n_kp = np.array([len(k) for k in match_set.keypoints], dtype=np.int64)
    return np.concatenate([[0], np.cumsum(n_kp)])


def _edges(match_set, off):
    us, vs = [], []
    for p in match_set.pairs:
        c = np.asarray(p.correspondences, dtype=np.int64).reshape(-1, 2)
        us.append(off[p.i] + c[:, 0])
        vs.append(off[p.j] + c[:, 1])
    if not us:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(us), np.concatenate(vs)


def component_labels(n_nodes, u, v):
    """Device connected components: label = smallest node id of the component."""
    if n_nodes >= 2**31 - 1:
        raise ValueError("more than 2^31 keypoints")
    device = N.require_cuda()
    U = torch.as_tensor(u.astype(np.int32), device=device)
    V = torch.as_tensor(v.astype(np.int32), device=device)
    lab = torch.empty(max(n_nodes, 1), dtype=torch.int32, device=device)
    N.check(N.lib().fm_cc_labels(int(n_nodes), len(u), N.ptr(U), N.ptr(V), N.ptr(lab),
                                 N.stream_handle()))
    return lab.cpu().numpy()[:n_nodes].astype(np.int64)


def build_tracks(match_set):
    """ref/tracks.py:38-56: components of size >= 2 without two keypoints of
    one image, each sorted, in the reference's order."""
    off = _node_offsets(match_set)
    n_nodes = int(off[-1])
    u, v = _edges(match_set, off)
    if not len(u):
        return TrackSet(tracks=[])
    lab = component_labels(n_nodes, u, v)
    touched = _sorted_unique(np.concatenate([u, v]))
    order = np.lexsort((touched, lab[touched]))
    nodes = touched[order]
    labels = lab[nodes]
    starts = np.flatnonzero(np.r_[True, labels[1:] != labels[:-1]])
    sizes = np.diff(np.r_[starts, len(nodes)])
    image = np.searchsorted(off, nodes, side="right") - 1
    kp = nodes - off[image]
    # same-image conflict: two consecutive members of a track share the image
    dup = np.r_[False, (image[1:] == image[:-1]) & (labels[1:] == labels[:-1])]
    bad = np.zeros(len(starts), dtype=bool)
    if dup.any():
        bad[np.searchsorted(starts, np.flatnonzero(dup), side="right") - 1] = True
    keep = (sizes >= 2) & ~bad
    # disjoint tracks: lexicographic order == order of first members
    ks, kn = starts[keep], sizes[keep]
    o = np.lexsort((kp[ks], image[ks]))
    ks, kn = ks[o], kn[o]
    sel = np.repeat(ks - np.r_[0, np.cumsum(kn)[:-1]], kn) + np.arange(int(kn.sum()))
    img_k, kp_k = image[sel], kp[sel]
    members = list(zip(img_k.tolist(), kp_k.tolist()))
    bounds = np.r_[0, np.cumsum(kn)].tolist()
    tracks = [members[a:b] for a, b in zip(bounds[:-1], bounds[1:])]
    index = dict(zip(members, np.repeat(np.arange(len(kn)), kn).tolist()))
    ts = TrackSet(tracks=tracks, index=index)
    # the same tracks as arrays, for complete_matches (checked against `tracks`)
    ts._fm_arrays = (img_k, kp_k, np.asarray(bounds[:-1], dtype=np.int64), kn, tracks)
    return ts


def _track_arrays(track_set):
    arr = getattr(track_set, "_fm_arrays", None)
    if arr is not None and arr[4] is track_set.tracks:  # not rebound since build_tracks
        return arr[:4]
    lens = np.array([len(t) for t in track_set.tracks], dtype=np.int64)
    flat = np.array([x for t in track_set.tracks for x in t], dtype=np.int64).reshape(-1, 2)
    return flat[:, 0], flat[:, 1], np.r_[0, np.cumsum(lens)[:-1]].astype(np.int64), lens


def complete_matches(track_set, match_set, max_track_size=200):
    """ref/tracks.py:59-106: add every correspondence implied by a track of
    at most max_track_size members that is not already present; new ones go
    after a pair's originals in sorted order, new pairs are FUNDAMENTAL and
    synthetic; pairs are returned sorted by (i, j)."""
    pairs_in = list(match_set.pairs)
    n_img = len(match_set.images)
    kmax = max([len(k) for k in match_set.keypoints] + [1])
    if float(n_img) ** 2 * float(kmax) ** 2 >= 2.0 ** 62:
        raise ValueError("image / keypoint counts too large for 64-bit correspondence keys")

    def key(i, j, ka, kb):
        return ((i * n_img + j) * kmax + ka) * kmax + kb

    ex = [key(p.i, p.j, *np.asarray(p.correspondences, dtype=np.int64).reshape(-1, 2).T)
          for p in pairs_in]
    existing = _sorted_unique(np.concatenate(ex)) if ex else np.zeros(0, np.int64)
    cand = []
    t_img, t_kp, t_start, t_len = _track_arrays(track_set)
    for s in np.unique(t_len[(t_len >= 2) & (t_len <= max_track_size)]).tolist():
        st = t_start[t_len == s]
        at = st[:, None] + np.arange(s)  # (n, s): members sorted, images distinct
        a, b = np.triu_indices(s, 1)
        ia, ka = t_img[at[:, a]].ravel(), t_kp[at[:, a]].ravel()
        ib, kb = t_img[at[:, b]].ravel(), t_kp[at[:, b]].ravel()
        cand.append(key(ia, ib, ka, kb))
    new = _sorted_unique(np.concatenate(cand)) if cand else np.zeros(0, np.int64)
    if len(existing) and len(new):
        at = np.minimum(np.searchsorted(existing, new), len(existing) - 1)
        new = new[existing[at] != new]
    kb = new % kmax
    rest = new // kmax
    ka = rest % kmax
    ij = rest // kmax
    # group the sorted keys by pair: (i, j) ascending, corr ascending within
    pstart = np.flatnonzero(np.r_[True, ij[1:] != ij[:-1]]) if len(new) else np.zeros(0, np.int64)
    pend = np.r_[pstart[1:], len(new)]
    added = {}
    for s0, s1 in zip(pstart.tolist(), pend.tolist()):
        k = int(ij[s0])
        added[(k // n_img, k % n_img)] = np.stack([ka[s0:s1], kb[s0:s1]], axis=1)
    out = []
    pair_cls = type(pairs_in[0]) if pairs_in else None
    for p in pairs_in:
        extra = added.pop((p.i, p.j), None)
        if extra is None:
            out.append(p)
            continue
        corr = np.concatenate([np.asarray(p.correspondences).reshape(-1, 2), extra.astype(np.int64)])
        out.append(pair_cls(i=p.i, j=p.j, geometry_class=p.geometry_class, correspondences=corr,
                            synthetic_from_tracks=p.synthetic_from_tracks))
    if added:
        fundamental = type(pairs_in[0].geometry_class).FUNDAMENTAL
        for (i, j) in sorted(added):
            out.append(pair_cls(i=i, j=j, geometry_class=fundamental,
                                correspondences=added[(i, j)].astype(np.int64),
                                synthetic_from_tracks=True))
    out.sort(key=lambda p: (p.i, p.j))
    return type(match_set)(images=match_set.images, keypoints=match_set.keypoints, pairs=out)


__all__ = ["TrackSet", "component_labels", "build_tracks", "complete_matches"]
