"""Input construction of the hot path: the direction graph and the epipolar
pairs the pipeline hands to ``multi_init_align`` and ``irls_refine``
(ref/pipeline.py:188-228).

In the reference this is a loop inside ``run_pipeline`` that, per completed
image pair, picks the points, runs one relative-translation sphere search and
appends an edge and an ``EpipolarPair``.  ``select_epipolar_pairs`` is the
same selection as one call: the point choice uses the reference's own numpy
expressions (so every point array is bitwise the reference's), all sphere
searches run as one batched device search per level
(``translation.reestimate_relative_batch``, the single-call decisions), and
the outputs come back in the reference's order.  A maintainer replaces the
loop with one call.
"""

import numpy as np

from . import translation as T
from .epipolar import EpipolarPair


def select_epipolar_pairs(completed_pairs, registered, norm_kps, pair_points, rotations,
                          camera_ids, cfg):
    """ref/pipeline.py:188-228 as one batched call.

    completed_pairs: the completed match set's pairs (``.i``, ``.j``,
    ``.correspondences`` (M, 2), ``.synthetic_from_tracks``), in order;
    registered: (n_images,) bool; norm_kps: per image (K, 3) normalised
    keypoints; pair_points: {(i, j): (x1, x2)} verified inliers; rotations:
    (n_images, 3, 3); camera_ids: per image camera id; cfg: sphere_samples,
    sphere_refine_levels.

    Returns (DirectionGraph over the registered images in sorted order,
    list of EpipolarPair, the sorted registered image ids).  Raises
    ValueError when no pair keeps a direction (ref/pipeline.py:221-223)."""
    reg = np.asarray(registered, dtype=bool)
    active = sorted(np.flatnonzero(reg))
    remap = {int(img): k for k, img in enumerate(active)}
    cand, x1s, x2s, rels = [], [], [], []
    for pair in completed_pairs:
        if not (reg[pair.i] and reg[pair.j]):
            continue
        if pair.synthetic_from_tracks or (pair.i, pair.j) not in pair_points:
            x1 = norm_kps[pair.i][pair.correspondences[:, 0]]
            x2 = norm_kps[pair.j][pair.correspondences[:, 1]]
            ok = np.all(np.isfinite(x1), axis=1) & np.all(np.isfinite(x2), axis=1)
            x1, x2 = x1[ok], x2[ok]
        else:
            x1, x2 = pair_points[(pair.i, pair.j)]
        if len(x1) < 2:
            continue
        cand.append(pair)
        x1s.append(x1)
        x2s.append(x2)
        rels.append(rotations[pair.j] @ rotations[pair.i].T)
    found = T.reestimate_relative_batch(x1s, x2s, rels, cfg) if cand else []
    edges_i, edges_j, directions, epi_pairs = [], [], [], []
    for pair, x1, x2, t_ij in zip(cand, x1s, x2s, found):
        if isinstance(t_ij, T.PairRejected):
            continue
        edges_i.append(remap[pair.i])
        edges_j.append(remap[pair.j])
        directions.append(T.world_direction(t_ij, rotations[pair.j]))
        epi_pairs.append(EpipolarPair(i=pair.i, j=pair.j, cam_i=int(camera_ids[pair.i]),
                                      cam_j=int(camera_ids[pair.j]), x1=x1, x2=x2))
    if not edges_i:
        raise ValueError("no pair kept a usable translation direction")
    graph = T.DirectionGraph(n=len(active), edges_i=np.array(edges_i, dtype=np.int64),
                             edges_j=np.array(edges_j, dtype=np.int64),
                             directions=np.stack(directions))
    return graph, epi_pairs, active


__all__ = ["select_epipolar_pairs"]
