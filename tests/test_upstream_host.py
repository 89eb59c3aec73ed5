"""Host-side logic of the upstream stages, on CPU (no kernel runs):
the vectorised candidate prep of search_alpha against a per-pair loop with
the reference's expressions, the LMedS sample tables, and build_tracks /
complete_matches against the reference's golden outputs with the device
connected-components step replaced by a union-find (test infrastructure)."""

import os

import numpy as np
import pytest

from tests.test_distortion_gpu import _match_set as dist_match_set
from tests.test_tracks_gpu import _match_set as track_match_set

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_distortion.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_candidate_prep_equals_per_pair_loop(golden):
    from paper_2505_04612_b200 import distortion as D
    ms = dist_match_set(golden, "b_")
    pairs = D.ready_fundamental_pairs(ms, 1, {0: -0.15})
    alphas = [-0.3, 0.1]
    cand, lens, p1, p2 = D._jobs(alphas, ms, pairs, 1, {0: -0.15})
    # per pair, as ref/distortion.py:99-118 writes it
    want = []
    for c, a in enumerate(alphas):
        for p in pairs:
            kp_i = ms.keypoints[p.i][p.correspondences[:, 0]]
            kp_j = ms.keypoints[p.j][p.correspondences[:, 1]]
            u = []
            for im_id, kp in ((p.i, kp_i), (p.j, kp_j)):
                im = ms.images[im_id]
                s = 0.5 * float(np.hypot(im.width, im.height))
                center = np.array([im.width / 2.0, im.height / 2.0])
                al = a if im.camera_id == 1 else -0.15
                u.append(D.undistort_normalized((kp - center) / s, al) * s + center)
            ok = np.all(np.isfinite(u[0]), axis=1) & np.all(np.isfinite(u[1]), axis=1)
            if ok.sum() < 8:
                continue
            si = 0.5 * float(np.hypot(ms.images[p.i].width, ms.images[p.i].height))
            want.append((c, u[0][ok] / si, u[1][ok] / si))
    assert cand.tolist() == [c for c, _, _ in want]
    assert lens.tolist() == [len(a) for _, a, _ in want]
    assert np.array_equal(p1, np.concatenate([a for _, a, _ in want]))  # bit-identical
    assert np.array_equal(p2, np.concatenate([b for _, _, b in want]))


def test_lmeds_tables_are_seeded_samples():
    from paper_2505_04612_b200 import distortion as D
    t8, t4 = D.lmeds_samples(50), D.lmeds_samples4(50)
    assert t8.shape == (64, 8) and t4.shape == (64, 4)
    assert all(len(set(r)) == len(r) for r in t8.tolist() + t4.tolist())  # without replacement
    assert t8.min() >= 0 and t8.max() < 50 and t4.max() < 50
    rng = np.random.default_rng(12345)  # ref/twoview.py:86-88
    assert np.array_equal(t8[0], rng.choice(50, 8, replace=False))


def _union_find_labels(n, u, v):
    parent = np.arange(n)

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for a, b in zip(u.tolist(), v.tolist()):
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[max(ra, rb)] = min(ra, rb)
    return np.array([find(a) for a in range(n)], dtype=np.int64)


@pytest.mark.parametrize("scene,src,cap", [("a_", "a_", 200), ("d_", "d_", 200), ("d3_", "d_", 4)])
def test_track_host_logic_matches_reference(golden, monkeypatch, scene, src, cap):
    from paper_2505_04612_b200 import tracks
    monkeypatch.setattr(tracks, "component_labels", _union_find_labels)
    ms = track_match_set(golden, src)
    ts = tracks.build_tracks(ms)
    assert [len(t) for t in ts.tracks] == golden[scene + "track_len"].tolist()
    assert [x for t in ts.tracks for x in t] == \
        [tuple(r) for r in golden[scene + "track_nodes"].tolist()]
    done = tracks.complete_matches(ts, ms, max_track_size=cap)
    assert [[p.i, p.j] for p in done.pairs] == golden[scene + "done_ij"].tolist()
    assert np.array_equal(np.concatenate([p.correspondences for p in done.pairs]),
                          golden[scene + "done_corr"])
    assert [p.synthetic_from_tracks for p in done.pairs] == golden[scene + "done_synth"].tolist()
