"""inputs.select_epipolar_pairs vs the selection inside the REFERENCE pipeline
(ref/pipeline.py:188-228) on NOISY_SPEC: the fixture
(tests/golden/make_select_golden.py) holds the stage inputs the reference
had and its outputs -- the DirectionGraph fed to multi_init_align and the
EpipolarPair list fed to irls_refine.

Tolerances: edges, pair order, cameras and point arrays identical (the point
arrays bitwise); directions within 1e-6 (the sphere search sums its mean
errors in a different order than the reference, so near-tied candidates may
swap; tests/test_pipeline_golden_gpu.py), most of them bitwise."""

import os
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

I = pytest.importorskip("paper_2505_04612_b200.inputs")


@pytest.fixture(scope="module")
def sel():
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_select.npz")))
    kp = [g["kp"][g["kp_off"][k]:g["kp_off"][k + 1]] for k in range(len(g["kp_off"]) - 1)]
    pairs = [SimpleNamespace(i=int(i), j=int(j), synthetic_from_tracks=bool(s),
                             correspondences=g["cp_corr"][g["cp_off"][k]:g["cp_off"][k + 1]].astype(np.int64))
             for k, ((i, j), s) in enumerate(zip(g["cp_ij"], g["cp_synth"]))]
    pp = {}
    for k, (i, j) in enumerate(g["pp_ij"]):
        c = g["pp_corr"][g["pp_off"][k]:g["pp_off"][k + 1]].astype(np.int64)
        pp[(int(i), int(j))] = (kp[i][c[:, 0]], kp[j][c[:, 1]])
    cfg = SimpleNamespace(sphere_samples=int(g["cfg"][0]), sphere_refine_levels=int(g["cfg"][1]))
    return g, kp, pairs, pp, cfg


def test_selection_matches_reference_pipeline(sel):
    g, kp, pairs, pp, cfg = sel
    graph, epi, active = I.select_epipolar_pairs(pairs, g["registered"], kp, pp, g["rotations"],
                                                 g["cams"], cfg)
    assert graph.n == int(g["out_n"][0]) and active == sorted(np.flatnonzero(g["registered"]))
    np.testing.assert_array_equal(graph.edges_i, g["out_ei"])
    np.testing.assert_array_equal(graph.edges_j, g["out_ej"])
    err = np.abs(graph.directions - g["out_dirs"]).max(axis=1)
    assert err.max() < 1e-6 and (err == 0).mean() > 0.5, err.max()
    assert [[p.i, p.j] for p in epi] == g["out_ij"].tolist()
    assert [[p.cam_i, p.cam_j] for p in epi] == g["out_cams"].tolist()
    assert [len(p.x1) for p in epi] == g["out_len"].tolist()
    kpall = g["kp"]
    np.testing.assert_array_equal(np.concatenate([p.x1 for p in epi]), kpall[g["out_rows1"]])
    np.testing.assert_array_equal(np.concatenate([p.x2 for p in epi]), kpall[g["out_rows2"]])


def test_selection_paths_synthetic_missing_nonfinite_unregistered(sel):
    """The branches NOISY_SPEC does not reach: track-completion pairs and
    pairs without verified inliers take the completed correspondences with
    non-finite rows dropped (ref/pipeline.py:197-202); pairs left with < 2
    points and pairs touching an unregistered image are skipped (:195-196,
    :205-206); edges use the registered-image remap (:189-191)."""
    g, kp, pairs, pp, cfg = sel
    kp = [k.copy() for k in kp]
    pairs = [SimpleNamespace(**vars(p)) for p in pairs]
    pp = dict(pp)
    reg = g["registered"].copy()
    reg[7] = False
    pairs[0].synthetic_from_tracks = True
    for p in pairs[1:6]:
        pp.pop((p.i, p.j))
    c = pairs[2].correspondences
    kp[pairs[2].i][c[::3, 0]] = np.nan  # a third of pair 2's points non-finite
    pairs[4].correspondences = pairs[4].correspondences[:1]  # one point left
    graph, epi, active = I.select_epipolar_pairs(pairs, reg, kp, pp, g["rotations"], g["cams"], cfg)
    remap = {img: k for k, img in enumerate(sorted(np.flatnonzero(reg)))}
    want = []
    for p in pairs:
        if not (reg[p.i] and reg[p.j]):
            continue
        if p.synthetic_from_tracks or (p.i, p.j) not in pp:
            x1 = kp[p.i][p.correspondences[:, 0]]
            x2 = kp[p.j][p.correspondences[:, 1]]
            ok = np.all(np.isfinite(x1), axis=1) & np.all(np.isfinite(x2), axis=1)
            x1, x2 = x1[ok], x2[ok]
        else:
            x1, x2 = pp[(p.i, p.j)]
        if len(x1) >= 2:
            want.append((p, x1, x2))
    assert len(epi) == len(want) == len(graph.edges_i)
    assert not any(p.i == 7 or p.j == 7 for p in epi)
    for got, (p, x1, x2) in zip(epi, want):
        assert (got.i, got.j) == (p.i, p.j)
        np.testing.assert_array_equal(got.x1, x1)
        np.testing.assert_array_equal(got.x2, x2)
    np.testing.assert_array_equal(graph.edges_i, [remap[p.i] for p, _, _ in want])
    np.testing.assert_array_equal(graph.edges_j, [remap[p.j] for p, _, _ in want])
    p2, p4 = pairs[2], pairs[4]
    assert reg[p2.i] and reg[p2.j] and reg[p4.i] and reg[p4.j]
    got = next(e for e in epi if (e.i, e.j) == (p2.i, p2.j))
    assert 2 <= len(got.x1) < len(p2.correspondences)  # lost its non-finite rows
    assert not any((e.i, e.j) == (p4.i, p4.j) for e in epi)  # one point left: skipped


def test_selection_nothing_usable_raises(sel):
    g, kp, pairs, pp, cfg = sel
    with pytest.raises(ValueError, match="no pair kept a usable translation direction"):
        I.select_epipolar_pairs(pairs, np.zeros(len(g["registered"]), dtype=bool), kp, pp,
                                g["rotations"], g["cams"], cfg)
