"""Track building and match completion (SURVEY 8f "next" #2) against the
reference: its own unit cases (pkg/tests/test_tracks.py, restated) and
golden outputs of build_tracks / complete_matches recorded on synthetic
match sets, including a thinned scene with missing pairs, missing
correspondences and same-image conflicts (make_distortion_golden.py)."""

import enum
import os
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_distortion.npz")


class GC(enum.Enum):
    FUNDAMENTAL = "F"
    HOMOGRAPHY = "H"


@dataclass(frozen=True)
class Pair:
    i: int
    j: int
    geometry_class: GC
    correspondences: np.ndarray
    synthetic_from_tracks: bool = False


@dataclass
class MS:
    images: list
    keypoints: list
    pairs: list

    def pair_index(self):
        return {(p.i, p.j): p for p in self.pairs}


def make_set(pairs):
    images = [SimpleNamespace(image_id=i) for i in range(4)]
    keypoints = [np.full((5, 2), 10.0) for _ in range(4)]
    objs = [Pair(i, j, GC.FUNDAMENTAL, np.array(c, dtype=np.int64).reshape(-1, 2))
            for (i, j), c in pairs.items()]
    return MS(images, keypoints, objs)


def test_reference_unit_cases():
    from paper_2505_04612_b200.tracks import build_tracks, complete_matches
    assert build_tracks(make_set({(0, 1): [[0, 0]], (1, 2): [[0, 0]]})).tracks == \
        [[(0, 0), (1, 0), (2, 0)]]
    assert len(build_tracks(make_set({(0, 1): [[0, 0], [1, 1]]})).tracks) == 2
    assert build_tracks(make_set({(0, 1): [[0, 0], [1, 0]]})).tracks == []
    ts = build_tracks(make_set({(0, 1): [[2, 3]]}))
    assert ts.index[(0, 2)] == ts.index[(1, 3)]
    ms = make_set({(0, 1): [[0, 0]], (1, 2): [[0, 0]]})
    idx = complete_matches(build_tracks(ms), ms).pair_index()
    assert idx[(0, 2)].synthetic_from_tracks and idx[(0, 2)].correspondences.tolist() == [[0, 0]]
    assert not idx[(0, 1)].synthetic_from_tracks and idx[(0, 1)].correspondences.tolist() == [[0, 0]]
    assert idx[(0, 2)].geometry_class is GC.FUNDAMENTAL
    ms = make_set({(0, 1): [[0, 0]], (1, 2): [[0, 0]], (2, 3): [[0, 0]]})
    once = complete_matches(build_tracks(ms), ms)
    twice = complete_matches(build_tracks(once), once)
    assert {(p.i, p.j): p.correspondences.tolist() for p in once.pairs} == \
        {(p.i, p.j): p.correspondences.tolist() for p in twice.pairs}
    ms = make_set({(0, 1): [[0, 0]], (1, 2): [[0, 0]]})
    assert (0, 2) not in complete_matches(build_tracks(ms), ms, max_track_size=2).pair_index()
    ms = make_set({(1, 2): [[0, 0]], (0, 1): [[0, 0]]})
    keys = [(p.i, p.j) for p in complete_matches(build_tracks(ms), ms).pairs]
    assert keys == sorted(keys)


def _match_set(g, p):
    kp = np.split(g[p + "kp"], np.cumsum(g[p + "kp_len"])[:-1])
    corr = np.split(g[p + "corr"], np.cumsum(g[p + "pair_len"])[:-1])
    images = [SimpleNamespace(image_id=k) for k in range(len(kp))]
    pairs = [Pair(int(i), int(j), GC.HOMOGRAPHY if h else GC.FUNDAMENTAL, c)
             for (i, j), c, h in zip(g[p + "pair_ij"], corr, g[p + "homography"])]
    return MS(images, kp, pairs)


@pytest.mark.parametrize("scene,src,cap", [("a_", "a_", 200), ("b_", "b_", 200),
                                           ("d_", "d_", 200), ("d3_", "d_", 4)])
def test_tracks_and_completion_match_reference(scene, src, cap):
    from paper_2505_04612_b200.tracks import build_tracks, complete_matches
    g = np.load(GOLDEN)
    ms = _match_set(g, src)
    ts = build_tracks(ms)
    assert [len(t) for t in ts.tracks] == g[scene + "track_len"].tolist()
    assert [x for t in ts.tracks for x in t] == [tuple(r) for r in g[scene + "track_nodes"].tolist()]
    done = complete_matches(ts, ms, max_track_size=cap)
    assert [[p.i, p.j] for p in done.pairs] == g[scene + "done_ij"].tolist()
    assert [len(p.correspondences) for p in done.pairs] == g[scene + "done_len"].tolist()
    assert np.array_equal(np.concatenate([p.correspondences for p in done.pairs]),
                          g[scene + "done_corr"])
    assert [p.synthetic_from_tracks for p in done.pairs] == g[scene + "done_synth"].tolist()
    assert [p.geometry_class is GC.HOMOGRAPHY for p in done.pairs] == g[scene + "done_homog"].tolist()


def test_integration_stub_components():
    """The fm_cc_labels ctypes stub in INTEGRATION.md works as written."""
    import re
    from paper_2505_04612_b200 import _native
    from tests.conftest import ROOT
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"could replace its union-find.*?```python\n(.*?)```", text, re.S).group(1)
    os.environ["FASTMAP_B200_LIB"] = _native.lib_path()
    ns = {}
    try:
        exec(compile(code, "INTEGRATION.md", "exec"), ns)
    finally:
        os.environ.pop("FASTMAP_B200_LIB", None)
    lab = ns["component_labels_gpu"](7, [0, 1, 4, 6], [1, 2, 5, 4])
    assert lab.tolist() == [0, 0, 0, 3, 4, 4, 4]
