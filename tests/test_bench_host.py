"""Host-side pieces of bench.py (no GPU): the config-1 problem the two arms
time, and the stage table parsing of the pipeline run."""
import numpy as np

import bench
from tests.helpers import Poses


class _Pair:
    def __init__(self, i, j, cam_i, cam_j, x1, x2):
        self.i, self.j, self.cam_i, self.cam_j, self.x1, self.x2 = i, j, cam_i, cam_j, x1, x2


class _Graph:
    def __init__(self, n, edges_i, edges_j, directions):
        self.n, self.edges_i, self.edges_j, self.directions = n, edges_i, edges_j, directions


def test_c1_problem_is_config1():
    g, pairs, graph = bench.c1_problem(_Pair, _Graph)
    assert len(pairs) == 1225 and sum(len(p.x1) for p in pairs) == 223241
    assert all(p.x1.shape[1] == 3 and np.all(p.x1[:, 2] == 1.0) for p in pairs[:50])
    assert graph.n == 50 and len(graph.edges_i) == 1225
    np.testing.assert_array_equal(np.c_[graph.edges_i, graph.edges_j], g["c1_ij"])
    p0 = pairs[0]
    np.testing.assert_array_equal(p0.x1[:, :2], g["c1_x1"][:len(p0.x1)].astype(np.float64))
    assert isinstance(bench.Poses(g["c1_R_in"], g["c1_c_in"]).registered, np.ndarray)
    assert Poses is not None


def test_pipeline_stage_table_parsing():
    report = ("stage                          seconds  details\n"
              "distortion.search                 2.083  cameras=1 fallback=0\n"
              "epipolar.adjust                   0.014  \n"
              "total                             5.000\n")
    rows = [l.split() for l in report.splitlines()[1:]]
    got = {r[0]: float(r[1]) for r in rows if len(r) >= 2 and r[1].replace(".", "", 1).isdigit()}
    assert got == {"distortion.search": 2.083, "epipolar.adjust": 0.014, "total": 5.0}
    assert "str(report).splitlines()[1:]" in bench.PIPELINE_SCRIPT
