"""The sharded epipolar engine (parallel.ShardedIrlsEngine) on one GPU with
several shards: same schedule, same decisions and the same poses as the
single-store engine and the reference (config 1)."""

import numpy as np
import pytest
import torch

from oracle import fastmap_oracle as O
from tests.helpers import Cfg

pytestmark = pytest.mark.gpu

P_ = pytest.importorskip("paper_2505_04612_b200.parallel")


@pytest.mark.parametrize("world,precision", [(1, "fp64"), (3, "fp64"), (1, "fp32"), (3, "fp32")])
def test_sharded_config1_matches_reference(golden_c1, world, precision):
    """fp64 moments: L1 history within 1e-6; fp32 moments (shifted model, the
    default): within the north-star 1e-4.  Decisions and RRA/RTA identical."""
    g = golden_c1
    dev = torch.device("cuda")
    lengths = g["c1_len"].astype(np.int64)
    ij = g["c1_ij"].astype(np.int64)
    x1 = np.column_stack([g["c1_x1"].astype(np.float64), np.ones(len(g["c1_x1"]))])
    x2 = np.column_stack([g["c1_x2"].astype(np.float64), np.ones(len(g["c1_x2"]))])
    cams = np.zeros_like(ij)
    n = int(ij.max()) + 1
    bounds = P_.partition_pairs(lengths, world)
    shards = P_.make_shards(x1, x2, lengths, ij, cams, n, 1, True, bounds, dev, precision=precision)
    R = g["c1_R_in"]
    params = torch.as_tensor(np.concatenate([np.concatenate([R[:, :, 0], R[:, :, 1]], 1).ravel(),
                                             g["c1_c_in"].ravel(), [0.0]]), device=dev)
    eng = P_.ShardedIrlsEngine(shards, params, Cfg())
    l1 = eng.run()
    np.testing.assert_allclose(l1, g["c1_l1"], rtol=1e-6 if precision == "fp64" else 1e-4)
    assert [eng.dropped, eng.kept] == list(g["c1_counts"])
    p = params.cpu().numpy()
    rot = O.project_to_so3(O.rot6d_to_matrix(p[:6 * n].reshape(n, 6)))
    cen = p[6 * n:9 * n].reshape(n, 3)
    tol_r, tol_c = (2e-5, 5e-5) if precision == "fp64" else (1e-4, 2e-4)
    assert np.abs(rot - g["c1_R_out"]).max() < tol_r
    assert np.abs(cen - g["c1_c_out"]).max() < tol_c
    ours = O.pose_metrics(rot, cen, g["c1_R_gt"], g["c1_c_gt"])
    ref = O.pose_metrics(g["c1_R_out"], g["c1_c_out"], g["c1_R_gt"], g["c1_c_gt"])
    for k in ("RRA@1", "RRA@3", "RTA@1", "RTA@3"):
        assert ours[k] == ref[k]
    counts = np.concatenate([sh.buf.n_active[0 if True else 1].cpu().numpy()[:sh.graph.n_pairs]
                             for sh in shards])
    active = np.concatenate([sh.store.caller_masks() for sh in shards])
    start = np.concatenate([[0], np.cumsum(lengths)])
    per_pair = np.array([active[start[k]:start[k + 1]].sum() for k in range(len(lengths))])
    assert np.array_equal(per_pair, g["c1_active_count"])
    del counts
