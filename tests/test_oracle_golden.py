"""Pin the CPU oracle (oracle/fastmap_oracle.py) to the reference's own
outputs (tests/golden/*.npz made by tests/golden/make_golden.py from
/root/reference).  CPU only."""

import numpy as np
import pytest

from oracle import fastmap_oracle as O
from tests.helpers import Cfg, c1_pairs, SimplePair, pairs_from


def _case(g, k):
    pre = f"e{k}_"
    n, cams, rf = (int(x) for x in g[pre + "meta"])
    pairs = pairs_from(g, pre, SimplePair)
    ij = g[pre + "ij"]
    cc = g[pre + "cams"]
    flat = O.FlatPairs.from_pairs(pairs)
    return pre, n, cams, bool(rf), pairs, ij, cc, flat


@pytest.mark.parametrize("k", [0, 1, 2])
def test_epipolar_api_vectors(golden_small, k):
    g = golden_small
    pre, n, cams, rf, pairs, ij, cc, flat = _case(g, k)
    params = g[pre + "params"]
    f = O.pair_forward(params, n, ij[:, 0], ij[:, 1], cc[:, 0], cc[:, 1], rf)
    r = np.abs(O.signed_residuals(flat, f["ghat"]))
    np.testing.assert_allclose(r, g[pre + "residuals"], rtol=1e-12, atol=1e-14)
    # unweighted W over active points
    W = O.weights_per_pair(flat, flat.active.astype(float))
    np.testing.assert_allclose(W, g[pre + "W_unweighted"], rtol=1e-11, atol=1e-13)
    Wi = O.weights_per_pair(flat, O.irls_weights(r, flat.active))
    np.testing.assert_allclose(Wi, g[pre + "W_irls"], rtol=1e-10, atol=1e-10)
    Z = int(flat.active.sum())
    l1 = np.sum(np.where(flat.active, r, 0.0)) / Z
    np.testing.assert_allclose(l1, g[pre + "loss_l1"][0], rtol=1e-12)
    assert Z == int(g[pre + "loss_l1"][1])
    l2, _ = O.quad_loss_grad(params, n, ij[:, 0], ij[:, 1], cc[:, 0], cc[:, 1], rf, cams, W, Z)
    np.testing.assert_allclose(l2, g[pre + "loss_l2"][0], rtol=1e-10)
    loss, grad = O.quad_loss_grad(params, n, ij[:, 0], ij[:, 1], cc[:, 0], cc[:, 1], rf, cams,
                                  g[pre + "W_irls"], Z)
    np.testing.assert_allclose(loss, g[pre + "quad_loss"][0], rtol=1e-11)
    np.testing.assert_allclose(grad, g[pre + "quad_grad"], rtol=1e-9,
                               atol=1e-12 * np.abs(grad).max())


def test_point_pass_linearisation_identity(golden_small):
    """Shifted model: vgrad = W ghat0 and s0 = ghat0^T W ghat0 at the
    linearisation point (shifted quadratic model)."""
    g = golden_small
    pre, n, cams, rf, pairs, ij, cc, flat = _case(g, 1)
    gh = O.pair_forward(g[pre + "params"], n, ij[:, 0], ij[:, 1], cc[:, 0], cc[:, 1], rf)["ghat"]
    out = O.point_pass(flat, gh)
    np.testing.assert_allclose(out["vgrad"], np.einsum("pkl,pl->pk", out["W"], gh), rtol=1e-9,
                               atol=1e-9)
    np.testing.assert_allclose(out["s0"], np.einsum("pk,pkl,pl->p", gh, out["W"], gh), rtol=1e-9)


def test_irls_refine_small(golden_small):
    g = golden_small
    pairs = pairs_from(g, "irls_", SimplePair)
    flat = O.FlatPairs.from_pairs(pairs)
    R, c, fs, rep = O.irls_refine(g["irls_R_in"], g["irls_c_in"], g["irls_ij"], g["irls_cams"],
                                  flat, Cfg(epipolar_lr=1e-3), n_cameras=1)
    # 900 Adam steps amplify summation-order rounding: 1e-7 absolute
    np.testing.assert_allclose(R, g["irls_R_out"], atol=1e-7)
    np.testing.assert_allclose(c, g["irls_c_out"], atol=1e-7)
    np.testing.assert_allclose(fs, g["irls_focal"], rtol=1e-6)
    np.testing.assert_allclose(rep["l1_history"], g["irls_l1"], rtol=1e-6)
    assert [rep["dropped_pairs"], rep["active_pairs"]] == list(g["irls_counts"])
    assert np.array_equal(flat.active, g["irls_active_out"])


def test_optim_vectors(golden_small):
    g = golden_small
    np.testing.assert_allclose(O.rot6d_to_matrix(g["rot6d_in"]), g["rot6d_R"], atol=1e-14)
    np.testing.assert_allclose(O.rot6d_jacobian(g["rot6d_in"]), g["rot6d_J"], atol=1e-12)
    np.testing.assert_allclose(O.project_to_so3(g["so3_in"]), g["so3_out"], atol=1e-12)
    opt = O.Adam(g["adam_p0"], lr=0.05)
    for k, gr in enumerate(g["adam_grads"]):
        np.testing.assert_array_equal(opt.step(gr), g["adam_traj"][k])
    with pytest.raises(FloatingPointError):
        O.Adam(np.zeros(2)).step(np.array([1.0, np.nan]))
    with pytest.raises(ValueError):
        O.rot6d_to_matrix(np.array([0.0, 0, 0, 1, 0, 0]))


def test_translation_vectors(golden_small):
    """The oracle's translation functions keep numpy's operations in the
    reference's order: bitwise the reference's golden outputs."""
    g = golden_small
    n = int(g["tr_n"][0])
    ei, ej, dirs = g["tr_ei"], g["tr_ej"], g["tr_dirs"]
    loss, grad = O.translation_loss_grad(g["tr_start"], ei, ej, dirs)
    assert loss == g["tr_loss"][0]
    np.testing.assert_array_equal(grad, g["tr_grad"])
    np.testing.assert_array_equal(O.per_node_residuals(g["tr_start"], ei, ej, dirs), g["tr_node_res"])
    np.testing.assert_array_equal(O.canonicalize(g["tr_start"] * 3 + 1), g["tr_canon"])
    c, l = O.align_centers(n, ei, ej, dirs, Cfg(translation_steps=300), seed=4)
    np.testing.assert_array_equal(c, g["tr_align"])
    assert l == g["tr_align_loss"][0]
    c, l = O.multi_init_align(n, ei, ej, dirs, Cfg(translation_steps=400, translation_inits=3),
                              seed=1)
    np.testing.assert_array_equal(c, g["tr_multi"])
    assert l == g["tr_multi_loss"][0]


def test_config1_metrics_of_reference_output(golden_c1):
    """The reference's config-1 adjustment improves the perturbed poses; the
    oracle metrics reproduce that."""
    g = golden_c1
    before = O.pose_metrics(g["c1_R_in"], g["c1_c_in"], g["c1_R_gt"], g["c1_c_gt"])
    after = O.pose_metrics(g["c1_R_out"], g["c1_c_out"], g["c1_R_gt"], g["c1_c_gt"])
    assert after["ATE"] < before["ATE"]
    assert after["RRA@1"] >= before["RRA@1"]


@pytest.mark.slow
def test_config1_irls_oracle(golden_c1):
    """Full oracle adjustment on config 1 equals the reference's result."""
    g = golden_c1
    pairs = c1_pairs(g, SimplePair)
    flat = O.FlatPairs.from_pairs(pairs)
    cams = np.zeros((len(pairs), 2), dtype=np.int64)
    R, c, fs, rep = O.irls_refine(g["c1_R_in"], g["c1_c_in"], g["c1_ij"], cams, flat, Cfg())
    np.testing.assert_allclose(rep["l1_history"], g["c1_l1"], rtol=1e-6)
    np.testing.assert_allclose(R, g["c1_R_out"], atol=1e-7)
    np.testing.assert_allclose(c, g["c1_c_out"], atol=1e-7)
    assert [rep["dropped_pairs"], rep["active_pairs"]] == list(g["c1_counts"])
