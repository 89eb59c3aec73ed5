"""GPU Adam, 6D rotation maps and SO(3) projection vs the reference golden
vectors (Adam bit-exact: the kernel avoids FMA contraction)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

Op = pytest.importorskip("paper_2505_04612_b200.optim")
from paper_2505_04612_b200 import model  # noqa: E402


def test_adam_bit_exact(golden_small):
    g = golden_small
    opt = Op.Adam(g["adam_p0"], lr=0.05)
    for k, gr in enumerate(g["adam_grads"]):
        np.testing.assert_array_equal(opt.step(gr), g["adam_traj"][k])
    with pytest.raises(ValueError):
        opt.step(np.zeros(3))
    with pytest.raises(FloatingPointError):
        Op.Adam(np.zeros(2)).step(np.array([1.0, np.nan]))


def test_adam_minimizes_quadratic():
    opt = Op.Adam(np.array([5.0, -3.0]), lr=0.1)
    for _ in range(500):
        opt.step(2.0 * opt.params)
    assert np.linalg.norm(opt.params) < 1e-4


def test_rot6d_and_projection(golden_small):
    g = golden_small
    np.testing.assert_allclose(Op.rot6d_to_matrix(g["rot6d_in"]), g["rot6d_R"], atol=1e-14)
    np.testing.assert_allclose(Op.rot6d_jacobian(g["rot6d_in"]), g["rot6d_J"], atol=1e-12)
    np.testing.assert_allclose(model.project_to_so3(g["so3_in"]), g["so3_out"], atol=1e-11)
    with pytest.raises(ValueError, match="zero first half"):
        Op.rot6d_to_matrix(np.array([0.0, 0.0, 0.0, 1.0, 0.0, 0.0]))
    with pytest.raises(ValueError, match="collinear"):
        Op.rot6d_to_matrix(np.array([1.0, 0.0, 0.0, 2.0, 0.0, 0.0]))
