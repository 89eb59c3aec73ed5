"""GPU parity of the global translation alignment (fm_tr_* kernels) against
the reference's golden vectors.

Tolerances: loss/gradient/residuals fp64, <= 1e-12 rel; short descents
(300-400 steps) <= 1e-6 abs on centres; the config-1 multi-init run (3 x 6000
+ 6000 steps of sign-gradient Adam) is compared on the converged loss and the
canonical shape."""

import numpy as np
import pytest
import torch

from oracle import fastmap_oracle as O
from tests.helpers import Cfg

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2505_04612_b200.translation")


def _graph(g):
    return T.DirectionGraph(n=int(g["tr_n"][0]), edges_i=g["tr_ei"], edges_j=g["tr_ej"],
                            directions=g["tr_dirs"])


def test_loss_grad_residuals_canonicalize(golden_small):
    g = golden_small
    gr = _graph(g)
    loss, grad = T.translation_loss_and_grad(g["tr_start"], gr)
    np.testing.assert_allclose(loss, g["tr_loss"][0], rtol=1e-13)
    np.testing.assert_allclose(grad, g["tr_grad"], rtol=1e-11, atol=1e-15)
    np.testing.assert_allclose(T.per_node_residuals(g["tr_start"], gr), g["tr_node_res"], rtol=1e-12)
    np.testing.assert_allclose(T.canonicalize(g["tr_start"] * 3 + 1), g["tr_canon"], atol=1e-13)


def test_align_and_multi_init(golden_small):
    g = golden_small
    gr = _graph(g)
    c, l = T.align_centers(gr, Cfg(translation_steps=300), seed=4)
    np.testing.assert_allclose(c, g["tr_align"], atol=1e-6)
    np.testing.assert_allclose(l, g["tr_align_loss"][0], rtol=1e-6)
    c, l = T.multi_init_align(gr, Cfg(translation_steps=400, translation_inits=3), seed=1)
    np.testing.assert_allclose(c, g["tr_multi"], atol=1e-5)
    np.testing.assert_allclose(l, g["tr_multi_loss"][0], rtol=1e-5)


def test_edge_cases():
    # zero steps: the initialisation and an infinite loss (ref/translation.py:145-152)
    gr = T.DirectionGraph(n=3, edges_i=np.array([0, 1]), edges_j=np.array([1, 2]),
                          directions=np.array([[1.0, 0, 0], [0, 1.0, 0]]))
    init = np.arange(9.0).reshape(3, 3)
    c, l = T.align_centers(gr, Cfg(), init=init, steps=0)
    assert np.array_equal(c, init) and l == np.inf
    # isolated node: zero gradient, zero residual (degree-0 -> 0)
    gr = T.DirectionGraph(n=4, edges_i=np.array([0, 1]), edges_j=np.array([1, 2]),
                          directions=np.array([[1.0, 0, 0], [0, 1.0, 0]]))
    start = np.random.default_rng(0).normal(size=(4, 3))
    loss, grad = T.translation_loss_and_grad(start, gr)
    l_ref, g_ref = O.translation_loss_grad(start, gr.edges_i, gr.edges_j, gr.directions)
    np.testing.assert_allclose(loss, l_ref, rtol=1e-14)
    np.testing.assert_allclose(grad, g_ref, rtol=1e-12, atol=1e-16)
    assert np.all(grad[3] == 0)
    assert T.per_node_residuals(start, gr)[3] == 0.0
    # single init falls back to align_centers
    c1, l1 = T.multi_init_align(gr, Cfg(translation_steps=50, translation_inits=1), seed=3)
    c2, l2 = T.align_centers(gr, Cfg(translation_steps=50), seed=3)
    np.testing.assert_array_equal(c1, c2)


def test_config1_multi_init(golden_c1):
    g = golden_c1
    ij = g["c1_ij"].astype(np.int64)
    gr = T.DirectionGraph(n=len(g["c1_c_gt"]), edges_i=ij[:, 0], edges_j=ij[:, 1],
                          directions=g["c1_dirs"])
    c, loss = T.multi_init_align(gr, Cfg(), seed=0)
    ref_loss = g["c1_tr_loss"][0]
    assert abs(loss - ref_loss) <= 1e-3 * ref_loss
    a = O.canonicalize(c)
    b = O.canonicalize(g["c1_tr_centers"])
    s, R, t = O.umeyama(a, b)
    assert np.max(np.linalg.norm(a @ (s * R).T + t - b, axis=1)) < 1e-2


def test_sharded_inits_reproduce_the_batch():
    """Runs do not depend on their batch: starts split into blocks (as
    parallel.multi_init_align_sharded does over ranks) give bitwise the same
    runs, merge and final descent as the single batch."""
    from paper_2505_04612_b200 import parallel as P_

    rng = np.random.default_rng(5)
    n, m = 40, 300
    c = rng.normal(size=(n, 3))
    e = set()
    while len(e) < m:
        i, j = rng.integers(0, n, size=2)
        if i != j:
            e.add((min(i, j), max(i, j)))
    e = np.array(sorted(e))
    d = c[e[:, 1]] - c[e[:, 0]]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    g = T.DirectionGraph(n=n, edges_i=e[:, 0], edges_j=e[:, 1], directions=d)

    class C:
        translation_lr, translation_steps, translation_inits = 1e-2, 300, 7
        adam_beta1, adam_beta2, adam_eps = 0.9, 0.999, 1e-8
    full = T.init_runs(g, C, 3, range(7))
    for world in (2, 3):
        b = P_.init_blocks(7, world)
        parts = [T.init_runs(g, C, 3, range(b[r], b[r + 1])) for r in range(world)]
        assert torch.equal(torch.cat(parts, dim=1), full)
    c1, l1 = T.multi_init_align(g, C, seed=3)
    c2, l2 = T.merge_and_finish(g, C, torch.cat(parts, dim=1))
    assert np.array_equal(c1, c2) and l1 == l2
