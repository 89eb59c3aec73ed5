"""GPU parity of the global translation alignment (fm_tr_* kernels) against
the reference's golden vectors.

Tolerance: none.  The kernels perform numpy's operations in numpy's order
(fm_translation.cu header), so losses, gradients, node residuals, canonical
centres and whole descents -- including the config-1 multi-init run of
3 x 6000 + 6000 sign-gradient Adam steps and the 16-init C3 batch -- are
BITWISE the reference's."""

import hashlib
import os

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
    assert loss == g["tr_loss"][0]
    np.testing.assert_array_equal(grad, g["tr_grad"])
    np.testing.assert_array_equal(T.per_node_residuals(g["tr_start"], gr), g["tr_node_res"])
    np.testing.assert_array_equal(T.canonicalize(g["tr_start"] * 3 + 1), g["tr_canon"])


def test_align_and_multi_init(golden_small):
    g = golden_small
    gr = _graph(g)
    c, l = T.align_centers(gr, Cfg(translation_steps=300), seed=4)
    np.testing.assert_array_equal(c, g["tr_align"])
    assert l == g["tr_align_loss"][0]
    c, l = T.multi_init_align(gr, Cfg(translation_steps=400, translation_inits=3), seed=1)
    np.testing.assert_array_equal(c, g["tr_multi"])
    assert l == g["tr_multi_loss"][0]


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
    assert loss == l_ref
    np.testing.assert_array_equal(grad, g_ref)
    assert np.all(grad[3] == 0)
    assert T.per_node_residuals(start, gr)[3] == 0.0
    # single init falls back to align_centers
    c1, l1 = T.multi_init_align(gr, Cfg(translation_steps=50, translation_inits=1), seed=3)
    c2, l2 = T.align_centers(gr, Cfg(translation_steps=50), seed=3)
    np.testing.assert_array_equal(c1, c2)


def test_config1_multi_init(golden_c1):
    """BASELINE config 1: 3 inits x 6000 steps + merge + 6000 steps, bitwise the
    reference's centres and loss, hence the same translation-stage ATE and
    RTA (north star: "ATE and RRA/RTA equal to the reference")."""
    g = golden_c1
    ij = g["c1_ij"].astype(np.int64)
    gr = T.DirectionGraph(n=len(g["c1_c_gt"]), edges_i=ij[:, 0], edges_j=ij[:, 1],
                          directions=g["c1_dirs"])
    c, loss = T.multi_init_align(gr, Cfg(), seed=0)
    assert loss == g["c1_tr_loss"][0]
    np.testing.assert_array_equal(c, g["c1_tr_centers"])
    ours = O.pose_metrics(g["c1_R_in"], c, g["c1_R_gt"], g["c1_c_gt"])
    ref = O.pose_metrics(g["c1_R_in"], g["c1_tr_centers"], g["c1_R_gt"], g["c1_c_gt"])
    assert ours == ref, (ours, ref)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def c3():
    from paper_2505_04612_b200.scenes import translation_graph_c3
    f = os.path.join(os.path.dirname(__file__), "golden", "golden_c3.npz")
    gold = dict(np.load(f))
    ei, ej, d, _ = translation_graph_c3()
    return gold, T.DirectionGraph(n=2000, edges_i=ei, edges_j=ej, directions=d)


def test_c3_loss_grad_all_starts(c3):
    """BASELINE configs[2] (2,000 nodes, 200,000 edges): loss and gradient at
    the 16 seeded starts in ONE batched call, bitwise the reference's
    translation_loss_and_grad (ref/translation.py:112-125) for each start."""
    gold, gr = c3
    starts = np.stack([np.random.default_rng(k).standard_normal((gr.n, 3)) for k in range(16)], axis=1)
    dg = T.device_graph(gr)
    t = torch.as_tensor(np.ascontiguousarray(starts), device=dg.device).requires_grad_(True)
    loss = T.TranslationL1Loss.apply(t, dg)
    loss.sum().backward()
    loss = loss.detach().cpu().numpy()
    grad = t.grad.cpu().numpy()
    np.testing.assert_array_equal(loss, gold["c3_loss0"])
    for k in range(16):
        np.testing.assert_array_equal(grad[:, k][:64], gold["c3_grad0_prefix"][k])
        assert _sha(grad[:, k]) == gold["c3_grad0_sha"][k], k


def test_c3_batched_multi_init(c3):
    """multi_init_align with 16 inits (the C3 shape: 4 warp groups of runs)
    and 200 steps per descent: every run, the per-node residuals, the merge
    choice, the merged start and the final descent bitwise the reference's
    (ref/translation.py:169-186)."""
    gold, gr = c3
    steps = int(gold["c3_steps"][0])
    cfg = Cfg(translation_steps=steps, translation_inits=16)
    dg = T.device_graph(gr)
    runs = T.init_runs(gr, cfg, 0, range(16), dg)
    raw = runs.cpu().numpy()
    for k in range(16):
        np.testing.assert_array_equal(raw[:64, k], gold["c3_run_prefix"][k])
        assert _sha(raw[:, k]) == gold["c3_run_sha"][k], k
    c, loss, choice = T.merge_and_finish(gr, cfg, runs.clone(), dg, return_choice=True)
    np.testing.assert_array_equal(choice, gold["c3_choice"])
    np.testing.assert_array_equal(c, gold["c3_final"])
    assert loss == gold["c3_final_loss"][0]
    canon = torch.from_numpy(raw).clone().to(dg.device)
    from paper_2505_04612_b200 import _native as N_
    N_.check(N_.lib().fm_tr_canonicalize(N_.ptr(canon), gr.n, 16, None, 0, N_.stream_handle()))
    canon_np = canon.cpu().numpy()
    for k in range(16):
        assert _sha(canon_np[:, k]) == gold["c3_canon_sha"][k], k
        res = T.per_node_residuals(canon_np[:, k], gr)
        np.testing.assert_array_equal(res[:64], gold["c3_node_res_prefix"][k])
        assert _sha(res) == gold["c3_node_res_sha"][k], k
    c2, loss2 = T.multi_init_align(gr, cfg, seed=0)
    np.testing.assert_array_equal(c2, gold["c3_final"])
    assert loss2 == gold["c3_final_loss"][0]


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


def test_bitwise_over_wide_dynamic_range():
    """The shared-reciprocal division (Markstein correction) is the correctly
    rounded quotient: loss, gradient and node residuals bitwise the numpy
    restatement (oracle, itself pinned bitwise to the reference's golden
    vectors) for centres spread over 12 decades, coincident endpoints (the
    1e-8 length clamp), duplicate edges and self-loops."""
    rng = np.random.default_rng(11)
    n, m = 300, 4000
    scale = 10.0 ** rng.uniform(-6, 6, size=(n, 1))
    c = rng.normal(size=(n, 3)) * scale
    c[5] = c[6]                      # coincident pair -> clamped length
    c[7] = c[8] + 1e-12
    ei = rng.integers(0, n, size=m)
    ej = rng.integers(0, n, size=m)
    ei[:4], ej[:4] = [5, 6, 7, 9], [6, 5, 8, 9]      # clamp cases and a self-loop
    ei[10:20], ej[10:20] = 3, 4                      # duplicates
    d = rng.normal(size=(m, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    gr = T.DirectionGraph(n=n, edges_i=ei, edges_j=ej, directions=d)
    loss, grad = T.translation_loss_and_grad(c, gr)
    l_ref, g_ref = O.translation_loss_grad(c, ei, ej, d)
    assert loss == l_ref
    np.testing.assert_array_equal(grad, g_ref)
    np.testing.assert_array_equal(T.per_node_residuals(c, gr), O.per_node_residuals(c, ei, ej, d))


def _descent(graph, init, steps, cluster):
    """translation._align with the cluster-persistent path on or off."""
    old = os.environ.pop("FM_TR_NOCLUSTER", None)
    if not cluster:
        os.environ["FM_TR_NOCLUSTER"] = "1"
    try:
        c, loss = T._align(T.device_graph(graph), init, Cfg(), steps)
        return c.cpu().numpy(), loss
    finally:
        os.environ.pop("FM_TR_NOCLUSTER", None)
        if old is not None:
            os.environ["FM_TR_NOCLUSTER"] = old


@pytest.mark.parametrize("B,steps", [(1, 1), (1, 250), (2, 7), (3, 250), (5, 33)])
def test_cluster_descent_equals_per_step_launches(B, steps):
    """Small graphs run the whole descent as one thread-block-cluster launch
    (fm_translation.cu tr_steps_cluster_kernel); it must give the per-step
    launches' results bit for bit: odd and even step counts (the ping-pong
    parity), runs per warp 1 and 2 with idle run lanes (B = 3, 5), a hub
    node of degree 300 (several incidence batches), duplicate edges and a
    self-loop."""
    rng = np.random.default_rng(B * 1000 + steps)
    n, m = 48, 900
    ei = rng.integers(0, n, size=m)
    ej = rng.integers(0, n, size=m)
    ei[:300] = 0                     # hub
    ei[300:310], ej[300:310] = 4, 5  # duplicates
    ei[310], ej[310] = 6, 6          # self-loop
    d = rng.normal(size=(m, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    gr = T.DirectionGraph(n=n, edges_i=ei, edges_j=ej, directions=d)
    init = rng.normal(size=(n, B, 3))
    c1, l1 = _descent(gr, init, steps, cluster=True)
    c2, l2 = _descent(gr, init, steps, cluster=False)
    np.testing.assert_array_equal(c1, c2)
    np.testing.assert_array_equal(l1, l2)
    if B == 1 and steps == 1:  # and the numpy restatement of the reference
        c_ref, l_ref = O.align_centers(n, ei, ej, d, Cfg(), init=init[:, 0], steps=steps)
        np.testing.assert_array_equal(c1[:, 0], c_ref)
        assert l1[0] == l_ref


def test_cluster_descent_nonfinite_raises():
    """A NaN direction makes the loss non-finite at the first step: the
    cluster path raises the reference's error (ref/translation.py:150)."""
    gr = T.DirectionGraph(n=4, edges_i=np.array([0, 1, 2]), edges_j=np.array([1, 2, 3]),
                          directions=np.array([[1.0, 0, 0], [np.nan, 1.0, 0], [0, 0, 1.0]]))
    with pytest.raises(FloatingPointError, match="non-finite translation loss"):
        T.align_centers(gr, Cfg(translation_steps=20), seed=0)
