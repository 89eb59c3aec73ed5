"""GPU parity of the rotation refinement (fm_rot_*; SURVEY 8f "next" #3)
against the reference's golden vectors (tests/golden/make_rotation_golden.py).

Tolerances: loss 1e-13 and 6D gradient 1e-11 relative (fp64; the node
gather and the 6D vector-Jacobian product sum in a different order than the
reference's scatter + (9, 6) Jacobian).  refine_rotations: the same number
of recorded losses (the best-iterate / early-stop rules are the
reference's) and the first 150 losses within 1e-10 relative.  Past that the
run is chaotic -- the geodesic gradient is unbounded at zero error, so Adam
hovers around the optimum (the reference says so, ref/rotation.py:208-209)
and ulp-level differences grow ~10x per 30 steps (tools/rot_diff.py:
6e-13 at step 200, 2e-4 at step 500) -- so the final state is compared by
quality: best loss within 5% (or 1e-5 absolute near zero), rotations within
1e-3."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

Rm = pytest.importorskip("paper_2505_04612_b200.rotation")


class _Edge:
    def __init__(self, i, j, rel):
        self.i, self.j, self.rel_rotation = int(i), int(j), rel


class _Graph:
    def __init__(self, n, ei, ej, rel):
        self.n_images = n
        self.edges = [_Edge(i, j, r) for i, j, r in zip(ei, ej, rel)]
        self.registered = np.ones(n, dtype=bool)


class _Cfg:
    def __init__(self, steps, c):
        self.rotation_steps = int(steps)
        self.rotation_lr, self.adam_beta1, self.adam_beta2, self.adam_eps = (float(x) for x in c)


@pytest.mark.parametrize("k", [0, 1, 2])
def test_loss_grad_matches_reference(golden_rotation, k):
    g, pre = golden_rotation, f"r{k}_"
    loss, grad = Rm.rotation_loss_and_grad(g[pre + "p"], g[pre + "ei"], g[pre + "ej"], g[pre + "rel"])
    np.testing.assert_allclose(loss, g[pre + "loss"][0], rtol=1e-13)
    np.testing.assert_allclose(grad, g[pre + "grad"], rtol=1e-11, atol=1e-14 * np.abs(grad).max())


@pytest.mark.parametrize("k", [0, 1, 2])
def test_refine_rotations_matches_reference(golden_rotation, k):
    g, pre = golden_rotation, f"r{k}_"
    graph = _Graph(int(g[pre + "n"][0]), g[pre + "ei"], g[pre + "ej"], g[pre + "rel"])
    out, hist = Rm.refine_rotations(g[pre + "init"], graph, _Cfg(g[pre + "steps"][0], g[pre + "cfg"]))
    ref = g[pre + "hist"]
    print(f"rotation graph {k}: {len(hist)} steps (ref {len(ref)}), max |dR| "
          f"{np.abs(out - g[pre + 'out']).max():.2e}")
    assert len(hist) == len(ref)
    np.testing.assert_allclose(hist[:150], ref[:150], rtol=1e-10)
    assert abs(min(hist) - ref.min()) <= max(0.05 * ref.min(), 1e-5)
    assert np.abs(out - g[pre + "out"]).max() < 1e-3
