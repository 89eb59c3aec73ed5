"""The point-pair store built on the device (fm_store_build) against a host
restatement of the layout: every caller point at slot
pair_off[rank[k]] + m, fp32 (x, y) (and z when z != 1) or the caller's fp64
(x, y, z), zeros on padding, packed active bits; sanitising of non-finite
points; the caller-order maps (mask write-back, slot gathers / scatters).
Bit-exact throughout (integer and copy work)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2505_04612_b200.store")


def ragged(seed, homog=False, nan=True):
    rng = np.random.default_rng(seed)
    lens = np.array([0, 1, 17, 33, 500, 16, 15, 64, 3, 129, 0, 250], dtype=np.int64)
    P = len(lens)
    ij = rng.integers(0, 6, size=(P, 2))
    ij[:, 1] = ij[:, 0] + 1 + rng.integers(0, 3, size=P)   # duplicates and unsorted pairs
    Z = int(lens.sum())
    x1 = rng.normal(size=(Z, 3))
    x2 = rng.normal(size=(Z, 3))
    if not homog:
        x1[:, 2] = x2[:, 2] = 1.0
    if nan:
        x1[5, 0] = np.nan
        x2[40, 1] = np.inf
    act = rng.random(Z) > 0.2
    return lens, ij, x1, x2, act


def host_layout(store, lens, x1, x2, act, sanitize, fp64):
    n = store.n_slots
    start = store.caller_start
    if fp64:
        e1 = np.zeros((n, 3))
        e2 = np.zeros((n, 3))
    else:
        e1 = np.zeros((n, 2), np.float32)
        e2 = np.zeros((n, 2), np.float32)
        z1 = np.zeros(n, np.float32)
        z2 = np.zeros(n, np.float32)
    bits = np.zeros(n, bool)
    for k in range(len(lens)):
        for m in range(lens[k]):
            z = start[k] + m
            sl = store.pair_off[store.rank[k]] + m
            a, c, on = x1[z].copy(), x2[z].copy(), act[z]
            if sanitize and not (np.all(np.isfinite(a)) and np.all(np.isfinite(c))):
                a[:] = c[:] = [0.0, 0.0, 1.0]
                on = False
            if fp64:
                e1[sl], e2[sl] = a, c
            else:
                e1[sl], e2[sl] = a[:2], c[:2]
                z1[sl], z2[sl] = a[2], c[2]
            bits[sl] = on
    words = np.packbits(bits, bitorder="little").view(np.int32)
    return e1, e2, (z1, z2) if not fp64 else None, words


@pytest.mark.parametrize("homog,fp64,sanitize", [(False, False, True), (False, False, False),
                                                  (True, False, False), (True, True, False)])
def test_device_store_build_matches_host_layout(homog, fp64, sanitize):
    lens, ij, x1, x2, act = ragged(3, homog=homog)
    dev = torch.device("cuda")
    st = S.PointPairStore(x1, x2, lens, ij[:, 0], ij[:, 1], active=act, device=dev,
                          sanitize=sanitize, fp64=fp64)
    assert np.array_equal(st.order, S.pair_order(ij[:, 0], ij[:, 1]))
    e1, e2, zz, words = host_layout(st, lens, x1, x2, act, sanitize, fp64)
    if fp64:
        assert np.array_equal(st.x1d.cpu().numpy(), e1, equal_nan=True)
        assert np.array_equal(st.x2d.cpu().numpy(), e2, equal_nan=True)
    else:
        assert np.array_equal(st.x1.cpu().numpy(), e1, equal_nan=True)
        assert np.array_equal(st.x2.cpu().numpy(), e2, equal_nan=True)
        assert st.homogeneous == homog
        if homog:
            assert np.array_equal(st.x1z.cpu().numpy(), zz[0], equal_nan=True)
    assert np.array_equal(st.active.cpu().numpy(), words)
    # caller-order maps
    expect = act.copy()
    if sanitize:
        bad = ~(np.isfinite(x1).all(1) & np.isfinite(x2).all(1))
        expect &= ~bad
    assert np.array_equal(st.caller_masks(), expect)
    vals = np.random.default_rng(0).normal(size=int(lens.sum()))
    slots = st.scatter_slots(vals)
    assert np.array_equal(st.gather_slots(slots).cpu().numpy(), vals)


def test_empty_and_all_active():
    dev = torch.device("cuda")
    st = S.PointPairStore(np.zeros((0, 3)), np.zeros((0, 3)), [0, 0], [1, 0], [2, 1], device=dev)
    assert st.n_points == 0 and np.all(st.active.cpu().numpy() == 0)
    lens, ij, x1, x2, _ = ragged(4, nan=False)
    st = S.PointPairStore(x1, x2, lens, ij[:, 0], ij[:, 1], device=dev)
    assert st.caller_masks().all()
    assert int(st.active_bits().sum().item()) == int(lens.sum())


def test_from_pairs_input_forms_build_the_same_store():
    """from_pairs concatenates straight into the pinned staging when every
    pair holds (n, 3) arrays numpy can cast safely; other forms (fp32 arrays,
    nested lists, integer masks) take the checked path.
    All give the same device store, bit for bit."""
    from types import SimpleNamespace as NS
    dev = torch.device("cuda")
    lens, ij, x1, x2, act = ragged(7, nan=False)
    x1 = x1.astype(np.float32).astype(np.float64)  # exact in fp32 for the fp32 form
    x2 = x2.astype(np.float32).astype(np.float64)
    start = np.concatenate([[0], np.cumsum(lens)])

    def pairs(f1, f2, fa):
        return [NS(i=int(ij[k, 0]), j=int(ij[k, 1]), x1=f1(x1[start[k]:start[k + 1]]),
                   x2=f2(x2[start[k]:start[k + 1]]), active=fa(act[start[k]:start[k + 1]]))
                for k in range(len(lens))]

    ident = lambda a: a.copy()  # noqa: E731
    # the reference's EpipolarPair holds (M, 3) homogeneous x1 / x2 (ref/epipolar.py:26-27)
    forms = {
        "fp64": pairs(ident, ident, ident),
        "fp32": pairs(lambda a: a.astype(np.float32), ident, ident),
        "lists": pairs(lambda a: a.tolist(), ident, lambda a: a.tolist()),
        "int_mask": pairs(ident, ident, lambda a: a.astype(np.int64)),
    }
    ref = None
    for name, ps in forms.items():
        st = S.PointPairStore.from_pairs(ps, device=dev)
        got = (st.x1.cpu().numpy(), st.x2.cpu().numpy(), st.active.cpu().numpy(), st.homogeneous)
        if ref is None:
            ref = got
            continue
        for a, b in zip(ref[:3], got[:3]):
            assert np.array_equal(a, b), name
        assert got[3] is False, name
