"""Drop-in for ``fastmap.epipolar`` (ref/epipolar.py) on the B200.

Same names, signatures, return types and exceptions as the reference; the
arithmetic runs in the C-ABI CUDA library:

* point-pair level (O(point pairs)): ``current_residuals``,
  ``precompute_weights``, ``epipolar_loss`` and the passes inside
  ``irls_refine`` -> ``fm_point_pass`` (fused residual / prune / L1 / IRLS
  moments kernel);
* image-pair level (O(image pairs) per step): ``quadratic_loss_and_grad`` ->
  ``fm_epi_loss_grad`` behind the ``EpipolarQuadraticLoss`` autograd
  function, and the 100-step inner loop of ``irls_refine`` ->
  ``fm_epi_adam_steps`` (loss + gradient + Adam per step, replayed from a
  CUDA graph).

``irls_refine`` uploads the point pairs once, keeps every pass, step and
mask update on the device, synchronises once per prune round and once per
IRLS iteration (error flag), and writes the pruned masks back into the
caller's ``EpipolarPair.active`` arrays in place, as the reference does
(ref/epipolar.py:283).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .model import PoseState  # noqa: F401  (re-exported for API parity)
from .optim import matrix_to_rot6d, skew  # noqa: F401
from .store import PairGraph, PointPairStore

_HUBER_EPS = 1e-6
# Moment precision of the IRLS point passes: "fp32" = fp32 Kronecker moments
# about the linearisation point (shifted quadratic model) with
# exact fp64 residuals / prune decisions; "fp64" = exact fp64 moments.
DEFAULT_PRECISION = "fp32"

SYM = [[0, 1, 2], [1, 3, 4], [2, 4, 5]]


@dataclass
class EpipolarPair:
    """One image pair entering the adjustment (ref/epipolar.py:19-36)."""

    i: int
    j: int
    cam_i: int
    cam_j: int
    x1: np.ndarray  # (M, 3) normalized homogeneous, image i
    x2: np.ndarray  # (M, 3) normalized homogeneous, image j
    terms: np.ndarray = field(default=None)  # (M, 9) flatten(x2 x1^T)
    active: np.ndarray = field(default=None)  # (M,) bool

    def __post_init__(self):
        if self.terms is None:
            self.terms = point_weight_vectors(self.x1, self.x2) if len(self.x1) else np.zeros((0, 9))
        if self.active is None:
            self.active = np.ones(len(self.x1), dtype=bool)


def point_weight_vectors(x1, x2):
    """flatten(x2 x1^T) rows, one per point pair (ref/epipolar.py:39-43)."""
    x1 = np.atleast_2d(np.asarray(x1, dtype=np.float64))
    x2 = np.atleast_2d(np.asarray(x2, dtype=np.float64))
    return (x2[:, :, None] * x1[:, None, :]).reshape(len(x1), 9)


def moments_to_weights(mom):
    """Expand Kronecker moments (36, P) into dense W (P, 9, 9):
    W[3p+r, 3q+s] = mom[sym(p,q)*6 + sym(r,s)]."""
    mom = np.asarray(mom, dtype=np.float64)
    idx = np.empty((9, 9), dtype=np.int64)
    for p in range(3):
        for r in range(3):
            for q in range(3):
                for s in range(3):
                    idx[3 * p + r, 3 * q + s] = SYM[p][q] * 6 + SYM[r][s]
    return np.moveaxis(mom[idx], -1, 0)


def _pass(store, mode, threshold=0.0, ghat=None, res_in=None, prev_active=None, out=None,
          scratch=None):
    out = out or {}
    po = N.PassOut(**{k: (v.data_ptr() if v is not None else None) for k, v in out.items()})
    if scratch is None:
        scratch = store.scratch()
    N.check(N.lib().fm_point_pass(ctypes.byref(store.struct()), mode, float(threshold),
                                  N.ptr(ghat), N.ptr(res_in), N.ptr(prev_active),
                                  ctypes.byref(po), N.ptr(scratch), scratch.numel(),
                                  N.stream_handle()))


def precompute_weights(x1, x2, residuals=None):
    """9x9 PSD matrix W = sum_m w_m t_m t_m^T, optionally IRLS-weighted
    (ref/epipolar.py:46-59); fp64 accumulation on the device."""
    x1 = np.atleast_2d(np.asarray(x1, dtype=np.float64))
    x2 = np.atleast_2d(np.asarray(x2, dtype=np.float64))
    if len(x1) == 0:
        return np.zeros((9, 9))
    device = N.require_cuda()
    store = PointPairStore(x1, x2, [len(x1)], [0], [0], device=device, fp64=True)
    P = 1
    mom = torch.zeros((36, P), dtype=torch.float64, device=device)
    mode = N.FM_PASS_MOMENTS | N.FM_PASS_ALL_POINTS | N.FM_PASS_F64
    res = None
    if residuals is not None:
        res = store.scatter_slots(np.asarray(residuals, dtype=np.float64).reshape(-1))
        mode |= N.FM_PASS_RES_IN
    _pass(store, mode, res_in=res, out={"mom64": mom})
    return moments_to_weights(mom.cpu().numpy())[0]


def compose_essential(R_i, R_j, o_i, o_j):
    """E = [t]x R_j R_i^T, t = -R_j (o_j - o_i) (ref/epipolar.py:62-70)."""
    device = N.require_cuda()
    args = [torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(1, -1)),
                            device=device) for a in (R_i, R_j, o_i, o_j)]
    out = torch.empty((1, 9), dtype=torch.float64, device=device)
    N.check(N.lib().fm_compose_essential(*[N.ptr(a) for a in args], 1, N.ptr(out), N.stream_handle()))
    return out.cpu().numpy().reshape(3, 3)


@dataclass
class AdjustmentState:
    """Optimization variables (ref/epipolar.py:73-106): 6D rotations,
    centers, per-camera log-focal corrections."""

    image_ids: np.ndarray
    rot6d: np.ndarray
    centers: np.ndarray
    log_focal: np.ndarray
    refine_focal: bool

    @classmethod
    def from_poses(cls, poses, image_ids, n_cameras, refine_focal):
        ids = np.asarray(image_ids, dtype=np.int64)
        return cls(image_ids=ids, rot6d=matrix_to_rot6d(poses.rotations[ids]),
                   centers=poses.centers[ids].copy(), log_focal=np.zeros(n_cameras),
                   refine_focal=refine_focal)

    def pack(self):
        parts = [self.rot6d.ravel(), self.centers.ravel()]
        if self.refine_focal:
            parts.append(self.log_focal.ravel())
        return np.concatenate(parts)

    def unpack(self, flat):
        n = len(self.image_ids)
        self.rot6d = flat[: 6 * n].reshape(n, 6)
        self.centers = flat[6 * n: 9 * n].reshape(n, 3)
        if self.refine_focal:
            self.log_focal = flat[9 * n:].copy()


def _pair_indices(state, pairs):
    """Dense image indices / camera ids per pair (ref/epipolar.py:163-169);
    raises KeyError for images missing from state.image_ids."""
    ids = np.asarray(state.image_ids, dtype=np.int64)
    pi = np.array([p.i for p in pairs], dtype=np.int64)
    pj = np.array([p.j for p in pairs], dtype=np.int64)
    order = np.argsort(ids, kind="stable")
    sorted_ids = ids[order]

    def remap(v):
        if len(v) == 0:
            return v
        pos = np.clip(np.searchsorted(sorted_ids, v), 0, max(len(ids) - 1, 0))
        if len(ids) == 0 or np.any(sorted_ids[pos] != v):
            bad = v[(len(ids) == 0) | (sorted_ids[pos] != v)][0]
            raise KeyError(int(bad))
        return order[pos]

    cam_i = np.array([p.cam_i for p in pairs], dtype=np.int64)
    cam_j = np.array([p.cam_j for p in pairs], dtype=np.int64)
    return remap(pi), remap(pj), cam_i, cam_j


def _state_params(state, device):
    packed = np.asarray(state.pack(), dtype=np.float64)
    if not state.refine_focal:
        return torch.as_tensor(packed, device=device)
    return torch.as_tensor(packed, device=device)


class _Problem:
    """Store + graph + parameters of one (state, pairs) API call."""

    def __init__(self, state, pairs, need_points=True):
        self.device = N.require_cuda()
        idx_i, idx_j, cam_i, cam_j = _pair_indices(state, pairs)
        n_cams = len(state.log_focal)
        if need_points:
            self.store = PointPairStore.from_pairs(pairs, device=self.device, fp64=True)
            order = self.store.order
        else:
            self.store = None
            from .store import pair_order
            order = pair_order([p.i for p in pairs], [p.j for p in pairs])
        self.order = order
        self.graph = PairGraph(idx_i[order], idx_j[order], cam_i[order], cam_j[order],
                               len(state.image_ids), n_cams, state.refine_focal, device=self.device)
        self.params = _state_params(state, self.device)
        self.gscratch = self.graph.scratch()
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)

    def ghat(self):
        P = self.graph.n_pairs
        gh = torch.empty((9, max(P, 1)), dtype=torch.float64, device=self.device)
        self.flag.zero_()
        N.check(N.lib().fm_epi_pair_ghat(ctypes.byref(self.graph.struct()), N.ptr(self.params),
                                         N.ptr(gh), N.ptr(self.flag), N.ptr(self.gscratch),
                                         self.gscratch.numel(), N.stream_handle()))
        N.raise_flag(self.flag.item())
        return gh


class EpipolarQuadraticLoss(torch.autograd.Function):
    """loss = (2/Z) sum_n ghat_n^T W_n ghat_n as a function of the packed
    parameters; forward and backward come from one fm_epi_loss_grad call."""

    @staticmethod
    def forward(ctx, params, graph, quad, scale, scratch):
        device = params.device
        loss = torch.empty(1, dtype=torch.float64, device=device)
        grad = torch.empty(graph.n_params, dtype=torch.float64, device=device)
        flag = torch.zeros(1, dtype=torch.int32, device=device)
        N.check(N.lib().fm_epi_loss_grad(ctypes.byref(graph.struct()), ctypes.byref(quad),
                                         N.ptr(params.detach()), float(scale), N.ptr(loss),
                                         N.ptr(grad), N.ptr(flag), N.ptr(scratch), scratch.numel(),
                                         N.stream_handle()))
        N.raise_flag(flag.item())
        ctx.save_for_backward(grad)
        return loss[0]

    @staticmethod
    def backward(ctx, grad_out):
        (grad,) = ctx.saved_tensors
        return grad_out * grad, None, None, None, None


def _quad_loss_grad(prob, quad, scale):
    params = prob.params.clone().requires_grad_(True)
    loss = EpipolarQuadraticLoss.apply(params, prob.graph, quad, scale, prob.gscratch)
    loss.backward()
    return float(loss.item()), params.grad.cpu().numpy()


def _dense_quad(prob, weights):
    W = np.stack([np.asarray(w, dtype=np.float64).reshape(9, 9) for w in weights])[prob.order]
    w81 = torch.as_tensor(np.ascontiguousarray(W.reshape(len(W), 81).T), device=prob.device)
    quad = N.QuadModel(kind=N.FM_QUAD_W64, w81=w81.data_ptr())
    return quad, w81


def epipolar_loss(state, pairs, weights=None, mode="l2"):
    """(2/Z) sum e^T W e ("l2") or the direct mean absolute residual ("l1")
    at the current state (ref/epipolar.py:141-160).  Returns (loss, Z)."""
    prob = _Problem(state, pairs, need_points=(mode != "l2" or weights is None))
    gh = prob.ghat()  # validates the rotations like the reference does
    Z = sum(int(np.count_nonzero(p.active)) for p in pairs)
    if Z == 0:
        raise ValueError("no active point pairs")
    if mode == "l2":
        if weights is None:
            P = prob.graph.n_pairs
            mom = torch.zeros((36, P), dtype=torch.float64, device=prob.device)
            _pass(prob.store, N.FM_PASS_MOMENTS | N.FM_PASS_F64, out={"mom64": mom})
            quad = N.QuadModel(kind=N.FM_QUAD_MOM64, mom64=mom.data_ptr())
            keep = mom
        else:
            quad, keep = _dense_quad(prob, weights)
        loss, _ = _quad_loss_grad(prob, quad, 2.0 / Z)
        del keep
        return loss, Z
    P = prob.graph.n_pairs
    l1 = torch.zeros(P, dtype=torch.float64, device=prob.device)
    _pass(prob.store, N.FM_PASS_L1, ghat=gh, out={"l1": l1})
    return float(l1.sum().item()) / Z, Z


def quadratic_loss_and_grad(state, pairs, weights, Z):
    """Loss (2/Z) sum ghat^T W ghat and its packed gradient
    (ref/epipolar.py:172-232)."""
    prob = _Problem(state, pairs, need_points=False)
    quad, keep = _dense_quad(prob, weights)
    out = _quad_loss_grad(prob, quad, 2.0 / Z)
    del keep
    return out


def current_residuals(state, pairs):
    """Per-pair |terms @ ghat| over all points (ref/epipolar.py:251-255)."""
    prob = _Problem(state, pairs)
    gh = prob.ghat()
    store = prob.store
    res = torch.zeros(store.n_slots, dtype=torch.float64, device=prob.device)
    _pass(store, N.FM_PASS_ALL_POINTS | N.FM_PASS_RES_OUT, ghat=gh, out={"residual": res})
    flat = store.gather_slots(res).cpu().numpy()
    return [flat[store.caller_start[k]:store.caller_start[k + 1]] for k in range(len(pairs))]


def prune_thresholds(cfg):
    """Linear threshold schedule (ref/epipolar.py:258-262)."""
    if cfg.prune_rounds == 1:
        return [cfg.prune_threshold_start]
    return list(np.linspace(cfg.prune_threshold_start, cfg.prune_threshold_end, cfg.prune_rounds))


class IrlsBuffers:
    """Device buffers of one irls_refine run (per image pair, store order).

    precision "fp32" (default, DEFAULT_PRECISION): fp32 moments + the
    shifted-model terms (exact fp64 residuals and prune decisions).
    precision "fp64": exact fp64 W moments, unshifted model."""

    def __init__(self, P, device, precision=None):
        precision = precision or DEFAULT_PRECISION
        Pm = max(P, 1)
        self.precision = precision
        self.ghat0 = torch.zeros((9, Pm), dtype=torch.float64, device=device)
        self.l1 = torch.zeros(Pm, dtype=torch.float64, device=device)
        self.n_active = [torch.zeros(Pm, dtype=torch.int32, device=device) for _ in range(2)]
        if precision == "fp64":
            self.mom64 = torch.zeros((36, Pm), dtype=torch.float64, device=device)
            self.quad = N.QuadModel(kind=N.FM_QUAD_MOM64, mom64=self.mom64.data_ptr())
            self.flags = N.FM_PASS_F64
        elif precision == "fp32":
            self.mom32 = torch.zeros((36, Pm), dtype=torch.float32, device=device)
            self.vgrad = torch.zeros((9, Pm), dtype=torch.float32, device=device)
            self.s0 = torch.zeros(Pm, dtype=torch.float64, device=device)
            self.quad = N.QuadModel(kind=N.FM_QUAD_SHIFTED32, mom32=self.mom32.data_ptr(),
                                    vgrad=self.vgrad.data_ptr(), s0=self.s0.data_ptr(),
                                    ghat0=self.ghat0.data_ptr())
            self.flags = 0
        else:
            raise ValueError(f"unknown precision {precision!r}")

        # {L1 sum, Z, kept pairs} of the last pass, fused into the pass kernel
        self.tot = torch.zeros(3, dtype=torch.float64, device=device)

    def out(self, k):
        o = {"l1": self.l1, "n_active": self.n_active[k], "totals": self.tot}
        if self.precision == "fp64":
            o["mom64"] = self.mom64
        else:
            o.update(mom32=self.mom32, vgrad=self.vgrad, s0=self.s0)
        return o

    def outputs(self):
        """Per-pair result tensors of a pass (for the e2e benchmark)."""
        return [t for t in self.out(0).values()]


class IrlsEngine:
    """The device-resident schedule of ``irls_refine`` (ref/epipolar.py:265-319)
    over an already-built store and pair graph.  Used by ``irls_refine`` and
    directly by the benchmark (store built on the device)."""

    def __init__(self, store, graph, params, cfg, use_graph=True, precision=None):
        precision = precision or DEFAULT_PRECISION
        if not getattr(store, "sanitized", False):
            raise ValueError("IrlsEngine needs a sanitized store (finite coordinates on every "
                             "slot; build it with sanitize=True)")
        self.store = store
        self.graph = graph
        self.device = store.device
        self.cfg = cfg
        self.params = params
        self.use_graph = use_graph
        P = graph.n_pairs
        self.buf = IrlsBuffers(P, self.device, precision)
        self.pscratch = store.scratch()
        self.gscratch = graph.scratch()
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.adam_m = torch.zeros_like(params)
        self.adam_v = torch.zeros_like(params)
        self.lib = N.lib()

    def _ghat(self):
        lib = self.lib
        N.check(lib.fm_epi_pair_ghat(ctypes.byref(self.graph.struct()), N.ptr(self.params),
                                     N.ptr(self.buf.ghat0), N.ptr(self.flag), N.ptr(self.gscratch),
                                     self.gscratch.numel(), N.stream_handle()))

    def point_pass(self, mode, threshold, cur, prev, totals=None, stop=None):
        """One fused pass into buffer `cur`; its {L1, Z, kept} go to `totals`
        (default buf.tot).  stop: a device error word that, when raised,
        makes the pass a no-op (the asynchronous schedule in _run)."""
        if mode & N.FM_PASS_MOMENTS:
            mode |= self.buf.flags
        torch.cuda.nvtx.range_push(f"fm.point_pass 0x{mode:x}")
        out = self.buf.out(cur)
        if totals is not None:
            out["totals"] = totals
        if stop is not None:
            out["stop"] = stop
        _pass(self.store, mode, threshold, ghat=self.buf.ghat0,
              prev_active=self.buf.n_active[prev] if (mode & N.FM_PASS_SKIP_DROPPED) else None,
              out=out, scratch=self.pscratch)
        torch.cuda.nvtx.range_pop()

    def run(self):
        torch.cuda.nvtx.range_push("fm.irls_refine")
        try:
            return self._run()
        finally:
            torch.cuda.nvtx.range_pop()

    def _run(self):
        """The schedule of ref/epipolar.py:278-319, enqueued without a host
        round trip: every pass writes its {L1, Z, kept} into its own row of
        a device history, each epoch reads its round's 2/Z on the device
        (fm_epi_adam_steps_z), the error word is snapshotted after every
        stage, and a raised word turns the later passes into no-ops (masks
        stay as at the first error).  One synchronisation at the end then
        replays the reference's checks in its order."""
        cfg = self.cfg
        P = self.graph.n_pairs
        thresholds = prune_thresholds(cfg)
        iters = cfg.irls_iters_between_prunes
        steps = cfg.epipolar_epoch_steps
        n_pass = len(thresholds) * iters + 1
        hist = torch.zeros((n_pass, 3), dtype=torch.float64, device=self.device)
        flags = torch.zeros(2 * n_pass, dtype=torch.int32, device=self.device)
        k = f = 0
        lr = cfg.epipolar_lr
        cur = 0
        for rnd, th in enumerate(thresholds):
            self._ghat()
            mode = N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS
            if rnd > 0:
                mode |= N.FM_PASS_L1 | N.FM_PASS_SKIP_DROPPED
            prev = cur
            cur = 1 - cur
            round_tot = hist[k]
            self.point_pass(mode, th, cur, prev, totals=round_tot, stop=self.flag)
            k += 1
            flags[f].copy_(self.flag[0])
            f += 1
            self.adam_m.zero_()
            self.adam_v.zero_()
            for it in range(iters):
                if it > 0:
                    self._ghat()
                    self.point_pass(N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED,
                                    0.0, 1 - cur, cur, totals=hist[k], stop=self.flag)
                    k += 1
                    # counts unchanged (no prune); keep the current buffer authoritative
                    self.buf.n_active[cur], self.buf.n_active[1 - cur] = \
                        self.buf.n_active[1 - cur], self.buf.n_active[cur]
                    flags[f].copy_(self.flag[0])
                    f += 1
                torch.cuda.nvtx.range_push("fm.adam_steps")
                N.check(self.lib.fm_epi_adam_steps_z(
                    ctypes.byref(self.graph.struct()), ctypes.byref(self.buf.quad),
                    N.ptr(self.params), N.ptr(self.adam_m), N.ptr(self.adam_v),
                    it * steps, steps, lr, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps,
                    N.ptr(round_tot), N.ptr(self.flag), int(self.use_graph), N.ptr(self.gscratch),
                    self.gscratch.numel(), N.stream_handle()))
                torch.cuda.nvtx.range_pop()
                flags[f].copy_(self.flag[0])
                f += 1
            lr /= cfg.lr_decay
        self._ghat()
        self.point_pass(N.FM_PASS_L1 | N.FM_PASS_SKIP_DROPPED, 0.0, 1 - cur, cur, totals=hist[k],
                        stop=self.flag)
        self.buf.n_active[cur], self.buf.n_active[1 - cur] = \
            self.buf.n_active[1 - cur], self.buf.n_active[cur]
        flags[f].copy_(self.flag[0])
        self.buf.tot.copy_(hist[k])
        # the one synchronisation; the reference's checks in its order
        H = hist.cpu().numpy()
        F = flags.cpu().numpy()
        l1_history = []
        k = f = 0
        Z = None
        kept = P
        for rnd in range(len(thresholds)):
            l1_sum, z, kept_r = H[k]
            k += 1
            if rnd > 0:
                l1_history.append(float(l1_sum) / Z)
            Z, kept = int(z), int(kept_r)
            N.raise_flag(int(F[f]))
            f += 1
            if kept == 0:
                self.dropped = P
                raise ValueError("all pairs pruned away")
            for it in range(iters):
                if it > 0:
                    k += 1
                    N.raise_flag(int(F[f]))
                    f += 1
                N.raise_flag(int(F[f]))
                f += 1
        N.raise_flag(int(F[f]))
        l1_history.append(float(H[k][0]) / Z)
        self.dropped = P - kept
        self.kept = kept
        return l1_history


def irls_refine(poses, pairs, cfg, n_cameras=1, use_graph=True, precision=None):
    """Scheduled IRLS refinement of global poses (and optionally focals)
    (ref/epipolar.py:265-319).  Mutates pair ``active`` masks during pruning.
    Returns (poses, focal_scale per camera, report dict)."""
    image_ids = sorted({p.i for p in pairs} | {p.j for p in pairs})
    state = AdjustmentState.from_poses(poses, image_ids, n_cameras, cfg.refine_focal)
    device = N.require_cuda()
    idx_i, idx_j, cam_i, cam_j = _pair_indices(state, pairs)
    store = PointPairStore.from_pairs(pairs, device=device, sanitize=True)
    o = store.order
    graph = PairGraph(idx_i[o], idx_j[o], cam_i[o], cam_j[o], len(image_ids), n_cameras,
                      cfg.refine_focal, device=device)
    params = torch.as_tensor(state.pack(), device=device)
    engine = IrlsEngine(store, graph, params, cfg, use_graph=use_graph,
                        precision=precision or DEFAULT_PRECISION)
    try:
        l1_history = engine.run()
    finally:
        store.write_back(pairs)
    state.unpack(params.cpu().numpy())
    out = poses_from_state(poses, state)
    focal_scale = np.exp(state.log_focal) if cfg.refine_focal else np.ones(n_cameras)
    report = {"l1_history": l1_history, "dropped_pairs": engine.dropped,
              "active_pairs": engine.kept}
    return out, focal_scale, report


def poses_from_state(poses, state):
    """Copy of ``poses`` with the state's rotations (projected onto SO(3))
    and centers written back (ref/epipolar.py:322-332)."""
    device = N.require_cuda()
    out = type(poses)(rotations=poses.rotations.copy(), centers=poses.centers.copy(),
                      registered=poses.registered.copy())
    n = len(state.image_ids)
    if n == 0:
        return out
    v6 = torch.as_tensor(np.ascontiguousarray(state.rot6d, dtype=np.float64), device=device)
    R = torch.empty((n, 9), dtype=torch.float64, device=device)
    flag = torch.zeros(1, dtype=torch.int32, device=device)
    N.check(N.lib().fm_rot6d_to_matrix(N.ptr(v6), n, 1, N.ptr(R), N.ptr(flag), N.stream_handle()))
    N.raise_flag(flag.item())
    ids = np.asarray(state.image_ids, dtype=np.int64)
    out.rotations[ids] = R.cpu().numpy().reshape(n, 3, 3)
    out.centers[ids] = state.centers
    return out


__all__ = ["EpipolarPair", "point_weight_vectors", "precompute_weights", "compose_essential",
           "AdjustmentState", "epipolar_loss", "quadratic_loss_and_grad", "current_residuals",
           "prune_thresholds", "irls_refine", "poses_from_state", "IrlsEngine",
           "EpipolarQuadraticLoss", "moments_to_weights"]
