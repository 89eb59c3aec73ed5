"""Drop-in for the global-alignment half of ``fastmap.translation``
(ref/translation.py:98-186) on the B200.

``translation_loss_and_grad`` -> ``fm_tr_loss_grad`` (behind the
``TranslationL1Loss`` autograd function); ``align_centers`` ->
``fm_tr_align`` (fused loss + gradient + Adam per step, CUDA-graph replay);
``multi_init_align`` runs all ``translation_inits`` random starts in
lock-step as one batched descent (one read of every edge serves all runs),
merges them on the device (``fm_tr_merge``) and finishes with the final
descent.  The random starts are drawn with the reference's own seeded numpy
generator, so run k starts from bit-identical centres.

``reestimate_relative`` (ref/translation.py:19-95, SURVEY 8f "next" #1) is
the per-image-pair sphere search that produces the graph's directions: the
candidate lattices are the reference's (same numpy expressions), the mean
epipolar errors of every candidate run on the device (``fm_sphere_errors``)
and so do the cheirality counts (``fm_depth_counts``).
"""

import ctypes
import functools
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .store import DirGraphDevice

_NORM_EPS = 1e-8
_GOLDEN_ANGLE = np.pi * (3.0 - np.sqrt(5.0))


class PairRejected(ValueError):
    """The pair carries no usable translation signal (ref/translation.py:19-20).
    install() rebinds this name to the reference's class, so the pipeline's
    ``except translation.PairRejected`` catches ours."""


@functools.lru_cache(maxsize=8)
def _fibonacci_sphere(n):
    k = np.arange(n, dtype=np.float64) + 0.5
    z = 1.0 - 2.0 * k / n
    r = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    phi = _GOLDEN_ANGLE * k
    out = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)
    out.setflags(write=False)
    return out


def fibonacci_sphere(n):
    """The reference's deterministic unit-sphere lattice of n points
    (ref/translation.py:23-29); computed once per n."""
    return _fibonacci_sphere(int(n)).copy()


_LATTICE_DEV = {}


def _lattice_on(device, n):
    """fibonacci_sphere(n) resident on the device (uploaded once)."""
    key = (str(device), int(n))
    t = _LATTICE_DEV.get(key)
    if t is None:
        t = _LATTICE_DEV[key] = torch.as_tensor(_fibonacci_sphere(int(n)).copy(), device=device)
    return t


@functools.lru_cache(maxsize=32)
def _cap_local(radius, n):
    """The axis-independent spiral of _cap_samples (cached per radius / n)."""
    k = np.arange(n, dtype=np.float64) + 0.5
    theta = radius * np.sqrt(k / n)
    phi = _GOLDEN_ANGLE * k
    out = np.stack([np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi), np.cos(theta)],
                   axis=1)
    out.setflags(write=False)
    return out


def _cross(a, b):
    # np.cross of two 3-vectors: the same products and differences
    return np.array([a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]])


def _cap_samples(axis, radius, n):
    """Spiral of n directions within angle `radius` of `axis`
    (ref/translation.py:32-49)."""
    local = _cap_local(float(radius), int(n))
    axis = axis / np.linalg.norm(axis)
    ref = np.array([1.0, 0.0, 0.0]) if abs(axis[2]) > 0.9 else np.array([0.0, 0.0, 1.0])
    u = _cross(ref, axis)
    u /= np.linalg.norm(u)
    v = _cross(axis, u)
    return local @ np.stack([u, v, axis], axis=1).T


def reestimate_relative(x1, x2, rel_rotation, cfg):
    """Unit relative translation of an image pair by sphere search
    (ref/translation.py:58-95): mean |x2^T [t]_x R x1| over a Fibonacci
    lattice of cfg.sphere_samples directions, refined cfg.sphere_refine_levels
    times on shrinking caps around the best, sign by cheirality on the first
    200 points.  Raises PairRejected for empty, flat (near-zero baseline) or
    cheirality-tied pairs, with the reference's messages."""
    out = reestimate_relative_batch([x1], [x2], [rel_rotation], cfg)[0]
    if isinstance(out, Exception):
        raise out
    return out


def reestimate_relative_batch(x1s, x2s, rel_rotations, cfg):
    """reestimate_relative for many image pairs at once: one device launch
    per search level for all pairs (fm_sphere_errors_batch) and one for the
    cheirality counts (fm_depth_counts_batch).  Returns, per pair, the unit
    direction or the PairRejected instance the single call would raise; the
    per-pair lattices and decisions are exactly those of the single call."""
    P = len(x1s)
    out = [None] * P
    x1s = [np.asarray(a, dtype=np.float64).reshape(-1, 3) for a in x1s]
    x2s = [np.asarray(b, dtype=np.float64).reshape(-1, 3) for b in x2s]
    live = [k for k in range(P) if len(x1s[k])]
    for k in range(P):
        if not len(x1s[k]):
            out[k] = PairRejected("no inlier point pairs")
    if not live:
        return out
    device = N.require_cuda()
    lib = N.lib()
    n = int(cfg.sphere_samples)
    for lo in range(0, len(live), 65535):
        ks = live[lo:lo + 65535]
        lens = np.array([len(x1s[k]) for k in ks], dtype=np.int64)
        off = torch.as_tensor(np.concatenate([[0], np.cumsum(lens)]), device=device)
        Z, B = int(lens.sum()), len(ks)
        # points of both sides and the rotations in one upload
        host = np.concatenate([np.concatenate([x1s[k] for k in ks]).ravel(),
                               np.concatenate([x2s[k] for k in ks]).ravel(),
                               np.ascontiguousarray(np.stack([rel_rotations[k] for k in ks]),
                                                    dtype=np.float64).ravel()])
        dev = torch.as_tensor(host, device=device)
        X1, X2, R = dev[:3 * Z], dev[3 * Z:6 * Z], dev[6 * Z:]
        e = torch.empty((B, n), dtype=torch.float64, device=device)

        def errors(d, stride):
            if not isinstance(d, torch.Tensor):
                d = torch.as_tensor(np.ascontiguousarray(d), device=device)
            N.check(lib.fm_sphere_errors_batch(N.ptr(X1), N.ptr(X2), N.ptr(off), B, N.ptr(R),
                                               N.ptr(d), stride, n, N.ptr(e), N.stream_handle()))
            return e.cpu().numpy()

        lattice = _fibonacci_sphere(n)
        err = errors(_lattice_on(device, n), 0)
        med = np.median(err, axis=1)
        flat = (med < 1e-15) | (np.min(err, axis=1) > 0.9 * med)
        best = lattice[np.argmin(err, axis=1)]
        radius = 2.0 * np.sqrt(4.0 * np.pi / n)
        for _ in range(int(cfg.sphere_refine_levels)):
            cands = np.stack([_cap_samples(best[q], radius, n) for q in range(B)])
            err_l = errors(cands, 3 * n)
            best = cands[np.arange(B), np.argmin(err_l, axis=1)]
            radius *= 2.0 * np.sqrt(np.pi / n)
        t = torch.as_tensor(np.ascontiguousarray(best), device=device)
        counts = torch.empty((B, 2), dtype=torch.int32, device=device)
        N.check(lib.fm_depth_counts_batch(N.ptr(R), N.ptr(t), N.ptr(X1), N.ptr(X2), N.ptr(off), B,
                                          200, N.ptr(counts), N.stream_handle()))
        counts = counts.cpu().numpy()
        for q, k in enumerate(ks):
            if flat[q]:
                out[k] = PairRejected("flat epipolar landscape (near-zero baseline)")
            elif counts[q, 0] == counts[q, 1]:
                out[k] = PairRejected("cheirality tie")
            else:
                out[k] = best[q] if counts[q, 0] > counts[q, 1] else -best[q]
    return out


def world_direction(t_ij, R_j):
    """Unit vector from camera center i to j in world coordinates
    (ref/translation.py:98-101; input construction helper)."""
    d = -np.asarray(R_j).T @ np.asarray(t_ij)
    return d / np.linalg.norm(d)


@dataclass
class DirectionGraph:
    n: int  # number of registered nodes (dense indices)
    edges_i: np.ndarray  # (m,)
    edges_j: np.ndarray  # (m,)
    directions: np.ndarray  # (m, 3) unit o^{i->j}


_GRAPH_CACHE = {}


def _graph_digest(graph):
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    h.update(np.int64(graph.n).tobytes())
    for a, dt in ((graph.edges_i, np.int64), (graph.edges_j, np.int64), (graph.directions, np.float64)):
        h.update(np.ascontiguousarray(np.asarray(a, dtype=dt)).tobytes())
    return h.digest()


def device_graph(graph):
    """Upload the direction graph, memoised per graph object AND content (an
    in-place edit of the arrays re-uploads)."""
    key = id(graph)
    digest = _graph_digest(graph)
    hit = _GRAPH_CACHE.get(key)
    if hit is not None and hit[0] is graph and hit[1] == digest:
        return hit[2]
    dg = DirGraphDevice(graph)
    if len(_GRAPH_CACHE) > 8:
        _GRAPH_CACHE.clear()
    _GRAPH_CACHE[key] = (graph, digest, dg)
    return dg


class TranslationL1Loss(torch.autograd.Function):
    """Mean per-edge L1 direction loss of B runs; forward and backward from
    one fm_tr_loss_grad call.  centers: (n, B, 3) fp64 device tensor."""

    @staticmethod
    def forward(ctx, centers, dg):
        B = centers.shape[1]
        loss = torch.empty(B, dtype=torch.float64, device=centers.device)
        grad = torch.empty_like(centers)
        scratch = dg.scratch(B)
        N.check(N.lib().fm_tr_loss_grad(ctypes.byref(dg.struct()), N.ptr(centers.detach()), B,
                                        N.ptr(loss), N.ptr(grad), N.ptr(scratch), scratch.numel(),
                                        N.stream_handle()))
        ctx.save_for_backward(grad)
        return loss

    @staticmethod
    def backward(ctx, grad_out):
        (grad,) = ctx.saved_tensors
        return grad * grad_out.view(1, -1, 1), None


def translation_loss_and_grad(centers, graph):
    """Mean per-edge L1 direction loss and its gradient w.r.t. centers
    (ref/translation.py:112-125)."""
    dg = device_graph(graph)
    c = np.asarray(centers, dtype=np.float64)
    t = torch.as_tensor(np.ascontiguousarray(c.reshape(graph.n, 1, 3)), device=dg.device)
    t.requires_grad_(True)
    loss = TranslationL1Loss.apply(t, dg)
    loss.sum().backward()
    return float(loss[0].item()), t.grad.reshape(c.shape).cpu().numpy()


def canonicalize(centers):
    """Centroid to the origin, unit mean norm (ref/translation.py:128-134)."""
    device = N.require_cuda()
    c = np.asarray(centers, dtype=np.float64)
    t = torch.as_tensor(np.ascontiguousarray(c.reshape(-1, 1, 3)).copy(), device=device)
    N.check(N.lib().fm_tr_canonicalize(N.ptr(t), t.shape[0], 1, None, 0, N.stream_handle()))
    return t.reshape(c.shape).cpu().numpy()


def _align(dg, init, cfg, steps):
    """Batched descent of B runs from init (n, B, 3); returns (centers, loss[B])."""
    B = init.shape[1]
    if isinstance(init, torch.Tensor):
        c = init.to(dg.device, torch.float64).contiguous().clone()
    else:
        c = torch.as_tensor(np.ascontiguousarray(init, dtype=np.float64), device=dg.device).clone()
    if steps == 0:
        return c, np.full(B, np.inf)
    loss = torch.empty(B, dtype=torch.float64, device=dg.device)
    flag = dg.flag()
    scratch = dg.scratch(B)
    N.check(N.lib().fm_tr_align(ctypes.byref(dg.struct()), N.ptr(c), B, int(steps),
                                cfg.translation_lr, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps,
                                N.ptr(loss), N.ptr(flag), N.ptr(scratch), scratch.numel(),
                                N.stream_handle()))
    N.raise_flag(flag.item(), "translation")
    return c, loss.cpu().numpy()


def align_centers(graph, cfg, seed=0, init=None, steps=None):
    """Adam descent of the L1 direction loss from a random (or given)
    initialization (ref/translation.py:137-152).  Returns (centers, loss)."""
    rng = np.random.default_rng(seed)
    if init is None:
        init = rng.standard_normal((graph.n, 3))
    dg = device_graph(graph)
    n_steps = steps if steps is not None else cfg.translation_steps
    c, loss = _align(dg, np.asarray(init, dtype=np.float64).reshape(graph.n, 1, 3), cfg, n_steps)
    return c.reshape(graph.n, 3).cpu().numpy(), float(loss[0])


def per_node_residuals(centers, graph):
    """Mean incident-edge L1 residual per node (ref/translation.py:155-166)."""
    dg = device_graph(graph)
    c = torch.as_tensor(np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(graph.n, 1, 3)),
                        device=dg.device)
    out = torch.empty(graph.n, dtype=torch.float64, device=dg.device)
    N.check(N.lib().fm_tr_node_residuals(ctypes.byref(dg.struct()), N.ptr(c), 1, N.ptr(out),
                                         N.stream_handle()))
    return out.cpu().numpy()


def init_runs(graph, cfg, seed, ks, dg=None):
    """Descents of the random starts seed + k, k in ks, as one batch; returns
    the final centres (n, len(ks), 3) on the device.  A run's trajectory does
    not depend on which other runs share its batch (fm_tr_align), so
    batches of any split reproduce the full batch."""
    dg = dg or device_graph(graph)
    init = np.stack([np.random.default_rng(seed + k).standard_normal((graph.n, 3)) for k in ks],
                    axis=1)
    runs, _ = _align(dg, init, cfg, cfg.translation_steps)
    return runs


def merge_and_finish(graph, cfg, runs, dg=None, return_choice=False):
    """Canonicalise the runs (n, B, 3), take per node the run with the lowest
    mean incident residual (first minimum), and descend from the merged
    centres (ref/translation.py:181-186)."""
    dg = dg or device_graph(graph)
    B = runs.shape[1]
    runs = runs.contiguous()
    merged = torch.empty((graph.n, 1, 3), dtype=torch.float64, device=dg.device)
    choice = torch.empty(graph.n, dtype=torch.int32, device=dg.device)
    scratch = dg.scratch(B)
    N.check(N.lib().fm_tr_merge(ctypes.byref(dg.struct()), N.ptr(runs), B, N.ptr(merged),
                                N.ptr(choice), N.ptr(scratch), scratch.numel(), N.stream_handle()))
    c, loss = _align(dg, merged, cfg, cfg.translation_steps)
    out = (c.reshape(graph.n, 3).cpu().numpy(), float(loss[0]))
    if return_choice:
        return out + (choice.cpu().numpy(),)
    return out


def multi_init_align(graph, cfg, seed=0, return_choice=False):
    """Independent random-seed runs merged per image, then a final descent
    (ref/translation.py:169-186).  All runs execute as one batched descent
    (parallel.multi_init_align_sharded splits them over ranks)."""
    if cfg.translation_inits == 1:
        return align_centers(graph, cfg, seed=seed)
    dg = device_graph(graph)
    runs = init_runs(graph, cfg, seed, range(cfg.translation_inits), dg)
    return merge_and_finish(graph, cfg, runs, dg, return_choice)


__all__ = ["PairRejected", "fibonacci_sphere", "reestimate_relative", "reestimate_relative_batch",
           "world_direction",
           "DirectionGraph", "translation_loss_and_grad", "canonicalize",
           "align_centers", "per_node_residuals", "multi_init_align", "TranslationL1Loss"]
