"""Drop-in for the Adam refinement half of ``fastmap.rotation``
(ref/rotation.py:162-230; SURVEY 8f "next" #3) on the B200.

``rotation_loss_and_grad`` -> ``fm_rot_loss_grad`` (mean geodesic loss and
its 6D gradient: per-node fixed-order gather of the edge terms, no
scatter); ``refine_rotations`` -> ``fm_rot_refine`` (the whole descent with
the reference's best-iterate and early-stopping rules on the device, in
CUDA-graph chunks of 100 steps).  Filtering / initialisation
(ref/rotation.py:56-149) stay out of scope.
"""

import ctypes

import numpy as np
import torch

from . import _native as N
from .model import project_to_so3
from .optim import matrix_to_rot6d
from .store import csr


class RotGraphDevice:
    """Relative-rotation edges over dense node indices, with the per-node
    incidence list (edge << 1 | side) of the deterministic gather."""

    def __init__(self, n, edges_i, edges_j, rel, device=None):
        device = device or N.require_cuda()
        ei = np.asarray(edges_i, dtype=np.int64)
        ej = np.asarray(edges_j, dtype=np.int64)
        m = len(ei)
        if m and (min(ei.min(), ej.min()) < 0 or max(ei.max(), ej.max()) >= n):
            raise IndexError("edge endpoint out of range")
        inc = np.concatenate([np.arange(m) * 2, np.arange(m) * 2 + 1])
        off, incs = csr(np.concatenate([ei, ej]), n, inc)
        self.n, self.m, self.device = int(n), m, device
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt), device=device)
        self.t = dict(ei=t(ei, np.int32), ej=t(ej, np.int32),
                      rel=t(np.asarray(rel, dtype=np.float64).reshape(m, 9), np.float64),
                      off=t(off, np.int32), inc=t(incs if m else np.zeros(1), np.int32))
        self._struct = N.RotGraph(n_nodes=self.n, n_edges=m, edge_i=self.t["ei"].data_ptr(),
                                  edge_j=self.t["ej"].data_ptr(), rel=self.t["rel"].data_ptr(),
                                  node_off=self.t["off"].data_ptr(), node_inc=self.t["inc"].data_ptr())

    def struct(self):
        return self._struct

    def scratch(self):
        nbytes = N.lib().fm_rot_scratch_bytes(self.n, self.m)
        return torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)


def rotation_loss_and_grad(params6d, edges_i, edges_j, rel_rotations):
    """Mean geodesic loss over edges and its gradient w.r.t. the 6D
    parameters (ref/rotation.py:162-194).  Returns (loss, grad (n, 6))."""
    p = np.asarray(params6d, dtype=np.float64)
    n = p.shape[0]
    g = RotGraphDevice(n, edges_i, edges_j, rel_rotations)
    P = torch.as_tensor(np.ascontiguousarray(p), device=g.device)
    loss = torch.empty(1, dtype=torch.float64, device=g.device)
    grad = torch.empty((n, 6), dtype=torch.float64, device=g.device)
    flag = torch.zeros(1, dtype=torch.int32, device=g.device)
    sc = g.scratch()
    N.check(N.lib().fm_rot_loss_grad(ctypes.byref(g.struct()), N.ptr(P), N.ptr(loss), N.ptr(grad),
                                     N.ptr(flag), N.ptr(sc), sc.numel(), N.stream_handle()))
    N.raise_flag(flag.item(), "rotation")
    return float(loss.item()), grad.cpu().numpy()


def refine_rotations(init, graph, cfg):
    """Adam descent of the mean geodesic loss from an initialization, keeping
    the best iterate and stopping early when the relative loss change over a
    100-step window falls below 1e-9 (ref/rotation.py:197-230).  ``graph``
    is the reference's RelPoseGraph (edges with i, j, rel_rotation;
    registered mask).  Returns (rotations, loss history)."""
    init = np.asarray(init, dtype=np.float64)
    active = np.flatnonzero(graph.registered)
    remap = {int(img): k for k, img in enumerate(active)}
    ei = np.array([remap[e.i] for e in graph.edges], dtype=np.int64)
    ej = np.array([remap[e.j] for e in graph.edges], dtype=np.int64)
    rel = np.stack([e.rel_rotation for e in graph.edges])
    g = RotGraphDevice(len(active), ei, ej, rel)
    params = torch.as_tensor(np.ascontiguousarray(matrix_to_rot6d(init[active])), device=g.device)
    steps = int(cfg.rotation_steps)
    history = torch.empty(max(steps, 1), dtype=torch.float64, device=g.device)
    done = ctypes.c_int32(0)
    flag = torch.zeros(1, dtype=torch.int32, device=g.device)
    sc = g.scratch()
    N.check(N.lib().fm_rot_refine(ctypes.byref(g.struct()), N.ptr(params), steps, cfg.rotation_lr,
                                  cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps, N.ptr(history),
                                  ctypes.byref(done), N.ptr(flag), N.ptr(sc), sc.numel(),
                                  N.stream_handle()))
    N.raise_flag(flag.item(), "rotation")
    out = init.copy()
    from .optim import rot6d_to_matrix
    final = project_to_so3(rot6d_to_matrix(params.cpu().numpy()))
    out[active] = final
    return out, [float(x) for x in history[:done.value].cpu().numpy()]


__all__ = ["rotation_loss_and_grad", "refine_rotations", "RotGraphDevice"]
