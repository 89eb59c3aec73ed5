"""Drop-in for ``fastmap.optim`` (ref/optim.py): Adam, the 6D rotation maps
and the finite-difference checker.

``Adam`` keeps its state on the GPU and steps with the fp64 kernel of the C
ABI (``fm_adam_step``, ref/optim.py:24-36 rounding-for-rounding: no FMA
contraction).  ``rot6d_to_matrix`` / ``rot6d_jacobian`` run the device
Gram-Schmidt map and its Jacobian (ref/optim.py:39-110).  ``matrix_to_rot6d``
and ``skew`` are pure data rearrangements and ``fd_check`` is the reference's
test oracle (it evaluates a caller-supplied function); those stay on the host.
"""

import ctypes

import numpy as np
import torch

from . import _native as N


def _to_dev(a, device):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)


class Adam:
    """Standard Adam with bias correction on a flat fp64 vector (device state)."""

    def __init__(self, params, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        self.device = N.require_cuda()
        p = np.asarray(params, dtype=np.float64)
        self._shape = p.shape
        self._p = _to_dev(p.ravel().copy(), self.device)
        self._m = torch.zeros_like(self._p)
        self._v = torch.zeros_like(self._p)
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.lr = lr
        self.beta1 = beta1
        self.beta2 = beta2
        self.eps = eps
        self.t = 0

    @property
    def params(self):
        return self._p.cpu().numpy().reshape(self._shape)

    @params.setter
    def params(self, value):
        v = np.asarray(value, dtype=np.float64)
        self._shape = v.shape
        self._p = _to_dev(v.ravel().copy(), self.device)

    @property
    def m(self):
        return self._m.cpu().numpy().reshape(self._shape)

    @property
    def v(self):
        return self._v.cpu().numpy().reshape(self._shape)

    def step(self, grads):
        if isinstance(grads, torch.Tensor):
            g = grads.to(self.device, torch.float64).reshape(-1).contiguous()
            shape = tuple(grads.shape)
        else:
            ga = np.asarray(grads, dtype=np.float64)
            shape = ga.shape
            g = _to_dev(ga.ravel(), self.device)
        if shape != tuple(self._shape):
            raise ValueError("gradient shape mismatch")
        self._flag.zero_()
        N.check(N.lib().fm_adam_step(N.ptr(self._p), N.ptr(self._m), N.ptr(self._v), N.ptr(g),
                                     self._p.numel(), self.t + 1, self.lr, self.beta1, self.beta2,
                                     self.eps, N.ptr(self._flag), N.stream_handle()))
        N.raise_flag(self._flag.item())
        self.t += 1
        return self.params


def rot6d_to_matrix(v):
    """Map 6-vectors (..., 6) to rotation matrices (..., 3, 3) on the GPU."""
    device = N.require_cuda()
    v = np.asarray(v, dtype=np.float64)
    batch = v.shape[:-1]
    flat = _to_dev(v.reshape(-1, 6), device)
    n = flat.shape[0]
    out = torch.empty((n, 9), dtype=torch.float64, device=device)
    flag = torch.zeros(1, dtype=torch.int32, device=device)
    N.check(N.lib().fm_rot6d_to_matrix(N.ptr(flat), n, 0, N.ptr(out), N.ptr(flag), N.stream_handle()))
    N.raise_flag(flag.item())
    return out.cpu().numpy().reshape(batch + (3, 3))


def matrix_to_rot6d(R):
    """First two columns of R (ref/optim.py:62-65)."""
    R = np.asarray(R, dtype=np.float64)
    return np.concatenate([R[..., :, 0], R[..., :, 1]], axis=-1)


def rot6d_jacobian(v):
    """Jacobian of rot6d_to_matrix, shape (..., 9, 6), computed on the GPU."""
    device = N.require_cuda()
    v = np.asarray(v, dtype=np.float64)
    batch = v.shape[:-1]
    flat = _to_dev(v.reshape(-1, 6), device)
    n = flat.shape[0]
    out = torch.empty((n, 54), dtype=torch.float64, device=device)
    N.check(N.lib().fm_rot6d_jacobian(N.ptr(flat), n, N.ptr(out), N.stream_handle()))
    return out.cpu().numpy().reshape(batch + (9, 6))


def skew(t):
    """Cross-product matrices [t]_x for vectors of shape (..., 3)."""
    t = np.asarray(t, dtype=np.float64)
    S = np.zeros(t.shape[:-1] + (3, 3))
    S[..., 0, 1] = -t[..., 2]
    S[..., 0, 2] = t[..., 1]
    S[..., 1, 0] = t[..., 2]
    S[..., 1, 2] = -t[..., 0]
    S[..., 2, 0] = -t[..., 1]
    S[..., 2, 1] = t[..., 0]
    return S


def fd_check(f, theta, h=1e-6, grad=None):
    """Max relative discrepancy between an analytic gradient and central
    finite differences of ``f`` at ``theta`` (ref/optim.py:126-153)."""
    theta = np.asarray(theta, dtype=np.float64)
    if grad is None:
        _, grad = f(theta)

        def value(x):
            return f(x)[0]
    else:
        value = f
    grad = np.asarray(grad, dtype=np.float64).ravel()
    fd = np.zeros_like(grad)
    flat = theta.ravel().copy()
    for k in range(flat.size):
        orig = flat[k]
        flat[k] = orig + h
        fp = value(flat.reshape(theta.shape))
        flat[k] = orig - h
        fm = value(flat.reshape(theta.shape))
        flat[k] = orig
        fd[k] = (fp - fm) / (2.0 * h)
    scale = np.maximum(np.abs(fd), np.abs(grad))
    scale = np.maximum(scale, np.max(scale) * 1e-6 + 1e-12)
    return float(np.max(np.abs(fd - grad) / scale))


__all__ = ["Adam", "rot6d_to_matrix", "matrix_to_rot6d", "rot6d_jacobian", "skew", "fd_check"]
