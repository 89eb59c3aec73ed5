"""Domain types the hot path consumes and returns (ref/model.py:112-143).

``PoseState`` mirrors the reference dataclass; the hot-path functions accept
the reference's own ``PoseState`` too (duck typing) and return the caller's
class.  ``project_to_so3`` runs the batched polar projection kernel.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


@dataclass
class PoseState:
    """Per-image world-to-camera rotations and camera centers in the world frame."""

    rotations: np.ndarray  # (n, 3, 3)
    centers: np.ndarray  # (n, 3)
    registered: np.ndarray  # (n,) bool

    @classmethod
    def identity(cls, n):
        return cls(rotations=np.broadcast_to(np.eye(3), (n, 3, 3)).copy(),
                   centers=np.zeros((n, 3)), registered=np.ones(n, dtype=bool))


def project_to_so3(R):
    """Nearest rotation matrix in Frobenius norm, for (3, 3) or (..., 3, 3)."""
    device = N.require_cuda()
    M = np.asarray(R, dtype=np.float64)
    batch = M.shape[:-2]
    flat = torch.as_tensor(np.ascontiguousarray(M.reshape(-1, 9)), device=device)
    out = torch.empty_like(flat)
    N.check(N.lib().fm_project_to_so3(N.ptr(flat), flat.shape[0], N.ptr(out), N.stream_handle()))
    return out.cpu().numpy().reshape(batch + (3, 3))


__all__ = ["PoseState", "project_to_so3"]
