"""ctypes binding of the C ABI in ``include/fastmap_b200.h``.

The library is loaded from the package directory (built in-tree by
``paper_2505_04612_b200.build``).  There is no CPU fallback: every product
entry point calls :func:`lib` which raises if the shared library is missing,
and :func:`require_cuda` which raises when no CUDA device is visible.
"""

import ctypes
import os

import torch

from . import build as _build

_LIB = None

FM_OK = 0
FM_ERR_INVALID = 1
FM_ERR_CUDA = 2
FM_ERR_NONFINITE_LOSS = 3
FM_ERR_NONFINITE_GRAD = 4
FM_ERR_ROT6D_ZERO = 5
FM_ERR_ROT6D_COLLINEAR = 6
FM_ERR_NO_ACTIVE = 7
FM_ERR_ALL_PRUNED = 8
FM_ERR_NONFINITE_TRANSLATION = 9
FM_ERR_NONFINITE_ROTATION = 10

FM_PASS_PRUNE = 1
FM_PASS_L1 = 2
FM_PASS_MOMENTS = 4
FM_PASS_IRLS = 8
FM_PASS_ALL_POINTS = 16
FM_PASS_RES_OUT = 32
FM_PASS_RES_IN = 64
FM_PASS_F64 = 128
FM_PASS_SKIP_DROPPED = 256

FM_QUAD_SHIFTED32 = 0
FM_QUAD_W64 = 1
FM_QUAD_MOM64 = 2

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
ABI_VERSION = 6
_F64 = ctypes.c_double
_SZ = ctypes.c_size_t


class PointStore(ctypes.Structure):
    _fields_ = [("n_pairs", _I64), ("n_slots", _I64), ("n_items", _I64), ("chunk", _I64),
                ("pair_off", _P), ("pair_len", _P), ("pair_item_off", _P), ("item_pair", _P),
                ("x1", _P), ("x2", _P), ("x1z", _P), ("x2z", _P), ("active", _P),
                ("item_desc", _P), ("slot_align", _I64), ("x1d", _P), ("x2d", _P)]


class PassOut(ctypes.Structure):
    _fields_ = [("mom32", _P), ("mom64", _P), ("vgrad", _P), ("s0", _P), ("l1", _P),
                ("n_active", _P), ("residual", _P), ("totals", _P), ("stop", _P)]


class PairGraph(ctypes.Structure):
    _fields_ = [("n_images", _I32), ("n_cameras", _I32), ("refine_focal", _I32),
                ("n_cam_chunks", _I32), ("n_pairs", _I64),
                ("pair_i", _P), ("pair_j", _P), ("pair_ci", _P), ("pair_cj", _P),
                ("img_off", _P), ("img_inc", _P), ("cam_off", _P), ("cam_inc", _P),
                ("cam_chunk_lo", _P), ("cam_chunk_cam", _P), ("cam_chunk_off", _P)]


class RotGraph(ctypes.Structure):
    _fields_ = [("n_nodes", _I32), ("n_edges", _I64), ("edge_i", _P), ("edge_j", _P), ("rel", _P),
                ("node_off", _P), ("node_inc", _P)]


class QuadModel(ctypes.Structure):
    _fields_ = [("kind", _I32), ("mom32", _P), ("vgrad", _P), ("s0", _P), ("ghat0", _P),
                ("w81", _P), ("mom64", _P)]


class PeerGroup(ctypes.Structure):
    _fields_ = [("n_ranks", _I32), ("rank", _I32), ("part", _P), ("ready", _P), ("epoch", _I64),
                ("max_blocks", _I32), ("system_scope", _I32)]


class DirGraph(ctypes.Structure):
    _fields_ = [("n_nodes", _I32), ("n_edges", _I64), ("edge_i", _P), ("edge_j", _P),
                ("dirs", _P), ("node_off", _P), ("node_inc", _P)]


# name -> (restype, argtypes); every symbol declared in include/fastmap_b200.h
SIGNATURES = {
    "fm_abi_version": (ctypes.c_int, []),
    "fm_last_error": (ctypes.c_char_p, []),
    "fm_device_count": (ctypes.c_int, []),
    "fm_point_pass_scratch_bytes": (_SZ, [ctypes.POINTER(PointStore)]),
    "fm_point_store_describe": (ctypes.c_int, [ctypes.POINTER(PointStore), _P]),
    "fm_store_build": (ctypes.c_int, [ctypes.POINTER(PointStore), _P, _P, _I32, _P, _P, _P, _I32, _P]),
    "fm_store_gather_mask": (ctypes.c_int, [ctypes.POINTER(PointStore), _P, _P, _P, _P]),
    "fm_store_gather_slots": (ctypes.c_int, [ctypes.POINTER(PointStore), _P, _P, _P, _P, _P]),
    "fm_store_scatter_slots": (ctypes.c_int, [ctypes.POINTER(PointStore), _P, _P, _P, _P, _P]),
    "fm_pass_totals_scratch_bytes": (_SZ, []),
    "fm_pass_totals": (ctypes.c_int, [_P, _P, _I64, _P, _P, _SZ, _P]),
    "fm_point_pass": (ctypes.c_int, [ctypes.POINTER(PointStore), ctypes.c_uint, _F64, _P, _P, _P,
                                     ctypes.POINTER(PassOut), _P, _SZ, _P]),
    "fm_epi_scratch_bytes": (_SZ, [ctypes.POINTER(PairGraph)]),
    "fm_epi_pair_ghat": (ctypes.c_int, [ctypes.POINTER(PairGraph), _P, _P, _P, _P, _SZ, _P]),
    "fm_epi_loss_grad": (ctypes.c_int, [ctypes.POINTER(PairGraph), ctypes.POINTER(QuadModel), _P,
                                        _F64, _P, _P, _P, _P, _SZ, _P]),
    "fm_epi_adam_steps": (ctypes.c_int, [ctypes.POINTER(PairGraph), ctypes.POINTER(QuadModel), _P,
                                         _P, _P, _I64, _I32, _F64, _F64, _F64, _F64, _F64, _P,
                                         _I32, _P, _SZ, _P]),
    "fm_epi_adam_steps_z": (ctypes.c_int, [ctypes.POINTER(PairGraph), ctypes.POINTER(QuadModel), _P,
                                           _P, _P, _I64, _I32, _F64, _F64, _F64, _F64, _P, _P,
                                           _I32, _P, _SZ, _P]),
    "fm_epi_adam_steps_nccl": (ctypes.c_int, [ctypes.POINTER(PairGraph), ctypes.POINTER(QuadModel),
                                              _P, _P, _P, _I64, _I32, _F64, _F64, _F64, _F64, _F64,
                                              _P, _P, _P, _I32, _P, _SZ, _P]),
    "fm_peer_part_len": (_SZ, [ctypes.POINTER(PairGraph)]),
    "fm_peer_flag_len": (_SZ, [ctypes.POINTER(PairGraph)]),
    "fm_epi_adam_steps_peer": (ctypes.c_int, [ctypes.POINTER(PairGraph), ctypes.POINTER(QuadModel),
                                              _P, _P, _P, _I64, _I32, _F64, _F64, _F64, _F64, _F64,
                                              _P, ctypes.POINTER(PeerGroup), _I32, _P, _SZ, _P]),
    "fm_peer_buffers_alloc": (ctypes.c_int, [_SZ, _SZ, ctypes.POINTER(ctypes.c_void_p),
                                             ctypes.POINTER(ctypes.c_void_p)]),
    "fm_peer_buffers_free": (ctypes.c_int, [_P, _P]),
    "fm_peer_sum_f64": (ctypes.c_int, [_P, _I32, ctypes.POINTER(PeerGroup), _P, _P]),
    "fm_ipc_get_handle": (ctypes.c_int, [_P, _P]),
    "fm_ipc_open_handle": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_void_p)]),
    "fm_ipc_close_handle": (ctypes.c_int, [_P]),
    "fm_release_cached_graphs": (None, []),
    "fm_nccl_available": (ctypes.c_int, []),
    "fm_nccl_unique_id": (ctypes.c_int, [_P]),
    "fm_nccl_comm_init": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), _I32, _P, _I32]),
    "fm_nccl_comm_destroy": (ctypes.c_int, [_P]),
    "fm_nccl_allreduce_sum_f64": (ctypes.c_int, [_P, _I64, _P, _P]),
    "fm_nccl_allgather_f64": (ctypes.c_int, [_P, _P, _I64, _P, _P]),
    "fm_rot6d_to_matrix": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P]),
    "fm_rot6d_jacobian": (ctypes.c_int, [_P, _I64, _P, _P]),
    "fm_project_to_so3": (ctypes.c_int, [_P, _I64, _P, _P]),
    "fm_compose_essential": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _P]),
    "fm_adam_step": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _F64, _F64, _F64, _F64, _P, _P]),
    "fm_tr_scratch_bytes": (_SZ, [_I32, _I64, _I32]),
    "fm_tr_loss_grad": (ctypes.c_int, [ctypes.POINTER(DirGraph), _P, _I32, _P, _P, _P, _SZ, _P]),
    "fm_tr_align": (ctypes.c_int, [ctypes.POINTER(DirGraph), _P, _I32, _I32, _F64, _F64, _F64,
                                   _F64, _P, _P, _P, _SZ, _P]),
    "fm_tr_canonicalize": (ctypes.c_int, [_P, _I32, _I32, _P, _SZ, _P]),
    "fm_tr_node_residuals": (ctypes.c_int, [ctypes.POINTER(DirGraph), _P, _I32, _P, _P]),
    "fm_tr_merge": (ctypes.c_int, [ctypes.POINTER(DirGraph), _P, _I32, _P, _P, _P, _SZ, _P]),
    "fm_sphere_errors": (ctypes.c_int, [_P, _P, _I64, _P, _P, _I32, _P, _P]),
    "fm_rot_scratch_bytes": (_SZ, [_I32, _I64]),
    "fm_rot_loss_grad": (ctypes.c_int, [ctypes.POINTER(RotGraph), _P, _P, _P, _P, _P, _SZ, _P]),
    "fm_rot_refine": (ctypes.c_int, [ctypes.POINTER(RotGraph), _P, _I32, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, _P,
                                     ctypes.POINTER(_I32), _P, _P, _SZ, _P]),
    "fm_depth_counts": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _P]),
    "fm_sphere_errors_batch": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P, _I64, _I32, _P, _P]),
    "fm_depth_counts_batch": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _I64, _P, _P]),
    "fm_fund_scratch_bytes": (ctypes.c_size_t, [_I64]),
    "fm_cc_labels": (ctypes.c_int, [_I32, _I64, _P, _P, _P, _P]),
    "fm_focal_votes": (ctypes.c_int, [_I32, _I32, _P, _P, _P, ctypes.c_double, _P, _P]),
    "fm_homog_fit": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _I64, _P]),
    "fm_fund_score": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t,
                                     _I64, _P]),
}


def lib_path():
    # FASTMAP_B200_LIB: alternative build of the same ABI (kernel tuning runs)
    return os.environ.get("FASTMAP_B200_LIB") or _build.LIB_PATH


def lib():
    """The loaded C-ABI library (raises if it is missing: no fallback)."""
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            raise RuntimeError(
                f"FastMap B200 native library not built ({path}); run "
                "`python -m paper_2505_04612_b200.build` (there is no CPU fallback)")
        handle = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.fm_abi_version() != ABI_VERSION:
            raise RuntimeError("FastMap B200 native library ABI mismatch")
        _LIB = handle
    return _LIB


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("the FastMap B200 hot path needs a CUDA device (no CPU fallback)")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t):
    """Device/host pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def last_error():
    msg = lib().fm_last_error()
    return msg.decode() if msg else ""


def check(rc):
    """Map an fm_status return code onto the reference's exception types."""
    if rc == FM_OK:
        return
    msg = last_error()
    if rc == FM_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"fastmap_b200 error {rc}: {msg}")


def raise_flag(code, context="epipolar"):
    """Raise the reference exception for a device flag value (0 = no error)."""
    code = int(code)
    if code == 0:
        return
    if code == FM_ERR_NONFINITE_LOSS:
        raise FloatingPointError("non-finite epipolar loss")
    if code == FM_ERR_NONFINITE_TRANSLATION:
        raise FloatingPointError("non-finite translation loss")
    if code == FM_ERR_NONFINITE_ROTATION:
        raise FloatingPointError("non-finite rotation loss")
    if code == FM_ERR_NONFINITE_GRAD:
        raise FloatingPointError("non-finite gradients")
    if code == FM_ERR_ROT6D_ZERO:
        raise ValueError("degenerate 6D rotation input: zero first half")
    if code == FM_ERR_ROT6D_COLLINEAR:
        raise ValueError("degenerate 6D rotation input: collinear halves")
    if code == FM_ERR_NO_ACTIVE:
        raise ValueError("no active point pairs")
    if code == FM_ERR_ALL_PRUNED:
        raise ValueError("all pairs pruned away")
    raise RuntimeError(f"fastmap_b200 device error code {code} ({context})")


def exported_symbols():
    return sorted(SIGNATURES)
