"""B200-native FastMap hot path (arXiv 2505.04612).

Drop-in replacements for the reference package's epipolar adjustment
(``fastmap.epipolar``), global translation alignment (the
``DirectionGraph`` half of ``fastmap.translation``) and optimizer kernel
(``fastmap.optim``), running on hand-written sm_100a CUDA kernels behind the
C ABI in ``include/fastmap_b200.h``.  See DESIGN.md / INTEGRATION.md.
"""

from . import build  # noqa: F401

__version__ = "0.1.0"

__all__ = ["epipolar", "translation", "optim", "model", "config", "store", "inputs", "install", "native_library"]


def native_library():
    """Path of the loaded C-ABI shared library (loads it; raises if missing)."""
    from . import _native
    _native.lib()
    return _native.lib_path()


def install(fastmap_module=None):
    """Route a loaded reference ``fastmap`` package through this hot path.

    Rebinds ``irls_refine`` and ``translation.multi_init_align`` where
    ``fastmap.pipeline`` looks them up (ref/pipeline.py:233, :248), plus the
    hot-path functions of ``fastmap.epipolar`` / ``fastmap.translation`` /
    ``fastmap.optim``.  Returns the dict of replaced originals.
    """
    import importlib

    from . import epipolar, optim, translation
    fm = fastmap_module or importlib.import_module("fastmap")
    pipeline = importlib.import_module(fm.__name__ + ".pipeline")
    ref_epi = importlib.import_module(fm.__name__ + ".epipolar")
    ref_tr = importlib.import_module(fm.__name__ + ".translation")
    ref_opt = importlib.import_module(fm.__name__ + ".optim")
    saved = {}

    def swap(mod, name, new):
        saved[(mod.__name__, name)] = getattr(mod, name)
        setattr(mod, name, new)

    swap(pipeline, "irls_refine", epipolar.irls_refine)
    for name in ("precompute_weights", "epipolar_loss", "quadratic_loss_and_grad",
                 "current_residuals", "irls_refine", "poses_from_state"):
        swap(ref_epi, name, getattr(epipolar, name))
    for name in ("translation_loss_and_grad", "canonicalize", "align_centers",
                 "per_node_residuals", "multi_init_align", "reestimate_relative"):
        swap(ref_tr, name, getattr(translation, name))
    # ref/pipeline.py:170 calls rotation.refine_rotations through the module
    ref_rot = importlib.import_module(fm.__name__ + ".rotation")
    from . import rotation
    for name in ("rotation_loss_and_grad", "refine_rotations"):
        swap(ref_rot, name, getattr(rotation, name))
    # raise the reference's PairRejected, which ref/pipeline.py:210 catches
    swap(translation, "PairRejected", ref_tr.PairRejected)
    for name in ("rot6d_to_matrix", "rot6d_jacobian"):
        swap(ref_opt, name, getattr(optim, name))
    # ref/pipeline.py:94 -> schedule_cameras -> search_alpha (module globals)
    ref_dist = importlib.import_module(fm.__name__ + ".distortion")
    ref_two = importlib.import_module(fm.__name__ + ".twoview")
    from . import distortion
    for name in ("score_alpha", "search_alpha"):
        swap(ref_dist, name, getattr(distortion, name))
    swap(distortion, "DegenerateGeometryError", ref_two.DegenerateGeometryError)
    # ref/pipeline.py:105 calls focal.undistorted_fundamentals through the module
    ref_focal = importlib.import_module(fm.__name__ + ".focal")
    from . import focal
    # vote_focal_multi (ref/pipeline.py:106) finds vote_focal through the module
    for name in ("undistorted_fundamentals", "apply_calibration", "vote_focal"):  # :105, :123
        swap(ref_focal, name, getattr(focal, name))
    swap(focal, "FocalUnderdeterminedError", ref_focal.FocalUnderdeterminedError)
    # ref/pipeline.py:178-181 calls tracks.build_tracks / complete_matches
    ref_tracks = importlib.import_module(fm.__name__ + ".tracks")
    from . import tracks
    for name in ("build_tracks", "complete_matches"):
        swap(ref_tracks, name, getattr(tracks, name))
    swap(tracks, "TrackSet", ref_tracks.TrackSet)
    return saved
