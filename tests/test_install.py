"""install() rebinds the reference package's hot-path names (CPU: no kernel
runs).  Needs the reference package: the source tree here, else the
unmodified install in baseline/_ref (tools/install_reference.sh), which
travels to the GPU box."""

import importlib
import os
import sys

import pytest

_HERE = os.path.dirname(os.path.abspath(__file__))
REF = next((p for p in ("/root/reference/pkg/src",
                        os.path.join(os.path.dirname(_HERE), "baseline", "_ref"))
            if os.path.isdir(os.path.join(p, "fastmap"))), "/root/reference/pkg/src")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "fastmap")),
                    reason="reference package not present")
def test_install_swaps_the_pipeline_call_sites():
    sys.path.insert(0, REF)
    try:
        fastmap = importlib.import_module("fastmap")
        pipeline = importlib.import_module("fastmap.pipeline")
        ref_tr = importlib.import_module("fastmap.translation")
        ref_epi = importlib.import_module("fastmap.epipolar")
        ref_rot = importlib.import_module("fastmap.rotation")
        ref_dist = importlib.import_module("fastmap.distortion")
        ref_two = importlib.import_module("fastmap.twoview")
        ref_focal = importlib.import_module("fastmap.focal")
        ref_tracks = importlib.import_module("fastmap.tracks")
    except ImportError as exc:  # reference dependencies missing
        pytest.skip(str(exc))
    finally:
        sys.path.remove(REF)
    import paper_2505_04612_b200 as b200
    from paper_2505_04612_b200 import distortion, epipolar, focal, rotation, tracks, translation
    saved = b200.install(fastmap)
    try:
        assert pipeline.irls_refine is epipolar.irls_refine          # ref/pipeline.py:248
        assert ref_tr.multi_init_align is translation.multi_init_align  # ref/pipeline.py:233
        assert ref_tr.reestimate_relative is translation.reestimate_relative  # :209
        assert translation.PairRejected is ref_tr.PairRejected       # caught at :210
        assert ref_epi.quadratic_loss_and_grad is epipolar.quadratic_loss_and_grad
        assert ref_rot.refine_rotations is rotation.refine_rotations     # ref/pipeline.py:170
        assert ref_dist.search_alpha is distortion.search_alpha          # via schedule_cameras
        assert distortion.DegenerateGeometryError is ref_two.DegenerateGeometryError
        assert ref_focal.undistorted_fundamentals is focal.undistorted_fundamentals  # :105
        assert ref_focal.apply_calibration is focal.apply_calibration  # :123
        assert ref_focal.vote_focal is focal.vote_focal  # via vote_focal_multi, :106
        assert ref_tracks.complete_matches is tracks.complete_matches  # :179
        assert tracks.TrackSet is ref_tracks.TrackSet
    finally:
        for (mod, name), obj in saved.items():
            setattr(sys.modules[mod], name, obj)
    assert translation.PairRejected is not ref_tr.PairRejected
    assert distortion.DegenerateGeometryError is not ref_two.DegenerateGeometryError
