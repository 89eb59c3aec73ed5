"""The C-ABI library builds, loads on a CPU-only host and exports every
symbol declared in include/fastmap_b200.h; product entry points fail loudly
without a GPU (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fastmap_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(fm_[a-z0-9_]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_2505_04612_b200 import _native, build
    build.build()
    lib = ctypes.CDLL(build.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    # and the Python binding covers exactly the header
    assert sorted(_native.SIGNATURES) == names


def test_abi_version_and_device_count():
    from paper_2505_04612_b200 import _native
    lib = _native.lib()
    assert lib.fm_abi_version() == 6
    n = lib.fm_device_count()
    assert n == torch.cuda.device_count() or (n == 0 and not torch.cuda.is_available())


def test_invalid_arguments_are_reported_without_a_device():
    from paper_2505_04612_b200 import _native
    lib = _native.lib()
    rc = lib.fm_point_pass(None, 0, 0.0, None, None, None, None, None, 0, None)
    assert rc == _native.FM_ERR_INVALID
    assert "null" in _native.last_error()
    with pytest.raises(ValueError):
        _native.check(rc)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_cuda():
    from paper_2505_04612_b200 import epipolar, translation
    with pytest.raises(RuntimeError, match="CUDA"):
        epipolar.precompute_weights(np.ones((3, 3)), np.ones((3, 3)))
    g = translation.DirectionGraph(n=2, edges_i=np.array([0]), edges_j=np.array([1]),
                                   directions=np.array([[1.0, 0, 0]]))
    with pytest.raises(RuntimeError, match="CUDA"):
        translation.translation_loss_and_grad(np.zeros((2, 3)), g)


def test_raise_flag_maps_reference_exceptions():
    from paper_2505_04612_b200 import _native as N
    with pytest.raises(FloatingPointError, match="non-finite epipolar loss"):
        N.raise_flag(N.FM_ERR_NONFINITE_LOSS)
    with pytest.raises(FloatingPointError, match="non-finite gradients"):
        N.raise_flag(N.FM_ERR_NONFINITE_GRAD)
    with pytest.raises(FloatingPointError, match="non-finite translation loss"):
        N.raise_flag(N.FM_ERR_NONFINITE_TRANSLATION)
    with pytest.raises(ValueError, match="zero first half"):
        N.raise_flag(N.FM_ERR_ROT6D_ZERO)
    with pytest.raises(ValueError, match="all pairs pruned away"):
        N.raise_flag(N.FM_ERR_ALL_PRUNED)
    N.raise_flag(0)
