"""pytest plugin: import the installed reference package (baseline/_ref)
and route it through the B200 drop-in (paper_2505_04612_b200.install) BEFORE
the reference's own test modules are collected, so their
``from fastmap.epipolar import ...`` lines bind our functions.

    python -m pytest -p tests.ref_dropin_plugin baseline/_ref/fastmap_tests/test_epipolar.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def pytest_configure(config):
    for p in (ROOT, REF):
        if p not in sys.path:
            sys.path.insert(0, p)
    import fastmap

    import paper_2505_04612_b200 as b200
    b200.install(fastmap)
    config._fm_dropin = fastmap.__file__


def pytest_report_header(config):
    return f"fastmap reference at {getattr(config, '_fm_dropin', '?')}, routed through the B200 drop-in"
