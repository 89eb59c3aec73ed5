#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored;
# it travels to the GPU box with the gpurun snapshot).  Offline: no index,
# --no-deps (numpy / scipy / opencv are already in the image).  The source is
# copied to /tmp first because the build writes into its tree and
# /root/reference is read-only.  The reference's own test files are copied
# next to the package so tests/test_reference_suite_gpu.py can run them
# against the installed drop-in on a box without /root/reference.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
rm -rf /tmp/fastmap_ref_src "$REPO/baseline/_ref"
cp -r "$SRC" /tmp/fastmap_ref_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" /tmp/fastmap_ref_src
cp -r "$SRC/tests" "$REPO/baseline/_ref/fastmap_tests"
echo "installed: $(ls "$REPO/baseline/_ref")"
