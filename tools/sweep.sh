#!/bin/bash
# Variant sweep (under gpurun): default lib with forced L, then build_variants/*.so.
for L in 4 8; do echo "== default L=$L"; FM_HOT_L=$L timeout 120 python tools/bench_modes.py c2 2>&1 | grep -oE '"precision.*"l1": [0-9.]+'; done
echo "== default auto"; timeout 120 python tools/bench_modes.py c2 2>&1 | grep -oE '"precision.*"l1": [0-9.]+'
for f in build_variants/*.so; do echo "== $f"; FASTMAP_B200_LIB=$PWD/$f timeout 120 python tools/bench_modes.py c2 2>&1 | grep -oE '"precision.*"l1": [0-9.]+|Error.*'; done
