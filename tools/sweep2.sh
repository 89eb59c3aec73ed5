#!/bin/bash
# per-variant wave probe at C2 and at 100k pairs (steady state)
echo "== default"; timeout 200 python tools/wave_probe.py 500,50,400 2000,50,400 2>&1 | grep pairs
for f in build_variants/*.so; do echo "== $f"; FASTMAP_B200_LIB=$PWD/$f timeout 200 python tools/wave_probe.py 500,50,400 2000,50,400 2>&1 | grep -E "pairs|Error"; done
