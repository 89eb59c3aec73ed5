#!/bin/bash
echo "== default"; timeout 200 python tools/size_probe.py 400 1600
for f in build_variants/*.so; do echo "== $f"; FASTMAP_B200_LIB=$PWD/$f timeout 200 python tools/size_probe.py 400 1600; done
