for f in build_variants/*.so; do echo "== $f"; FASTMAP_B200_LIB=$PWD/$f python tools/bench_modes.py c2 2>&1 | grep -E "pass_us|Error"; done
