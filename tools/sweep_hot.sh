python tools/pass_probe.py c2 -
for f in build_variants/hot_*.so; do echo "== $f"; FASTMAP_B200_LIB=$f python tools/pass_probe.py c2 -; done
python tools/pass_probe.py c2 -
