for L in 4 8 16; do echo "L=$L"; FM_HOT_L=$L python tools/bench_modes.py c2 2>&1 | grep pass_us; done
echo auto; python tools/bench_modes.py c2 2>&1 | grep pass_us
