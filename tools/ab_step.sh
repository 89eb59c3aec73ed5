for r in 1 2; do for f in build_variants/hot_auto2.so build_variants/hot_ticket.so; do printf "%s %s " $r $(basename $f); FASTMAP_B200_LIB=$f python tools/pass_probe_batch.py c2 20 10 | tail -1; done; done
for f in build_variants/hot_auto2.so build_variants/hot_ticket.so; do printf "ev %s " $(basename $f); FASTMAP_B200_LIB=$f python tools/pass_probe.py c2 - | tail -1 | cut -c1-120; done
FASTMAP_B200_LIB=build_variants/hot_ticket.so python -m pytest tests/test_epipolar_gpu.py tests/test_parallel_gpu.py tests/test_mixed_launch_gpu.py -q -m gpu -x 2>&1 | tail -2
