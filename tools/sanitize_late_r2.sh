#!/bin/bash
# compute-sanitizer over the late round-2 changes: the cluster-persistent
# translation descent, the one-sync irls_refine schedule (stop word,
# device 2/Z, pinned schedule ring)
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --leak-check no python -m pytest -q -m gpu -x \
  tests/test_translation_gpu.py tests/test_epipolar_gpu.py -k "cluster or align_and_multi or config1_multi or mid_schedule or pruned or irls_refine_small or config1_pose_parity" \
  > gpurun_out/san2_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san2_memcheck.log | tail -3
timeout 900 compute-sanitizer --tool racecheck python -m pytest -q -m gpu -x \
  tests/test_translation_gpu.py -k "cluster_descent_equals and 3-250" > gpurun_out/san2_racecheck.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/san2_racecheck.log | tail -3
timeout 900 compute-sanitizer --tool synccheck python -m pytest -q -m gpu -x \
  tests/test_translation_gpu.py -k "cluster_descent_equals and 3-250" > gpurun_out/san2_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san2_synccheck.log | tail -3
