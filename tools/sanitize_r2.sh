#!/bin/bash
# compute-sanitizer over the kernels added / changed in round 2
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python -m pytest -q -m gpu -x \
  tests/test_epipolar_gpu.py tests/test_store_gpu.py tests/test_inputs_gpu.py \
  tests/test_parallel_gpu.py -k "not gloo" > gpurun_out/san_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_memcheck.log | tail -4
timeout 900 compute-sanitizer --tool racecheck python -m pytest -q -m gpu -x \
  tests/test_epipolar_gpu.py -k "config1_pose_parity or irls_refine_small or ragged" > gpurun_out/san_racecheck.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/san_racecheck.log | tail -4
timeout 600 compute-sanitizer --tool synccheck python -m pytest -q -m gpu -x \
  tests/test_epipolar_gpu.py -k "config1_pose_parity" > gpurun_out/san_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_synccheck.log | tail -3
