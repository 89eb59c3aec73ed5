#!/bin/bash
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --leak-check no python -m pytest -q -m gpu -x \
  tests/test_parallel_gpu.py -k "peer or nccl" > gpurun_out/san_peer_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_peer_memcheck.log | tail -3
timeout 900 compute-sanitizer --tool synccheck python -m pytest -q -m gpu -x \
  tests/test_parallel_gpu.py -k "peer" > gpurun_out/san_peer_sync.log 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_peer_sync.log | tail -3
