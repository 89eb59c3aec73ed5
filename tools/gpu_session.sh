#!/bin/bash
# Under gpurun: bash tools/gpu_session.sh STEP [STEP ...]
mkdir -p gpurun_out
for what in "$@"; do
  echo "=== $what"
  case $what in
    tests) timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -30 ;;
    tests_tr) timeout 900 python -m pytest tests/test_translation_gpu.py tests/test_pipeline_golden_gpu.py -q -m gpu 2>&1 | tail -30 ;;
    tests_ref) timeout 1500 python -m pytest tests/test_reference_suite_gpu.py -q -m gpu -s 2>&1 | tail -60 ;;
    trbench) timeout 600 python -c "
import torch, bench
s = torch.cuda.Stream()
print(bench.translation_bench(torch.device('cuda'), s))" 2>&1 | tail -3 ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err ;;
    benchref) timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/benchref.json 2> gpurun_out/benchref.err; tail -c 3000 gpurun_out/benchref.json; tail -5 gpurun_out/benchref.err ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 ;;
  esac
done
