#!/bin/bash
# One GPU iteration (under gpurun): tests, per-mode timings, ncu of the hot pass.
#   bash tools/cycle.sh TAG [notests] [noncu]
TAG=$1; shift
mkdir -p gpurun_out
if [[ " $* " != *" notests "* ]]; then
  timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
fi
timeout 300 python tools/bench_modes.py c2 2>&1 | tail -3
if [[ " $* " != *" noncu "* ]]; then
  for prec in fp64 fp32; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_$prec python tools/one_pass.py full $prec > gpurun_out/ncu_${TAG}_$prec.log 2>&1
    tail -1 gpurun_out/ncu_${TAG}_$prec.log
  done
fi
