#!/bin/bash
# Round-2 profiling session (under gpurun): bench, launch list of the bench
# command, ncu --set full of the hot pass (C2) and of the Adam-step kernels.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
tail -c 600 gpurun_out/bench_r2.json; tail -3 gpurun_out/bench_r2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fm_timed/" --csv \
  --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 3 --skip-cpu --skip-strong \
  > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 \
  -o gpurun_out/prof_r2_pass_c2 python tools/one_pass.py full fp32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 \
  -o gpurun_out/prof_r2_pass_c4 python tools/one_pass.py full fp32 c4 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none --graph-profiling node \
  -k regex:"pair_grad|image_reduce" -s 50 -c 2 -o gpurun_out/prof_r2_adam_c2 python tools/irls_run.py c2 fp32 > /dev/null 2>&1
ls gpurun_out
