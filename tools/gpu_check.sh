#!/bin/bash
# Usage (under gpurun): bash tools/gpu_check.sh TAG [tests] [bench] [ncu]
TAG=$1; shift
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests) timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 ;;
    alltests) timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -25 ;;
    bench) timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 2500 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err ;;
    quickbench) timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu --skip-optimize 2>&1 | tail -c 1500 ;;
    launches) timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --skip-cpu --skip-optimize > /dev/null 2>&1; wc -l gpurun_out/launches_$TAG.csv ;;
    ncu) timeout 600 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --skip-cpu --skip-optimize > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log ;;
    smoke) python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 ;;
  esac
done
