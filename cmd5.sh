set -x
python tools_debug_c2.py 2>&1 | tail -8
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -c 3000 gpurun_out/bench5.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python bench.py --steps 3 --warmup 3 --skip-cpu --skip-optimize > /dev/null 2>&1; wc -l gpurun_out/launches5.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 -o gpurun_out/prof5 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-optimize > gpurun_out/ncu5.log 2>&1; tail -3 gpurun_out/ncu5.log
