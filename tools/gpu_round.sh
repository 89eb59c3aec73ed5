timeout 300 python -m pytest tests/test_parallel_gpu.py -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r1s2b.json 2> gpurun_out/bench_r1s2b.err; tail -c 3000 gpurun_out/bench_r1s2b.json; tail -3 gpurun_out/bench_r1s2b.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 -o gpurun_out/prof_r1s2b python bench.py --steps 3 --warmup 3 --skip-cpu --skip-optimize > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1s2b.csv python bench.py --steps 10 --warmup 3 --skip-cpu --skip-optimize > /dev/null 2>&1
ls -la gpurun_out | tail -5
