timeout 300 python -m pytest tests/test_parallel_gpu.py -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r1s3.json 2> gpurun_out/bench_r1s3.err; tail -c 3000 gpurun_out/bench_r1s3.json; tail -3 gpurun_out/bench_r1s3.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 -o gpurun_out/prof_r1s3 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-optimize > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1s3.csv python bench.py --steps 10 --warmup 3 --skip-cpu --skip-optimize > /dev/null 2>&1
ls -la gpurun_out | tail -5
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --skip-cpu > gpurun_out/bench_c4_r1s3.json 2>/dev/null; tail -c 600 gpurun_out/bench_c4_r1s3.json
